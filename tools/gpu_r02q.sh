set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/r02q_pytest.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02q_smoke.txt 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/r02q_bench.txt 2> gpurun_out/r02q_bench.err
for e in 1e-5 1e-6 1e-7; do timeout 300 python tools/c4_trace.py $e 1024 --twice > gpurun_out/r02q_c4_$e.txt 2>&1; done
cat gpurun_out/r02q_pytest.txt gpurun_out/r02q_smoke.txt; head -c 1500 gpurun_out/r02q_bench.txt
