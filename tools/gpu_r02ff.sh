set -x
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02ff_gpu.txt 2>&1; tail -3 gpurun_out/r02ff_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for e in 1e-7 1e-8; do FC_PHASES=1 timeout 300 python tools/c4_trace.py $e 1024 > gpurun_out/r02ff_phases_$e.txt 2>&1; done
grep -h "fc phases\|\"rc\"" gpurun_out/r02ff_phases_*.txt | cut -c1-120 | grep -E "rc|total|dd factor"
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r02ff_bench.txt 2> gpurun_out/r02ff_bench.err; tail -c 600 gpurun_out/r02ff_bench.txt
