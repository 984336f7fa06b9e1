# round 2, session 4: baseline of the restored tree (GPU suite, smoke, bench)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s4_gputest.log 2>&1; echo "pytest exit $?"
tail -5 gpurun_out/s4_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s4_smoke.log 2>&1; echo "smoke exit $?"; tail -2 gpurun_out/s4_smoke.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/s4_bench.jsonl 2> gpurun_out/s4_bench.err; echo "bench exit $?"
head -c 600 gpurun_out/s4_bench.jsonl
