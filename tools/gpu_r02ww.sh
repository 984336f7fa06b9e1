set -x
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r02ww_gpu.txt 2>&1; tail -3 gpurun_out/r02ww_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r02ww_bench.txt 2> gpurun_out/r02ww_bench.err; tail -c 1500 gpurun_out/r02ww_bench.txt
timeout 900 python tools/eps_sweep.py > gpurun_out/r02ww_eps_sweep.jsonl 2>&1; cut -c1-200 gpurun_out/r02ww_eps_sweep.jsonl
timeout 300 python tools/timeline.py 1024 1e-6 > gpurun_out/r02ww_timeline.txt 2>&1; sed -n 3,16p gpurun_out/r02ww_timeline.txt
FC_PHASES=1 timeout 300 python tools/c4_trace.py 1e-6 > gpurun_out/r02ww_phases.txt 2>&1; grep "fc phases" gpurun_out/r02ww_phases.txt | head -20
