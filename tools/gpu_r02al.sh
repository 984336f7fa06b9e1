set -x
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r02g_gpu.txt 2>&1; tail -3 gpurun_out/r02g_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/r02g_bench.txt 2> gpurun_out/r02g_bench.err; tail -c 300 gpurun_out/r02g_bench.txt
timeout 900 python tools/eps_sweep.py > gpurun_out/r02g_eps_sweep.jsonl 2>&1; cut -c1-130 gpurun_out/r02g_eps_sweep.jsonl
