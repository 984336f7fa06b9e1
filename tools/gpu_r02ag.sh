set -x
timeout 900 python tools/eps_sweep.py > gpurun_out/r02ag_eps_sweep.jsonl 2>&1; cut -c1-160 gpurun_out/r02ag_eps_sweep.jsonl
FC_PHASES=1 timeout 300 python tools/c4_trace.py 1e-8 1024 > gpurun_out/r02ag_phases_1e-8.txt 2>&1; grep "fc phases" gpurun_out/r02ag_phases_1e-8.txt | head -8
timeout 1500 python -m pytest tests/test_gpu_parity_fullsize.py tests/test_gpu_determinism.py -q -x > gpurun_out/r02ag_gpu.txt 2>&1; tail -3 gpurun_out/r02ag_gpu.txt
