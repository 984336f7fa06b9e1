mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_truncate_pcg.py -q --tb=short > gpurun_out/pytest_gpu.log 2>&1
tail -1 gpurun_out/pytest_gpu.log
timeout 1200 python tools/eps_sweep.py > gpurun_out/eps_sweep.jsonl 2>&1
cat gpurun_out/eps_sweep.jsonl | tail -4
