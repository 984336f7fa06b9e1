mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_state.py -q -s --tb=short > gpurun_out/pytest_gpu.log 2>&1
tail -1 gpurun_out/pytest_gpu.log
