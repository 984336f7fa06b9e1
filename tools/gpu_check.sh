mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_caseA.py tests/test_gpu_setup.py -q -s --tb=short > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
