mkdir -p gpurun_out
timeout 600 python tools/diag_eig.py 2048 > gpurun_out/diag_eig.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_setup.py -q --tb=line > gpurun_out/pytest_gpu.log 2>&1
tail -2 gpurun_out/pytest_gpu.log
