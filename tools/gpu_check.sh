mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_als.py -q -m gpu -x 2>&1 | tail -25
