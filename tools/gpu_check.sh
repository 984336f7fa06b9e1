mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_lr2d.py -q -m gpu -s -x 2>&1 | tail -40
