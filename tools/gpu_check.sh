set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_truncate_pcg.py tests/test_gpu_apply.py -x -q 2>&1 | tail -40
