mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_lr2d.py -q -m gpu -x -s > gpurun_out/pt.log 2>&1 || { echo "pytest failed/timeout"; tail -15 gpurun_out/pt.log; exit 1; }
grep -a "2D n=1024" gpurun_out/pt.log; tail -1 gpurun_out/pt.log
