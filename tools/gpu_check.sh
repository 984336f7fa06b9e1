mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_truncate_pcg.py -q -m gpu -x -k "k13 or small_eps" 2>&1 | tail -15
FC_TRUNC_QR=0 timeout 600 python -m pytest tests/test_gpu_truncate_pcg.py -q -m gpu -k "k13" 2>&1 | tail -4
