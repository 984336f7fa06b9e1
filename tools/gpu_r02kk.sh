set -x
timeout 900 python -m pytest tests -m gpu -q -x --deselect "tests/test_gpu_parity_fullsize.py" -k "not parity_fullsize" > gpurun_out/r02kk_gpu.txt 2>&1; tail -3 gpurun_out/r02kk_gpu.txt
timeout 600 python tools/diag_kr_drop.py 6 1e-6 2>&1 | tail -9
timeout 600 python tools/diag_kr_drop.py 10 1e-6 2>&1 | tail -9
