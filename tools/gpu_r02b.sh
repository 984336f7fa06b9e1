set -x
python -m pytest tests/test_gpu_apply.py -x -q 2>&1 | tail -5
timeout 300 python tools/c4_trace.py 1e-6 1024 --twice > gpurun_out/r02b_c4_1e6.txt 2>&1
timeout 600 python tools/diag_spectral_eps.py 1024 > gpurun_out/r02b_spectral.txt 2>&1
timeout 600 python tools/diag_spectral_eps.py 1024 --sinc >> gpurun_out/r02b_spectral.txt 2>&1
cat gpurun_out/r02b_spectral.txt
