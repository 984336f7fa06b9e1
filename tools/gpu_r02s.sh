set -x
FC_PHASES=1 timeout 300 python tools/c4_trace.py 1e-7 1024 > gpurun_out/r02s_phases_1e7.txt 2>&1
FC_PHASES=1 FC_TRACE=1 timeout 300 python tools/c4_trace.py 1e-8 1024 --kmax=6 > gpurun_out/r02s_phases_1e8.out 2> gpurun_out/r02s_phases_1e8.err
grep "fc phases" gpurun_out/r02s_phases_1e8.err
grep "fc phases" gpurun_out/r02s_phases_1e7.txt
python -m pytest tests/test_gpu_apply.py tests/test_gpu_determinism.py -q -x 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_truncate_pcg.py -q -x -s 2>&1 | tail -30 > gpurun_out/r02s_trunc_pcg.txt
tail -30 gpurun_out/r02s_trunc_pcg.txt
