set -x
python -m pytest tests/test_gpu_linalg.py tests/test_gpu_determinism.py tests/test_gpu_truncate_pcg.py -q -x 2>&1 | tail -3
FC_TRACE=1 timeout 600 python tools/diag_plain8.py 1e-8 > gpurun_out/r02w_plain8.txt 2> gpurun_out/r02w_plain8.err
cat gpurun_out/r02w_plain8.txt; grep "refined\|terms=" gpurun_out/r02w_plain8.err | tail -12
for e in 1e-7 1e-8; do FC_PHASES=1 timeout 300 python tools/c4_trace.py $e 1024 > gpurun_out/r02w_phases_$e.txt 2>&1; done
grep -h "fc phases\|\"rc\"" gpurun_out/r02w_phases_*.txt | cut -c1-200
