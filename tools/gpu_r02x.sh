set -x
python -m pytest tests/test_gpu_apply.py -q -x 2>&1 | tail -2
timeout 600 python tools/diag_plain8.py 1e-8 > gpurun_out/r02x_plain8.txt 2>&1; cat gpurun_out/r02x_plain8.txt | grep -v "^\[fc"
for e in 1e-7 1e-8; do FC_PHASES=1 timeout 300 python tools/c4_trace.py $e 1024 > gpurun_out/r02x_phases_$e.txt 2>&1; done
grep -h "fc phases\|\"rc\"" gpurun_out/r02x_phases_*.txt | cut -c1-160
timeout 300 python tools/bench_apply.py --no-trunc > gpurun_out/r02x_c5_apply.txt 2>&1; cat gpurun_out/r02x_c5_apply.txt
ncu --set full --import-source on -k regex:dgemm_big --launch-count 1 -o gpurun_out/r02x_kr python tools/profile_apply.py > gpurun_out/r02x_ncu.log 2>&1; tail -3 gpurun_out/r02x_ncu.log
