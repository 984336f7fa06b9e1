set -x
python -m pytest tests/test_gpu_linalg.py tests/test_gpu_determinism.py -q -x 2>&1 | tail -3
for e in 1e-7 1e-8; do FC_PHASES=1 timeout 300 python tools/c4_trace.py $e 1024 > gpurun_out/r02u_phases_$e.txt 2>&1; done
grep -h "fc phases\|\"rc\"" gpurun_out/r02u_phases_*.txt | cut -c1-300
timeout 1200 python -m pytest tests/test_gpu_parity_fullsize.py -q -s -x --durations=20 > gpurun_out/r02u_parity.txt 2>&1
grep -E "rank history|reldiff|passed|failed|Error|assert|apply-trunc|cp_truncate|fused|C4 eps|S0|Z0|s call" gpurun_out/r02u_parity.txt | head -60
