set -x
python -m pytest tests/test_gpu_truncate_pcg.py tests/test_gpu_determinism.py -q -x 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_parity_fullsize.py -q -x -s -k "c4_iterate or fused or eps_sweep" 2>&1 | grep -E "reldiff|passed|failed|C4 eps|eps=1e-8" | head -12
for e in 1e-7 1e-8; do FC_PHASES=1 timeout 300 python tools/c4_trace.py $e 1024 > gpurun_out/r02dd_phases_$e.txt 2>&1; done
grep -h "fc phases\|\"rc\"" gpurun_out/r02dd_phases_*.txt | cut -c1-120 | head -24
