set -x
python -m pytest tests/test_gpu_apply.py tests/test_gpu_truncate_pcg.py -q -x 2>&1 | tail -2
timeout 300 python tools/bench_apply.py --no-trunc > gpurun_out/r02y_c5_apply.txt 2>&1; python -c "
import json
for l in open('gpurun_out/r02y_c5_apply.txt'):
    d=json.loads(l); print(d['n'],d['R'],d['r'],round(d['inv_kernel_ms'],4),round(d['inv_tflops'],2),round(d['inv_frac_dmma'],3))"
for e in 1e-8; do FC_PHASES=1 timeout 300 python tools/c4_trace.py $e 1024 > gpurun_out/r02y_phases_$e.txt 2>&1; done
grep -h "fc phases\|\"rc\"" gpurun_out/r02y_phases_*.txt | cut -c1-160 | head -14
timeout 900 python -m pytest tests/test_gpu_parity_fullsize.py -q -x -s -k "c4_iterate or C4 or eps_sweep" 2>&1 | grep -E "reldiff|passed|failed|C4 eps|rank history" | head -20
