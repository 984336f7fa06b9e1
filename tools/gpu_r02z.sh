set -x
python -m pytest tests/test_gpu_apply.py -q -x 2>&1 | tail -2
for sk in 0 1 2 3 4 6; do echo "sk=$sk"; FC_APPLY_SPLITK=$sk timeout 300 python tools/bench_apply.py --no-trunc 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if d['n']>=1024 and d['r']*d['R']>=512: print(d['n'],d['R'],d['r'],round(d['inv_kernel_ms'],4),round(d['inv_frac_dmma'],3))"; done
FC_PHASES=1 timeout 300 python tools/c4_trace.py 1e-8 1024 > gpurun_out/r02z_phases_1e-8.txt 2>&1
grep -h "fc phases\|\"rc\"" gpurun_out/r02z_phases_1e-8.txt | cut -c1-160 | head -16
timeout 900 python tools/fidelity_sweep.py > gpurun_out/r02z_fidelity.txt 2>&1; cat gpurun_out/r02z_fidelity.txt
