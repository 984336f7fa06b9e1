set -x
timeout 900 python -m pytest tests/test_gpu_apply.py -q -x > gpurun_out/r02xx_apply_tests.txt 2>&1; tail -5 gpurun_out/r02xx_apply_tests.txt
for v in 1 0; do
FC_STREAMK=$v timeout 900 python tools/bench_apply.py --no-trunc > gpurun_out/r02xx_c5_streamk$v.jsonl 2>&1
done
python - <<'PY'
import json
def load(p):
    return {(r['n'],r['R'],r['r']): r for r in (json.loads(l) for l in open(p) if l.startswith('{'))}
a=load('gpurun_out/r02xx_c5_streamk1.jsonl'); b=load('gpurun_out/r02xx_c5_streamk0.jsonl')
for k in sorted(a):
    print(k, 'streamk %.1f%% (%.3f ms)  tiles-only %.1f%% (%.3f ms)' % (100*a[k]['inv_frac_dmma'], a[k]['inv_kernel_ms'], 100*b[k]['inv_frac_dmma'], b[k]['inv_kernel_ms']))
PY
