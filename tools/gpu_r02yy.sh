set -x
for cfg in "1.01 32" "1.01 8" "1.01 16"; do
set -- $cfg
FC_STREAMK_EFF=$1 FC_STREAMK_MINIT=$2 timeout 900 python tools/bench_apply.py --no-trunc > gpurun_out/r02yy_c5_eff$1_min$2.jsonl 2>&1
done
python - <<'PY'
import json
def load(p):
    return {(r['n'],r['R'],r['r']): r for r in (json.loads(l) for l in open(p) if l.startswith('{'))}
fs=['gpurun_out/r02xx_c5_streamk0.jsonl','gpurun_out/r02xx_c5_streamk1.jsonl','gpurun_out/r02yy_c5_eff1.01_min32.jsonl','gpurun_out/r02yy_c5_eff1.01_min16.jsonl','gpurun_out/r02yy_c5_eff1.01_min8.jsonl']
import os
t=[load(f) for f in fs if os.path.exists(f)]
for k in sorted(t[-1]):
    print(k, ' '.join('%5.1f' % (100*x[k]['inv_frac_dmma']) for x in t if k in x))
PY
