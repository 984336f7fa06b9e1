# Knob sweep on the C4 bench: one bench line per environment setting (diagnostics only).
# usage: bash tools/knob_sweep.sh "BASE=1" "FC_POLAR_WAVES=4" ...
mkdir -p gpurun_out
for kv in "$@"; do
  env $kv timeout 240 python bench.py --steps 5 --warmup 3 > gpurun_out/ks.log 2>&1
  python - "$kv" <<'PY'
import json, sys
try:
    d = json.loads(open("gpurun_out/ks.log").read().strip().splitlines()[-1])
    print(sys.argv[1], "%.2f iters/s" % d["value"], "iters", d["iters_per_solve"], "rel_res %.3e" % d["final_rel_res"], "sm_mhz", d["clocks"]["sm_mhz"])
except Exception as e:
    print(sys.argv[1], "FAILED", e)
PY
done
