# Knob sweep on the C4 bench: one bench line per environment setting (diagnostics only).
mkdir -p gpurun_out
for kv in "BASE=1" "FC_TRI_THREADS=256" "FC_TRI_THREADS=384" "FC_TRI_PACKED_THREADS=512" "FC_SKINNY_WAVES=1" "FC_SKINNY_WAVES=4" "BASE=2"; do
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
