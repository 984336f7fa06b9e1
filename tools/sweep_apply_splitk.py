"""FC_APPLY_SPLITK sweep of the inverse mode transform over the 27 C5 cells: one subprocess per
split (the knob is read once per process), one JSON line per (cell, split) with the transform's
TFLOP/s and fraction of the measured DMMA peak.  `python tools/sweep_apply_splitk.py [splits]`"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
splits = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "0,1,2,3,4,5,6,8").split(",")]
for sk in splits:
    env = dict(os.environ)
    if sk > 0:
        env["FC_APPLY_SPLITK"] = str(sk)
    else:
        env.pop("FC_APPLY_SPLITK", None)    # 0: the library's own choice
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "bench_apply.py"), "--no-trunc"],
                         env=env, capture_output=True, text=True)
    for line in out.stdout.splitlines():
        if line.startswith("{"):
            row = json.loads(line)
            row["splitk"] = sk
            print(json.dumps(row), flush=True)
    if out.returncode != 0:
        print(json.dumps({"splitk": sk, "error": out.stderr[-400:]}), flush=True)
