"""C4 solve trace: per-iteration rel_res, ranks and times at a given eps (and n); optionally two
back-to-back solves compared bit for bit (reproducibility).  `python tools/c4_trace.py EPS [N] [--twice] [--kmax=K]`"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2006_09314_b200.binding import DeviceCP, Library, make_params  # noqa: E402
from synth import make_problem  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
eps = float(args[0]) if args else 1e-8
n = int(args[1]) if len(args) > 1 else 1024
p = make_problem("C4", n=n, eps=eps)
L = Library()
ctx = L.context(torch.cuda.current_stream().cuda_stream)
kmax = next((int(a.split("=")[1]) for a in sys.argv if a.startswith("--kmax=")), 0)
prm = make_params(p.alpha, p.beta, p.eps, p.tol_stop, kmax=kmax)
ctx.sl_setup(p.n, p.a_mid, prm)
b = DeviceCP.from_numpy(p.b_w, p.b_U)
runs = []
for _ in range(2 if "--twice" in sys.argv else 1):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    u, rep, rc = ctx.pcg_solve(b, prm)
    e1.record()
    torch.cuda.synchronize()
    rep["rc"] = rc
    rep["time_ms"] = e0.elapsed_time(e1)
    runs.append(rep)
    print(json.dumps({"eps": eps, "n": n, "rc": rc, "iters": rep["iters"], "time_ms": rep["time_ms"],
                      "rel_res": [float(f"{x:.6e}") for x in rep["rel_res"]],
                      "rank_R": rep["rank_R"], "rank_S": rep["rank_S"], "rank_Z": rep["rank_Z"],
                      "rank_P": rep["rank_P"], "rank_X": rep["rank_X"], "tucker_S": rep["tucker_S"],
                      "t_iter_ms": [round(t, 1) for t in rep["t_iter_ms"]]}), flush=True)
if len(runs) == 2:
    a, b2 = runs
    same = all(a[k] == b2[k] for k in ("rel_res", "rank_R", "rank_S", "rank_Z", "rank_P", "rank_X"))
    print(json.dumps({"bit_identical": same}))
