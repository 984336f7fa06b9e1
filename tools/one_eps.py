"""One C4 solve (n = 1024) at a given eps: iterations, time to eps, final residual (FC_* env honoured)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2006_09314_b200.binding import DeviceCP, Library, make_params  # noqa: E402
from synth import make_problem  # noqa: E402

eps = float(sys.argv[1]) if len(sys.argv) > 1 else 1e-7
p = make_problem("C4", n=1024, eps=eps)
L = Library()
ctx = L.context(torch.cuda.current_stream().cuda_stream)
prm = make_params(p.alpha, p.beta, p.eps, p.tol_stop)
ctx.sl_setup(p.n, p.a_mid, prm)
b = DeviceCP.from_numpy(p.b_w, p.b_U)
ctx.pcg_solve(b, prm)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
u, rep, rc = ctx.pcg_solve(b, prm)
e1.record()
torch.cuda.synchronize()
print(json.dumps({"eps": eps, "rc": rc, "iters": rep["iters"], "time_ms": e0.elapsed_time(e1),
                  "final_rel_res": rep["rel_res"][rep["iters"] - 1], "rank_X": u.rank}))
