import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2006_09314_b200.binding import FC_F, FC_G, DeviceCP, Library, make_params  # noqa: E402
from synth import make_problem  # noqa: E402

L = Library()
p = make_problem("C4", n=512, eps=1e-8)
ctx = L.context()
prm = make_params(p.alpha, p.beta, p.eps, p.tol_stop, kmax=6)
ctx.sl_setup(p.n, p.a_mid, prm)
b = DeviceCP.from_numpy(p.b_w, p.b_U)
for which in (FC_G, FC_F):
    y1, i1 = ctx.fracop_apply_truncate(which, b, p.eps)
    yu = ctx.fracop_apply(which, b)
    y2, i2 = ctx.cp_truncate(yu, p.eps)
    d = ctx.cp_axpy(y1, -1.0, y2)
    rel = math.sqrt(max(ctx.cp_dot(d, d), 0) / ctx.cp_dot(y2, y2))
    print("which %d fused tucker %s rank %d | plain tucker %s rank %d | rel diff %.2e" % (
        which, list(i1.tucker_rank), y1.rank, list(i2.tucker_rank), y2.rank, rel), flush=True)
u, rep, rc = ctx.pcg_solve(b, prm)
print("pcg", rc, ["%.1e" % x for x in rep["rel_res"]], flush=True)
