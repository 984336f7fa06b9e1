import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_09314_b200.binding import DeviceCP, Library, make_params  # noqa: E402
from synth import make_problem  # noqa: E402

L = Library()
for n, rg in ((512, 24), (512, 12), (1024, 24)):
    p = make_problem("C4", n=n, eps=1e-8)
    ctx = L.context()
    prm = make_params(p.alpha, p.beta, p.eps, p.tol_stop, kmax=25, precond_rank=rg)
    ctx.sl_setup(p.n, p.a_mid, prm)
    u, rep, rc = ctx.pcg_solve(DeviceCP.from_numpy(p.b_w, p.b_U), prm)
    print("n=%d r_G=%d rc=%d" % (n, rg, rc), ["%.1e" % x for x in rep["rel_res"]], "%.0f ms" % rep["t_total_ms"], flush=True)
