import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_09314_b200.binding import DeviceCP, Library, make_params  # noqa: E402
from synth import make_problem  # noqa: E402

L = Library()
for n in (512, 1024):
    p = make_problem("C4", n=n, eps=1e-8)
    ctx = L.context()
    prm = make_params(p.alpha, p.beta, p.eps, p.tol_stop, kmax=8)
    ctx.sl_setup(p.n, p.a_mid, prm)
    print("n=%d F rank %s G rank %s" % (n, ctx.op_spectral_rank(0), ctx.op_spectral_rank(1)), flush=True)
    u, rep, rc = ctx.pcg_solve(DeviceCP.from_numpy(p.b_w, p.b_U), prm)
    print("device n=%d" % n, rc, ["%.2e" % x for x in rep["rel_res"]], rep["rank_R"], rep["rank_S"], rep["t_iter_ms"], flush=True)
