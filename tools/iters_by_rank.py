"""Case-(A) / case-(B) PCG iterations by preconditioner rank r_G and grid (beta = 1, alpha = 1/2)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_09314_b200.binding import DeviceCP, Library, make_params  # noqa: E402
from synth import make_problem  # noqa: E402

L = Library()
for case in ("A", "B"):
    for alpha in (1.0, 0.5):
        for rg in (6, 12, 24):
            row = {}
            for n in (64, 128, 256, 512, 1024):
                p = make_problem("C4", n=n, alpha=alpha, beta=1.0, precond=case)
                ctx = L.context()
                prm = make_params(p.alpha, p.beta, p.eps, p.tol_stop, precond_rank=rg,
                                  precond_case=1 if case == "A" else 0)
                ctx.sl_setup(p.n, p.a_mid, prm)
                u, rep, rc = ctx.pcg_solve(DeviceCP.from_numpy(p.b_w, p.b_U), prm)
                row[n] = rep["iters"] if rc == 0 else f"rc{rc}"
            print(json.dumps({"case": case, "alpha": alpha, "r_G": rg, "iters": row}), flush=True)
