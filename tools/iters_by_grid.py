"""PCG iterations of the C4 workload by grid, preconditioner case and alpha (the paper's Table
iter_3d / iternums_precond_3d setting: beta = 1, eps = 1e-6, rank-6 preconditioner)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_09314_b200.binding import DeviceCP, Library, make_params  # noqa: E402
from synth import make_problem  # noqa: E402

L = Library()
for case in ("A", "B"):
    for alpha in (1.0, 0.5, 0.1):
        row = {}
        for n in (64, 128, 256, 512, 1024):
            p = make_problem("C4", n=n, alpha=alpha, beta=1.0, precond=case)
            ctx = L.context()
            prm = make_params(p.alpha, p.beta, p.eps, p.tol_stop, precond_case=1 if case == "A" else 0)
            ctx.sl_setup(p.n, p.a_mid, prm)
            u, rep, rc = ctx.pcg_solve(DeviceCP.from_numpy(p.b_w, p.b_U), prm)
            row[n] = rep["iters"] if rc == 0 else f"rc{rc}"
        print(json.dumps({"case": case, "alpha": alpha, "beta": 1.0, "iters": row}), flush=True)
