"""Small cases for compute-sanitizer (racecheck / synccheck / memcheck): smoke() (C1 n = 16 solve
through the C-ABI) and fc_syev at N = 600 (the 16-CTA cluster tridiagonalisation) plus N = 80
(packed path) and N = 1000 (global path).  `python tools/sanitize_case.py [smoke|syev|all]`"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "all"
if what in ("smoke", "all"):
    from paper_2006_09314_b200.binding import DeviceCP, Library, make_params
    from synth import make_problem
    p = make_problem("C1", n=16)
    ctx = Library().context()
    prm = make_params(p.alpha, p.beta, p.eps, p.tol_stop)
    ctx.sl_setup(p.n, p.a_mid, prm)
    u, rep, rc = ctx.pcg_solve(DeviceCP.from_numpy(p.b_w, p.b_U), prm)
    assert rc == 0, rc
    print("smoke solve ok", rep["iters"], flush=True)
if what in ("syev", "all"):
    from paper_2006_09314_b200.binding import Library
    ctx = Library().context()
    for N in (80, 600, 1000):
        rng = np.random.default_rng(N)
        A = rng.standard_normal((N, N))
        M = A @ A.T / N
        (lam, Y), = ctx.syev([torch.tensor(M, device="cuda")], [min(N, 64)])
        torch.cuda.synchronize()
        ref = np.linalg.eigvalsh(M)[::-1]
        err = float(np.max(np.abs(lam.cpu().numpy()[:N] - ref)))
        print(f"syev N={N} max eig err {err:.2e}", flush=True)
