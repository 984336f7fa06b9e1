"""True residual ||b - F~ X_k|| / ||b|| of the PCG iterate after k iterations (pcg_solve with
kmax = k), against the recursively updated ||R_k|| / ||b|| the solver reports.  The true residual
uses the untruncated apply and Gaussian rank-1 probes (no cancellation floor).
`python tools/diag_true_res.py [n] [eps] [kmax]`"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2006_09314_b200.binding import FC_F, DeviceCP, Library, make_params  # noqa: E402
from synth import make_problem  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
eps = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-8
kmax = int(sys.argv[3]) if len(sys.argv) > 3 else 4
NP = 32
rng = np.random.default_rng(9)
probes = [rng.standard_normal((n, NP)) for _ in range(3)]


def pv(y: DeviceCP):
    w, U = y.to_numpy()
    P = [U[l].T @ probes[l] for l in range(3)]
    return (w[:, None] * P[0] * P[1] * P[2]).sum(axis=0)


p = make_problem("C4", n=n, eps=eps)
L = Library()
ctx = L.context()
ctx.sl_setup(p.n, p.a_mid, make_params(p.alpha, p.beta, p.eps, p.tol_stop))
b = DeviceCP.from_numpy(p.b_w, p.b_U)
pb = pv(b)
nb = np.sqrt(np.mean(pb ** 2))
for k in range(1, kmax + 1):
    prm = make_params(p.alpha, p.beta, p.eps, p.tol_stop, kmax=k)
    u, rep, rc = ctx.pcg_solve(b, prm)
    fu = ctx.fracop_apply(FC_F, u)
    tr = np.sqrt(np.mean((pb - pv(fu)) ** 2)) / nb
    print(f"n={n} eps={eps:g} k={k}: reported rel_res {rep['rel_res'][-1]:.4e}  true {tr:.4e}  rank_X {u.rank}", flush=True)
