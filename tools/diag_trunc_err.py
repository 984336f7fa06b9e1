"""Truncation error at C4 size, measured with Gaussian rank-1 probes (no cancellation floor):
for y0 = F x (untruncated) and y = trunc(F x), e = y0 - y,  E[<e, g1 (x) g2 (x) g3>^2] = ||e||^2
for iid N(0,1) probes g.  Prints ||e|| / ||y0|| for the fused (eigen-coordinate, structured)
route and the CP route (cp_truncate of the untruncated apply), per eps.
`python tools/diag_trunc_err.py [n] [iters]` (iters: also the R/Z/P/S iterates of the first PCG
iterations via kmax)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2006_09314_b200.binding import FC_F, FC_G, DeviceCP, Library, make_params  # noqa: E402
from synth import make_problem  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
NP = 24
rng = np.random.default_rng(7)
probes = [rng.standard_normal((n, NP)) for _ in range(3)]


def probe_vals(y: DeviceCP):
    w, U = y.to_numpy()
    P = [U[l].T @ probes[l] for l in range(3)]          # R x NP
    return (w[:, None] * P[0] * P[1] * P[2]).sum(axis=0)


def rel_err(y_ref: DeviceCP, y: DeviceCP):
    a, b = probe_vals(y_ref), probe_vals(y)
    return float(np.sqrt(np.mean((a - b) ** 2)) / np.sqrt(np.mean(a ** 2)))


L = Library()
for eps in (1e-6, 1e-7, 1e-8):
    p = make_problem("C4", n=n, eps=eps)
    ctx = L.context()
    ctx.sl_setup(p.n, p.a_mid, make_params(p.alpha, p.beta, p.eps, p.tol_stop))
    b = DeviceCP.from_numpy(p.b_w, p.b_U)
    rows = []
    for which, name in ((FC_G, "G"), (FC_F, "F")):
        y0 = ctx.fracop_apply(which, b)
        y1, i1 = ctx.fracop_apply_truncate(which, b, eps)
        y2, i2 = ctx.cp_truncate(y0, eps)
        rows.append(f"{name}b: apply rank {y0.rank} | fused -> {y1.rank} (tucker {list(i1.tucker_rank)}) err {rel_err(y0, y1):.2e}"
                    f" | cp -> {y2.rank} (tucker {list(i2.tucker_rank)}) err {rel_err(y0, y2):.2e}")
        # second level: apply to the truncated output (the next iterate's shape)
        z0 = ctx.fracop_apply(which, y1)
        z1, j1 = ctx.fracop_apply_truncate(which, y1, eps)
        z2, j2 = ctx.cp_truncate(z0, eps)
        rows.append(f"{name}{name}b: apply rank {z0.rank} | fused -> {z1.rank} (tucker {list(j1.tucker_rank)}) err {rel_err(z0, z1):.2e}"
                    f" | cp -> {z2.rank} (tucker {list(j2.tucker_rank)}) err {rel_err(z0, z2):.2e}")
        torch.cuda.synchronize()
    print(f"n={n} eps={eps:g}\n  " + "\n  ".join(rows), flush=True)
