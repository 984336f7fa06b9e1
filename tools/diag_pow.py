"""Consistency of the spectral CPs F, lam^alpha, lam^-alpha (F = beta lam^a + lam^-a) on the device."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2006_09314_b200.binding import FC_F, FC_POW_MINUS, FC_POW_PLUS, DeviceCP, Library, make_params  # noqa: E402
from synth import make_problem, random_cp  # noqa: E402

L = Library()
for n in (64, 256, 1024):
    p = make_problem("C4", n=n)
    ctx = L.context()
    ctx.sl_setup(p.n, p.a_mid, make_params(p.alpha, p.beta, p.eps, p.tol_stop))
    w, U = random_cp(n, 2, 3)
    x = DeviceCP.from_numpy(np.array([1.0, 0.7]), U)
    Fx = ctx.fracop_apply(FC_F, x)
    Px = ctx.fracop_apply(FC_POW_PLUS, x)
    Mx = ctx.fracop_apply(FC_POW_MINUS, x)
    z = ctx.cp_axpy(ctx.cp_axpy(Fx, -p.beta, Px), -1.0, Mx)
    rel = math.sqrt(max(ctx.cp_dot(z, z), 0) / ctx.cp_dot(Fx, Fx))
    lams = [ctx.sl_get_eigen(l)[0].cpu().numpy() for l in range(3)]
    rng = np.random.default_rng(1)
    idx = rng.integers(0, n, size=(3, 20000))
    lsum = (lams[0][idx[0]] + lams[1][idx[1]]) + lams[2][idx[2]]
    out = [f"n={n} ||Fx - b P+x - P-x||/||Fx|| = {rel:.2e}"]
    for which, f in ((FC_F, lambda l: p.beta * l ** p.alpha + l ** -p.alpha), (FC_POW_PLUS, lambda l: l ** p.alpha),
                     (FC_POW_MINUS, lambda l: l ** -p.alpha)):
        cw, cU = ctx.op_get_spectral_cp(which).to_numpy()
        val = np.einsum("t,st,st,st->s", cw, cU[0][idx[0]], cU[1][idx[1]], cU[2][idx[2]])
        ref = f(lsum)
        r, tk = ctx.op_spectral_rank(which)
        out.append(f"kind {which}: rank {r} tucker {tk} rms rel err {math.sqrt(np.mean((val - ref) ** 2) / np.mean(ref ** 2)):.2e} max rel {np.max(np.abs(val - ref) / np.abs(ref)):.2e}")
    print(" | ".join(out), flush=True)
