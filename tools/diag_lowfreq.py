"""Relative error of the device spectral CPs on the lowest frequencies (i, j, k < 8) vs random."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2006_09314_b200.binding import FC_F, FC_POW_MINUS, FC_POW_PLUS, FC_G, Library, make_params  # noqa: E402
from synth import make_problem  # noqa: E402

L = Library()
for n in (64, 256, 1024):
    p = make_problem("C4", n=n)
    ctx = L.context()
    ctx.sl_setup(p.n, p.a_mid, make_params(p.alpha, p.beta, p.eps, p.tol_stop))
    lams = [ctx.sl_get_eigen(l)[0].cpu().numpy() for l in range(3)]
    g = np.arange(8)
    I, J, K = np.meshgrid(g, g, g, indexing="ij")
    idx = [I.ravel(), J.ravel(), K.ravel()]
    lsum = (lams[0][idx[0]] + lams[1][idx[1]]) + lams[2][idx[2]]
    row = [f"n={n}"]
    for which, f in ((FC_F, lambda l: p.beta * l ** p.alpha + l ** -p.alpha), (FC_POW_PLUS, lambda l: l ** p.alpha),
                     (FC_POW_MINUS, lambda l: l ** -p.alpha)):
        cw, cU = ctx.op_get_spectral_cp(which).to_numpy()
        val = np.einsum("t,st,st,st->s", cw, cU[0][idx[0]], cU[1][idx[1]], cU[2][idx[2]])
        ref = f(lsum)
        row.append(f"kind {which}: low-freq max rel err {np.max(np.abs(val - ref) / np.abs(ref)):.2e}")
    print(" | ".join(row), flush=True)
