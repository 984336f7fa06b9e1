import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2006_09314_b200.binding import FC_F, FC_G, Library, make_params  # noqa: E402
from synth import make_problem  # noqa: E402

L = Library()
for n, eps in ((256, 1e-8), (512, 1e-8), (512, 1e-6)):
    p = make_problem("C4", n=n, eps=eps)
    ctx = L.context()
    ctx.sl_setup(p.n, p.a_mid, make_params(p.alpha, p.beta, p.eps, p.tol_stop))
    lams = [ctx.sl_get_eigen(l)[0].cpu().numpy() for l in range(3)]
    g = np.arange(12)
    I, J, K = np.meshgrid(g, g, g, indexing="ij")
    rng = np.random.default_rng(5)
    idx = [np.concatenate([I.ravel(), rng.integers(0, n, 50000)]), np.concatenate([J.ravel(), rng.integers(0, n, 50000)]),
           np.concatenate([K.ravel(), rng.integers(0, n, 50000)])]
    ls = (lams[0][idx[0]] + lams[1][idx[1]]) + lams[2][idx[2]]
    out = []
    for which, f in ((FC_F, lambda l: p.beta * l ** p.alpha + l ** -p.alpha), (FC_G, lambda l: 1 / (p.beta * l ** p.alpha + l ** -p.alpha))):
        w, U = ctx.op_get_spectral_cp(which).to_numpy()
        val = np.einsum("t,st,st,st->s", w, U[0][idx[0]], U[1][idx[1]], U[2][idx[2]])
        ref = f(ls)
        rel = np.abs(val - ref) / ref
        out.append("kind %d rank %d: low max rel %.2e, random max rel %.2e, min value %.3e (exact min %.3e)" % (
            which, len(w), rel[:1728].max(), rel[1728:].max(), val.min(), ref.min()))
    print("n=%d eps=%g | " % (n, eps) + " | ".join(out), flush=True)
