"""Device spectral CPs at C4 (n = 1024) for each eps of the sweep: ranks, max relative error on the
lowest 8^3 modes and on random samples, min values (F~ must stay positive for an SPD operator)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2006_09314_b200.binding import FC_F, FC_G, Library, make_params  # noqa: E402
from synth import make_problem  # noqa: E402

L = Library()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
sinc = "--sinc" in sys.argv
for eps in (1e-6, 1e-7, 1e-8):
    p = make_problem("C4", n=n, eps=eps)
    ctx = L.context()
    ctx.sl_setup(p.n, p.a_mid, make_params(p.alpha, p.beta, p.eps, p.tol_stop))
    if sinc:
        ctx.op_build_spectral_sinc(FC_F, eps)
    lams = [ctx.sl_get_eigen(l)[0].cpu().numpy() for l in range(3)]
    g = np.arange(8)
    I, J, K = np.meshgrid(g, g, g, indexing="ij")
    rng = np.random.default_rng(5)
    m = 200000
    idx = [np.concatenate([I.ravel(), rng.integers(0, n, m)]), np.concatenate([J.ravel(), rng.integers(0, n, m)]),
           np.concatenate([K.ravel(), rng.integers(0, n, m)])]
    ls = (lams[0][idx[0]] + lams[1][idx[1]]) + lams[2][idx[2]]
    out = []
    for which, f in ((FC_F, lambda l: p.beta * l ** p.alpha + l ** -p.alpha),
                     (FC_G, lambda l: 1 / (p.beta * l ** p.alpha + l ** -p.alpha))):
        w, U = ctx.op_get_spectral_cp(which).to_numpy()
        val = np.einsum("t,st,st,st->s", w, U[0][idx[0]], U[1][idx[1]], U[2][idx[2]])
        ref = f(ls)
        rel = np.abs(val - ref) / ref
        out.append("%s rank %d: low max rel %.2e, random max rel %.2e, rms rel %.2e, min %.3e (exact %.3e)" % (
            "F" if which == FC_F else "G", len(w), rel[:512].max(), rel[512:].max(), np.sqrt(np.mean(rel ** 2)),
            val.min(), ref.min()))
    print("n=%d eps=%g%s | " % (n, eps, " sinc" if sinc else "") + " | ".join(out), flush=True)
