"""Full-grid spectrum of the preconditioned operator.  F~ and G~ are diagonal in the same
eigenbasis (case B), so G~F~ has the eigenvalues G~_ijk F~_ijk exactly: min / max over all n^3
grid points give kappa(G~F~) and show any indefiniteness (F~ <= 0 or G~ <= 0 somewhere).
Slices k = 0..n-1: F~[:, :, k] = U0 diag(w U2[k, :]) U1^T (torch GEMMs on the GPU; diagnostic
only, not the product path).  `python tools/diag_precond_spectrum.py [n] [eps ...]`"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2006_09314_b200.binding import FC_F, FC_G, Library, make_params  # noqa: E402
from synth import make_problem  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
epss = [float(x) for x in sys.argv[2:]] or [1e-6, 1e-7, 1e-8]
L = Library()
for eps in epss:
    p = make_problem("C4", n=n, eps=eps)
    ctx = L.context()
    ctx.sl_setup(p.n, p.a_mid, make_params(p.alpha, p.beta, p.eps, p.tol_stop))
    lam = [ctx.sl_get_eigen(l)[0] for l in range(3)]
    cps = {}
    for which in (FC_F, FC_G):
        y = ctx.op_get_spectral_cp(which)
        R = y.rank
        cps[which] = (y.w[:R].clone(), [y.U[l][:R].T.contiguous() for l in range(3)])
    st = {k: [float("inf"), -float("inf")] for k in ("F/Fex", "G*Fex", "G*F", "F", "G")}
    l12 = lam[0][:, None] + lam[1][None, :]
    for k in range(n):
        Fex = p.beta * (l12 + lam[2][k]) ** p.alpha + (l12 + lam[2][k]) ** -p.alpha
        sl = {}
        for which in (FC_F, FC_G):
            w, U = cps[which]
            sl[which] = (U[0] * (w * U[2][k])[None, :]) @ U[1].T
        vals = {"F/Fex": sl[FC_F] / Fex, "G*Fex": sl[FC_G] * Fex, "G*F": sl[FC_G] * sl[FC_F], "F": sl[FC_F],
                "G": sl[FC_G]}
        for key, v in vals.items():
            st[key][0] = min(st[key][0], float(v.min()))
            st[key][1] = max(st[key][1], float(v.max()))
    kap = st["G*F"][1] / st["G*F"][0] if st["G*F"][0] > 0 else float("inf")
    print(f"n={n} eps={eps:g} rF={cps[FC_F][0].numel()} rG={cps[FC_G][0].numel()} | " +
          " | ".join(f"{k} [{a:.4e}, {b:.4e}]" for k, (a, b) in st.items()) + f" | kappa(G~F~)={kap:.3e}", flush=True)
