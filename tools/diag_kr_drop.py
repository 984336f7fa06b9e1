"""Diagnostic: how much of the eigen-coordinate Khatri-Rao basis K_l = [w_a (.) zhat_b] of an
apply output carries energy below delta (eps/2)^2 E (the truncation cut's resolution)?  Column
(a, b)'s side-matrix coefficient row norm: w_ab^2 = sum_{k,j} (E[a,k] w_F[k])^2 (C_x[b,j] w_x[j])^2
prod_{m != l} n_m(k,j)^2 (n_m: the term's mode-m factor norm).  C4 n=1024 iterate after K iterations.
`python tools/diag_kr_drop.py [K] [eps]`"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402

from _parity import as_cp, device_setup_to_oracle  # noqa: E402
from paper_2006_09314_b200.binding import DeviceCP, Library, make_params  # noqa: E402
from synth import make_problem  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 6
eps = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-6
p = make_problem("C4", n=1024, eps=eps)
prm = make_params(p.alpha, p.beta, p.eps, p.tol_stop, kmax=K)
ctx = Library().context()
st = device_setup_to_oracle(ctx, p, prm)
u, rep, rc = ctx.pcg_solve(DeviceCP.from_numpy(p.b_w, p.b_U), prm)
x = as_cp(u)
F = st.F
for l in range(3):
    # F's Tucker basis W (SVD of the factor matrix), E = W^T U_F; x's basis and coefficients
    Wf, sf, _ = np.linalg.svd(F.U[l], full_matrices=False)
    sF = int(np.sum(sf > 1e-14 * sf[0]))
    Wf = Wf[:, :sF]
    E = Wf.T @ F.U[l]
    Xh = st.V[l].T @ x.U[l]                               # eigen coordinates
    Qx, sx, _ = np.linalg.svd(Xh, full_matrices=False)
    tX = int(np.sum(sx > 1e-14 * sx[0]))
    Qx = Qx[:, :tX]
    Cx = Qx.T @ Xh
    # term norms n_m(k, j) per mode m
    n2 = []
    for m in range(3):
        Xm = st.V[m].T @ x.U[m]
        n2.append((F.U[m] ** 2).T @ (Xm ** 2))            # r x Rx
    P2 = n2[(l + 1) % 3] * n2[(l + 2) % 3]                # prod_{m != l} n_m^2
    A = (E ** 2) * (F.w ** 2)[None, :]                    # s x r
    B = (Cx ** 2) * (x.w ** 2)[None, :]                   # t x Rx
    omega2 = A @ P2 @ B.T                                 # s x t
    Etot = float(np.sum(np.outer(F.w ** 2, x.w ** 2) * n2[0] * n2[1] * n2[2]))
    thr = (eps / 2) ** 2 * Etot
    o = np.sort(omega2.ravel())
    cum = np.cumsum(o)
    for delta in (1e-2, 1e-3, 1e-4):
        ndrop = int(np.searchsorted(cum, delta * thr, side="right"))
        print(f"mode {l}: s={sF} t={tX} cols={o.size} delta={delta:g}: droppable {ndrop} ({ndrop / o.size:.0%})")
