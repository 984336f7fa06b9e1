"""Algorithm 1 [P:1825-1872] driven from Python through the C-ABI (fracop_apply_truncate,
cp_axpy, cp_truncate, cp_dot) with per-step diagnostics: a_k, b_k, and the error of every
truncation measured against its untruncated input with Gaussian rank-1 probes.
`python tools/diag_pcg_by_hand.py [n] [eps] [kmax]`"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2006_09314_b200.binding import FC_F, FC_G, DeviceCP, Library, make_params  # noqa: E402
from synth import make_problem  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
eps = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-8
kmax = int(sys.argv[3]) if len(sys.argv) > 3 else 6
NP = 32
rng = np.random.default_rng(9)
probes = [rng.standard_normal((n, NP)) for _ in range(3)]


def pv(y: DeviceCP):
    w, U = y.to_numpy()
    P = [U[l].T @ probes[l] for l in range(3)]
    return (w[:, None] * P[0] * P[1] * P[2]).sum(axis=0)


def err(ref, y):
    a, b = pv(ref), pv(y)
    return np.sqrt(np.mean((a - b) ** 2)) / np.sqrt(np.mean(a ** 2))


p = make_problem("C4", n=n, eps=eps)
L = Library()
ctx = L.context()
ctx.sl_setup(p.n, p.a_mid, make_params(p.alpha, p.beta, p.eps, p.tol_stop))
B = DeviceCP.from_numpy(p.b_w, p.b_U)
nB = np.sqrt(ctx.cp_dot(B, B))
R = B
Z, _ = ctx.fracop_apply_truncate(FC_G, R, eps)
print(f"Z0 rank {Z.rank} err {err(ctx.fracop_apply(FC_G, R), Z):.2e}", flush=True)
P = Z
X = None
rz = ctx.cp_dot(R, Z)
for k in range(kmax):
    S, iS = ctx.fracop_apply_truncate(FC_F, P, eps)
    eS = err(ctx.fracop_apply(FC_F, P), S)
    ps = ctx.cp_dot(P, S)
    a = rz / ps
    RS = ctx.cp_axpy(R, -a, S)
    Rn, iR = ctx.cp_truncate(RS, eps)
    eR = err(RS, Rn)
    rr = ctx.cp_dot(Rn, Rn)
    Zn, iZ = ctx.fracop_apply_truncate(FC_G, Rn, eps)
    eZ = err(ctx.fracop_apply(FC_G, Rn), Zn)
    rz_new = ctx.cp_dot(Rn, Zn)
    b = rz_new / rz
    ZP = ctx.cp_axpy(Zn, b, P)
    Pn, iP = ctx.cp_truncate(ZP, eps)
    eP = err(ZP, Pn)
    print(f"k={k} rel_res {np.sqrt(max(rr, 0)) / nB:.4e} a={a:.4e} b={b:.4e} <R,Z>={rz:.4e} <P,S>={ps:.4e} | "
          f"S {S.rank} tk{list(iS.tucker_rank)} err {eS:.1e} | R {Rn.rank} tk{list(iR.tucker_rank)} err {eR:.1e} | "
          f"Z {Zn.rank} err {eZ:.1e} | P {Pn.rank} err {eP:.1e}", flush=True)
    R, Z, P, rz = Rn, Zn, Pn, rz_new
