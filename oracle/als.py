"""C2T with ALS refinement: the canonical-to-Tucker algorithm [P:1060,
P:1792-1803] refines the RHOSVD bases by alternating least squares (HOOI) before the
Tucker-to-canonical step.  (Oracle: test-only; imports nothing from the CUDA path.)

Reading ALS (the paper gives the algorithm only by citation [KhKh:06]):
  1. RHOSVD of x (O9 steps 1-4): ranks r_l from the (eps/2)^2 tail rule, initial bases Z_l;
  2. `sweeps` HOOI sweeps, modes l = 0, 1, 2 in order, ranks fixed:
       A_m = Z_m^T U_m (m != l),  W_l = U_l diag(w) (A_a (.) A_b)^T   (n x r_a r_b; (.) = Khatri-Rao),
       Z_l <- the leading r_l left singular vectors of W_l;
     (each step maximises ||x x_1 Z_1^T x_2 Z_2^T x_3 Z_3^T|| over Z_l: the Tucker error is
     non-increasing);
  3. core = x x_l Z_l^T, then T2C with the (eps/2) cut (O9 step 5).
"""
from __future__ import annotations

import numpy as np

from .cp import CP, zeros
from .truncate import rank_cut, tucker_to_canonical


def rhosvd(x: CP, eps: float):
    """O9 steps 1-4 (zero terms dropped): (w, U, Z, ranks)."""
    keep = x.w != 0
    for l in range(3):
        keep &= np.any(x.U[l] != 0, axis=0)
    w = x.w[keep]
    U = [u[:, keep] for u in x.U]
    thr = (eps / 2.0) ** 2 * float(np.sum(w * w))
    Z, ranks = [], []
    for l in range(3):
        Zf, s, _ = np.linalg.svd(U[l] * w[None, :], full_matrices=False)
        r = rank_cut(s ** 2, thr)
        Z.append(Zf[:, :r])
        ranks.append(r)
    return w, U, Z, ranks


def hooi_sweep(w, U, Z):
    """One ALS sweep over l = 0, 1, 2 (ranks fixed)."""
    Z = [z.copy() for z in Z]
    for l in range(3):
        a, b = [m for m in range(3) if m != l]
        Aa, Ab = Z[a].T @ U[a], Z[b].T @ U[b]                    # r_a x R, r_b x R
        KR = (Aa[:, None, :] * Ab[None, :, :]).reshape(-1, w.size)   # (r_a r_b) x R
        W = (U[l] * w[None, :]) @ KR.T                            # n x r_a r_b
        Uf, _, _ = np.linalg.svd(W, full_matrices=False)
        Z[l] = Uf[:, :Z[l].shape[1]]
    return Z


def tucker_core(w, U, Z):
    C = [Z[l].T @ U[l] for l in range(3)]
    return np.einsum("t,at,bt,ct->abc", w, C[0], C[1], C[2])


def c2t_als(x: CP, eps: float, sweeps: int = 2, info: dict | None = None) -> CP:
    if not np.any(x.w != 0):
        return zeros(x.shape)
    w, U, Z, ranks = rhosvd(x, eps)
    if w.size == 0:
        return zeros(x.shape)
    for _ in range(sweeps):
        Z = hooi_sweep(w, U, Z)
    core = tucker_core(w, U, Z)
    if info is not None:
        info["tucker_rank"] = ranks
        info["core_norm2"] = float(np.sum(core * core))
    return tucker_to_canonical(core, Z, eps, info=info)
