"""Canonical (CP) tensors and O6 apply, O7 dot, O8 axpy.  (Oracle: test-only.)

CP format [P:1706-1712]: T = sum_k xi_k u_k^(1) (x) u_k^(2) (x) u_k^(3), unit columns,
signed weights; rank 0 is the zero tensor (reading A18).
"""
from __future__ import annotations

from dataclasses import dataclass
import numpy as np


@dataclass
class CP:
    w: np.ndarray            # (R,)
    U: list                  # 3 arrays (n_l, R)

    @property
    def rank(self) -> int:
        return int(self.w.size)

    @property
    def shape(self):
        return tuple(u.shape[0] for u in self.U)

    def copy(self) -> "CP":
        return CP(self.w.copy(), [u.copy() for u in self.U])


def zeros(shape) -> CP:
    return CP(np.zeros(0), [np.zeros((n, 0)) for n in shape])


def normalized(w, U) -> CP:
    """Fold column norms into the weights (unit-column convention [P:1711])."""
    w = np.asarray(w, dtype=np.float64).copy()
    U = [np.array(u, dtype=np.float64, copy=True) for u in U]
    for l in range(3):
        nrm = np.linalg.norm(U[l], axis=0)
        U[l] = U[l] / np.where(nrm > 0, nrm, 1.0)
        w = w * nrm
    return CP(w, U)


def full(x: CP) -> np.ndarray:
    """Dense tensor sum_k xi_k u1_k (x) u2_k (x) u3_k (tiny n only)."""
    return np.einsum("k,ik,jk,lk->ijl", x.w, x.U[0], x.U[1], x.U[2])


def dot(x: CP, y: CP) -> float:
    """O7: <x,y> = sum_{k,m} xi_k zeta_m prod_l <u_k^l, v_m^l> [P:1748-1755]."""
    if x.rank == 0 or y.rank == 0:
        return 0.0
    H = np.ones((x.rank, y.rank))
    for l in range(3):
        H = H * (x.U[l].T @ y.U[l])
    return float(x.w @ H @ y.w)


def norm(x: CP) -> float:
    return float(np.sqrt(max(dot(x, x), 0.0)))


def axpy(x: CP, a: float, y: CP) -> CP:
    """O8: x + a*y by concatenation [x terms ; a*y terms] (ranks add) [P:1845-1866]."""
    return CP(np.concatenate([x.w, a * y.w]),
              [np.concatenate([x.U[l], y.U[l]], axis=1) for l in range(3)])


def scale(a: float, x: CP) -> CP:
    return CP(a * x.w, [u.copy() for u in x.U])


def hadamard(x: CP, y: CP) -> CP:
    """Hadamard product [P:1756-1763]; term t = k*R_y + m (reading A19)."""
    Rx, Ry = x.rank, y.rank
    w = np.outer(x.w, y.w).reshape(-1)
    U = [(x.U[l][:, :, None] * y.U[l][:, None, :]).reshape(x.U[l].shape[0], Rx * Ry)
         for l in range(3)]
    return normalized(w, U)


def apply(V: list, spec: CP, x: CP) -> CP:
    """O6: F(A) x = sum_k sum_j (x)_l G_l^T (u_l^k . G_l x_l^j), G_l = V_l^T [P:614-623].

    Steps per mode (reading A4, A19): W = V^T X (forward transform); Yhat[:, k*R+j] =
    U_F[:, k] * W[:, j] (Khatri-Rao / Hadamard); Y = V Yhat (inverse transform); weights
    w_F[k]*zeta_j; then columns are normalised with norms folded into the weights.
    The output rank is r*R, untruncated [P:615-621].
    """
    if x.rank == 0:
        return zeros(x.shape)
    r, R = spec.rank, x.rank
    U = []
    for l in range(3):
        W = V[l].T @ x.U[l]                                             # S5
        Yh = (spec.U[l][:, :, None] * W[:, None, :]).reshape(-1, r * R)  # S6
        U.append(V[l] @ Yh)                                             # S7
    w = np.outer(spec.w, x.w).reshape(-1)
    return normalized(w, U)                                             # S8
