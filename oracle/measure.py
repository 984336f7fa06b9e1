"""O12 reldiff(x, y) = ||x - y|| / ||y|| in a common orthonormal basis.  (Oracle: test-only.)

The inner-product identity ||x-y||^2 = <x,x> - 2<x,y> + <y,y> floors at ~1e-8 relative,
so per mode a Householder QR of [U_x, U_y] gives Q_l, both tensors are projected to dense
cores and the difference is taken there (floor ~ eps * sqrt(R_x + R_y)).
"""
from __future__ import annotations

import numpy as np

from .cp import CP, dot


def _core(x: CP, Q: list) -> np.ndarray:
    C = [Q[l].T @ x.U[l] for l in range(3)]
    return np.einsum("t,at,bt,ct->abc", x.w, C[0], C[1], C[2])


def diff_norm(x: CP, y: CP, max_core: int = 2 ** 26) -> float:
    if x.rank == 0 and y.rank == 0:
        return 0.0
    Q = [np.linalg.qr(np.concatenate([x.U[l], y.U[l]], axis=1))[0] for l in range(3)]
    if np.prod([q.shape[1] for q in Q]) > max_core:
        v = dot(x, x) - 2 * dot(x, y) + dot(y, y)
        return float(np.sqrt(max(v, 0.0)))
    return float(np.linalg.norm(_core(x, Q) - _core(y, Q)))


def reldiff(x: CP, y: CP) -> float:
    ny = float(np.sqrt(max(dot(y, y), 0.0)))
    return diff_norm(x, y) / ny
