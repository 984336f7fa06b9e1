"""O12 reldiff(x, y) = ||x - y|| / ||y|| in a common orthonormal basis.  (Oracle: test-only.)

The inner-product identity ||x-y||^2 = <x,x> - 2<x,y> + <y,y> floors at ~1e-8 relative, so the
difference is taken between dense cores in a common orthonormal basis per mode (floor ~ eps *
sqrt(R_x + R_y)).  The basis is the left singular vectors of the weighted factors
[U_x |w_x|, U_y |w_y|] above 1e-15 of the largest singular value: the span is that of the factors
(up to parts carrying < 1e-15 of the largest weighted column), so it stays small for low-rank
Tucker-structured tensors (truncation outputs at n = 1024: ~100 per mode instead of min(n, R_x +
R_y)), and the core path applies at every size the tests use.
"""
from __future__ import annotations

import numpy as np

from .cp import CP, dot

BASIS_CUT = 1e-15


def _basis(x: CP, y: CP, l: int) -> np.ndarray:
    A = np.concatenate([x.U[l] * np.abs(x.w)[None, :], y.U[l] * np.abs(y.w)[None, :]], axis=1)
    U, s, _ = np.linalg.svd(A, full_matrices=False)
    k = int(np.sum(s > BASIS_CUT * s[0])) if s.size and s[0] > 0 else 0
    return U[:, :max(k, 1)]


def _core(x: CP, Q: list) -> np.ndarray:
    """sum_t w_t (Q0^T u0_t) (x) (Q1^T u1_t) (x) (Q2^T u2_t), as one matrix product."""
    C = [Q[l].T @ x.U[l] for l in range(3)]
    kr = (C[1][:, None, :] * C[2][None, :, :]).reshape(-1, x.rank)      # Khatri-Rao (b, c) x t
    return ((C[0] * x.w[None, :]) @ kr.T).reshape(C[0].shape[0], C[1].shape[0], C[2].shape[0])


def diff_norm(x: CP, y: CP, max_core: int = 2 ** 26) -> float:
    if x.rank == 0 and y.rank == 0:
        return 0.0
    if x.rank == 0 or y.rank == 0:
        z = y if x.rank == 0 else x
        return float(np.sqrt(max(dot(z, z), 0.0)))
    Q = [_basis(x, y, l) for l in range(3)]
    if np.prod([q.shape[1] for q in Q]) > max_core:
        v = dot(x, x) - 2 * dot(x, y) + dot(y, y)
        return float(np.sqrt(max(v, 0.0)))
    return float(np.linalg.norm(_core(x, Q) - _core(y, Q)))


def reldiff(x: CP, y: CP) -> float:
    ny = float(np.sqrt(max(dot(y, y), 0.0)))
    return diff_norm(x, y) / ny
