"""D0: dense n^3 x n^3 reference for tiny n (n <= 10).  (Oracle: test-only.)

A = T1 (x) I (x) I + I (x) T2 (x) I + I (x) I (x) T3 [P:449-452] assembled densely,
F(A) = Q F(Lambda) Q^T by a full symmetric eigendecomposition (the spectral definition
of the fractional power [P:261-268, P:363-365]), and u* = F(A)^{-1} b by a direct solve.
Vectorisation is NumPy C-order: index (i, j, k) -> i n2 n3 + j n3 + k.
"""
from __future__ import annotations

import numpy as np

from .sturm import dense_tridiagonal


def dense_A(a_mid, boundary=0) -> np.ndarray:
    T = [dense_tridiagonal(a_mid[l], boundary) for l in range(3)]
    n = [t.shape[0] for t in T]
    I = [np.eye(k) for k in n]
    return (np.kron(np.kron(T[0], I[1]), I[2]) + np.kron(np.kron(I[0], T[1]), I[2])
            + np.kron(np.kron(I[0], I[1]), T[2]))


def dense_fn(A: np.ndarray, f) -> np.ndarray:
    lam, Q = np.linalg.eigh(A)
    return (Q * f(lam)[None, :]) @ Q.T


def dense_solve(A: np.ndarray, f, b: np.ndarray) -> np.ndarray:
    return np.linalg.solve(dense_fn(A, f), b.reshape(-1)).reshape(b.shape)


def dense_pcg(Fm, Gm, b, tol, kmax=100):
    """Textbook dense PCG (for the eps = 0 equivalence pin [S:425])."""
    x = np.zeros_like(b)
    r = b.copy()
    z = Gm @ r
    p = z.copy()
    rz = r @ z
    hist = []
    for k in range(kmax):
        s = Fm @ p
        a = rz / (p @ s)
        x = x + a * p
        r = r - a * s
        hist.append((x.copy(), np.linalg.norm(r) / np.linalg.norm(b)))
        if hist[-1][1] <= tol:
            break
        z = Gm @ r
        rzn = r @ z
        p = z + (rzn / rz) * p
        rz = rzn
    return x, hist
