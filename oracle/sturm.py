"""O1-O3: grid, 1D Sturm-Liouville FD operator and its eigenpairs.  (Oracle: test-only.)

Paper: Section "Finite difference scheme" [P:443-519] and "Stiffness matrix in the
low-rank Kronecker form" [P:524-561].  Readings: A1 (h = 1/(n+1)), A2 (paper
boundary rule), A3 (SPD sign), A4 (T = V diag(lam) V^T, columns of V are eigenvectors,
lam ascending; sign rule: the entry of largest magnitude of each column is positive, ties
-> lowest index.  SURVEY's V[0, j] > 0 is ill-posed here: for strongly varying a (C3) the
first component underflows to exactly 0).
"""
from __future__ import annotations

import numpy as np


def effective_midpoints(a_mid: np.ndarray, boundary: int = 0) -> np.ndarray:
    """Midpoint coefficients entering the weak form [P:471-480].

    a_mid[i] = a((i+1/2)h), i = 0..n.  The paper's case formula [P:513-519] puts
    -2 a_{3/2} and -2 a_{n-1/2} on the boundary diagonals, i.e. (reading A2) the outer
    midpoint values are replaced: a~_{1/2} := a_{3/2}, a~_{n+1/2} := a_{n-1/2}.
    boundary=1 keeps the standard a_{1/2}, a_{n+1/2}.
    """
    a = np.array(a_mid, dtype=np.float64, copy=True)
    if not np.all(np.isfinite(a)) or np.any(a <= 0):
        raise ValueError("NONPOS_COEF: midpoint coefficient <= 0 or non-finite")
    if boundary == 0:
        a[0] = a[1]
        a[-1] = a[-2]
    return a


def bidiagonal_factor(a_mid: np.ndarray, boundary: int = 0) -> np.ndarray:
    """O2: the (n+1) x n weighted difference matrix C with T = C^T C [P:477].

    Row r (0-based, r = 0..n) is sqrt(a~_{r+1/2}) (y_{r+1} - y_r)/h with y_0 = y_{n+1} = 0
    [P:469]; column c holds y_{c+1}.
    """
    a = effective_midpoints(a_mid, boundary)
    n = a.size - 1
    h = 1.0 / (n + 1)
    C = np.zeros((n + 1, n))
    s = np.sqrt(a) / h
    for r in range(n + 1):
        if r <= n - 1:
            C[r, r] = s[r]
        if r >= 1:
            C[r, r - 1] = -s[r]
    return C


def tridiagonal(a_mid: np.ndarray, boundary: int = 0):
    """(d, e) of the SPD tridiagonal T = -(1/h^2)[a_ij] of [P:491-519] (sign: reading A3).

    1-based: d_i = (a~_{i-1/2} + a~_{i+1/2})/h^2, e_i = -a~_{i+1/2}/h^2.
    """
    a = effective_midpoints(a_mid, boundary)
    n = a.size - 1
    h2 = (1.0 / (n + 1)) ** 2
    d = (a[:-1] + a[1:]) / h2
    e = -a[1:-1] / h2
    return d, e


def dense_tridiagonal(a_mid, boundary=0):
    d, e = tridiagonal(a_mid, boundary)
    return np.diag(d) + np.diag(e, 1) + np.diag(e, -1)


def eigenpairs(a_mid: np.ndarray, boundary: int = 0):
    """O3: lam (ascending), V (n x n, column j = eigenvector j, max-|.| entry > 0) [P:532-542].

    lam = sigma(C)^2 and V = right singular vectors of C (LAPACK gesdd), which is the
    paper's own weak-form factorisation T = C^T C [P:477].
    """
    C = bidiagonal_factor(a_mid, boundary)
    _, s, Vt = np.linalg.svd(C, full_matrices=False)
    order = np.argsort(s)                      # ascending lambda
    lam = s[order] ** 2
    V = Vt[order].T.copy()
    piv = np.argmax(np.abs(V), axis=0)
    V *= np.sign(V[piv, np.arange(V.shape[1])])[None, :]
    return lam, V


def laplace_eigenvalues(n: int) -> np.ndarray:
    """Closed form 4/h^2 sin^2(k pi h/2), k = 1..n [P:781-785] (sign per reading A3)."""
    h = 1.0 / (n + 1)
    k = np.arange(1, n + 1)
    return 4.0 / h**2 * np.sin(k * np.pi * h / 2.0) ** 2


def dst1_basis(n: int) -> np.ndarray:
    """Orthonormal sine (DST-I) eigenbasis of the 1D Dirichlet Laplacian [P:778-780]."""
    h = 1.0 / (n + 1)
    i = np.arange(1, n + 1)
    return np.sqrt(2.0 * h) * np.sin(np.outer(i, i) * np.pi * h)
