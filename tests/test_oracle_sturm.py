"""Pins for oracle O1-O3 (grid, FD assembly, 1D eigenpairs) against closed forms and
independent routines.  CPU only."""
import os

import numpy as np
import pytest
from scipy.linalg import eigh_tridiagonal

from oracle import sturm
from oracle.dense import dense_A
from synth import make_problem, midpoints

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _golden(name):
    out = {}
    for line in open(os.path.join(GOLD, name)):
        if line.startswith("#") or not line.strip():
            continue
        k, *v = line.split()
        out[k] = [float(x) for x in v]
    return out


def test_n3_spec_example():
    g = _golden("spec_n3_laplace.txt")
    lam, _ = sturm.eigenpairs(np.ones(4))
    assert np.allclose(lam, g["eigenvalues"], atol=g["tol"][0])


@pytest.mark.parametrize("n", [5, 32, 128, 1024])
def test_laplace_closed_form(n):
    """a = 1: lam_k = 4/h^2 sin^2(k pi h/2) [P:781-785]; paper boundary rule is exact here."""
    lam, V = sturm.eigenpairs(np.ones(n + 1))
    ref = sturm.laplace_eigenvalues(n)
    assert np.max(np.abs(lam - ref) / ref) < 1e-13
    if n <= 128:
        S = sturm.dst1_basis(n)
        S = S * np.sign(np.sum(S * V, axis=0))[None, :]      # up to sign (reading A25)
        assert np.max(np.abs(V - S)) < 1e-12


def test_assembly_matches_paper_case_formula():
    """Entries of -(1/h^2)[a_ij] [P:513-519] for a non-constant a, both boundary rules."""
    n = 7
    h = 1.0 / (n + 1)
    a = 1.0 + midpoints(n) ** 2            # a_mid[i] = a_{i+1/2}
    d, e = sturm.tridiagonal(a, boundary=0)
    # interior diagonal a_{i+1/2} + a_{i-1/2}; boundary rows 2 a_{3/2}, 2 a_{n-1/2}
    assert np.isclose(d[0], 2 * a[1] / h**2) and np.isclose(d[-1], 2 * a[n - 1] / h**2)
    for i in range(1, n - 1):               # 0-based row i <-> paper row i+1
        assert np.isclose(d[i], (a[i] + a[i + 1]) / h**2)
    for i in range(n - 1):
        assert np.isclose(e[i], -a[i + 1] / h**2)
    d1, _ = sturm.tridiagonal(a, boundary=1)
    assert np.isclose(d1[0], (a[0] + a[1]) / h**2)
    # T = C^T C with the bidiagonal factor [P:477]
    C = sturm.bidiagonal_factor(a, 0)
    assert np.allclose(C.T @ C, sturm.dense_tridiagonal(a, 0), rtol=1e-14, atol=1e-10)


@pytest.mark.parametrize("c", [0.37, 2.5])
def test_constant_scaling(c):
    lam1, _ = sturm.eigenpairs(np.ones(65))
    lamc, _ = sturm.eigenpairs(c * np.ones(65))
    assert np.max(np.abs(lamc / (c * lam1) - 1)) < 1e-14


@pytest.mark.parametrize("name,n", [("C1", 64), ("C3a", 96)])
def test_eigen_invariants(name, n):
    p = make_problem(name, n=n)
    for l in range(3):
        a = p.a_mid[l]
        lam, V = sturm.eigenpairs(a)
        T = sturm.dense_tridiagonal(a)
        assert np.all(np.diff(lam) > 0)
        assert np.max(np.abs(V.T @ V - np.eye(n))) < 1e-13
        assert np.max(np.abs(T @ V - V * lam[None, :])) < 1e-13 * np.max(lam)
        assert np.all(V[np.argmax(np.abs(V), axis=0), np.arange(n)] > 0)
        # bracketing by the unit-coefficient spectrum [S:223], 1D form of [P:912-916]
        ae = sturm.effective_midpoints(a)
        lap = sturm.laplace_eigenvalues(n)
        assert np.all(lam >= ae.min() * lap * (1 - 1e-13))
        assert np.all(lam <= ae.max() * lap * (1 + 1e-13))
        # independent LAPACK tridiagonal solver (stebz/stemr), index-by-index
        d, e = sturm.tridiagonal(a)
        ref = eigh_tridiagonal(d, e, eigvals_only=True)
        assert np.max(np.abs(lam - ref) / ref) < 1e-10


def test_kronecker_sum_additivity():
    """eig(T1 (+) T2 (+) T3) = {lam1_i + lam2_j + lam3_k} [P:555-561, P:684]."""
    p = make_problem("C1", n=5)
    lams = [sturm.eigenpairs(p.a_mid[l])[0] for l in range(3)]
    ref = np.sort((lams[0][:, None, None] + lams[1][None, :, None] + lams[2][None, None, :]).ravel())
    got = np.linalg.eigvalsh(dense_A(p.a_mid))
    assert np.max(np.abs(got - ref) / ref) < 1e-12


def test_nonpositive_coefficient_rejected():
    a = np.ones(9)
    a[3] = 0.0
    with pytest.raises(ValueError):
        sturm.eigenpairs(a)
