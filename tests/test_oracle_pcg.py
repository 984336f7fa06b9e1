"""Pins for oracle O10 (Algorithm 1) against dense PCG / direct solves.  CPU only."""
import numpy as np
import pytest

from oracle import cp as cpm
from oracle import pcg as P
from oracle import spectral as sp
from oracle import sturm
from oracle.dense import dense_A, dense_fn, dense_pcg
from oracle.measure import reldiff
from synth import make_problem


def _setup_exact(p):
    lams, V = [], []
    for l in range(3):
        lam, Vl = sturm.eigenpairs(p.a_mid[l])
        lams.append(lam)
        V.append(Vl)
    return lams, V


def _B(p):
    return cpm.normalized(p.b_w, p.b_U)


def test_identity_operator_one_iteration():
    """[S:420]: fun = precond = I gives 1 iteration with X = B."""
    p = make_problem("C1", n=8)
    B = _B(p)
    ident = lambda x: x.copy()
    X, rep = P.pcg(ident, ident, B, 1e-10, 1e-8)
    assert rep["iters"] == 1 and rep["converged"]
    assert reldiff(X, B) < 1e-12


def test_exact_preconditioner_one_iteration():
    """G = F^{-1} exactly (rank-n^2 CPs): CG converges in one step."""
    p = make_problem("C1", n=5)
    lams, V = _setup_exact(p)
    F = sp.exact_spectral_cp(lams, sp.FC_F, p.alpha, p.beta)
    G = sp.exact_spectral_cp(lams, sp.FC_G, p.alpha, p.beta)
    X, rep = P.pcg(lambda x: cpm.apply(V, F, x), lambda x: cpm.apply(V, G, x), _B(p),
                   1e-12, 1e-9)
    assert rep["iters"] == 1


def test_untruncated_matches_textbook_dense_pcg():
    """eps -> 0 (truncation exact) reproduces dense PCG iterates [S:425]."""
    p = make_problem("C1", n=4)
    lams, V = _setup_exact(p)
    F = sp.exact_spectral_cp(lams, sp.FC_F, p.alpha, p.beta)
    G = sp.spectral_cp(lams, sp.FC_G, p.alpha, p.beta, 1e-6, rank=2, spd_guard=True)
    A = dense_A(p.a_mid)
    Fm = dense_fn(A, sp.spectral_fn(sp.FC_F, p.alpha, p.beta))
    # dense preconditioner = the same rank-2 CP, as a matrix in the eigenbasis
    Q = np.kron(np.kron(V[0], V[1]), V[2])
    Gm = Q @ np.diag(cpm.full(G).ravel()) @ Q.T
    B = _B(p)
    tol = 1e-9
    X, rep = P.pcg(lambda x: cpm.apply(V, F, x), lambda x: cpm.apply(V, G, x), B, 1e-15, tol)
    xd, hist = dense_pcg(Fm, Gm, cpm.full(B).ravel(), tol)
    assert rep["iters"] == len(hist)
    assert np.allclose(rep["rel_res"], [h[1] for h in hist], rtol=1e-6, atol=1e-12)
    assert np.linalg.norm(cpm.full(X).ravel() - xd) <= 1e-10 * np.linalg.norm(xd)


@pytest.mark.parametrize("name", ["C1", "C3b"])
def test_solution_vs_direct_solve(name):
    """Final u vs D0 u* = F(A)^{-1} b at n = 8: within kappa(F)*(eps_D + tol_stop)."""
    p = make_problem(name, n=8)
    u, rep, st = P.solve(p, with_true_residual=True)
    assert rep["converged"]
    A = dense_A(p.a_mid)
    fn = sp.spectral_fn(sp.FC_F, p.alpha, p.beta)
    ustar = np.linalg.solve(dense_fn(A, fn), cpm.full(_B(p)).ravel())
    lam = np.linalg.eigvalsh(A)
    kappa = fn(lam).max() / fn(lam).min()
    err = np.linalg.norm(cpm.full(u).ravel() - ustar) / np.linalg.norm(ustar)
    assert err <= kappa * (p.eps + p.tol_stop) * 3
    assert rep["true_residual"] <= 10 * p.tol_stop


def test_grid_independence_qualitative():
    """Iteration counts vary little with n at fixed alpha, beta ([P:1399-1401], Table iter_3d)."""
    its = []
    for n in (12, 24):
        p = make_problem("C1", n=n)
        _, rep, _ = P.solve(p)
        its.append(rep["iters"])
    assert abs(its[0] - its[1]) <= 2
