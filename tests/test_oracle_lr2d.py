"""Pins of the 2D oracle (oracle/lr2d.py) against closed forms, the
dense Kronecker-sum operator and the paper's 2D iteration table — nothing here re-runs the
oracle's own formulas."""
import numpy as np
import pytest

from oracle import lr2d
from oracle.dense import dense_fn, dense_pcg
from oracle.spectral import FC_F, FC_G, spectral_fn
from oracle.sturm import dense_tridiagonal, eigenpairs
from synth import make_problem2
from synth.configs import midpoints, _coef_c1


def _orth(n, k, seed):
    q, _ = np.linalg.qr(np.random.default_rng(seed).standard_normal((n, k)))
    return q


def test_truncate2_eckart_young():
    """X = Q1 diag(s) Q2^T with s_k = 2^-k (k < 10), stored redundantly (each term split in two
    halves plus a cancelling pair): the reduced SVD keeps the closed-form minimal rank
    r* = min{r : sum_{k>=r} 4^-k <= eps^2 sum 4^-k} and returns the leading r* terms exactly;
    the error is sqrt(tail(r*)) (Eckart-Young, [P:973-976])."""
    n1, n2, K = 20, 15, 10
    s = 2.0 ** -np.arange(K)
    Q1, Q2 = _orth(n1, K, 1), _orth(n2, K, 2)
    v, w = np.random.default_rng(3).standard_normal(n1), np.random.default_rng(4).standard_normal(n2)
    U1 = np.concatenate([Q1, Q1, v[:, None], v[:, None]], axis=1)
    U2 = np.concatenate([Q2, Q2, w[:, None], w[:, None]], axis=1)
    wts = np.concatenate([s / 2, s / 2, [1.0, -1.0]])
    x = lr2d.normalized2(wts, [U1, U2])
    X = (Q1 * s) @ Q2.T
    tot = float(np.sum(s ** 2))
    for eps in (1e-1, 1e-2, 1e-3, 3e-5):
        tails = [float(np.sum(s[r:] ** 2)) for r in range(K + 1)]
        r_star = next(r for r in range(1, K + 1) if tails[r] <= eps * eps * tot)
        y = lr2d.truncate2(x, eps)
        assert y.rank == r_star
        Xr = (Q1[:, :r_star] * s[:r_star]) @ Q2[:, :r_star].T
        assert np.abs(lr2d.full2(y) - Xr).max() < 1e-13
        assert np.linalg.norm(X - lr2d.full2(y)) == pytest.approx(np.sqrt(tails[r_star]), rel=1e-9, abs=1e-14)
        assert np.allclose(y.U[0].T @ y.U[0], np.eye(r_star), atol=1e-13)


def test_truncate2_zero_and_exact_rank():
    x = lr2d.LR2(np.zeros(3), [np.eye(5)[:, :3], np.eye(4)[:, :3]])
    assert lr2d.truncate2(x, 1e-6).rank == 0
    # an exactly rank-2 input keeps 2 terms for any eps below the smaller term's share
    Q1, Q2 = _orth(7, 2, 5), _orth(6, 2, 6)
    y = lr2d.truncate2(lr2d.LR2(np.array([3.0, 1.0]), [Q1, Q2]), 1e-8)
    assert y.rank == 2 and np.allclose(y.w, [3.0, 1.0])


def _dense2(a_mid):
    T = [dense_tridiagonal(a_mid[l]) for l in range(2)]
    n1, n2 = T[0].shape[0], T[1].shape[0]
    return np.kron(T[0], np.eye(n2)) + np.kron(np.eye(n1), T[1])


def test_apply2_equals_dense_operator():
    """apply2 with the exact (full-rank) factorisation of D2 equals F(A) vec(X) with
    A = T1 (x) I + I (x) T2 assembled densely and F(A) from its eigendecomposition
    (the spectral definition [P:261-268]); C-order vec: X[i, j] -> i n2 + j."""
    n = 6
    a_mid = _coef_c1(midpoints(n))[:2]
    lams, V = zip(*[eigenpairs(a_mid[l]) for l in range(2)])
    F = lr2d.spectral2(list(lams), FC_F, 0.5, 0.01, 1e-16, rank=n)
    rng = np.random.default_rng(7)
    x = lr2d.normalized2(np.array([1.0, -0.5, 0.25]), [rng.standard_normal((n, 3)) for _ in range(2)])
    y = lr2d.apply2(list(V), F, x)
    Fd = dense_fn(_dense2(a_mid), spectral_fn(FC_F, 0.5, 0.01))
    ref = (Fd @ lr2d.full2(x).reshape(-1)).reshape(n, n)
    assert np.abs(lr2d.full2(y) - ref).max() <= 1e-11 * np.abs(ref).max()
    assert y.rank == F.rank * x.rank


def test_dot2_equals_dense():
    rng = np.random.default_rng(8)
    x = lr2d.normalized2(rng.standard_normal(4), [rng.standard_normal((9, 4)), rng.standard_normal((7, 4))])
    y = lr2d.normalized2(rng.standard_normal(3), [rng.standard_normal((9, 3)), rng.standard_normal((7, 3))])
    assert lr2d.dot2(x, y) == pytest.approx(float(np.sum(lr2d.full2(x) * lr2d.full2(y))), rel=1e-13)
    z = lr2d.axpy2(x, -2.0, y)
    assert np.abs(lr2d.full2(z) - (lr2d.full2(x) - 2.0 * lr2d.full2(y))).max() < 1e-13


def test_spectral2_rank_one_special_case():
    """lam1 constant: D2[i, j] = F(c + lam2_j) has rank exactly 1 (a closed form); the
    factorisation keeps 1 term and reproduces D2 to rounding."""
    n = 16
    lam2 = eigenpairs(_coef_c1(midpoints(n))[1])[0]
    lam1 = np.full(n, 50.0)
    F = lr2d.spectral2([lam1, lam2], FC_F, 0.5, 0.01, 1e-10)
    assert F.rank == 1
    D = spectral_fn(FC_F, 0.5, 0.01)(lam1[:, None] + lam2[None, :])
    assert np.abs(lr2d.full2(F) - D).max() <= 1e-13 * np.abs(D).max()
    G = lr2d.spectral2([lam1, lam2], FC_G, 0.5, 0.01, 1e-10, rank=1, spd_guard=True)
    assert G.rank == 1 and np.min(lr2d.full2(G)) > 0


def test_spectral2_error_bound_and_guard():
    """Reading 2D-S: ||D2 - F~||_F <= eps_D ||D2||_F; the rank-r_G preconditioner is positive
    on the grid after the guard (A7')."""
    p = make_problem2("D1", n=48)
    st = lr2d.setup2(p)
    D = lr2d.coefficient_matrix(st.lams, FC_F, p.alpha, p.beta)
    assert np.linalg.norm(D - lr2d.full2(st.F)) <= p.eps * np.linalg.norm(D)
    assert st.G.rank >= 6 and np.min(lr2d.full2(st.G)) > 0


def test_pcg2_equals_dense_pcg():
    """With eps -> 0 the rank-structured PCG is textbook PCG on the dense F~, G~ (the same
    residual history) and u solves F~ u = b to the stopping tolerance."""
    p = make_problem2("D1", n=8, eps=1e-13)
    p.tol_stop = 1e-10
    st = lr2d.setup2(p, F_rank=8, G_rank=2, eps_D=1e-13)
    u, rep, _ = lr2d.solve2(p, st)
    Vk = np.kron(st.V[0], st.V[1])
    dF = lr2d.full2(st.F).reshape(-1)
    dG = lr2d.full2(st.G).reshape(-1)
    Fm = (Vk * dF[None, :]) @ Vk.T
    Gm = (Vk * dG[None, :]) @ Vk.T
    b = lr2d.full2(lr2d.normalized2(p.b_w, p.b_U)).reshape(-1)
    x, hist = dense_pcg(Fm, Gm, b, p.tol_stop)
    assert rep["iters"] == len(hist)
    assert np.allclose(rep["rel_res"], [h[1] for h in hist], rtol=1e-6, atol=1e-12)
    ustar = np.linalg.solve(Fm, b)
    assert np.linalg.norm(lr2d.full2(u).reshape(-1) - ustar) <= 1e-8 * np.linalg.norm(ustar)


def test_pcg2_iteration_counts_like_the_paper():
    """Table iter_2d [P:1198-1225] ((A^alpha + A^-alpha) u = y, case-(B) preconditioner):
    2 iterations for alpha = 1/2 at n = 64..1024; the seeded stand-in right-hand side gives
    the same count at n = 64 and 128 (beta = 1 as in the table)."""
    for n in (64, 128):
        p = make_problem2("D1", n=n, beta=1.0)
        _, rep, _ = lr2d.solve2(p)
        assert rep["converged"] and rep["iters"] == 2
