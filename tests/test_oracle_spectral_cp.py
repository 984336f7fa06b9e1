"""Pins for oracle O4-O9 (spectral CP, apply, dot, truncation) against the dense D0
reference, closed forms and invariants.  CPU only."""
import os

import numpy as np
import pytest

from oracle import cp as cpm
from oracle import spectral as sp
from oracle import sturm
from oracle.dense import dense_A, dense_fn
from oracle.measure import reldiff
from oracle.truncate import truncate, rank_cut, tail_sums
from synth import make_problem, random_cp

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _eig(p):
    lams, V = [], []
    for l in range(3):
        lam, Vl = sturm.eigenpairs(p.a_mid[l])
        lams.append(lam)
        V.append(Vl)
    return lams, V


def _rand(n, R, seed):
    w, U = random_cp(n, R, seed)
    return cpm.CP(np.random.default_rng(seed + 100).uniform(0.5, 1.5, R) * w, U)


# ---- O4 -------------------------------------------------------------------------------

def test_spec_entry_alpha1():
    """[S:271]: alpha=1, beta=gamma=1: F(3*9.3726) = 28.1533 (eq. [P:693])."""
    g = {}
    for line in open(os.path.join(GOLD, "spec_n3_laplace.txt")):
        if not line.startswith("#") and line.strip():
            k, *v = line.split()
            g[k] = float(v[0])
    lam, _ = sturm.eigenpairs(np.ones(4))
    D = sp.coefficient_tensor([lam, lam, lam], sp.FC_F, 1.0, 1.0)
    assert abs(D[0, 0, 0] - g["f_entry_111_alpha1"]) < g["f_tol"]


def test_spectral_functions():
    lam = np.array([0.5, 1.0, 7.0])
    a, b = 0.3, 0.2
    F = sp.spectral_fn(sp.FC_F, a, b)(lam)
    assert np.allclose(F, b * lam**a + lam**(-a), rtol=1e-15)
    assert np.allclose(sp.spectral_fn(sp.FC_G, a, b)(lam) * F, 1.0, rtol=1e-15)
    assert np.allclose(sp.spectral_fn(sp.FC_POW_PLUS, a, b)(lam) *
                       sp.spectral_fn(sp.FC_POW_MINUS, a, b)(lam), 1.0, rtol=1e-15)
    assert F[1] == pytest.approx(b + 1.0)


# ---- O5 -------------------------------------------------------------------------------

def test_lambda_tensor_is_tucker_222_rank3():
    """F(lam) = lam: D_A = lam1 (+) lam2 (+) lam3 has Tucker ranks (2,2,2) [P:670-674, P:752]."""
    p = make_problem("C1", n=12)
    lams, _ = _eig(p)
    info = {}
    x = sp.spectral_cp(lams, sp.FC_LAMBDA, 0.5, 0.01, 1e-10, info=info)
    assert info["tucker_rank"] == [2, 2, 2]
    assert x.rank <= 4                                      # T2C of a 2x2x2 core: <= 2*2
    assert info["max_abs_err"] <= 1e-13 * info["max_F"] * 100


def test_alpha_to_zero_rank1():
    """alpha -> 0: F -> (beta + 1) * 1, rank 1 ([P:1512-1519] mapped)."""
    p = make_problem("C1", n=10)
    lams, _ = _eig(p)
    x = sp.spectral_cp(lams, sp.FC_F, 1e-9, 0.01, 1e-6)
    assert x.rank == 1
    assert np.allclose(cpm.full(x), 1.01, rtol=1e-6)


@pytest.mark.parametrize("eps", [1e-4, 1e-6])
def test_spectral_cp_entries_and_monotone_rank(eps):
    p = make_problem("C1", n=24)
    lams, _ = _eig(p)
    info = {}
    sp.spectral_cp(lams, sp.FC_F, p.alpha, p.beta, eps, info=info)
    # HOSVD bound sum_l tail_l <= 3 (eps^2/3)||D||^2 plus the T2C cut (eps/2)^2||core||^2
    assert info["fro_rel_err"] <= np.sqrt(1.25) * eps
    info2 = {}
    sp.spectral_cp(lams, sp.FC_F, p.alpha, p.beta, eps / 100, info=info2)
    assert info2["rank"] >= info["rank"]
    assert all(a >= b for a, b in zip(info2["tucker_rank"], info["tucker_rank"]))


def test_preconditioner_spd_guard():
    """C3b's alpha=0.75, beta=0.1 is the stiff case; the guarded rank-6 G is positive."""
    p = make_problem("C3b", n=20)
    lams, _ = _eig(p)
    G = sp.spectral_cp(lams, sp.FC_G, p.alpha, p.beta, p.eps, rank=6, spd_guard=True)
    assert G.rank >= 6
    assert sp.cp_min_entry(G) > 0


# ---- O6 apply ---------------------------------------------------------------------------

def test_apply_matches_dense_D0():
    """Factored apply with the exact (rank n^2) spectral CP equals dense F(A)x [P:600-621]."""
    p = make_problem("C1", n=6)
    lams, V = _eig(p)
    A = dense_A(p.a_mid)
    x = _rand(6, 3, 7)
    for kind in (sp.FC_F, sp.FC_G, sp.FC_POW_PLUS):
        spec = sp.exact_spectral_cp(lams, kind, p.alpha, p.beta)
        y = cpm.apply(V, spec, x)
        assert y.rank == spec.rank * x.rank
        ref = dense_fn(A, sp.spectral_fn(kind, p.alpha, p.beta)) @ cpm.full(x).ravel()
        got = cpm.full(y).ravel()
        assert np.linalg.norm(got - ref) / np.linalg.norm(ref) < 1e-13


def test_apply_invariants():
    p = make_problem("C1", n=8)
    lams, V = _eig(p)
    x, y = _rand(8, 3, 1), _rand(8, 2, 2)
    spec = sp.exact_spectral_cp(lams, sp.FC_F, p.alpha, p.beta)
    # symmetry <Fx, y> = <x, Fy>
    a = cpm.dot(cpm.apply(V, spec, x), y)
    b = cpm.dot(x, cpm.apply(V, spec, y))
    assert abs(a - b) <= 1e-13 * abs(a)
    # identity CP (F = 1): apply(x) = x
    one = sp.exact_spectral_cp(lams, sp.FC_ONE, p.alpha, p.beta)
    assert reldiff(cpm.apply(V, one, x), x) < 1e-13
    # POW+ o POW- = I with exact CPs
    pp = sp.exact_spectral_cp(lams, sp.FC_POW_PLUS, p.alpha, p.beta)
    pm = sp.exact_spectral_cp(lams, sp.FC_POW_MINUS, p.alpha, p.beta)
    z = cpm.apply(V, pp, cpm.apply(V, pm, x))
    assert np.linalg.norm(cpm.full(z) - cpm.full(x)) / np.linalg.norm(cpm.full(x)) < 1e-12


# ---- O7 dot / O8 axpy / O12 -----------------------------------------------------------------

def test_dot_and_axpy_dense():
    x, y = _rand(9, 4, 3), _rand(9, 5, 4)
    X, Y = cpm.full(x), cpm.full(y)
    assert abs(cpm.dot(x, y) - np.sum(X * Y)) < 1e-13 * np.linalg.norm(X) * np.linalg.norm(Y)
    assert abs(cpm.dot(x, y)) <= cpm.norm(x) * cpm.norm(y) * (1 + 1e-12)
    z = cpm.axpy(x, -0.7, y)
    assert np.allclose(cpm.full(z), X - 0.7 * Y, atol=1e-14)
    h = cpm.hadamard(x, y)
    assert np.allclose(cpm.full(h), X * Y, atol=1e-14)
    assert abs(reldiff(z, z)) < 1e-14
    assert reldiff(x, y) == pytest.approx(np.linalg.norm(X - Y) / np.linalg.norm(Y), rel=1e-10)


# ---- O9 truncation ---------------------------------------------------------------------------

def test_tail_and_rank_cut():
    s2 = np.array([1.0, 1e-3, 1e-6, 1e-9, 1e-12])
    t = tail_sums(s2)
    assert t[5] == 0 and t[4] == 1e-12 and t[0] == pytest.approx(np.sum(s2))
    assert rank_cut(s2, 2e-9) == 3          # tail after 3 = 1e-9 + 1e-12 <= 2e-9
    assert rank_cut(s2, 1e-10) == 4
    assert rank_cut(np.array([1.0, 0.5, 0.5, 1e-20]), 0.3) == 3   # tie kept together


def test_truncate_duplicates_collapse():
    x = _rand(10, 2, 5)
    d = cpm.CP(np.concatenate([x.w, x.w]), [np.concatenate([u, u], axis=1) for u in x.U])
    info = {}
    y = truncate(d, 1e-8, info)
    assert info["tucker_rank"] == [2, 2, 2]
    assert np.linalg.norm(cpm.full(y) - 2 * cpm.full(x)) <= 1e-12 * np.linalg.norm(cpm.full(x))


@pytest.mark.parametrize("eps", [1e-2, 1e-4, 1e-6])
def test_truncate_error_bound_and_orthogonality(eps):
    p = make_problem("C1", n=16)
    lams, V = _eig(p)
    F = sp.spectral_cp(lams, sp.FC_F, p.alpha, p.beta, 1e-8)
    x = cpm.apply(V, F, _rand(16, 3, 9))                  # a realistic apply output
    y = truncate(x, eps)
    X, Y = cpm.full(x), cpm.full(y)
    assert np.linalg.norm(X - Y) <= eps * np.linalg.norm(x.w)     # RHOSVD bound vs ||xi||
    assert y.rank <= x.rank
    # orthogonal CP: xi^T (G1 o G2 o G3) xi = sum xi^2
    assert cpm.dot(y, y) == pytest.approx(np.sum(y.w ** 2), rel=1e-12)
    # idempotence (up to the second cut)
    z = truncate(y, eps)
    assert np.linalg.norm(cpm.full(z) - Y) <= eps * np.linalg.norm(Y)


def test_truncate_zero_and_weights():
    x = _rand(6, 3, 11)
    x.w[:] = 0
    assert truncate(x, 1e-6).rank == 0
