"""Pins of the oracle's state recovery [P:287-289, P:969-972]:
y = beta_paper A^-alpha u, i.e. y = A^-alpha u under reading A5 (beta_paper = 1, gamma = beta).

  * the exact-rank CP of lam^-alpha applied in the SL eigenbasis is the dense A^-alpha (D0);
  * A^alpha A^-alpha = I with exact CPs (SURVEY O6 pin);
  * at the exact solution u* of F(A) u = b the optimality system gives b - y* = beta A^alpha u*
    (algebra of F = beta lam^alpha + lam^-alpha), and the low-rank oracle chain (solve, then state)
    reproduces y* to the PCG/truncation accuracy."""
import numpy as np
import pytest

from oracle import cp as cpm
from oracle import pcg as P
from oracle import spectral as sp
from oracle.dense import dense_A, dense_fn, dense_solve
from synth import make_problem


def _rand_cp(n, R, seed):
    rng = np.random.default_rng(seed)
    return cpm.CP(rng.uniform(0.5, 1.5, R), [rng.standard_normal((n, R)) for _ in range(3)])


def test_exact_pow_minus_is_dense_A_to_minus_alpha():
    p = make_problem("C1", n=5)
    st = P.setup(p)
    Pm = sp.exact_spectral_cp(st.lams, sp.FC_POW_MINUS, p.alpha, p.beta)
    x = _rand_cp(p.n, 2, 1)
    A = dense_A(p.a_mid, p.boundary)
    ref = dense_fn(A, lambda lam: np.power(lam, -p.alpha)) @ cpm.full(x).reshape(-1)
    got = cpm.full(cpm.apply(st.V, Pm, x)).reshape(-1)
    assert np.max(np.abs(got - ref)) <= 1e-13 * np.max(np.abs(ref))


def test_pow_plus_after_pow_minus_is_identity():
    p = make_problem("C3a", n=5)
    st = P.setup(p)
    Pp = sp.exact_spectral_cp(st.lams, sp.FC_POW_PLUS, p.alpha, p.beta)
    Pm = sp.exact_spectral_cp(st.lams, sp.FC_POW_MINUS, p.alpha, p.beta)
    x = _rand_cp(p.n, 2, 2)
    y = cpm.apply(st.V, Pp, cpm.apply(st.V, Pm, x))
    assert np.max(np.abs(cpm.full(y) - cpm.full(x))) <= 1e-12 * np.max(np.abs(cpm.full(x)))


@pytest.mark.parametrize("alpha,beta", [(0.5, 0.01), (0.75, 1.0)])
def test_state_of_the_solution(alpha, beta):
    p = make_problem("C1", n=6, alpha=alpha, beta=beta, eps=1e-9)
    A = dense_A(p.a_mid, p.boundary)
    B = cpm.normalized(p.b_w, p.b_U)
    Bd = cpm.full(B)
    f = sp.spectral_fn(sp.FC_F, p.alpha, p.beta)
    u_star = dense_solve(A, f, Bd)
    y_star = (dense_fn(A, lambda lam: np.power(lam, -p.alpha)) @ u_star.reshape(-1)).reshape(u_star.shape)
    Aa = dense_fn(A, lambda lam: np.power(lam, p.alpha))
    assert np.max(np.abs((Bd - y_star).reshape(-1) - p.beta * Aa @ u_star.reshape(-1))) <= 1e-12 * np.max(np.abs(Bd))
    # the oracle chain: low-rank PCG solve, then the state
    u, rep, st = P.solve(p)
    y = P.state(p, st, u)
    lams = np.concatenate(st.lams)
    kappa = f(lams.max() * 3) / min(f(lams.min() * 3), f(lams.max() * 3), 2 * np.sqrt(p.beta))
    err = np.linalg.norm(cpm.full(y) - y_star) / np.linalg.norm(y_star)
    assert err <= kappa * 10 * p.tol_stop
