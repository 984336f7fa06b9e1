"""Pins of the truncation thresholds (reading A11/A12: per-mode cut (eps/2)^2 sum xi^2, T2C cut
(eps/2)^2 ||beta||^2) and of the rank cap (reading A26), on orthogonally decomposable tensors
where every quantity has a closed form.

x = sum_k s_k e_k (x) e_k (x) e_k (orthonormal e_k; canonical terms mutually orthogonal):
  * each mode's side matrix U_l diag(xi) has singular values exactly s_k;
  * the Tucker core in the kept bases is diag(s_1..s_r), its slices have the single singular
    values s_k, so T2C keeps terms by the same tail rule;
  * the truncation error is exactly sqrt(sum of the dropped s_k^2) (Pythagoras).
The tails are placed between (eps/2)^2 E and eps^2 E, so the (eps/2) constant and a plain eps^2
reading give different ranks and different errors: a swapped constant fails here even though it
keeps ||x - trunc x|| <= eps ||x||.  [P:187-190] ("controlled by the given eps-threshold"),
[P:1802-1816] (T2C of the mixed Tucker-canonical core)."""
import numpy as np
import pytest

from oracle import cp as cpm
from oracle.truncate import truncate, tucker_to_canonical


def _odeco(s, n=24, seed=0):
    """Orthogonally decomposable CP with weights s (descending), random orthonormal e_k per mode,
    terms shuffled and duplicated halves (the cut must not depend on the term order)."""
    rng = np.random.default_rng(seed)
    K = s.size
    E = [np.linalg.qr(rng.standard_normal((n, K)))[0] for _ in range(3)]
    perm = rng.permutation(K)
    # split every term into two equal halves: same tensor, 2K canonical terms
    w = np.concatenate([0.5 * s[perm], 0.5 * s[perm]])
    U = [np.concatenate([e[:, perm], e[:, perm]], axis=1) for e in E]
    return cpm.CP(w, U), E


def _spectrum_between(eps, K=12, r0=5):
    """s_1..s_K with tail(r0) = sum_{k>r0} s_k^2 = 0.5 eps^2 E (between (eps/2)^2 E and eps^2 E)
    and tail(r0 + 1) = 0.2 eps^2 E (below (eps/2)^2 E = 0.25 eps^2 E)."""
    head = np.linspace(1.0, 0.5, r0)
    Eh = np.sum(head ** 2)
    # tail energies as fractions f of the total E: E = Eh / (1 - f0), f0 = 0.5 eps^2
    f0, f1 = 0.5 * eps ** 2, 0.2 * eps ** 2
    E = Eh / (1.0 - f0)
    t0, t1 = f0 * E, f1 * E
    s_r0 = np.sqrt(t0 - t1)                       # term r0+1 carries tail(r0) - tail(r0+1)
    rest = np.full(K - r0 - 1, np.sqrt(t1 / (K - r0 - 1)))
    s = np.concatenate([head, [s_r0], rest])
    assert np.all(np.diff(s) <= 0)
    return s, r0


@pytest.mark.parametrize("eps", [1e-2, 1e-3, 1e-4])
def test_eps_half_constant_decides_the_rank(eps):
    s, r0 = _spectrum_between(eps)
    x, E = _odeco(s)
    info = {}
    y = truncate(x, eps, info)
    # (eps/2)^2: tail(r0) = 0.5 eps^2 E > 0.25 eps^2 E -> keep r0 + 1; an eps^2 reading keeps r0
    assert info["tucker_rank"] == [r0 + 1] * 3
    assert y.rank == r0 + 1
    # the error is exactly the dropped energy (orthogonal terms): sqrt(0.2) eps ||x||
    err = np.sqrt(max(cpm.dot(cpm.axpy(x, -1.0, y), cpm.axpy(x, -1.0, y)), 0.0))
    nx = np.sqrt(np.sum(s ** 2))
    assert err == pytest.approx(np.sqrt(0.2) * eps * nx, rel=1e-6)
    assert err <= 0.5 * eps * nx               # the (eps/2) constants' bound, not just eps
    # the kept weights are the s_k themselves (up to sign: factors' signs are free)
    assert np.allclose(np.sort(np.abs(y.w))[::-1], s[:r0 + 1], rtol=1e-10)


def test_t2c_cut_uses_eps_half_of_the_core_norm():
    """T2C alone on a diagonal core: the pooled cut keeps the smallest R with the dropped
    sum s^2 <= (eps/2)^2 ||core||_F^2."""
    eps = 1e-3
    s, r0 = _spectrum_between(eps)
    K = s.size
    core = np.zeros((K, K, K))
    core[np.arange(K), np.arange(K), np.arange(K)] = s
    Z = [np.eye(K)] * 3
    y = tucker_to_canonical(core, Z, eps)
    assert y.rank == r0 + 1
    y = tucker_to_canonical(core, Z, 2 * eps)        # (2 eps / 2)^2 = eps^2: tail(r0) fits
    assert y.rank == r0


def test_rank_cap_keeps_the_top_triples():
    """A26: a truncation whose eps-cut keeps more than rank_cap triples keeps the top rank_cap
    ones (largest s), and reports the clip."""
    s = np.geomspace(1.0, 1e-3, 10)
    x, _ = _odeco(s, seed=3)
    info = {}
    y = truncate(x, 1e-8, info, rank_cap=4)
    assert info["clipped"] and y.rank == 4
    assert np.allclose(np.sort(np.abs(y.w))[::-1], s[:4], rtol=1e-10)
    info = {}
    y = truncate(x, 1e-8, info, rank_cap=50)
    assert not info["clipped"] and y.rank == 10
