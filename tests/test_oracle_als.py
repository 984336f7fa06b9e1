"""Pins of the C2T-ALS oracle (oracle/als.py): exact recovery of an exact
Tucker tensor, the HOOI monotonicity theorem and stationarity, checked on dense tensors."""
import numpy as np

from oracle import als
from oracle import cp as cpm


def _orth(n, k, rng):
    q, _ = np.linalg.qr(rng.standard_normal((n, k)))
    return q


def _tucker_as_cp(n, r, seed, noise=0.0):
    """x = core x_l Q_l (exact multilinear rank r) written as a CP (one term per core entry),
    plus an optional random rank-4 perturbation."""
    rng = np.random.default_rng(seed)
    Q = [_orth(n, r[l], rng) for l in range(3)]
    core = rng.standard_normal(r) * np.exp(-0.5 * np.arange(r[0]))[:, None, None]
    idx = np.argwhere(np.ones(r, dtype=bool))
    w = np.array([core[tuple(i)] for i in idx])
    U = [Q[l][:, idx[:, l]] for l in range(3)]
    x = cpm.normalized(w, U)
    if noise:
        y = cpm.normalized(noise * np.ones(4), [rng.standard_normal((n, 4)) for _ in range(3)])
        x = cpm.axpy(x, 1.0, y)
    return x


def _proj_err(x, Z):
    """|| x - x x_l Z_l Z_l^T ||_F on the dense tensor"""
    X = cpm.full(x)
    P = [z @ z.T for z in Z]
    Y = np.einsum("abc,ia,jb,kc->ijk", X, P[0], P[1], P[2])
    return float(np.linalg.norm(X - Y))


def test_als_recovers_exact_tucker_tensor():
    x = _tucker_as_cp(10, (3, 4, 2), seed=1)
    y = als.c2t_als(x, 1e-10, sweeps=2)
    assert np.abs(cpm.full(y) - cpm.full(x)).max() <= 1e-12 * np.abs(cpm.full(x)).max()


def test_hooi_monotone_and_stationary():
    """Each ALS step maximises the projected norm over one basis: the Tucker projection error
    never increases; after a few sweeps the projectors stop moving (stationary point)."""
    x = _tucker_as_cp(11, (3, 3, 3), seed=2, noise=0.05)
    w, U, Z, ranks = als.rhosvd(x, 0.3)
    errs = [_proj_err(x, Z)]
    Ps = []
    for _ in range(6):
        Z = als.hooi_sweep(w, U, Z)
        errs.append(_proj_err(x, Z))
        Ps.append([z @ z.T for z in Z])
    assert all(errs[k + 1] <= errs[k] * (1 + 1e-12) + 1e-14 for k in range(len(errs) - 1))
    assert errs[-1] < errs[0]                      # the refinement does something here
    assert max(np.abs(Ps[-1][l] - Ps[-2][l]).max() for l in range(3)) < 1e-6


def test_als_output_within_eps():
    """The O9 bound holds with the refined bases: the Tucker stage loses at most its RHOSVD
    error (HOOI only lowers it) and T2C at most (eps/2)||core||."""
    x = _tucker_as_cp(12, (4, 4, 3), seed=3, noise=0.02)
    X = cpm.full(x)
    for eps in (1e-1, 1e-2):
        y = als.c2t_als(x, eps, sweeps=3)
        assert np.linalg.norm(cpm.full(y) - X) <= eps * np.linalg.norm(X)
