"""GPU parity of cp_truncate_als (C2T-ALS refinement) against the oracle
(oracle/als.py, pinned by tests/test_oracle_als.py)."""
import numpy as np
import pytest

from oracle import als
from oracle import cp as cpm
from oracle.measure import reldiff

pytestmark = pytest.mark.gpu


def _tucker_cp(n, r, seed, noise):
    rng = np.random.default_rng(seed)
    Q = [np.linalg.qr(rng.standard_normal((n, r[l])))[0] for l in range(3)]
    core = rng.standard_normal(r) * np.exp(-0.7 * np.arange(r[0]))[:, None, None]
    idx = np.argwhere(np.ones(r, dtype=bool))
    w = np.array([core[tuple(i)] for i in idx])
    x = cpm.normalized(w, [Q[l][:, idx[:, l]] for l in range(3)])
    y = cpm.normalized(noise * np.ones(6), [rng.standard_normal((n, 6)) for _ in range(3)])
    return cpm.axpy(x, 1.0, y)


@pytest.mark.parametrize("n,r,eps,sweeps", [(16, (4, 3, 3), 1e-2, 2), (40, (6, 5, 4), 3e-3, 3), (96, (8, 8, 6), 1e-3, 2)])
def test_cp_truncate_als_parity(lib, n, r, eps, sweeps):
    """Tucker ranks and output rank as the oracle's; result within 1e-9 ||x|| of the oracle's
    and within eps of x.  (HOOI improves the Tucker projection — pinned in test_oracle_als — not
    necessarily the error after the T2C cut, so no comparison with cp_truncate's result.)"""
    from paper_2006_09314_b200.binding import DeviceCP, make_params
    x = _tucker_cp(n, r, seed=n, noise=2e-3)
    ctx = lib.context()
    ctx.sl_setup(n, np.ones((3, n + 1)), make_params(0.5, 0.01, 1e-6))
    info_ref = {}
    ref = als.c2t_als(x, eps, sweeps, info_ref)
    y, info = ctx.cp_truncate_als(DeviceCP.from_numpy(x.w, x.U), eps, sweeps)
    w, U = y.to_numpy()
    yd = cpm.CP(w, U)
    assert list(info.tucker_rank) == info_ref["tucker_rank"]
    assert y.rank == ref.rank
    assert reldiff(yd, ref) <= 1e-9
    assert reldiff(yd, x) <= eps


def test_cp_truncate_als_zero_sweeps_is_cp_truncate(lib):
    from paper_2006_09314_b200.binding import DeviceCP, make_params
    n = 24
    x = _tucker_cp(n, (5, 4, 4), seed=5, noise=1e-3)
    ctx = lib.context()
    ctx.sl_setup(n, np.ones((3, n + 1)), make_params(0.5, 0.01, 1e-6))
    a, _ = ctx.cp_truncate_als(DeviceCP.from_numpy(x.w, x.U), 1e-3, 0)
    b, _ = ctx.cp_truncate(DeviceCP.from_numpy(x.w, x.U), 1e-3)
    wa, Ua = a.to_numpy()
    wb, Ub = b.to_numpy()
    assert a.rank == b.rank
    assert reldiff(cpm.CP(wa, Ua), cpm.CP(wb, Ub)) <= 1e-13
