"""Pins of O12 reldiff (the parity measure): exact on a difference with a closed form, and
resolving differences far below the ~1e-8 floor of the inner-product identity at sizes where
the common span is low-rank but min(n, R_x + R_y) is not (the full-size parity regime)."""
import numpy as np
import pytest

from oracle import cp as cpm
from oracle.measure import diff_norm, reldiff


def _tucker_cp(n, r, R, seed):
    """A CP with R terms whose factors lie in an r-dimensional subspace per mode (like a
    truncation output), unit columns."""
    rng = np.random.default_rng(seed)
    Q = [np.linalg.qr(rng.standard_normal((n, r)))[0] for _ in range(3)]
    U = [q @ rng.standard_normal((r, R)) for q in Q]
    return cpm.normalized(rng.standard_normal(R), U), Q


@pytest.mark.parametrize("delta", [1e-6, 1e-10, 1e-13])
def test_reldiff_resolves_small_differences(delta):
    n, r, R = 600, 20, 700                     # R_x + R_y = 1401 > n: the naive basis is n-dimensional
    x, Q = _tucker_cp(n, r, R, 1)
    # y = x + delta * (unit rank-1 term inside the span): ||y - x|| = delta exactly
    e = [q[:, 0] for q in Q]
    y = cpm.CP(np.concatenate([x.w, [delta]]), [np.concatenate([x.U[l], e[l][:, None]], axis=1) for l in range(3)])
    got = diff_norm(x, y)
    assert got == pytest.approx(delta, rel=1e-3, abs=1e-15 * np.sqrt(cpm.dot(x, x)) * 50)
    assert reldiff(x, x) == 0.0


def test_reldiff_matches_dense_difference():
    n = 12
    rng = np.random.default_rng(5)
    x = cpm.CP(rng.standard_normal(7), [rng.standard_normal((n, 7)) for _ in range(3)])
    y = cpm.CP(rng.standard_normal(5), [rng.standard_normal((n, 5)) for _ in range(3)])
    X, Y = cpm.full(x), cpm.full(y)
    assert reldiff(x, y) == pytest.approx(np.linalg.norm(X - Y) / np.linalg.norm(Y), rel=1e-12)
