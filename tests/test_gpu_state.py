"""GPU parity of state recovery, state_recover: y = A^-alpha u truncated at
eps [P:287-289, P:969-972] (reading A5), against the oracle (tests/test_oracle_state.py pins it)."""
import math

import numpy as np
import pytest

from oracle import cp as cpm
from oracle import pcg as P
from oracle.measure import reldiff
from synth import make_problem, random_cp

pytestmark = pytest.mark.gpu


def _cp(y):
    w, U = y.to_numpy()
    return cpm.CP(w, U)


@pytest.mark.parametrize("name,n", [("C1", 16), ("C1", 32), ("C3b", 20)])
def test_state_shared(lib, name, n):
    """Shared eigenpairs and spectral CP of lam^-alpha: ranks as the oracle's, y within eps."""
    from paper_2006_09314_b200.binding import FC_POW_MINUS, DeviceCP, make_params
    p = make_problem(name, n=n)
    st = P.setup(p)
    ctx = lib.context()
    prm = make_params(p.alpha, p.beta, p.eps)
    for l in range(3):
        ctx.sl_set_eigen(p.n, l, st.lams[l], st.V[l], prm)
    Pm = P.state_cp(p, st)
    ctx.op_set_spectral_cp(FC_POW_MINUS, DeviceCP.from_numpy(Pm.w, Pm.U))
    u = P.solve(p, st)[0]
    y, info = ctx.state_recover(DeviceCP.from_numpy(u.w, u.U), p.eps)
    ref_info = {}
    from oracle.truncate import truncate
    ref = truncate(cpm.apply(st.V, Pm, u), p.eps, ref_info)
    assert list(info.tucker_rank) == ref_info["tucker_rank"]
    assert y.rank == ref.rank
    assert reldiff(_cp(y), ref) <= p.eps


def test_state_lazy_build_independent(lib):
    """sl_setup + state_recover (the lambda^-alpha CP built on first use on the device) vs the whole
    oracle: both CPs are eps_D-accurate, so y agrees to ~kappa(A^-alpha) * eps."""
    from paper_2006_09314_b200.binding import DeviceCP, make_params
    p = make_problem("C1", n=24)
    ctx = lib.context()
    ctx.sl_setup(p.n, p.a_mid, make_params(p.alpha, p.beta, p.eps, p.tol_stop))
    st = P.setup(p)
    w, U = random_cp(p.n, 3, 21)
    u = cpm.CP(np.array([1.0, 0.5, -0.25]), U)
    y, _ = ctx.state_recover(DeviceCP.from_numpy(u.w, u.U), p.eps)
    ref = P.state(p, st, u)
    lam_min = sum(l[0] for l in st.lams)
    lam_max = sum(l[-1] for l in st.lams)
    kappa = (lam_max / lam_min) ** p.alpha
    assert reldiff(_cp(y), ref) <= kappa * 10 * p.eps


def probe_reldiff(ctx, y, yu, n, K=256, seed=7):
    """||y - yu|| / ||yu|| estimated with K Gaussian rank-1 probes g = g1 (x) g2 (x) g3:
    E<d, g>^2 = ||d||^2 for iid N(0, 1) factors, and <y, g>, <yu, g> are each computed to ~eps
    (no cancellation of squares: cp_dot(d, d) of the CP difference has a floor of ~sqrt(eps)
    relative, exactly the level tested here).  The mean of <d, g>^2 over K rank-1 probes has
    relative standard deviation <= sqrt(26 / K) (E X^4 <= 27 (E X^2)^2 for products of 3 Gaussian
    factors): ~0.3 at K = 256, i.e. ~15 % on the norm ratio."""
    from paper_2006_09314_b200.binding import DeviceCP
    rng = np.random.default_rng(seed)
    num = den = 0.0
    for _ in range(K):
        g = DeviceCP.from_numpy(np.ones(1), [rng.standard_normal((n, 1)) for _ in range(3)])
        a, b = ctx.cp_dot(y, g), ctx.cp_dot(yu, g)
        num += (a - b) ** 2
        den += b * b
    return math.sqrt(num / den)


def test_state_fullsize(lib):
    """C4, n = 1024: the state of the solved control, y = A^-alpha u (state_recover, fused
    apply -> truncate at 1e-8), equals the untruncated apply of the lambda^-alpha CP to the
    truncation accuracy, measured with Gaussian rank-1 probes (probe_reldiff; the CP difference's
    own cp_dot cancels to ~1e-8 and gave 0 .. 4e-8 for the same code).  A check of
    b - y - beta A^alpha u against b - F(u) is NOT used: the eps_D spectral CPs are Frobenius-
    accurate, and on the lowest frequencies (where a smooth u lives) lambda^alpha's CP is off by up
    to 84 % at n = 1024 ('Spectral-CP accuracy on smooth modes')."""
    from paper_2006_09314_b200.binding import FC_POW_MINUS, DeviceCP, make_params
    p = make_problem("C4", n=1024)
    ctx = lib.context()
    prm = make_params(p.alpha, p.beta, p.eps, p.tol_stop)
    ctx.sl_setup(p.n, p.a_mid, prm)
    u, rep, rc = ctx.pcg_solve(DeviceCP.from_numpy(p.b_w, p.b_U), prm)
    assert rc == 0
    y, info = ctx.state_recover(u, 1e-8)
    yu = ctx.fracop_apply(FC_POW_MINUS, u)
    rel = probe_reldiff(ctx, y, yu, p.n)
    print(f"C4 n=1024 state: rank {y.rank} (untruncated {yu.rank}), ||y - A^-a u|| / ||A^-a u|| = {rel:.2e}")
    assert rel <= 1.5e-8      # eps = 1e-8 plus the estimator's spread (measured 6.96e-9)
