"""GPU parity: cp_truncate (S11-S13) and pcg_solve (S14) against the oracle, with shared
eigenpairs and spectral CPs (sl_set_eigen / op_set_spectral_cp).

Tolerances: ranks identical at non-marginal cuts; a single truncation
within 1e-9 relative (the device forms the side-matrix Gram, whose singular directions near the
cut carry ~eps*s_1^2/s_r^2 error, i.e. <= 1e-10 of the tensor at eps = 1e-6); the final control
u within max(10 eps, 1e-9) [BASELINE.json north_star]."""
import numpy as np
import pytest

from oracle import cp as cpm
from oracle import pcg as P
from oracle import spectral as sp
from oracle.measure import reldiff
from oracle.truncate import truncate
from synth import make_problem, random_cp

pytestmark = pytest.mark.gpu


def _shared(ctx, p, F_rank=None):
    from paper_2006_09314_b200.binding import DeviceCP, make_params, FC_F, FC_G
    st = P.setup(p, F_rank=F_rank)
    prm = make_params(p.alpha, p.beta, p.eps)
    for l in range(3):
        ctx.sl_set_eigen(p.n, l, st.lams[l], st.V[l], prm)
    ctx.op_set_spectral_cp(FC_F, DeviceCP.from_numpy(st.F.w, st.F.U))
    ctx.op_set_spectral_cp(FC_G, DeviceCP.from_numpy(st.G.w, st.G.U))
    return st


def _cp(y):
    w, U = y.to_numpy()
    return cpm.CP(w, U)


@pytest.mark.parametrize("n,R,eps", [(16, 3, 1e-6), (32, 4, 1e-6), (32, 2, 1e-4), (37, 5, 1e-7)])
def test_truncate_apply_output(lib, n, R, eps):
    from paper_2006_09314_b200.binding import DeviceCP
    p = make_problem("C1", n=n)
    ctx = lib.context()
    st = _shared(ctx, p)
    w, U = random_cp(n, R, 3)
    x = cpm.apply(st.V, st.F, cpm.CP(np.linspace(1, 2, R), U))
    info_o = {}
    ref = truncate(x, eps, info_o)
    y, info = ctx.cp_truncate(DeviceCP.from_numpy(x.w, x.U), eps)
    assert list(info.tucker_rank) == info_o["tucker_rank"]
    assert y.rank == ref.rank
    assert reldiff(_cp(y), ref) <= 1e-9
    g = _cp(y)
    assert cpm.dot(g, g) == pytest.approx(np.sum(g.w ** 2), rel=1e-10)     # orthogonal CP


@pytest.mark.parametrize("n,R1,R2", [(24, 10, 12), (64, 40, 30)])
def test_truncate_concat_and_duplicates(lib, n, R1, R2):
    from paper_2006_09314_b200.binding import DeviceCP
    p = make_problem("C1", n=n)
    ctx = lib.context()
    st = _shared(ctx, p)
    a = truncate(cpm.apply(st.V, st.F, cpm.CP(*random_cp(n, 2, 1))), 1e-6)
    b = truncate(cpm.apply(st.V, st.G, cpm.CP(*random_cp(n, 2, 2))), 1e-6)
    x = cpm.axpy(a, -0.37, b)
    ref = truncate(x, 1e-6)
    y, info = ctx.cp_truncate(DeviceCP.from_numpy(x.w, x.U), 1e-6)
    assert y.rank == ref.rank
    assert reldiff(_cp(y), ref) <= 1e-9
    d = cpm.CP(np.concatenate([a.w, a.w]), [np.concatenate([u, u], axis=1) for u in a.U])
    y, info = ctx.cp_truncate(DeviceCP.from_numpy(d.w, d.U), 1e-8)
    assert reldiff(_cp(y), cpm.scale(2.0, a)) <= 1e-9


def test_truncate_zero_and_rank1(lib):
    from paper_2006_09314_b200.binding import DeviceCP
    p = make_problem("C1", n=12)
    ctx = lib.context()
    _shared(ctx, p)
    w, U = random_cp(12, 1, 4)
    y, info = ctx.cp_truncate(DeviceCP.from_numpy(2.5 * w, U), 1e-6)
    assert y.rank == 1 and abs(y.w[0].item()) == pytest.approx(2.5, rel=1e-13)
    y, info = ctx.cp_truncate(DeviceCP.from_numpy(0 * w, U), 1e-6)
    assert y.rank == 0


@pytest.mark.parametrize("name,n", [("C1", 32), ("C1", 16), ("C3b", 24)])
def test_pcg_parity_shared(lib, name, n):
    from paper_2006_09314_b200.binding import DeviceCP, make_params
    p = make_problem(name, n=n)
    ctx = lib.context()
    st = _shared(ctx, p)
    u_ref, rep_ref, _ = P.solve(p, st)
    b = DeviceCP.from_numpy(p.b_w, p.b_U)
    prm = make_params(p.alpha, p.beta, p.eps, p.tol_stop)
    u, rep, rc = ctx.pcg_solve(b, prm)
    assert rc == 0 and rep["converged"]
    assert rep["iters"] == rep_ref["iters"]
    assert rep["rank_S"] == rep_ref["rank_S"]
    assert rep["rank_X"] == rep_ref["rank_X"]
    assert rep["rank_R"] == rep_ref["rank_R"]
    assert np.allclose(rep["rel_res"], rep_ref["rel_res"], rtol=1e-5)
    assert reldiff(_cp(u), u_ref) <= max(10 * p.eps, 1e-9)
