"""GPU parity: cp_truncate (S11-S13) and pcg_solve (S14) against the oracle, with shared
eigenpairs and spectral CPs (sl_set_eigen / op_set_spectral_cp).

Tolerances: ranks identical at non-marginal cuts; a single truncation
within eps relative.  Typically the two agree to ~1e-10 (the device forms the side-matrix Gram,
whose singular directions near the cut carry ~eps_mach*s_1^2/s_r^2 error); when two T2C
candidates are near-tied at the cut, the two implementations may keep different members of the
tie, which changes the result by at most the dropped singular value, i.e. < eps/2 (reading A25).
The final control u within max(10 eps, 1e-9) [BASELINE.json north_star]."""
import numpy as np
import pytest

from oracle import cp as cpm
from oracle import pcg as P
from oracle import spectral as sp
from oracle.measure import reldiff
from oracle.truncate import truncate
from synth import make_problem, random_cp

from _parity import check_rank_history, trunc_tolerance

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
    tol, _ = trunc_tolerance(info_o, eps)
    assert reldiff(_cp(y), ref) <= tol
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
    info_o = {}
    ref = truncate(x, 1e-6, info_o)
    y, info = ctx.cp_truncate(DeviceCP.from_numpy(x.w, x.U), 1e-6)
    assert y.rank == ref.rank
    tol, _ = trunc_tolerance(info_o, 1e-6)
    assert reldiff(_cp(y), ref) <= tol
    # duplicated terms [a; a] = 2a: the Tucker ranks are exact, so the RHOSVD tails vanish and
    # the only loss is the T2C pooled cut of the recomputed core, <= (eps/2) ||2a|| (A10/A11)
    d = cpm.CP(np.concatenate([a.w, a.w]), [np.concatenate([u, u], axis=1) for u in a.U])
    y, info = ctx.cp_truncate(DeviceCP.from_numpy(d.w, d.U), 1e-8)
    assert reldiff(_cp(y), cpm.scale(2.0, a)) <= 0.5e-8 + 1e-12
    assert y.rank <= 2 * a.rank


@pytest.mark.parametrize("name,n,R,which", [("C1", 16, 2, 0), ("C1", 32, 3, 1), ("C3b", 24, 4, 0),
                                            ("C1", 40, 5, 0)])
def test_fused_apply_truncate(lib, name, n, R, which):
    """fracop_apply_truncate (the solver's operator step) vs trunc(apply(x)) of the oracle."""
    from paper_2006_09314_b200.binding import DeviceCP
    p = make_problem(name, n=n)
    ctx = lib.context()
    st = _shared(ctx, p)
    spec = st.F if which == 0 else st.G
    x = truncate(cpm.apply(st.V, st.F, cpm.CP(np.linspace(1, 2, R), random_cp(n, R, 9)[1])), p.eps)
    info_o = {}
    ref = truncate(cpm.apply(st.V, spec, x), p.eps, info_o)
    y, info = ctx.fracop_apply_truncate(which, DeviceCP.from_numpy(x.w, x.U), p.eps)
    assert list(info.tucker_rank) == info_o["tucker_rank"]
    assert y.rank == ref.rank
    tol, _ = trunc_tolerance(info_o, p.eps)
    assert reldiff(_cp(y), ref) <= tol


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


@pytest.mark.parametrize("name,n", [("C1", 32), ("C1", 16), ("C3b", 24), ("C4", 32)])
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
    check_rank_history(rep, rep_ref, f"{name} n={n}", floor_rank=0.95 * n * n)
    d = reldiff(_cp(u), u_ref)
    assert d <= max(10 * p.eps, 1e-9)
    # true residual ||B - F(u)||/||B|| (O11) on both sides: the two differ by at most
    # ||F(u_gpu - u_oracle)|| / ||B|| <= F_max ||u_gpu - u_oracle|| / ||B||  (+ dot rounding)
    from paper_2006_09314_b200.binding import FC_F
    from oracle.measure import diff_norm
    B = cpm.normalized(p.b_w, p.b_U)
    fun = lambda x: cpm.apply(st.V, st.F, x)
    true_ref = diff_norm(fun(u_ref), B) / cpm.norm(B)
    Fu = ctx.fracop_apply(FC_F, u)
    r = ctx.cp_axpy(b, -1.0, Fu)
    true_gpu = np.sqrt(max(ctx.cp_dot(r, r), 0.0) / ctx.cp_dot(b, b))
    f = sp.spectral_fn(sp.FC_F, p.alpha, p.beta)
    fmax = max(f(sum(l[-1] for l in st.lams)), f(sum(l[0] for l in st.lams)))
    slack = fmax * d * cpm.norm(u_ref) / cpm.norm(B) + 1e-7
    assert abs(true_gpu - true_ref) <= slack, (true_gpu, true_ref, slack)


@pytest.mark.parametrize("n,R,eps", [(48, 5, 1e-8), (40, 4, 1e-9), (64, 3, 1e-8)])
def test_truncate_small_eps_refined_cut(lib, n, R, eps):
    """Cuts below the Gram noise level ((eps/2)^2 E < k eps_mach lam_max): cp_truncate (CP route)
    takes the K13 path for eps < 1e-6 (SVD of the side matrix itself: rank-revealing basis of
    B^T + QR-preconditioned Jacobi, no squaring floor); apply outputs (structured route) take
    reading A11' (noise subspace re-diagonalised from the data).  Tucker ranks as the oracle's
    exact SVD cut (+-1 in the A23 band), result within 2 eps."""
    from paper_2006_09314_b200.binding import DeviceCP
    p = make_problem("C1", n=n)
    ctx = lib.context()
    st = _shared(ctx, p)
    w, U = random_cp(n, R, 17)
    x = cpm.apply(st.V, st.F, cpm.CP(np.linspace(1, 2, R), U))
    info_o = {}
    ref = truncate(x, eps, info_o)
    y, info = ctx.cp_truncate(DeviceCP.from_numpy(x.w, x.U), eps)
    for l in range(3):
        assert abs(info.tucker_rank[l] - info_o["tucker_rank"][l]) <= 1
    assert reldiff(_cp(y), ref) <= 2 * eps


@pytest.mark.parametrize("eps", [1e-9, 1e-10])
def test_truncate_k13_below_gram_floor(lib, eps):
    """K13 (SVD of the side matrix, no squaring): a CP whose mode spectra decay geometrically
    over 14 decades, cut at eps where the Gram eigenvalues (noise ~eps_mach s_max^2, i.e. a floor
    of ~1e-8 relative in s) cannot see the cut.  Tucker ranks equal the oracle's exact-SVD cut
    unless that cut is inside the A23 noise band; result within 2 eps."""
    from paper_2006_09314_b200.binding import DeviceCP, make_params
    n, R = 64, 48
    rng = np.random.default_rng(21)
    Q = [np.linalg.qr(rng.standard_normal((n, R)))[0] for _ in range(3)]
    decay = 10.0 ** (-np.linspace(0, 14, R))
    U = [Q[l] @ (np.diag(decay) @ rng.standard_normal((R, R))) for l in range(3)]
    x = cpm.normalized(np.ones(R), U)
    ctx = lib.context()
    ctx.sl_setup(n, np.ones((3, n + 1)), make_params(0.5, 0.01, 1e-6))
    info_o = {}
    ref = truncate(x, eps, info_o)
    y, info = ctx.cp_truncate(DeviceCP.from_numpy(x.w, x.U), eps)
    marginal = min(info_o["margins"]) < 5e-3
    for l in range(3):
        assert abs(info.tucker_rank[l] - info_o["tucker_rank"][l]) <= (1 if marginal else 0), (l, marginal)
    assert reldiff(_cp(y), ref) <= 2 * eps


@pytest.mark.parametrize("cap", [24, 60])
def test_pcg_rank_cap_hit(lib, cap):
    """A26: with params.rank_cap below the eps-cut ranks every truncation keeps its top rank_cap
    T2C triples; pcg_solve reports FC_RANK_CAP_HIT (2) when it converges anyway and counts the
    clipped truncations; the oracle with the same cap agrees rank by rank."""
    from paper_2006_09314_b200.binding import DeviceCP, make_params
    p = make_problem("C1", n=32)
    ctx = lib.context()
    st = _shared(ctx, p)
    prm = make_params(p.alpha, p.beta, p.eps, p.tol_stop, rank_cap=cap, kmax=12)
    u, rep, rc = ctx.pcg_solve(DeviceCP.from_numpy(p.b_w, p.b_U), prm)
    u_ref, rep_ref, _ = P.solve(p, st, kmax=12, rank_cap=cap)
    print(f"cap {cap}: rc {rc} iters {rep['iters']} cap_hits {rep['cap_hits']} / oracle {rep_ref['cap_hits']}")
    assert max(max(rep[k]) for k in ("rank_S", "rank_X", "rank_R", "rank_Z", "rank_P")) <= cap
    assert rep["cap_hits"] > 0
    if rep["converged"]:
        assert rc == 2
    else:
        assert rc == 1
    check_rank_history(rep, rep_ref, f"cap {cap}")
    if rep_ref["converged"] and rep["converged"]:
        assert reldiff(_cp(u), u_ref) <= max(10 * p.eps, 1e-9)
