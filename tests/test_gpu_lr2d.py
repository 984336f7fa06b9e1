"""GPU parity of the 2D variant against the 2D oracle (oracle/lr2d.py,
pinned by tests/test_oracle_lr2d.py): reduced-SVD truncation, factored apply, dot, the device
spectral factorisation, and the 2D PCG (shared inputs and independent setups)."""
import numpy as np
import pytest

from oracle import lr2d
from oracle.spectral import FC_F, FC_G
from synth import make_problem2

pytestmark = pytest.mark.gpu


def _dev(x):
    from paper_2006_09314_b200.binding import DeviceLR2
    return DeviceLR2.from_numpy(x.w, x.U)


def _host(y):
    w, U = y.to_numpy()
    return lr2d.LR2(w, U)


def _graded(n1, n2, s, R, seed):
    """X = Q1 diag(s) Q2^T stored redundantly as R >= len(s) terms (random mixing)."""
    rng = np.random.default_rng(seed)
    k = len(s)
    Q1, _ = np.linalg.qr(rng.standard_normal((n1, k)))
    Q2, _ = np.linalg.qr(rng.standard_normal((n2, k)))
    M = rng.standard_normal((k, R))
    Minv = np.linalg.pinv(M)                    # k x R -> R x k with M Minv = I_k
    U1 = (Q1 * s) @ M                           # n1 x R
    U2 = Q2 @ Minv.T                            # n2 x R ; U1 U2^T = Q1 diag(s) Q2^T
    return lr2d.normalized2(np.ones(R), [U1, U2])


@pytest.mark.parametrize("n,R,eps", [(64, 40, 1e-6), (37, 3, 1e-8), (257, 120, 1e-6), (1024, 200, 1e-7)])
def test_truncate2d_parity(lib, n, R, eps):
    """Ranks identical to the oracle's truncated SVD; reconstructions within 1e-10 ||X|| (the
    truncated SVD is unique for distinct singular values); orthonormal output factors."""
    ctx = lib.context()
    ctx.sl_setup_2d(n, np.ones((2, n + 1)), _params(eps))
    k = min(R, 60)
    s = 10.0 ** (-np.linspace(0, 12, k))        # graded, distinct
    x = _graded(n, n, s, R, seed=n + R)
    ref_info = {}
    ref = lr2d.truncate2(x, eps, ref_info)
    y = _host(ctx.cp_truncate_2d(_dev(x), eps))
    assert y.rank == ref.rank, (y.rank, ref.rank, ref_info["margins"])
    X = lr2d.full2(x)
    assert np.linalg.norm(lr2d.full2(y) - lr2d.full2(ref)) <= 1e-10 * np.linalg.norm(X)
    assert np.abs(y.U[0].T @ y.U[0] - np.eye(y.rank)).max() < 1e-12
    assert np.abs(y.U[1].T @ y.U[1] - np.eye(y.rank)).max() < 1e-12


def test_truncate2d_edge_cases(lib):
    """zero input -> rank 0; exact rank-1 -> rank 1 with its weight; duplicated terms collapse."""
    n = 33
    ctx = lib.context()
    ctx.sl_setup_2d(n, np.ones((2, n + 1)), _params(1e-6))
    z = lr2d.LR2(np.zeros(2), [np.eye(n)[:, :2], np.eye(n)[:, :2]])
    assert ctx.cp_truncate_2d(_dev(z), 1e-6).rank == 0
    rng = np.random.default_rng(1)
    a, b = rng.standard_normal(n), rng.standard_normal(n)
    one = lr2d.normalized2(np.array([2.0, 1.0, -0.5]), [np.stack([a, a, a], 1), np.stack([b, b, b], 1)])
    y = _host(ctx.cp_truncate_2d(_dev(one), 1e-10))
    assert y.rank == 1
    assert abs(abs(y.w[0]) - 2.5 * np.linalg.norm(a) * np.linalg.norm(b)) <= 1e-12 * abs(y.w[0])


def _params(eps, **kw):
    from paper_2006_09314_b200.binding import make_params
    return make_params(0.5, 0.01, eps, **kw)


def _shared_ctx(lib, p, st):
    """device context with the oracle's eigenpairs and spectral factorisations injected"""
    from paper_2006_09314_b200.binding import make_params
    ctx = lib.context()
    prm = make_params(p.alpha, p.beta, p.eps)
    for l in range(2):
        ctx.sl_set_eigen(p.n, l, st.lams[l], st.V[l], prm)
    ctx.op_set_spectral_2d(FC_F, _dev(st.F))
    ctx.op_set_spectral_2d(FC_G, _dev(st.G))
    return ctx, prm


def test_apply2d_and_dot_shared(lib):
    p = make_problem2("D1", n=48)
    st = lr2d.setup2(p)
    ctx, _ = _shared_ctx(lib, p, st)
    rng = np.random.default_rng(3)
    x = lr2d.normalized2(rng.standard_normal(5), [rng.standard_normal((p.n, 5)) for _ in range(2)])
    for which, sp in ((FC_F, st.F), (FC_G, st.G)):
        y = _host(ctx.fracop_apply_2d(which, _dev(x)))
        ref = lr2d.apply2(st.V, sp, x)
        assert y.rank == ref.rank
        assert np.abs(lr2d.full2(y) - lr2d.full2(ref)).max() <= 1e-12 * np.abs(lr2d.full2(ref)).max()
    v = lr2d.normalized2(rng.standard_normal(3), [rng.standard_normal((p.n, 3)) for _ in range(2)])
    assert ctx.cp_dot_2d(_dev(x), _dev(v)) == pytest.approx(lr2d.dot2(x, v), rel=1e-12, abs=1e-13)


@pytest.mark.parametrize("n", [64, 512])
def test_setup2d_independent(lib, n):
    """Device factorisation (range finder + SVD) vs the oracle's exact SVD of D2: F within
    2 eps_D ||D2|| of each other, ranks within 1; G rank-r_G (or guard-raised) positive."""
    p = make_problem2("D1", n=n)
    st = lr2d.setup2(p)
    ctx = lib.context()
    ctx.sl_setup_2d(p.n, p.a_mid, _params(p.eps))
    F = _host(ctx.op_get_spectral_2d(FC_F))
    G = _host(ctx.op_get_spectral_2d(FC_G))
    D = lr2d.coefficient_matrix(st.lams, FC_F, p.alpha, p.beta)
    assert abs(F.rank - st.F.rank) <= 1
    assert np.linalg.norm(lr2d.full2(F) - lr2d.full2(st.F)) <= 2 * p.eps * np.linalg.norm(D)
    assert np.linalg.norm(lr2d.full2(F) - D) <= 1.0000001 * p.eps * np.linalg.norm(D)
    assert G.rank == st.G.rank
    assert np.min(lr2d.full2(G)) > 0


@pytest.mark.parametrize("n", [32, 128])
def test_pcg2d_parity_shared(lib, n):
    """Shared eigenpairs and factorisations: iteration count and ranks as the oracle's,
    residual history within 1e-6 relative, u within 10 eps."""
    p = make_problem2("D1", n=n)
    st = lr2d.setup2(p)
    u_ref, rep_ref, _ = lr2d.solve2(p, st)
    ctx, prm = _shared_ctx(lib, p, st)
    from paper_2006_09314_b200.binding import make_params
    prm = make_params(p.alpha, p.beta, p.eps, p.tol_stop)
    u, rep, rc = ctx.pcg_solve_2d(_dev(lr2d.normalized2(p.b_w, p.b_U)), prm)
    assert rc == 0 and rep["iters"] == rep_ref["iters"]
    for key in ("rank_S", "rank_X", "rank_R"):
        assert rep[key] == rep_ref[key], key
    assert np.allclose(rep["rel_res"], rep_ref["rel_res"], rtol=1e-6)
    U = lr2d.full2(u_ref)
    assert np.linalg.norm(lr2d.full2(_host(u)) - U) <= 10 * p.eps * np.linalg.norm(U)


def test_pcg2d_fullsize_independent(lib):
    """D2 (n = 1024, rank-8 bumps): independent device setup and solve vs the whole oracle;
    both converge, iteration counts within 1, u within kappa * 10 eps (the two spectral
    factorisations are each eps_D-accurate)."""
    p = make_problem2("D2")
    u_ref, rep_ref, st = lr2d.solve2(p)
    ctx = lib.context()
    from paper_2006_09314_b200.binding import make_params
    prm = make_params(p.alpha, p.beta, p.eps, p.tol_stop)
    ctx.sl_setup_2d(p.n, p.a_mid, prm)
    u, rep, rc = ctx.pcg_solve_2d(_dev(lr2d.normalized2(p.b_w, p.b_U)), prm)
    print(f"2D n=1024: iters {rep['iters']} (oracle {rep_ref['iters']}), rank {u.rank}, "
          f"loop {rep['t_loop_ms']:.2f} ms")
    assert rc == 0 and abs(rep["iters"] - rep_ref["iters"]) <= 1
    lam_min = st.lams[0][0] + st.lams[1][0]
    lam_max = st.lams[0][-1] + st.lams[1][-1]
    f = lambda l: p.beta * l ** p.alpha + l ** -p.alpha
    kappa = max(f(lam_min), f(lam_max)) / min(f(lam_min), f(lam_max))
    U = lr2d.full2(u_ref)
    assert np.linalg.norm(lr2d.full2(_host(u)) - U) <= kappa * 10 * p.eps * np.linalg.norm(U)
