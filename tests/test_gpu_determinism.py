"""Run-to-run reproducibility of every stage of the hot path: the same call on the same inputs must
return bit-identical results (rank bookkeeping is only reproducible if every reduction has a fixed
order: split-K partial tiles, Gram partials, matvecs, pooled cuts).  North star: "bit-exact for
... rank bookkeeping"."""
import numpy as np
import pytest

from synth import make_problem, random_cp

pytestmark = pytest.mark.gpu


def _graded(N, seed):
    rng = np.random.default_rng(seed)
    Q, _ = np.linalg.qr(rng.standard_normal((N, N)))
    lam = 10.0 ** (-14.0 * np.arange(N) / N)
    M = (Q * lam) @ Q.T
    return 0.5 * (M + M.T)


@pytest.mark.parametrize("N", [40, 96, 97, 300, 600, 840, 1000])
def test_syev_bit_identical(lib, N):
    """fc_syev on every tridiagonalisation path (packed <= 96, 16-CTA cluster 97..840, global)."""
    import torch
    ctx = lib.context()
    M = _graded(N, N)
    outs = []
    for _ in range(2):
        (lam, Y), = ctx.syev([torch.tensor(M, device="cuda")], [min(N, 64)])
        outs.append((lam.cpu().numpy(), Y.cpu().numpy()))
    assert np.array_equal(outs[0][0], outs[1][0])
    assert np.array_equal(outs[0][1], outs[1][1])


@pytest.mark.parametrize("n,p,rank", [(1024, 300, 120), (512, 700, 400), (2048, 200, 200)])
def test_orthonormalize_bit_identical(lib, n, p, rank):
    import torch
    ctx = lib.context()
    rng = np.random.default_rng(n + p)
    K = (rng.standard_normal((n, rank)) @ rng.standard_normal((rank, p))) * np.logspace(0, -8, p)[None, :]
    outs = []
    for _ in range(2):
        A = torch.tensor(np.ascontiguousarray(K.T), device="cuda")
        outs.append(ctx.orthonormalize(A, 1e-13).cpu().numpy())
    assert outs[0].shape == outs[1].shape and np.array_equal(outs[0], outs[1])


def _cp_bits(y):
    w, U = y.to_numpy()
    return w, U


@pytest.mark.parametrize("n,R,eps", [(256, 300, 1e-6), (512, 150, 1e-8)])
def test_truncate_bit_identical(lib, n, R, eps):
    from paper_2006_09314_b200.binding import DeviceCP
    ctx = lib.context()
    p = make_problem("C1", n=n)
    from paper_2006_09314_b200.binding import make_params
    ctx.sl_setup(p.n, p.a_mid, make_params(p.alpha, p.beta, eps, 10 * eps))
    w, U = random_cp(n, R, 11)
    # a low-rank-ish CP: random terms mixed from 40 directions per mode
    rng = np.random.default_rng(3)
    U = [u[:, :40] @ rng.standard_normal((40, R)) for u in U]
    U = [u / np.linalg.norm(u, axis=0) for u in U]
    x = DeviceCP.from_numpy(np.linspace(1.0, 0.01, R), U)
    outs = [ctx.cp_truncate(x, eps) for _ in range(2)]
    (y0, i0), (y1, i1) = outs
    assert y0.rank == y1.rank and list(i0.tucker_rank) == list(i1.tucker_rank)
    for a, b in zip(_cp_bits(y0), _cp_bits(y1)):
        assert np.array_equal(np.asarray(a), np.asarray(b))
    outs = [ctx.fracop_apply_truncate(0, y0, eps) for _ in range(2)]
    (z0, _), (z1, _) = outs
    assert z0.rank == z1.rank
    for a, b in zip(_cp_bits(z0), _cp_bits(z1)):
        assert np.array_equal(np.asarray(a), np.asarray(b))


@pytest.mark.parametrize("n,eps", [(256, 1e-6), (1024, 1e-6)])
def test_pcg_solve_bit_identical(lib, n, eps):
    """Two back-to-back C4-shaped solves: identical residual history and all five rank histories."""
    from paper_2006_09314_b200.binding import DeviceCP, make_params
    p = make_problem("C4", n=n, eps=eps)
    ctx = lib.context()
    prm = make_params(p.alpha, p.beta, p.eps, p.tol_stop)
    ctx.sl_setup(p.n, p.a_mid, prm)
    b = DeviceCP.from_numpy(p.b_w, p.b_U)
    reps = []
    for _ in range(2):
        u, rep, rc = ctx.pcg_solve(b, prm)
        assert rc == 0
        reps.append((rep, u.to_numpy()))
    (r0, u0), (r1, u1) = reps
    for k in ("rel_res", "rank_X", "rank_R", "rank_S", "rank_Z", "rank_P", "tucker_S"):
        assert r0[k] == r1[k], k
    assert np.array_equal(u0[0], u1[0])


def test_streamk_solve_matches_whole_tile_launches():
    """The stream-K 128 x 128 GEMM in the truncation (per-term Grams, term-norm products and the
    core contraction once a Tucker rank exceeds 64, late in the C4 solve) against the same solve
    with every launch on whole tiles (FC_STREAMK=0, read once per process: two subprocesses):
    same iteration count, the five rank histories equal up to +-1 at a truncation (a different
    summation order may flip a marginal cut), residual histories equal to the 6 printed digits."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    reps = []
    for v in ("1", "0"):
        env = dict(os.environ, FC_STREAMK=v)
        out = subprocess.run([sys.executable, os.path.join(root, "tools", "c4_trace.py"), "1e-6", "1024"],
                             env=env, capture_output=True, text=True, timeout=600)
        assert out.returncode == 0, out.stderr[-2000:]
        reps.append(json.loads(next(l for l in out.stdout.splitlines() if l.startswith("{"))))
    a, b = reps
    assert a["rc"] == 0 and b["rc"] == 0 and a["iters"] == b["iters"]
    assert max(a["tucker_S"]) > 64, "the workload no longer reaches the stream-K Gram path"
    for k in ("rank_X", "rank_R", "rank_S", "rank_Z", "rank_P"):
        assert all(abs(x - y) <= 1 for x, y in zip(a[k], b[k])), (k, a[k], b[k])
    assert np.allclose(a["rel_res"], b["rel_res"], rtol=1e-5, atol=0.0)
