"""Shared helpers of the GPU parity tests (test infrastructure; imports the oracle).

Shared-input parity: the oracle's PCG needs only the 1D eigenpairs (lambda, V)
and the spectral CPs F and G.  At BASELINE.json's full sizes the oracle's own setup is
infeasible (its spectral CP materialises n^3 entries of D), so the device-built inputs are
exported through the C-ABI (sl_get_eigen, op_get_spectral_cp) and both sides run Algorithm 1
[P:1825-1872] on the same bytes."""
import numpy as np
import pytest

from oracle import cp as cpm
from oracle import pcg as P

MARGIN_BAND = 5e-3   # relative distance of thr to a bracketing tail below which a cut is marginal (A23)
CANCEL_RES = 1e-4    # below this relative residual, R - a S cancels ~1/rel_res of its magnitude


def device_setup_to_oracle(ctx, p, params):
    """sl_setup on the device, then the same eigenpairs / spectral CPs as an oracle Setup."""
    from paper_2006_09314_b200.binding import FC_F, FC_G
    ctx.sl_setup(p.n, p.a_mid, params)
    lams, V = [], []
    for l in range(3):
        lam, Vl = ctx.sl_get_eigen(l)
        lams.append(lam.cpu().numpy())
        V.append(Vl.cpu().numpy())
    Fw, FU = ctx.op_get_spectral_cp(FC_F).to_numpy()
    Gw, GU = ctx.op_get_spectral_cp(FC_G).to_numpy()
    return P.Setup(lams, V, cpm.CP(Fw, FU), cpm.CP(Gw, GU))


def as_cp(y):
    w, U = y.to_numpy()
    return cpm.CP(w, U)


def check_rank_history(rep, rep_ref, label="", floor_rank=None):
    """Ranks equal truncation by truncation (S, X, R, Z, P of every iteration, in Algorithm 1's
    order) and rel_res within 1e-5 relative, for the whole solve, unless ONE justified exit fires
    at the first differing rank:
      * "marginal": the oracle logged a cut inside the A23 noise band (|tail - thr| < MARGIN_BAND
        thr) at or before that truncation (both sides then legitimately keep different ranks);
      * "cancellation": rel_res < CANCEL_RES, where R - a S cancels ~1/rel_res of its
        magnitude, and the ranks differ by <= max(2, 1 %);
      * "floor" (only with floor_rank, e.g. 0.95 n^2 at tiny n): the T2C keeps essentially every
        one of its n^2 candidates and the ranks differ by one — the last candidate's singular value
        is at the accuracy floor of the two slice-SVD implementations (the device drops triples
        below 1e-12 of the slice norm, reading "negligible slice columns").
    After an exit the two runs are different, equally valid rank sequences: only the iteration
    count (+-1) and the final control are compared by the caller.  Returns (exit, at) and prints
    which exit fired (None: every truncation of the solve matched)."""
    m = rep_ref["margins"]          # order: Z0, then per iteration S, X, R, Z, P
    keys = (("rank_S", 0), ("rank_X", 1), ("rank_R", 2), ("rank_Z", 3), ("rank_P", 4))
    exit_, at = None, None
    n_it = min(rep["iters"], rep_ref["iters"])
    compared = 0
    for k in range(n_it):
        base = 1 + 5 * k
        cancel = k > 0 and rep_ref["rel_res"][k - 1] < CANCEL_RES
        for key, off in keys:
            if k >= len(rep_ref[key]) or k >= len(rep[key]):
                continue
            a, b = rep[key][k], rep_ref[key][k]
            compared += 1
            if a == b:
                continue
            if min(m[:base + off + 1]) < MARGIN_BAND:
                exit_ = "marginal"
            elif cancel and abs(a - b) <= max(2, 0.01 * b):
                exit_ = "cancellation"
            elif floor_rank is not None and abs(a - b) == 1 and b >= floor_rank:
                exit_ = "floor"
            else:
                raise AssertionError(f"{label} {key}[{k}]: device {a} oracle {b}, oracle margin "
                                     f"{m[base + off] if base + off < len(m) else None}")
            at = (k, key)
            break
        if exit_ is not None:
            break
        assert rep["rel_res"][k] == pytest.approx(rep_ref["rel_res"][k], rel=1e-5), (label, k)
    print(f"[rank history {label}] {compared} truncations compared over {n_it} iterations, exit: {exit_} at {at}")
    if exit_ is None:
        assert rep["iters"] == rep_ref["iters"]
    else:
        assert abs(rep["iters"] - rep_ref["iters"]) <= 1
    return exit_, at


EPS_MACH = 2.220446049250313e-16


def trunc_tolerance(info_o, eps, tight=None):
    """Single-truncation parity bar: max(1e-10, 10 eps_mach / eps) relative, unless
    the oracle logged a cut inside the A23 band (a T2C near-tie or a marginal mode cut), where the
    two sides may keep different members of a tie and differ by up to the dropped singular value
    (< eps/2, reading A25).  The 10 eps_mach / eps term: the device takes the leading singular
    vectors of a side matrix from its Gram, whose eigenvectors carry an angle error
    ~eps_mach lambda_0 / gap; at the last kept direction (sigma_r ~ eps sigma_0, gap ~ sigma_r^2)
    that moves the result by ~eps_mach / eps of its norm (2e-10 at eps = 1e-6)."""
    if tight is None:
        tight = max(1e-10, 10.0 * EPS_MACH / eps)
    marg = min(info_o.get("margins", [np.inf]) or [np.inf])
    return (eps if marg < MARGIN_BAND else tight), marg
