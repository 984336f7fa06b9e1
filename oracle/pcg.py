"""O10 Algorithm 1 (PCG in low-rank format) and O11 report; plus the setup chain
O1-O5 for a `synth.Problem`.  (Oracle: test-only.)

Algorithm 1 [P:1825-1872], verbatim line by line, with the readings:
A13 stop when ||R^{k+1}|| / ||B|| <= tol_stop (tol_stop = 10 eps), A14 X^0 = 0,
A15 R^0 = B untruncated, A16 beta_k's denominator reuses <R^k, Z^k>, A17 k_max = 100.
Scalars are named a_k, b_k so they cannot clash with the operator's alpha, beta.
"""
from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

from . import cp as cpm
from .cp import CP
from .sturm import dst1_basis, effective_midpoints, eigenpairs, laplace_eigenvalues
from .spectral import FC_F, FC_G, FC_POW_MINUS, spectral_cp
from .truncate import truncate


@dataclass
class Setup:
    lams: list
    V: list
    F: CP
    G: CP
    info: dict = field(default_factory=dict)
    lamsG: list = None         # eigenvalues G is a function of (= lams in case (B))
    VG: list = None            # basis G is applied in (= V in case (B))


def precond_basis_A(problem):
    """Case (A) [P:842-849]: b0_l = (max a_l + min a_l)/2 over the coefficient values the operator
    uses (majorant / minorant on the grid, A2's effective midpoints); B = sum_l b0_l (1D Laplacian)
    is diagonal in the DST-I basis [P:778-785]: lam_k = b0_l 4/h^2 sin^2(k pi h/2).
    Returns (b0, lams, V)."""
    b0, lams, V = [], [], []
    for l in range(3):
        a = effective_midpoints(problem.a_mid[l], problem.boundary)
        b0.append(0.5 * (a.max() + a.min()))
        lams.append(b0[-1] * laplace_eigenvalues(problem.n))
        V.append(dst1_basis(problem.n))
    return b0, lams, V


def setup(problem, F_rank=None, G_rank=None, eps_D=None) -> Setup:
    """sl_setup: O2/O3 per mode, then O5 for F (eps_D-driven) and G (rank r_G, SPD guard);
    in case (A) G = 1/F over the b0-Laplacian's eigenvalues, applied in the DST-I basis."""
    lams, V = [], []
    for l in range(3):
        lam, Vl = eigenpairs(problem.a_mid[l], problem.boundary)
        lams.append(lam)
        V.append(Vl)
    eps_D = problem.eps if eps_D is None else eps_D
    infoF, infoG = {}, {}
    F = spectral_cp(lams, FC_F, problem.alpha, problem.beta, eps_D, rank=F_rank, info=infoF)
    lamsG, VG = lams, V
    if getattr(problem, "precond", "B") == "A":
        _, lamsG, VG = precond_basis_A(problem)
    G = spectral_cp(lamsG, FC_G, problem.alpha, problem.beta, eps_D,
                    rank=problem.precond_rank if G_rank is None else G_rank,
                    spd_guard=True, info=infoG)
    return Setup(lams, V, F, G, {"F": infoF, "G": infoG}, lamsG, VG)


class NotSPD(RuntimeError):
    pass


def pcg(fun, precond, B: CP, eps: float, tol_stop: float, kmax: int = 100, trunc=None,
        rank_cap: int | None = None):
    """Algorithm 1.  fun/precond: CP -> CP (untruncated applies); trunc(x, eps) -> CP.
    rank_cap (A26): every truncation keeps at most rank_cap T2C triples; rep["cap_hits"] counts
    the truncations that were clipped."""
    rep = {"rel_res": [], "rank_X": [], "rank_R": [], "rank_Z": [], "rank_P": [],
           "rank_S": [], "t_iter": [], "converged": False, "iters": 0, "margins": [],
           "cap_hits": 0}
    if trunc is None:
        def trunc(x, e):                                      # logs the cut margins (A23)
            info = {}
            y = truncate(x, e, info, rank_cap=rank_cap)
            rep["margins"].append(min(info.get("margins", [np.inf]) or [np.inf]))
            rep["cap_hits"] += int(info.get("clipped", False))
            return y
    normB = cpm.norm(B)
    X = cpm.zeros(B.shape)                                   # X^(0) = 0          (A14)
    R = B.copy()                                             # line 1, R^0 = B    (A15)
    Z = trunc(precond(R), eps)                               # lines 2-3
    P = Z.copy()                                             # line 4
    rz = cpm.dot(R, Z)
    for k in range(kmax):                                    # lines 6..21
        t0 = time.perf_counter()
        S = trunc(fun(P), eps)                               # lines 7-8
        ps = cpm.dot(P, S)
        if not np.isfinite(ps) or ps <= 0:
            raise NotSPD(f"<P,S> = {ps} at iteration {k}")
        a_k = rz / ps                                        # line 9
        X = trunc(cpm.axpy(X, a_k, P), eps)                  # lines 10-11
        R = trunc(cpm.axpy(R, -a_k, S), eps)                 # lines 12-13
        rel = np.sqrt(max(cpm.dot(R, R), 0.0)) / normB       # line 14 (A13)
        rep["rel_res"].append(rel)
        rep["rank_S"].append(S.rank); rep["rank_X"].append(X.rank); rep["rank_R"].append(R.rank)
        rep["iters"] = k + 1
        if rel <= tol_stop:
            rep["converged"] = True
            rep["rank_Z"].append(Z.rank); rep["rank_P"].append(P.rank)
            rep["t_iter"].append(time.perf_counter() - t0)
            return X, rep
        Z = trunc(precond(R), eps)                           # lines 17-18
        rz_new = cpm.dot(R, Z)
        b_k = rz_new / rz                                    # line 19 (A16)
        P = trunc(cpm.axpy(Z, b_k, P), eps)                  # lines 20-21
        rz = rz_new
        rep["rank_Z"].append(Z.rank); rep["rank_P"].append(P.rank)
        rep["t_iter"].append(time.perf_counter() - t0)
    return X, rep


def solve(problem, st: Setup | None = None, kmax=None, with_true_residual=False, rank_cap=None):
    """pcg_solve for a synth.Problem: returns (u, report, setup)."""
    st = setup(problem) if st is None else st
    B = cpm.normalized(problem.b_w, problem.b_U)
    fun = lambda x: cpm.apply(st.V, st.F, x)
    pre = lambda x: cpm.apply(st.VG if st.VG is not None else st.V, st.G, x)
    u, rep = pcg(fun, pre, B, problem.eps, problem.tol_stop,
                 problem.kmax if kmax is None else kmax, rank_cap=rank_cap)
    if with_true_residual:                                   # O11
        from .measure import diff_norm
        rep["true_residual"] = diff_norm(fun(u), B) / cpm.norm(B)
    return u, rep, st


def state_cp(problem, st: Setup, eps_D=None) -> CP:
    """Spectral CP of lam^-alpha (FC_POW_MINUS) on the SL eigenvalues, eps_D-driven (O5)."""
    eps_D = problem.eps if eps_D is None else eps_D
    return spectral_cp(st.lams, FC_POW_MINUS, problem.alpha, problem.beta, eps_D)


def state(problem, st: Setup, u: CP, Pm: CP | None = None) -> CP:
    """State recovery [P:287-289, P:969-972]: y = beta_paper A^-alpha u; with reading A5
    (beta_paper = 1) y = A^-alpha u, truncated at eps (O6 apply, O9 truncate)."""
    Pm = state_cp(problem, st) if Pm is None else Pm
    return truncate(cpm.apply(st.V, Pm, u), problem.eps)
