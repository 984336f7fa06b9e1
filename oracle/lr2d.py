"""2D variant of the method: rank-structured PCG for the 2D control
equation (beta A^alpha + A^-alpha) u = b, A = T1 (x) I + I (x) T2 [P:449-452 with d = 2],
with the reduced-SVD truncation the paper uses for d = 2 [P:973-976].  (Oracle: test-only;
imports nothing from the CUDA path.)

Format [P:585-595]: x = sum_k w_k u1_k (x) u2_k, i.e. the n1 x n2 matrix X = U1 diag(w) U2^T,
unit columns, signed weights (reading A18).

  apply   F(A) x = sum_k sum_j G1^T (u1_k . G1 x1_j) (x) G2^T (u2_k . G2 x2_j)   [P:597-611]
          (G_l = V_l^T; term order t = k*R + j, reading A19; rank r*R, untruncated)
  trunc   reduced SVD [P:973-976]: the result is the truncated SVD of X (Eckart-Young), so
          the oracle takes the plain definition: SVD of the dense X, smallest r with
          sum_{k>r} s_k^2 <= eps^2 sum_k s_k^2 (reading 2D-T: one stage, relative Frobenius
          error eps; ties and zeros as A23)
  spectral  D2[i, j] = F(lam1_i + lam2_j) [P:693 with d = 2]; its low-rank factorisation is
          the truncated SVD of D2 with the same tail rule at eps_D (reading 2D-S), or the top
          `rank` terms for the preconditioner G = 1/F with the SPD guard of A7'/A7'' (rank
          raised to <= 64 while an entry is <= 0, then the constant-shift term)
  pcg     Algorithm 1 [P:1825-1872] verbatim, as oracle.pcg.pcg, with these 2D operations.
"""
from __future__ import annotations

from dataclasses import dataclass
import time

import numpy as np

from .spectral import spectral_fn, FC_F, FC_G
from .sturm import eigenpairs
from .truncate import rank_cut


@dataclass
class LR2:
    w: np.ndarray            # (R,)
    U: list                  # 2 arrays (n_l, R)

    @property
    def rank(self) -> int:
        return int(self.w.size)

    @property
    def shape(self):
        return tuple(u.shape[0] for u in self.U)

    def copy(self) -> "LR2":
        return LR2(self.w.copy(), [u.copy() for u in self.U])


def zeros2(shape) -> LR2:
    return LR2(np.zeros(0), [np.zeros((n, 0)) for n in shape])


def normalized2(w, U) -> LR2:
    """Fold column norms into the weights (unit-column convention [P:1711])."""
    w = np.asarray(w, dtype=np.float64).copy()
    U = [np.array(u, dtype=np.float64, copy=True) for u in U]
    for l in range(2):
        nrm = np.linalg.norm(U[l], axis=0)
        U[l] = U[l] / np.where(nrm > 0, nrm, 1.0)
        w = w * nrm
    return LR2(w, U)


def full2(x: LR2) -> np.ndarray:
    """X = U1 diag(w) U2^T."""
    return (x.U[0] * x.w[None, :]) @ x.U[1].T


def dot2(x: LR2, y: LR2) -> float:
    """<x, y> = sum_{k,m} w_k v_m <u1_k, y1_m> <u2_k, y2_m> [P:1748-1755 with d = 2]."""
    if x.rank == 0 or y.rank == 0:
        return 0.0
    H = (x.U[0].T @ y.U[0]) * (x.U[1].T @ y.U[1])
    return float(x.w @ H @ y.w)


def norm2(x: LR2) -> float:
    return float(np.sqrt(max(dot2(x, x), 0.0)))


def axpy2(x: LR2, a: float, y: LR2) -> LR2:
    """x + a*y by concatenation [x terms ; a*y terms] [P:1845-1866]."""
    return LR2(np.concatenate([x.w, a * y.w]), [np.concatenate([x.U[l], y.U[l]], axis=1) for l in range(2)])


def truncate2(x: LR2, eps: float, info: dict | None = None) -> LR2:
    """Reduced SVD truncation [P:973-976] = truncated SVD of the dense X (reading 2D-T)."""
    n1, n2 = x.shape
    if x.rank == 0:
        if info is not None:
            info.update(rank=0, margins=[])
        return zeros2((n1, n2))
    X = full2(x)
    Uf, s, Vt = np.linalg.svd(X, full_matrices=False)
    s2 = s * s
    margins = []
    r = rank_cut(s2, eps * eps * float(np.sum(s2)), margins=margins)
    if info is not None:
        info.update(rank=r, margins=margins, energy=float(np.sum(s2)))
    if s2.sum() == 0.0:
        return zeros2((n1, n2))
    return LR2(s[:r].copy(), [Uf[:, :r].copy(), Vt[:r].T.copy()])


def apply2(V: list, spec: LR2, x: LR2) -> LR2:
    """F(A) x in factored form [P:597-611]: per mode W = V^T X (forward), Yhat[:, k*R+j] =
    u_k . W[:, j] (Hadamard), Y = V Yhat (inverse); weights w_F[k] w_j; columns normalised."""
    if x.rank == 0:
        return zeros2(x.shape)
    r, R = spec.rank, x.rank
    U = []
    for l in range(2):
        W = V[l].T @ x.U[l]
        Yh = (spec.U[l][:, :, None] * W[:, None, :]).reshape(-1, r * R)
        U.append(V[l] @ Yh)
    return normalized2(np.outer(spec.w, x.w).reshape(-1), U)


def coefficient_matrix(lams, kind: int, alpha: float, beta: float) -> np.ndarray:
    """D2[i, j] = F(lam1_i + lam2_j) [P:693 with d = 2]."""
    return spectral_fn(kind, alpha, beta)(lams[0][:, None] + lams[1][None, :])


def spectral2(lams, kind: int, alpha: float, beta: float, eps: float, rank: int | None = None,
              spd_guard: bool = False, info: dict | None = None) -> LR2:
    """Low-rank factorisation of D2 (reading 2D-S): truncated SVD at eps (tail rule of
    truncate2), or the top `rank` terms; SPD guard as A7'/A7'' (rank <= 64, then a shift)."""
    D = coefficient_matrix(lams, kind, alpha, beta)
    Uf, s, Vt = np.linalg.svd(D, full_matrices=False)
    s2 = s * s
    r = rank_cut(s2, eps * eps * float(np.sum(s2))) if rank is None else min(rank, s.size)
    shift = 0.0
    if spd_guard:
        while True:
            mn = float(np.min((Uf[:, :r] * s[None, :r]) @ Vt[:r]))
            if mn > 0.0:
                break
            if r < min(64, s.size):
                r += 1
                continue
            shift = 2.0 * abs(mn) + 1e-15 * float(np.sum(np.abs(s[:r])))
            break
    out = LR2(s[:r].copy(), [Uf[:, :r].copy(), Vt[:r].T.copy()])
    if shift > 0.0:
        n1, n2 = D.shape
        one = LR2(np.array([shift * np.sqrt(n1 * n2)]),
                  [np.full((n1, 1), 1.0 / np.sqrt(n1)), np.full((n2, 1), 1.0 / np.sqrt(n2))])
        out = axpy2(out, 1.0, one)
    if info is not None:
        info.update(rank=out.rank, shift=shift,
                    rel_err=float(np.linalg.norm(D - full2(out)) / np.linalg.norm(D)))
    return out


@dataclass
class Setup2:
    lams: list
    V: list
    F: LR2
    G: LR2


def setup2(problem, F_rank=None, G_rank=None, eps_D=None) -> Setup2:
    """Eigenpairs of modes 1, 2 (O1-O3 on a_mid[0], a_mid[1]) and the spectral factorisations
    of F (eps_D) and G (rank r_G, SPD guard)."""
    eps_D = problem.eps if eps_D is None else eps_D
    lams, V = [], []
    for l in range(2):
        lam, Vl = eigenpairs(problem.a_mid[l], problem.boundary)
        lams.append(lam)
        V.append(Vl)
    F = spectral2(lams, FC_F, problem.alpha, problem.beta, eps_D, rank=F_rank)
    G = spectral2(lams, FC_G, problem.alpha, problem.beta, eps_D,
                  rank=problem.precond_rank if G_rank is None else G_rank, spd_guard=True)
    return Setup2(lams, V, F, G)


class NotSPD(RuntimeError):
    pass


def pcg2(fun, precond, B: LR2, eps: float, tol_stop: float, kmax: int = 100):
    """Algorithm 1 [P:1825-1872] with trunc = truncate2 (readings A13-A17 as in 3D)."""
    rep = {"rel_res": [], "rank_X": [], "rank_R": [], "rank_Z": [], "rank_P": [],
           "rank_S": [], "t_iter": [], "converged": False, "iters": 0, "margins": []}

    def trunc(x, e):
        info = {}
        y = truncate2(x, e, info)
        rep["margins"].append(min(info.get("margins", [np.inf]) or [np.inf]))
        return y

    normB = norm2(B)
    X = zeros2(B.shape)                                      # A14
    R = B.copy()                                             # A15
    Z = trunc(precond(R), eps)                               # lines 2-3
    P = Z.copy()                                             # line 4
    rz = dot2(R, Z)
    for k in range(kmax):
        t0 = time.perf_counter()
        S = trunc(fun(P), eps)                               # lines 7-8
        ps = dot2(P, S)
        if not np.isfinite(ps) or ps <= 0:
            raise NotSPD(f"<P,S> = {ps} at iteration {k}")
        a_k = rz / ps                                        # line 9
        X = trunc(axpy2(X, a_k, P), eps)                     # lines 10-11
        R = trunc(axpy2(R, -a_k, S), eps)                    # lines 12-13
        rel = np.sqrt(max(dot2(R, R), 0.0)) / normB          # line 14
        rep["rel_res"].append(rel)
        rep["rank_S"].append(S.rank); rep["rank_X"].append(X.rank); rep["rank_R"].append(R.rank)
        rep["iters"] = k + 1
        if rel <= tol_stop:
            rep["converged"] = True
            rep["rank_Z"].append(Z.rank); rep["rank_P"].append(P.rank)
            rep["t_iter"].append(time.perf_counter() - t0)
            return X, rep
        Z = trunc(precond(R), eps)                           # lines 17-18
        rz_new = dot2(R, Z)
        b_k = rz_new / rz                                    # line 19 (A16)
        P = trunc(axpy2(Z, b_k, P), eps)                     # lines 20-21
        rz = rz_new
        rep["rank_Z"].append(Z.rank); rep["rank_P"].append(P.rank)
        rep["t_iter"].append(time.perf_counter() - t0)
    return X, rep


def solve2(problem, st: Setup2 | None = None, kmax=None):
    """pcg_solve_2d for a synth.Problem2: returns (u, report, setup)."""
    st = setup2(problem) if st is None else st
    B = normalized2(problem.b_w, problem.b_U)
    fun = lambda x: apply2(st.V, st.F, x)
    pre = lambda x: apply2(st.V, st.G, x)
    u, rep = pcg2(fun, pre, B, problem.eps, problem.tol_stop, problem.kmax if kmax is None else kmax)
    return u, rep, st
