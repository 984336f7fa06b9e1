"""O4 spectral functions and O5 the spectral-diagonal CP.  (Oracle: test-only.)

The operator F(A) = (G1^T (x) G2^T (x) G3^T) F(Lambda) (G1 (x) G2 (x) G3) [P:706-716] is
fixed by the coefficient tensor D[i,j,k] = F(lam1_i + lam2_j + lam3_k) [P:666-694]; its
canonical approximation D ~ sum_k w_k u1_k (x) u2_k (x) u3_k is built by the
full-to-Tucker-to-canonical algorithm [P:720-722, P:1775-1789, P:1802-1812].  Readings:
A5 (F = beta*lam^alpha + lam^-alpha), A6/A7 (preconditioner G = 1/F, rank r_G = 6, SPD
guard), A8 (eps_D = eps), A9 (the oracle materialises D and runs a full HOSVD).
"""
from __future__ import annotations

import numpy as np

from .cp import CP
from .truncate import rank_cut, tucker_to_canonical

FC_F, FC_G, FC_POW_PLUS, FC_POW_MINUS, FC_LAMBDA, FC_ONE = 0, 1, 2, 3, 4, 5


def spectral_fn(kind: int, alpha: float, beta: float):
    """O4 [P:640-648] (mapped per A5): F = beta lam^a + lam^-a, G = 1/F, POW+- = lam^+-a."""
    if kind == FC_F:
        return lambda lam: beta * np.power(lam, alpha) + np.power(lam, -alpha)
    if kind == FC_G:
        return lambda lam: 1.0 / (beta * np.power(lam, alpha) + np.power(lam, -alpha))
    if kind == FC_POW_PLUS:
        return lambda lam: np.power(lam, alpha)
    if kind == FC_POW_MINUS:
        return lambda lam: np.power(lam, -alpha)
    if kind == FC_LAMBDA:
        return lambda lam: lam
    if kind == FC_ONE:
        return lambda lam: np.ones_like(lam)
    raise ValueError(kind)


def lambda_sum(lams) -> np.ndarray:
    """lam1_i + lam2_j + lam3_k formed as (lam1_i + lam2_j) + lam3_k (O4 order) [P:684]."""
    l1, l2, l3 = lams
    return (l1[:, None, None] + l2[None, :, None]) + l3[None, None, :]


def coefficient_tensor(lams, kind, alpha, beta) -> np.ndarray:
    """D[i,j,k] = F(lam1_i + lam2_j + lam3_k) [P:693] (materialised; n <= 256)."""
    return spectral_fn(kind, alpha, beta)(lambda_sum(lams))


def hosvd(D: np.ndarray, eps: float):
    """Full-to-Tucker: per-mode SVD of the unfoldings, r_l minimal with
    sum_{k>r} s^2 <= (eps^2/3)||D||^2, core = D x_l Z_l^T [P:1720-1737]."""
    nD2 = float(np.sum(D * D))
    Z = []
    for l in range(3):
        Dl = np.moveaxis(D, l, 0).reshape(D.shape[l], -1)
        Uf, s, _ = np.linalg.svd(Dl, full_matrices=False)
        r = rank_cut(s ** 2, eps * eps / 3.0 * nD2)
        Z.append(Uf[:, :r])
    core = np.einsum("ijk,ia,jb,kc->abc", D, Z[0], Z[1], Z[2])
    return core, Z


def cp_min_entry(x: CP) -> float:
    return float(np.min(np.einsum("k,ik,jk,lk->ijl", x.w, x.U[0], x.U[1], x.U[2])))


def spectral_cp(lams, kind: int, alpha: float, beta: float, eps: float,
                rank: int | None = None, spd_guard: bool = False, info: dict | None = None) -> CP:
    """O5: CP of D = F(lambda-sum): HOSVD at eps, then T2C (cut (eps/2) or top `rank`).

    SPD guard (readings A7/A7'/A7''): when `spd_guard`, the rank is raised (up to 64), then the
    Tucker tolerance tightened (down to eps/1e4), until the CP is positive on the whole grid;
    failing that, a constant term 2|min| + 1e-15 sum|w| makes it positive.
    """
    D = coefficient_tensor(lams, kind, alpha, beta)
    core, Z = hosvd(D, eps)
    if info is not None:
        info["tucker_rank"] = [z.shape[1] for z in Z]
    if rank is None:
        out = tucker_to_canonical(core, Z, eps)
    else:
        r = rank
        out = tucker_to_canonical(core, Z, None, keep=r)
        if spd_guard:
            # reading A7': raise the T2C rank (up to 64) until the CP is positive on the grid;
            # if the Tucker approximation itself is not positive at that accuracy, tighten its
            # tolerance tenfold and repeat (up to eps/1e4)
            e = eps
            shift = 0.0
            while (mn := cp_min_entry(out)) <= 0:
                if r < min(64, int(np.prod(core.shape))):
                    r += 1
                elif e > eps * 1e-4:
                    e /= 10.0
                    core, Z = hosvd(D, e)
                    r = rank
                else:
                    # reading A7'': still not positive (entries of D spanning many decades keep
                    # a rounding-level negative lobe): add the constant s (x) 1 (x) 1 (x) 1 with
                    # s = 2|min| + 1e-15 sum|w|  (sum|w| bounds the largest entry)
                    shift = 2.0 * abs(mn) + 1e-15 * float(np.sum(np.abs(out.w)))
                    n1 = [u.shape[0] for u in out.U]
                    one = [np.full((k, 1), 1.0 / np.sqrt(k)) for k in n1]
                    out = CP(np.append(out.w, shift * np.sqrt(float(np.prod(n1)))),
                             [np.hstack([u, o]) for u, o in zip(out.U, one)])
                    break
                out = tucker_to_canonical(core, Z, None, keep=r)
            if info is not None:
                info["guard_eps"] = e
                info["guard_shift"] = shift
    if info is not None:
        info["rank"] = out.rank
        diff = np.einsum("k,ik,jk,lk->ijl", out.w, out.U[0], out.U[1], out.U[2]) - D
        info["max_abs_err"] = float(np.max(np.abs(diff)))
        info["max_F"] = float(np.max(np.abs(D)))
        info["fro_rel_err"] = float(np.linalg.norm(diff) / np.linalg.norm(D))
    return out


def exact_spectral_cp(lams, kind, alpha, beta) -> CP:
    """The exact rank-n^2 CP of D: D = sum_{j,k} D[:, j, k] (x) e_j (x) e_k (tiny n)."""
    D = coefficient_tensor(lams, kind, alpha, beta)
    n1, n2, n3 = D.shape
    U1 = D.reshape(n1, n2 * n3)
    U2 = np.repeat(np.eye(n2), n3, axis=1)
    U3 = np.tile(np.eye(n3), (1, n2))
    nrm = np.linalg.norm(U1, axis=0)
    return CP(nrm.copy(), [U1 / nrm, U2, U3])
