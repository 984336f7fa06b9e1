"""O9: rank truncation trunc(x, eps) = RHOSVD (canonical-to-Tucker) + Tucker-to-canonical.
(Oracle: test-only.)

Paper: "reduced HOSVD (RHOSVD) ... does not require the construction of a full size
tensor", complexity O(d n^2 R) [P:1791-1796]; C2T combined with the Tucker-to-canonical
transform for a mixed Tucker-canonical core, canonical rank R <= r^2 in 3D [P:1802-1816];
"controlled by the given eps-threshold" [P:187-190]; used for d = 3 in Algorithm 1
[P:973-976, 1873-1876].  Readings: A10 (slice-SVD T2C along the min-rank
mode), A11 (side matrix U_l diag(xi), per-mode cut (eps/2)^2 sum xi^2), A12 (relative),
A23 (ties kept together; tails summed from the small end).
"""
from __future__ import annotations

import numpy as np

from .cp import CP, zeros


def tail_sums(s2: np.ndarray) -> np.ndarray:
    """t[r] = sum_{k >= r} s2[k] for r = 0..len (t[len] = 0), summed from the small end.

    s2 is sorted descending, so the running sum starts at the smallest value.
    """
    t = np.zeros(s2.size + 1)
    acc = 0.0
    for k in range(s2.size - 1, -1, -1):
        acc += s2[k]
        t[k] = acc
    return t


def rank_cut(s2: np.ndarray, thr: float, rmin: int = 1, margins: list | None = None) -> int:
    """min{ r >= rmin : sum_{k > r} s2_k <= thr }, ties at the cut kept together (A23).

    `margins` (logging only) receives the relative distance of thr to the two tails that
    bracket the decision, min(|t[r]-thr|, |t[r-1]-thr|)/thr: a small value marks a cut that
    rounding differences between two implementations may flip (the noise band of A23)."""
    t = tail_sums(s2)
    r = rmin
    while r < s2.size and t[r] > thr:
        r += 1
    while 0 < r < s2.size and s2[r] == s2[r - 1] and s2[r] > 0:   # A23: zero terms never bind
        r += 1
    r = min(r, s2.size)
    if margins is not None and thr > 0:
        m = abs(t[r] - thr) / thr
        if r - 1 >= rmin:
            m = min(m, abs(t[r - 1] - thr) / thr)
        margins.append(m)
    return r


def tucker_to_canonical(core: np.ndarray, Z: list, eps: float | None, keep: int | None = None,
                        info: dict | None = None, rank_cap: int | None = None) -> CP:
    """T2C of the Tucker tensor core x_1 Z1 x_2 Z2 x_3 Z3 [P:1804-1812] (reading A10).

    Slice along the min-rank mode c (ties -> lowest mode); a < b are the other modes.
    SVD of every slice core(:,:,nu) (r_a x r_b); pool (s, nu, m); sort by s descending,
    ties by (nu, m); keep the smallest R with sum_{dropped} s^2 <= (eps/2)^2 ||core||_F^2
    (or the top `keep` triples).  Output factors Z_a a_m, Z_b b_m, Z_c[:, nu], weight s.
    rank_cap (reading A26, the rank cap of Algorithm 1's iterates): R = min(R, rank_cap), i.e.
    the top rank_cap triples of the pooled order; info["clipped"] records it.
    """
    r = core.shape
    c = int(np.argmin(r))
    a, b = [l for l in range(3) if l != c]
    cp_ = np.moveaxis(core, (a, b, c), (0, 1, 2))
    trip = []
    for nu in range(r[c]):
        Ua, s, Vbt = np.linalg.svd(cp_[:, :, nu], full_matrices=False)
        for m in range(s.size):
            trip.append((s[m], nu, m, Ua[:, m], Vbt[m, :]))
    trip.sort(key=lambda t: (-t[0], t[1], t[2]))
    s_all = np.array([t[0] for t in trip])
    nb2 = float(np.sum(core * core))
    if nb2 == 0.0:
        return zeros(tuple(z.shape[0] for z in Z))
    margins = info.setdefault("margins", []) if info is not None else None
    if keep is not None:
        R = min(keep, len(trip))
    else:
        R = rank_cut(s_all ** 2, (eps / 2.0) ** 2 * nb2, margins=margins)
    clipped = rank_cap is not None and R > rank_cap
    if clipped:
        R = rank_cap
    if info is not None:
        info["clipped"] = clipped
        info["t2c_mode"] = c
        info["t2c_candidates"] = len(trip)
        info["out_rank"] = R
    U = [None, None, None]
    U[a] = np.stack([Z[a] @ t[3] for t in trip[:R]], axis=1)
    U[b] = np.stack([Z[b] @ t[4] for t in trip[:R]], axis=1)
    U[c] = np.stack([Z[c][:, t[1]] for t in trip[:R]], axis=1)
    return CP(s_all[:R].copy(), U)


def truncate(x: CP, eps: float, info: dict | None = None, rank_cap: int | None = None) -> CP:
    """O9 steps 1-5 (RHOSVD -> core -> T2C); rank_cap: see tucker_to_canonical (A26)."""
    # 1. drop terms with zero weight or a zero column
    keep = x.w != 0
    for l in range(3):
        keep &= np.any(x.U[l] != 0, axis=0)
    if not np.any(keep):
        return zeros(x.shape)
    w = x.w[keep]
    U = [u[:, keep] for u in x.U]
    E = float(np.sum(w * w))
    thr = (eps / 2.0) ** 2 * E
    Z, C, ranks = [], [], []
    margins = info.setdefault("margins", []) if info is not None else None
    for l in range(3):
        A = U[l] * w[None, :]                                  # side matrix U_l diag(xi)
        Zf, s, _ = np.linalg.svd(A, full_matrices=False)       # 2. singular values
        r = rank_cut(s ** 2, thr, margins=margins)             # 3. tail from the small end
        Z.append(Zf[:, :r])                                    # 4. Z_l
        C.append(Z[-1].T @ U[l])                               #    C_l = Z_l^T U_l
        ranks.append(r)
    core = np.einsum("t,at,bt,ct->abc", w, C[0], C[1], C[2])   # 4. beta
    if info is not None:
        info["tucker_rank"] = ranks
    return tucker_to_canonical(core, Z, eps, info=info, rank_cap=rank_cap)   # 5. T2C
