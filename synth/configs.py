"""BASELINE.json configs C1..C5 as seeded synthetic inputs (SURVEY.md §8(d) recipe).

Grid convention (reading A1): n interior points, h = 1/(n+1), x_i = i*h for
i = 1..n, midpoints x_{i+1/2} = (i+1/2)*h for i = 0..n.  The coefficient a_l is sampled at
the n+1 midpoints; that is the `a_mid` array handed to `sl_setup` [P:471-472].

Right-hand sides are canonical (CP) tensors b = sum_t w_t u1_t (x) u2_t (x) u3_t with unit
columns (the format convention of [P:1706-1712]); `normalize_cp` only moves column norms
into the weights.  The paper's own H-type design function exists only as a figure
[P:1024-1032], so these seeded shapes stand in for it.
"""
from __future__ import annotations

from dataclasses import dataclass, field
import numpy as np

TWO_PI = 2.0 * np.pi


def grid_points(n: int) -> np.ndarray:
    """x_i = i/(n+1), i = 1..n (interior Dirichlet grid)."""
    return np.arange(1, n + 1, dtype=np.float64) / (n + 1)


def midpoints(n: int) -> np.ndarray:
    """x_{i+1/2} = (i+1/2)/(n+1), i = 0..n."""
    return (np.arange(0, n + 1, dtype=np.float64) + 0.5) / (n + 1)


def normalize_cp(w, U):
    """Return (w', U') with unit columns; column norms are folded into the weights."""
    w = np.asarray(w, dtype=np.float64).copy()
    U = [np.array(u, dtype=np.float64, copy=True) for u in U]
    for l in range(len(U)):
        nrm = np.linalg.norm(U[l], axis=0)
        U[l] = U[l] / np.where(nrm > 0, nrm, 1.0)
        w = w * nrm
    return w, U


def random_cp(n: int, R: int, seed: int):
    """iid N(0,1) factor entries per (term, mode), columns normalised, weights 1 [BJ C3/C5]."""
    rng = np.random.default_rng(seed)
    U = [rng.standard_normal((n, R)) for _ in range(3)]
    for l in range(3):
        U[l] /= np.linalg.norm(U[l], axis=0)
    return np.ones(R), U


# ---- coefficient families -------------------------------------------------------------

def _coef_c1(x):
    """BJ configs[0]: a1 = 1+0.5 sin(2 pi x), a2 = 1+0.3 cos(2 pi y), a3 = 1+x(1-x)."""
    return np.stack([1.0 + 0.5 * np.sin(TWO_PI * x),
                     1.0 + 0.3 * np.cos(TWO_PI * x),
                     1.0 + x * (1.0 - x)])


def _coef_c3(x, seed=3):
    """BJ configs[2]: a_l = 1 + 0.9 sin(2 pi (x + phi_l)), phi_l ~ U(0,1) from seed 3."""
    phi = np.random.default_rng(seed).uniform(0.0, 1.0, size=3)
    return np.stack([1.0 + 0.9 * np.sin(TWO_PI * (x + phi[l])) for l in range(3)])


def _coef_unit(x):
    return np.ones((3, x.size))


# ---- right-hand sides -----------------------------------------------------------------

def _rhs_c1(n):
    x = grid_points(n)
    s = np.sin(np.pi * x)
    g = x * (1.0 - x) * np.exp(x)
    U = [np.stack([s, g], axis=1) for _ in range(3)]
    return normalize_cp(np.ones(2), U)


def _rhs_c2(n, seed=2):
    x = grid_points(n)
    w = np.random.default_rng(seed).uniform(0.5, 1.5, size=4)
    f = np.stack([np.sin(k * np.pi * x) * np.exp(-x) for k in range(1, 5)], axis=1)
    return normalize_cp(w, [f.copy(), f.copy(), f.copy()])


def _rhs_c4(n, R=16, seed=4):
    x = grid_points(n)
    rng = np.random.default_rng(seed)
    c = rng.uniform(0.2, 0.8, size=(3, R))
    wd = rng.uniform(0.05, 0.2, size=(3, R))
    U = [np.exp(-((x[:, None] - c[l][None, :]) ** 2) / (2.0 * wd[l][None, :] ** 2)) for l in range(3)]
    return normalize_cp(np.ones(R), U)


@dataclass
class Problem:
    name: str
    n: int
    a_mid: np.ndarray          # (3, n+1) midpoint samples a_l((i+1/2)h), i = 0..n
    alpha: float
    beta: float
    eps: float
    tol_stop: float
    b_w: np.ndarray
    b_U: list = field(default_factory=list)
    kmax: int = 100
    precond_rank: int = 6
    boundary: int = 0          # 0 = paper rule [P:517-518], 1 = standard
    precond: str = "B"         # preconditioner case (A) or (B) [P:758-768]; B = default (A6)


CONFIGS = {
    # name: (default n, coefficient fn, alpha, beta, eps, rhs fn)
    "C1": dict(n=32, coef=_coef_c1, alpha=0.5, beta=0.01, eps=1e-6, rhs=_rhs_c1),
    "C2": dict(n=128, coef=_coef_c1, alpha=0.5, beta=0.01, eps=1e-7, rhs=_rhs_c2),
    "C3a": dict(n=512, coef=_coef_c3, alpha=0.25, beta=0.1, eps=1e-6,
                rhs=lambda n: random_cp(n, 8, 13)),
    "C3b": dict(n=512, coef=_coef_c3, alpha=0.75, beta=0.1, eps=1e-6,
                rhs=lambda n: random_cp(n, 8, 13)),
    "C4": dict(n=1024, coef=_coef_c1, alpha=0.5, beta=0.01, eps=1e-6, rhs=_rhs_c4),
    "unit": dict(n=16, coef=_coef_unit, alpha=0.5, beta=0.01, eps=1e-6, rhs=_rhs_c1),
}


def make_problem(name: str, n: int | None = None, eps: float | None = None,
                 alpha: float | None = None, beta: float | None = None, precond: str = "B") -> Problem:
    """Build config `name` (optionally at another n / eps, e.g. C4's eps sweep; precond "A"
    selects the case-(A) anisotropic-Laplacian preconditioner)."""
    cfg = CONFIGS[name]
    n = cfg["n"] if n is None else n
    eps = cfg["eps"] if eps is None else eps
    a_mid = cfg["coef"](midpoints(n))
    w, U = cfg["rhs"](n)
    return Problem(name=name, n=n, a_mid=np.ascontiguousarray(a_mid),
                   alpha=cfg["alpha"] if alpha is None else alpha,
                   beta=cfg["beta"] if beta is None else beta,
                   eps=eps, tol_stop=10.0 * eps, b_w=w, b_U=U, precond=precond)


# C5 operator-apply sweep grid [BJ configs[4]]
C5_GRID = [(n, R, r) for n in (256, 1024, 2048) for R in (16, 64, 256) for r in (8, 16, 32)]


# ---- 2D variant --------------------------------------------------
# The paper's 2D tests [P:1068-1225] use a box / H-type design function given only as figures;
# these seeded stand-ins reuse C1's a1, a2 and rank-2 / rank-8 right-hand sides.

@dataclass
class Problem2:
    name: str
    n: int
    a_mid: np.ndarray          # (2, n+1) midpoint samples of a1, a2
    alpha: float
    beta: float
    eps: float
    tol_stop: float
    b_w: np.ndarray
    b_U: list = field(default_factory=list)
    kmax: int = 100
    precond_rank: int = 6
    boundary: int = 0


def _rhs2_smooth(n):
    x = grid_points(n)
    s = np.sin(np.pi * x)
    g = x * (1.0 - x) * np.exp(x)
    return normalize_cp(np.ones(2), [np.stack([s, g], axis=1), np.stack([s, g], axis=1)])


def _rhs2_bumps(n, R=8, seed=6):
    x = grid_points(n)
    rng = np.random.default_rng(seed)
    c = rng.uniform(0.2, 0.8, size=(2, R))
    wd = rng.uniform(0.05, 0.2, size=(2, R))
    U = [np.exp(-((x[:, None] - c[l][None, :]) ** 2) / (2.0 * wd[l][None, :] ** 2)) for l in range(2)]
    return normalize_cp(np.ones(R), U)


CONFIGS2 = {
    # D1: the paper's 2D n = 64 setting [P:1125-1152] (alpha sweep), smooth rank-2 right-hand side
    "D1": dict(n=64, alpha=0.5, beta=0.01, eps=1e-6, rhs=_rhs2_smooth),
    # D2: large 2D grid (the paper's 2D grids reach 2048 [P:1097-1123]), rank-8 bumps
    "D2": dict(n=1024, alpha=0.5, beta=0.01, eps=1e-6, rhs=_rhs2_bumps),
}


def make_problem2(name: str, n: int | None = None, eps: float | None = None, alpha: float | None = None,
                  beta: float | None = None) -> Problem2:
    cfg = CONFIGS2[name]
    n = cfg["n"] if n is None else n
    eps = cfg["eps"] if eps is None else eps
    a_mid = _coef_c1(midpoints(n))[:2]
    w, U = cfg["rhs"](n)
    return Problem2(name=name, n=n, a_mid=np.ascontiguousarray(a_mid),
                    alpha=cfg["alpha"] if alpha is None else alpha,
                    beta=cfg["beta"] if beta is None else beta,
                    eps=eps, tol_stop=10.0 * eps, b_w=w, b_U=U)
