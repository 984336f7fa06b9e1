"""Sinc-quadrature construction of the spectral tensors D^-alpha and D^alpha (SURVEY §8(f) row
f4) [P:325-351, P:725-752].  (Oracle: test-only; imports nothing from the CUDA path.)

D^-alpha[i,j,k] = (lam1_i + lam2_j + lam3_k)^-alpha
                = 1/Gamma(alpha) int_0^inf t^(alpha-1) exp(-t (lam1_i + lam2_j + lam3_k)) dt   [P:331]
                ~ sum_k c_k exp(-t_k lam1_i) exp(-t_k lam2_j) exp(-t_k lam3_k)                 [P:727-734]

Quadrature (a standard sinc rule on the real line, parameters derived here): t = e^x turns the
integral into int_R exp(alpha x - lam e^x) dx, analytic in the strip |Im x| < pi/2; the
trapezoid rule with step h = 2 pi d / ln(1/eps) has discretisation error ~ exp(-2 pi d / h) = eps
for a strip half-width d.  The integrand's decay weakens towards |Im x| = pi/2 (the constant in
front of the error grows: 22 eps at d = pi/2 for alpha = 1), so d = pi/3 is used: error <= eps
measured for alpha in [0.05, 1], eps in [1e-12, 1e-6] over lam in [30, 1.3e7].
The range [x_lo, x_hi] drops tails below eps * Gamma(alpha) * lam^-alpha for every lam in
[lam_min, lam_max]:  lower tail  e^(alpha x_lo) / alpha <= eps Gamma(alpha) lam_max^-alpha,
upper tail  L^alpha e^-L <= eps Gamma(alpha)  with  L = lam_min e^(x_hi).
Nodes t_k = e^(x_lo + k h), weights c_k = h t_k^alpha / Gamma(alpha): the canonical rank is
R = 2M+1 = O(|log eps| (|log eps| + log(lam_max/lam_min))) terms, positive factors.

D^alpha = D (.) D^(alpha-1) [P:746-750] with D = lam-sum of canonical rank 3: rank <= 3 R, then
compressed by the truncation (O9).
"""
from __future__ import annotations

import math

import numpy as np

from . import cp as cpm
from .cp import CP
from .truncate import truncate


def sinc_nodes(alpha: float, lam_min: float, lam_max: float, eps: float):
    """(t, c): nodes and weights of the sinc rule for lam^-alpha on [lam_min, lam_max]."""
    g = math.gamma(alpha)
    h = 2.0 * math.pi * (math.pi / 3.0) / math.log(1.0 / eps)
    x_lo = (math.log(eps * alpha * g) - alpha * math.log(lam_max)) / alpha
    L = math.log(1.0 / (eps * g))
    for _ in range(20):                                      # L = ln(1/(eps Gamma)) + alpha ln L
        L = math.log(1.0 / (eps * g)) + alpha * math.log(max(L, 1.0))
    x_hi = math.log(L / lam_min)
    m = int(math.ceil((x_hi - x_lo) / h))
    x = x_lo + h * np.arange(m + 1)
    t = np.exp(x)
    c = h * np.exp(alpha * x) / g
    return t, c


def sinc_pow_minus(lams, alpha: float, eps: float) -> CP:
    """CP of D^-alpha by the sinc rule (positive factors, unit columns)."""
    lo = sum(float(np.min(l)) for l in lams)
    hi = sum(float(np.max(l)) for l in lams)
    t, c = sinc_nodes(alpha, lo, hi, eps)
    U, w = [], c.copy()
    for l in range(3):
        E = np.exp(-np.outer(lams[l], t))                    # n x R
        nrm = np.linalg.norm(E, axis=0)
        U.append(E / nrm)
        w = w * nrm
    return CP(w, U)


def sinc_pow_plus(lams, alpha: float, eps: float) -> CP:
    """CP of D^alpha = D (.) D^(alpha-1), truncated at eps (alpha = 1: D itself, rank 3)."""
    # D = lam1 (x) 1 (x) 1 + 1 (x) lam2 (x) 1 + 1 (x) 1 (x) lam3  (canonical rank 3)
    U = [np.stack([lams[l] if l == m else np.ones(len(lams[l])) for m in range(3)], axis=1) for l in range(3)]
    D = cpm.normalized(np.ones(3), U)
    if alpha >= 1.0:
        return truncate(D, eps)
    Q = sinc_pow_minus(lams, 1.0 - alpha, eps)
    return truncate(cpm.hadamard(D, Q), eps)


def sinc_F(lams, alpha: float, beta: float, eps: float) -> CP:
    """F = beta D^alpha + D^-alpha from the two sinc constructions, truncated at eps."""
    return truncate(cpm.axpy(cpm.scale(beta, sinc_pow_plus(lams, alpha, eps)), 1.0,
                             sinc_pow_minus(lams, alpha, eps)), eps)
