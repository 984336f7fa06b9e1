"""Pins of the oracle's sinc-quadrature spectral CPs [P:325-351, P:725-752].

Pinned against the closed form lam^-alpha (the rule approximates Gamma(alpha) lam^-alpha pointwise),
against the exact tensor D^-alpha entrywise, and against the HOSVD route (O5) for F."""
import math

import numpy as np
import pytest

from oracle import cp as cpm
from oracle import sinc
from oracle import spectral as sp
from oracle.sturm import eigenpairs
from synth import make_problem


@pytest.mark.parametrize("alpha", [0.1, 0.25, 0.5, 0.75, 1.0])
@pytest.mark.parametrize("eps", [1e-6, 1e-10])
def test_sinc_rule_pointwise(alpha, eps):
    lo, hi = 30.0, 1.3e7                       # the C4 lam-sum range at n = 1024
    t, c = sinc.sinc_nodes(alpha, lo, hi, eps)
    lam = np.logspace(math.log10(lo), math.log10(hi), 400)
    approx = np.exp(-np.outer(lam, t)) @ c
    assert np.max(np.abs(approx - lam ** -alpha) * lam ** alpha) <= 2 * eps
    assert np.all(c > 0)


def test_sinc_rank_growth():
    """R = O(|log eps|^2 / alpha) for this (trapezoid) rule: from eps = 1e-6 to 1e-10 the rank grows
    at most by (10/6)^2 (+ 20 % for the range terms)."""
    r6 = len(sinc.sinc_nodes(0.5, 30.0, 1.3e7, 1e-6)[0])
    r10 = len(sinc.sinc_nodes(0.5, 30.0, 1.3e7, 1e-10)[0])
    assert r10 <= 1.2 * (10 / 6) ** 2 * r6


@pytest.mark.parametrize("name,n", [("C1", 12), ("C3b", 10)])
def test_sinc_cp_entries(name, n):
    p = make_problem(name, n=n)
    lams = [eigenpairs(p.a_mid[l])[0] for l in range(3)]
    for eps in (1e-6, 1e-10):
        Pm = sinc.sinc_pow_minus(lams, p.alpha, eps)
        D = sp.coefficient_tensor(lams, sp.FC_POW_MINUS, p.alpha, p.beta)
        assert np.max(np.abs(cpm.full(Pm) - D) / D) <= 5 * eps            # uniform relative accuracy
        Pp = sinc.sinc_pow_plus(lams, p.alpha, eps)
        Dp = sp.coefficient_tensor(lams, sp.FC_POW_PLUS, p.alpha, p.beta)
        assert np.linalg.norm(cpm.full(Pp) - Dp) <= 2 * eps * np.linalg.norm(Dp)


def test_sinc_F_agrees_with_hosvd_route():
    p = make_problem("C1", n=14)
    lams = [eigenpairs(p.a_mid[l])[0] for l in range(3)]
    Fs = sinc.sinc_F(lams, p.alpha, p.beta, p.eps)
    Fh = sp.spectral_cp(lams, sp.FC_F, p.alpha, p.beta, p.eps)
    D = sp.coefficient_tensor(lams, sp.FC_F, p.alpha, p.beta)
    assert np.linalg.norm(cpm.full(Fs) - D) <= 2 * p.eps * np.linalg.norm(D)
    assert np.linalg.norm(cpm.full(Fs) - cpm.full(Fh)) <= 3 * p.eps * np.linalg.norm(D)
