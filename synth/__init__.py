"""Seeded synthetic inputs shared by the oracle tests, the CUDA parity tests and bench.py.

This package holds NO arithmetic of the method (no operator assembly, no eigen-solve, no
spectral function, no truncation).  It only evaluates the coefficient functions and the
right-hand-side factor functions that BASELINE.json's configs name, on the grid, from
fixed seeds (NumPy PCG64 `default_rng`).  Both the oracle (`oracle/`) and the GPU path
(`paper_2006_09314_b200/`) consume the same bytes from here; neither imports the other.
"""
from .configs import (  # noqa: F401
    CONFIGS, Problem, grid_points, midpoints, make_problem, random_cp, normalize_cp,
    CONFIGS2, Problem2, make_problem2,
)
