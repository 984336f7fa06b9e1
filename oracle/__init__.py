"""ORACLE — test infrastructure only.

A plain, slow, obviously-correct CPU (NumPy/SciPy, FP64) implementation of the hot path of
Schmitt, Khoromskij, Khoromskaia, Schulz, arXiv 2006.09314, written from the
paper step by step.  It shares NO code with the CUDA path in
`paper_2006_09314_b200/` and neither imports the other.  Only `tests/`,
`__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` / `--impl reference` legs may
import it.  The product path never routes through here.

Modules
  sturm     O1 grid, O2 FD assembly, O3 1D eigenpairs               [P:443-542]
  spectral  O4 spectral functions, O5 spectral-diagonal CP (HOSVD+T2C) [P:640-722,1720-1812]
  cp        CP type, O6 apply, O7 dot, O8 axpy/scale                 [P:597-623,1706-1763]
  truncate  O9 RHOSVD (C2T) + Tucker-to-canonical                    [P:187-190,1791-1816]
  pcg       O10 Algorithm 1, O11 report                              [P:1825-1872]
  measure   O12 reldiff in a common orthonormal basis
  dense     D0 dense n^3 x n^3 reference (tiny n only)               [P:449-452,573-577]

Parity status: every function above is pinned by a
`-m "not gpu"` test against closed forms, the dense D0 reference or invariants, except
the items DESIGN.md lists as "parity unpinned": (1) the factor values of the spectral CP
(only its entries are pinned), (2) RHOSVD/T2C factors beyond the epsilon bound,
(3) absolute PCG iteration counts for the case-(B) preconditioner in 3D.
"""
