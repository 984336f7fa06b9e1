"""fc_orthonormalize on synthetic low-rank matrices of several shapes: accepted count, orthonormality."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2006_09314_b200.binding import Library  # noqa: E402

ctx = Library().context()
for n, p, r in ((1024, 600, 600), (1024, 800, 800), (1024, 1024, 1024), (1024, 1763, 724), (1024, 1763, 1024),
                (1024, 700, 520), (2048, 900, 900)):
    rng = np.random.default_rng(n + p + r)
    K = rng.standard_normal((n, r)) @ rng.standard_normal((r, p)) if r < p else rng.standard_normal((n, p))
    A = torch.tensor(np.ascontiguousarray(K.T), device="cuda")
    Q = ctx.orthonormalize(A, 1e-10).cpu().numpy().T
    err = np.abs(Q.T @ Q - np.eye(Q.shape[1]))
    bad = np.argwhere(err > 1e-8)
    print(f"n={n} p={p} r={r}: k={Q.shape[1]} orth err {err.max():.2e} first bad {bad[:4].tolist()}", flush=True)
