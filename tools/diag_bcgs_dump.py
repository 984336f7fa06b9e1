"""fc_orthonormalize on a dumped basis (gpurun_out/kdump.npy, n x p): accepted count and orthonormality."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2006_09314_b200.binding import Library  # noqa: E402

K = np.load(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/kdump.npy")
ctx = Library().context()
for tau in (1e-10, 1e-13):
    A = torch.tensor(np.ascontiguousarray(K.T), device="cuda")
    Q = ctx.orthonormalize(A, tau).cpu().numpy().T
    G = Q.T @ Q
    err = np.abs(G - np.eye(Q.shape[1]))
    bad = np.argwhere(err > 1e-8)
    print(f"tau {tau:g}: k = {Q.shape[1]}, orth err {err.max():.2e}, first bad pairs {bad[:6].tolist()}, "
          f"resid {np.linalg.norm(K - Q @ (Q.T @ K)) / np.linalg.norm(K):.2e}", flush=True)
