"""One fracop_apply at a C5 cell (for ncu captures of the fused inverse transform)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_09314_b200.binding import DeviceCP, Library, make_params, FC_F  # noqa: E402
from synth import random_cp  # noqa: E402


def main(n=1024, R=64, r=16, reps=3):
    L = Library()
    ctx = L.context()
    Q, _ = np.linalg.qr(np.random.default_rng(n).standard_normal((n, n)))
    prm = make_params(0.5, 0.01, 1e-6)
    for l in range(3):
        ctx.sl_set_eigen(n, l, np.linspace(1, 2, n), Q, prm)
    w, U = random_cp(n, r, 77)
    ctx.op_set_spectral_cp(FC_F, DeviceCP.from_numpy(w, U))
    w, U = random_cp(n, R, 5)
    x = DeviceCP.from_numpy(w, U)
    y = DeviceCP(n, r * R)
    for _ in range(reps):
        ctx.fracop_apply(FC_F, x, y)
    torch.cuda.synchronize()
    print("ok", ctx.last_kernel_stats())


if __name__ == "__main__":
    a = [int(v) for v in sys.argv[1:4]] if len(sys.argv) >= 4 else [1024, 64, 16]
    main(*a)
