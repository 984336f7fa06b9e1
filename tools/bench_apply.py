"""C5 operator-apply sweep (BASELINE.json configs[4]): fracop_apply timed with CUDA events
(dominant kernel = the fused Khatri-Rao inverse transform: achieved TFLOP/s and its fraction of
the measured DMMA peak, and the algorithmic GB/s), then the truncation of the r R product back to
eps = 1e-6 (fracop_apply_truncate) where reading A22 lets it run (Tucker core r1 r2 r3 <= 2^28
and T2C output <= 2^16 terms; otherwise the CAPACITY error is recorded).  Prints one JSON line per
(n, R, r) cell.  `python tools/bench_apply.py [--no-trunc]`"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_09314_b200.binding import DeviceCP, Library, make_params, FC_F  # noqa: E402
from synth import random_cp  # noqa: E402
from synth.configs import C5_GRID  # noqa: E402


def main(cells=None, reps=10):
    L = Library()
    ctx = L.context()
    peaks = {}
    for n, R, r in (cells or C5_GRID):
        rng = np.random.default_rng(n)
        Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
        prm = make_params(0.5, 0.01, 1e-6)
        for l in range(3):
            ctx.sl_set_eigen(n, l, np.linspace(1, 2, n), Q, prm)
        w, U = random_cp(n, r, 77)
        ctx.op_set_spectral_cp(FC_F, DeviceCP.from_numpy(w, U))
        w, U = random_cp(n, R, 5)
        x = DeviceCP.from_numpy(w, U)
        y = DeviceCP(n, r * R)
        for _ in range(3):
            ctx.fracop_apply(FC_F, x, y)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        kms = []
        e0.record()
        for _ in range(reps):
            ctx.fracop_apply(FC_F, x, y)
            kms.append(ctx.last_kernel_stats()["ms"])
        e1.record()
        torch.cuda.synchronize()
        st = ctx.last_kernel_stats()
        tot = e0.elapsed_time(e1) / reps
        kmed = float(np.median(kms))
        tf = st["flops"] / kmed / 1e9
        row = {"n": n, "R": R, "r": r, "apply_ms": tot, "inv_kernel_ms": kmed, "inv_tflops": tf,
               "inv_frac_dmma": tf / 37.16, "inv_gbs": st["bytes"] / kmed / 1e6,
               "inv_frac_hbm": st["bytes"] / kmed / 1e6 / 6554.9}
        if "--no-trunc" not in sys.argv:
            from paper_2006_09314_b200.binding import FCError
            try:
                t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                t0.record()
                z, info = ctx.fracop_apply_truncate(FC_F, x, 1e-6, cap=1 << 16)
                t1.record()
                torch.cuda.synchronize()
                row.update({"trunc_ms": t0.elapsed_time(t1), "trunc_tucker": list(info.tucker_rank),
                            "trunc_rank": z.rank, "trunc_basis": list(info.basis_dim)})
            except FCError as e:
                row.update({"trunc": f"not run (A22): {e}"})
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
