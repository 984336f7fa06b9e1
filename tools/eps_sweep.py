"""C4 (n = 1024) eps sweep {1e-5, 1e-6, 1e-7, 1e-8} (BASELINE configs[3]): iterations, time-to-eps,
ranks, final residual (one warm-up solve, then 3 timed)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2006_09314_b200.binding import DeviceCP, Library, make_params  # noqa: E402
from synth import make_problem  # noqa: E402

L = Library()
for eps in (1e-5, 1e-6, 1e-7, 1e-8):
    p = make_problem("C4", n=1024, eps=eps)
    ctx = L.context(torch.cuda.current_stream().cuda_stream)
    prm = make_params(p.alpha, p.beta, p.eps, p.tol_stop)
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    ctx.sl_setup(p.n, p.a_mid, prm)
    s1.record()
    torch.cuda.synchronize()
    setup = s0.elapsed_time(s1)
    b = DeviceCP.from_numpy(p.b_w, p.b_U)
    try:
        u, rep, rc = ctx.pcg_solve(b, prm)
        ts = []
        for _ in range(3):
            s0.record()
            u, rep, rc = ctx.pcg_solve(b, prm)
            s1.record()
            torch.cuda.synchronize()
            ts.append(s0.elapsed_time(s1))
        out = {"eps": eps, "rc": rc, "iters": rep["iters"], "time_to_eps_ms": float(np.median(ts)),
               "iters_per_s": rep["iters"] / (np.median(ts) / 1e3), "setup_ms": setup,
               "final_rel_res": rep["rel_res"][-1], "rank_X": rep["rank_X"][-1], "max_rank_R": max(rep["rank_R"]),
               "F_rank": ctx.op_spectral_rank(0)[0]}
    except Exception as e:
        out = {"eps": eps, "error": str(e)[:200]}
    print(json.dumps(out), flush=True)
