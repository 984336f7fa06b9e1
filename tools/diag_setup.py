"""Diagnostics: sl_setup at a config/n, spectral ranks, timings; then a pcg_solve with the
per-iteration ranks (JSON line per call)."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_09314_b200.binding import DeviceCP, FCError, Library, make_params, FC_F, FC_G  # noqa: E402
from synth import make_problem  # noqa: E402


def main(name, n, solve=True, eps=None):
    p = make_problem(name, n=n, eps=eps)
    L = Library()
    ctx = L.context()
    prm = make_params(p.alpha, p.beta, p.eps, p.tol_stop)
    out = {"name": name, "n": n, "eps": p.eps}
    t = time.time()
    try:
        ctx.sl_setup(n, p.a_mid, prm)
        torch.cuda.synchronize()
        out["setup_s"] = time.time() - t
        out["F"] = ctx.op_spectral_rank(FC_F)
        out["G"] = ctx.op_spectral_rank(FC_G)
    except FCError as e:
        out["setup_error"] = str(e)
        print(json.dumps(out), flush=True)
        return
    if solve:
        t = time.time()
        try:
            u, rep, rc = ctx.pcg_solve(DeviceCP.from_numpy(p.b_w, p.b_U), prm)
            out["solve_s"] = time.time() - t
            out["rc"] = rc
            out["rep"] = {k: rep[k] for k in ("iters", "converged", "rel_res", "rank_S", "rank_X", "rank_R",
                                                "rank_Z", "rank_P", "tucker_S", "t_iter_ms", "t_total_ms",
                                                "t_loop_ms")}
        except FCError as e:
            out["solve_error"] = str(e)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]), solve=(len(sys.argv) < 4 or sys.argv[3] != "nosolve"),
         eps=float(sys.argv[4]) if len(sys.argv) > 4 else None)
