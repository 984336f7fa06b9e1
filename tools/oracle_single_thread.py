"""BASELINE.md's CPU plan: the oracle (as it stands) on C1 (n = 32) and C2 (n = 128), full solves
with its own setup, on ONE host thread (threadpoolctl limits BLAS/LAPACK) and on all cores.
Prints one JSON line per (config, threads)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from threadpoolctl import threadpool_limits  # noqa: E402

from oracle import pcg as P  # noqa: E402
from synth import make_problem  # noqa: E402

for name in sys.argv[1:] or ["C1", "C2"]:
    for threads in (1, os.cpu_count()):
        with threadpool_limits(limits=threads):
            p = make_problem(name)
            t0 = time.perf_counter()
            st = P.setup(p)
            t1 = time.perf_counter()
            u, rep, _ = P.solve(p, st)
            t2 = time.perf_counter()
        print(json.dumps({"cfg": name, "n": p.n, "eps": p.eps, "threads": threads, "setup_s": t1 - t0,
                          "solve_s": t2 - t1, "iters": rep["iters"], "iters_per_s": rep["iters"] / (t2 - t1),
                          "rel_res": rep["rel_res"][-1], "rank_u": u.rank}), flush=True)
