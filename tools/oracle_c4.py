"""Time the oracle's PCG (Algorithm 1, oracle/pcg.py, as it stands) on a BASELINE config at full
size with device-built setup inputs injected (sl_get_eigen / op_get_spectral_cp: the oracle's own
setup materialises n^3 entries).  `python tools/oracle_c4.py [CFG] [N] [KMAX] [EPS]`"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import cp as cpm  # noqa: E402
from oracle import pcg as P  # noqa: E402
from paper_2006_09314_b200.binding import FC_F, FC_G, Library, make_params  # noqa: E402
from synth import make_problem  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
kmax = int(sys.argv[3]) if len(sys.argv) > 3 else 2
kw = {"eps": float(sys.argv[4])} if len(sys.argv) > 4 else {}
p = make_problem(cfg, n=n, **kw)
ctx = Library().context()
ctx.sl_setup(p.n, p.a_mid, make_params(p.alpha, p.beta, p.eps, p.tol_stop))
lams, V = [], []
for l in range(3):
    lam, Vl = ctx.sl_get_eigen(l)
    lams.append(lam.cpu().numpy())
    V.append(Vl.cpu().numpy())
Fw, FU = ctx.op_get_spectral_cp(FC_F).to_numpy()
Gw, GU = ctx.op_get_spectral_cp(FC_G).to_numpy()
st = P.Setup(lams, V, cpm.CP(Fw, FU), cpm.CP(Gw, GU))
t0 = time.perf_counter()
u, rep, _ = P.solve(p, st, kmax=kmax)
dt = time.perf_counter() - t0
print(json.dumps({"cfg": cfg, "n": n, "kmax": kmax, "cores": os.cpu_count(), "s_total": dt,
                  "t_iter_s": rep["t_iter"], "rel_res": rep["rel_res"], "rank_S": rep["rank_S"],
                  "rank_R": rep["rank_R"], "rank_Z": rep["rank_Z"], "rank_P": rep["rank_P"],
                  "F_rank": int(Fw.size), "G_rank": int(Gw.size)}))
