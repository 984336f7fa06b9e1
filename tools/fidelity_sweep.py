"""Spectral-CP fidelity on smooth modes vs solver cost: C4 (n = 1024,
eps = 1e-6) with the operator CP F built at eps_D in {1e-6, 1e-8, 1e-10} and the preconditioner
rank r_G in {6, 24}.  For each: the max relative error of F~ (and of G~ F) on the 8^3 lowest
eigen-modes against the exact F(lam1_i + lam2_j + lam3_k) (A5), the ranks, PCG iterations and
time-to-eps.  Prints one JSON line per setting.  `python tools/fidelity_sweep.py`"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2006_09314_b200.binding import FC_F, FC_G, DeviceCP, Library, make_params  # noqa: E402
from synth import make_problem  # noqa: E402


def cp_entries(w, U, idx):
    """CP value at the index triples idx (m x 3)."""
    return np.einsum("t,mt,mt,mt->m", w, U[0][idx[:, 0]], U[1][idx[:, 1]], U[2][idx[:, 2]])


p = make_problem("C4", n=1024)
L = Library()
K = 8
ii = np.stack(np.meshgrid(np.arange(K), np.arange(K), np.arange(K), indexing="ij"), -1).reshape(-1, 3)
for eps_D in (1e-6, 1e-8, 1e-10):
    for rG in (6, 24):
        ctx = L.context()
        prm = make_params(p.alpha, p.beta, p.eps, p.tol_stop, eps_D=eps_D, precond_rank=rG)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ctx.sl_setup(p.n, p.a_mid, prm)
        e1.record()
        torch.cuda.synchronize()
        lam = [ctx.sl_get_eigen(l)[0].cpu().numpy() for l in range(3)]
        Fw, FU = ctx.op_get_spectral_cp(FC_F).to_numpy()
        Gw, GU = ctx.op_get_spectral_cp(FC_G).to_numpy()
        s = lam[0][ii[:, 0]] + lam[1][ii[:, 1]] + lam[2][ii[:, 2]]
        Fex = p.beta * s ** p.alpha + s ** (-p.alpha)
        Ft, Gt = cp_entries(Fw, FU, ii), cp_entries(Gw, GU, ii)
        b = DeviceCP.from_numpy(p.b_w, p.b_U)
        u, rep, rc = ctx.pcg_solve(b, prm)
        u, rep, rc = ctx.pcg_solve(b, prm)          # second solve: warm
        print(json.dumps({"eps_D": eps_D, "r_G": rG, "rank_F": int(Fw.size), "rank_G": int(Gw.size),
                          "setup_ms": e0.elapsed_time(e1),
                          "lowmode_F_relerr_max": float(np.max(np.abs(Ft / Fex - 1))),
                          "lowmode_GF_range": [float(np.min(Gt * Fex)), float(np.max(Gt * Fex))],
                          "rc": rc, "iters": rep["iters"], "time_ms": rep["t_total_ms"],
                          "rank_R_last": rep["rank_R"][-1], "rel_res": rep["rel_res"][-1]}), flush=True)
        del ctx
