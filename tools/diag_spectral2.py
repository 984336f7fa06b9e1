"""Which path breaks G: the T2C keep path (test F with op_rank) or G-specific?"""
import json, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import cp as cpm
from oracle import spectral as sp
from paper_2006_09314_b200.binding import Library, make_params, FC_F, FC_G
from synth import make_problem
p = make_problem("C1", n=64)
L = Library()
for op_rank, prank in ((40, 6), (0, 121), (121, 6)):
    ctx = L.context()
    ctx.sl_setup(64, p.a_mid, make_params(p.alpha, p.beta, p.eps, p.tol_stop, op_rank=op_rank, precond_rank=prank))
    lams = [ctx.sl_get_eigen(l)[0].cpu().numpy() for l in range(3)]
    for which, kind in ((FC_F, sp.FC_F), (FC_G, sp.FC_G)):
        D = sp.coefficient_tensor(lams, kind, p.alpha, p.beta)
        w, U = ctx.op_get_spectral_cp(which).to_numpy()
        err = np.linalg.norm(cpm.full(cpm.CP(w, U)) - D) / np.linalg.norm(D)
        print(json.dumps({"op_rank": op_rank, "prank": prank, "which": which, "rank": int(w.size), "err": err}), flush=True)
