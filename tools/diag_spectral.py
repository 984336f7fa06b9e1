"""Device spectral CPs (F, G) vs the oracle's at small n: Tucker ranks, weights, errors."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import cp as cpm  # noqa: E402
from oracle import spectral as sp  # noqa: E402
from paper_2006_09314_b200.binding import Library, make_params, FC_F, FC_G  # noqa: E402
from synth import make_problem  # noqa: E402


def main(name="C1", n=64):
    p = make_problem(name, n=n)
    L = Library()
    for prank in (6, 40):
        ctx = L.context()
        ctx.sl_setup(n, p.a_mid, make_params(p.alpha, p.beta, p.eps, p.tol_stop, precond_rank=prank))
        lams = [ctx.sl_get_eigen(l)[0].cpu().numpy() for l in range(3)]
        for which, kind in ((FC_F, sp.FC_F), (FC_G, sp.FC_G)):
            D = sp.coefficient_tensor(lams, kind, p.alpha, p.beta)
            w, U = ctx.op_get_spectral_cp(which).to_numpy()
            err = np.linalg.norm(cpm.full(cpm.CP(w, U)) - D) / np.linalg.norm(D)
            info = {}
            o = sp.spectral_cp(lams, kind, p.alpha, p.beta, p.eps, rank=None if which == FC_F else prank,
                               spd_guard=(which == FC_G), info=info)
            erro = np.linalg.norm(cpm.full(o) - D) / np.linalg.norm(D)
            print(json.dumps({"which": which, "prank": prank, "gpu_rank_tucker": ctx.op_spectral_rank(which),
                              "orc_rank": o.rank, "orc_tucker": info["tucker_rank"], "gpu_err": err,
                              "orc_err": erro, "gpu_w": list(np.sort(np.abs(w))[::-1][:8]),
                              "orc_w": list(np.sort(np.abs(o.w))[::-1][:8])}), flush=True)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "C1", int(sys.argv[2]) if len(sys.argv) > 2 else 64)
