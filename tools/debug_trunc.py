"""Replay every truncation input of an oracle PCG run through the GPU cp_truncate and
compare Tucker ranks, output ranks and the result (debugging aid; prints JSON lines)."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import cp as cpm  # noqa: E402
from oracle import pcg as P  # noqa: E402
from oracle.measure import reldiff  # noqa: E402
from oracle.truncate import truncate  # noqa: E402
from paper_2006_09314_b200.binding import DeviceCP, Library, make_params, FC_F, FC_G  # noqa: E402
from synth import make_problem  # noqa: E402


def main(name="C1", n=16):
    p = make_problem(name, n=n)
    st = P.setup(p)
    L = Library()
    ctx = L.context()
    prm = make_params(p.alpha, p.beta, p.eps)
    for l in range(3):
        ctx.sl_set_eigen(p.n, l, st.lams[l], st.V[l], prm)
    ctx.op_set_spectral_cp(FC_F, DeviceCP.from_numpy(st.F.w, st.F.U))
    ctx.op_set_spectral_cp(FC_G, DeviceCP.from_numpy(st.G.w, st.G.U))
    calls = []
    last = {}

    def fun(x, which, spec):
        last["x"], last["which"] = x, which
        return cpm.apply(st.V, spec, x)

    def tr(x, eps):
        info = {}
        y = truncate(x, eps, info)
        g, ginfo = ctx.cp_truncate(DeviceCP.from_numpy(x.w, x.U), eps)
        w, U = g.to_numpy()
        rec = {"i": len(calls), "in_rank": x.rank, "tucker_o": info["tucker_rank"],
               "tucker_g": list(ginfo.tucker_rank), "out_o": y.rank, "out_g": g.rank,
               "margin_o": min(info.get("margins", [1.0])), "reldiff": reldiff(cpm.CP(w, U), y)}
        if "x" in last:                    # replay the fused device apply->truncate on the same P
            xin = last.pop("x")
            f, finfo = ctx.fracop_apply_truncate(last["which"], DeviceCP.from_numpy(xin.w, xin.U), eps)
            fw, fU = f.to_numpy()
            rec.update({"fused_tucker_g": list(finfo.tucker_rank), "fused_out_g": f.rank,
                        "fused_reldiff": reldiff(cpm.CP(fw, fU), y)})
        calls.append(rec)
        print(json.dumps(rec), flush=True)
        return y

    B = cpm.normalized(p.b_w, p.b_U)
    P.pcg(lambda x: fun(x, FC_F, st.F), lambda x: fun(x, FC_G, st.G), B, p.eps, p.tol_stop,
          kmax=3, trunc=tr)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "C1", int(sys.argv[2]) if len(sys.argv) > 2 else 16)
