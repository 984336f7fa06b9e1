"""Diagnostic: cp_truncate (CP route) of an untruncated apply output at C4 n = 1024, eps = 1e-8,
against the oracle's truncation of the same CP (and the fused route).  `python tools/diag_plain8.py`"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from _parity import as_cp, device_setup_to_oracle  # noqa: E402
from oracle import cp as cpm  # noqa: E402
from oracle.measure import reldiff  # noqa: E402
from oracle.truncate import truncate  # noqa: E402
from paper_2006_09314_b200.binding import FC_F, DeviceCP, Library, make_params  # noqa: E402
from synth import make_problem  # noqa: E402

eps = float(sys.argv[1]) if len(sys.argv) > 1 else 1e-8
p = make_problem("C4", n=1024)
prm = make_params(p.alpha, p.beta, p.eps, p.tol_stop, kmax=10)
ctx = Library().context()
st = device_setup_to_oracle(ctx, p, prm)
u, rep, rc = ctx.pcg_solve(DeviceCP.from_numpy(p.b_w, p.b_U), prm)
x = as_cp(u)
ax = cpm.apply(st.V, st.F, x)
info_o = {}
ref = truncate(ax, eps, info_o)
print("oracle tucker", info_o["tucker_rank"], "rank", ref.rank, "min margin", min(info_o["margins"]))
yd, info = ctx.cp_truncate(DeviceCP.from_numpy(ax.w, ax.U), eps)
print("plain(oracle apply) tucker", list(info.tucker_rank), "basis", list(info.basis_dim), "rank", yd.rank,
      "reldiff vs oracle", reldiff(as_cp(yd), ref))
ya = ctx.fracop_apply(FC_F, u)
print("device apply vs oracle apply", reldiff(as_cp(ya), ax))
yp, info = ctx.cp_truncate(ya, eps)
print("plain(device apply) tucker", list(info.tucker_rank), "rank", yp.rank, "reldiff vs oracle", reldiff(as_cp(yp), ref))
yf, info = ctx.fracop_apply_truncate(FC_F, u, eps)
print("fused tucker", list(info.tucker_rank), "rank", yf.rank, "reldiff vs oracle", reldiff(as_cp(yf), ref))
# truncation errors ||x - y|| / ||x|| of each route against the untruncated apply output x
# (common basis cut at 1e-12 of the largest weighted column: x's full span is ~n-dimensional)
import oracle.measure as M  # noqa: E402
M.BASIS_CUT = 1e-12
import numpy as np  # noqa: E402
nx = np.sqrt(cpm.dot(ax, ax))
for name, y in (("oracle", ref), ("plain", as_cp(yp)), ("fused", as_cp(yf))):
    print(f"||x - y_{name}|| / ||x|| = {M.diff_norm(ax, y) / nx:.3e}  (eps {eps:g})")
