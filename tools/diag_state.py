"""state_recover / POW_PLUS apply-truncate of the C4 solution vs the untruncated applies."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2006_09314_b200.binding import FC_F, FC_POW_MINUS, FC_POW_PLUS, DeviceCP, Library, make_params  # noqa: E402
from synth import make_problem  # noqa: E402

L = Library()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
p = make_problem("C4", n=n)
ctx = L.context()
prm = make_params(p.alpha, p.beta, p.eps, p.tol_stop)
ctx.sl_setup(p.n, p.a_mid, prm)
b = DeviceCP.from_numpy(p.b_w, p.b_U)
u, rep, rc = ctx.pcg_solve(b, prm)
print("u rank", u.rank, "iters", rep["iters"])


def rel(a, b_):
    d = ctx.cp_axpy(a, -1.0, b_)
    return math.sqrt(max(ctx.cp_dot(d, d), 0) / ctx.cp_dot(b_, b_))


for which, name in ((FC_F, "F"), (FC_POW_PLUS, "P+"), (FC_POW_MINUS, "P-")):
    yt, info = ctx.fracop_apply_truncate(which, u, 1e-10)
    yu = ctx.fracop_apply(which, u)
    print(name, "trunc rank", yt.rank, "tucker", list(info.tucker_rank), "untrunc rank", yu.rank,
          "||trunc - untrunc||/||untrunc|| = %.2e" % rel(yt, yu), "norms %.4e %.4e" % (math.sqrt(ctx.cp_dot(yt, yt)), math.sqrt(ctx.cp_dot(yu, yu))), flush=True)
ys, _ = ctx.state_recover(u, 1e-10)
yu = ctx.fracop_apply(FC_POW_MINUS, u)
print("state_recover vs untrunc P-: %.2e" % rel(ys, yu))

# the test's chain
nb = math.sqrt(ctx.cp_dot(b, b))
y, _ = ctx.state_recover(u, 1e-10)
t, _ = ctx.fracop_apply_truncate(FC_POW_PLUS, u, 1e-10)
Fu, _ = ctx.fracop_apply_truncate(FC_F, u, 1e-10)
print("||b|| %.4e ||y|| %.4e ||t|| %.4e ||Fu|| %.4e beta %g" % (nb, math.sqrt(ctx.cp_dot(y, y)), math.sqrt(ctx.cp_dot(t, t)),
      math.sqrt(ctx.cp_dot(Fu, Fu)), p.beta))
comb = ctx.cp_axpy(y, p.beta, t)          # A^-a u + beta A^a u
print("||Fu - (y + beta t)|| / ||Fu|| = %.3e" % rel(Fu, comb))
z = ctx.cp_axpy(ctx.cp_axpy(b, -1.0, y), -p.beta, t)
zz = ctx.cp_axpy(b, -1.0, comb)
print("||b - y - beta t|| / ||b|| = %.3e (chain)  %.3e (via comb)" % (math.sqrt(max(ctx.cp_dot(z, z), 0)) / nb,
      math.sqrt(max(ctx.cp_dot(zz, zz), 0)) / nb))
r, _ = ctx.cp_truncate(z, 1e-10)
print("truncated z: rank", r.rank, "norm from weights %.3e" % (math.sqrt(float(np.sum(r.w[:r.rank].cpu().numpy() ** 2))) / nb))
