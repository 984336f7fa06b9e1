"""C4 at eps = 1e-8: device vs oracle with shared inputs (n = 32), and the device alone at larger n."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from oracle import pcg as P  # noqa: E402
from paper_2006_09314_b200.binding import FC_F, FC_G, DeviceCP, Library, make_params  # noqa: E402
from synth import make_problem  # noqa: E402

L = Library()
p = make_problem("C4", n=32, eps=1e-8)
st = P.setup(p)
ctx = L.context()
prm = make_params(p.alpha, p.beta, p.eps)
for l in range(3):
    ctx.sl_set_eigen(p.n, l, st.lams[l], st.V[l], prm)
ctx.op_set_spectral_cp(FC_F, DeviceCP.from_numpy(st.F.w, st.F.U))
ctx.op_set_spectral_cp(FC_G, DeviceCP.from_numpy(st.G.w, st.G.U))
u_ref, rep_ref, _ = P.solve(p, st)
u, rep, rc = ctx.pcg_solve(DeviceCP.from_numpy(p.b_w, p.b_U), make_params(p.alpha, p.beta, p.eps, p.tol_stop, kmax=12))
print("oracle", ["%.2e" % x for x in rep_ref["rel_res"]], rep_ref["rank_R"], rep_ref["rank_X"])
print("device", ["%.2e" % x for x in rep["rel_res"]], rep["rank_R"], rep["rank_X"], flush=True)
for n in (64, 256):
    p = make_problem("C4", n=n, eps=1e-8)
    ctx = L.context()
    prm = make_params(p.alpha, p.beta, p.eps, p.tol_stop, kmax=15)
    ctx.sl_setup(p.n, p.a_mid, prm)
    u, rep, rc = ctx.pcg_solve(DeviceCP.from_numpy(p.b_w, p.b_U), prm)
    print("device n=%d" % n, rc, ["%.2e" % x for x in rep["rel_res"]], rep["rank_R"], flush=True)
