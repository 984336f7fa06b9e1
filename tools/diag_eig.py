import numpy as np, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_09314_b200.binding import Library, make_params
from oracle import sturm
from synth import make_problem
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
p = make_problem("C1", n=n)
ctx = Library().context()
ctx.sl_setup(n, p.a_mid, make_params(p.alpha, p.beta, p.eps))
for l in range(3):
    lam, V = ctx.sl_get_eigen(l); lam = lam.cpu().numpy(); V = V.cpu().numpy()
    T = sturm.dense_tridiagonal(p.a_mid[l])
    res = np.abs(T @ V - V * lam[None, :]).max(axis=0)
    bad = np.argsort(res)[-5:]
    gaps = np.minimum(np.diff(lam, prepend=-np.inf)[bad], np.diff(lam, append=np.inf)[bad])
    lo, _ = sturm.eigenpairs(p.a_mid[l])
    print("mode", l, "max res %.2e" % res.max(), "bad idx", bad.tolist(), "res", ["%.1e" % x for x in res[bad]],
          "lam", ["%.6e" % x for x in lam[bad]], "gaps", ["%.2e" % g for g in gaps], "orth %.1e" % np.abs(V.T @ V - np.eye(n)).max(),
          "lam err vs oracle", ["%.1e" % x for x in (np.abs(lam - lo) / lo)[bad]])
