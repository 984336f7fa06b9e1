import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import cp as cpm  # noqa: E402
from oracle.measure import reldiff  # noqa: E402
from oracle.truncate import truncate  # noqa: E402
from paper_2006_09314_b200.binding import DeviceCP, Library, make_params  # noqa: E402
from synth import make_problem  # noqa: E402

L = Library()
for n, R, eps in ((512, 300, 1e-8), (512, 300, 1e-6), (256, 200, 1e-8)):
    p = make_problem("C1", n=n)
    ctx = L.context()
    ctx.sl_setup(p.n, p.a_mid, make_params(p.alpha, p.beta, p.eps, p.tol_stop))
    rng = np.random.default_rng(7)
    x = np.arange(1, n + 1) / (n + 1)
    U = []
    for l in range(3):
        c = rng.uniform(0.1, 0.9, R)
        w = rng.uniform(0.02, 0.2, R)
        F = np.exp(-(x[:, None] - c[None, :]) ** 2 / (2 * w[None, :] ** 2))
        U.append(F / np.linalg.norm(F, axis=0))
    wts = np.exp(-np.arange(R) / 20.0) * rng.choice([-1, 1], R)
    X = cpm.CP(wts, U)
    info_o = {}
    ref = truncate(X, eps, info_o)
    y, info = ctx.cp_truncate(DeviceCP.from_numpy(X.w, X.U), eps)
    w2, U2 = y.to_numpy()
    print("n=%d R=%d eps=%g: oracle tucker %s rank %d | device tucker %s rank %d | reldiff %.2e" % (
        n, R, eps, info_o["tucker_rank"], ref.rank, list(info.tucker_rank), y.rank, reldiff(cpm.CP(w2, U2), ref)), flush=True)
