"""Debug: the Khatri-Rao basis K = W_G (.) V^T U_B of the first truncation at C4, built in
NumPy from the device's eigenpairs and spectral CP; inspect its columns and run the same
blocked Gram-Schmidt in NumPy; then call the device fused apply-truncate (FC_TRACE prints
the device basis orthogonality)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_09314_b200.binding import DeviceCP, Library, make_params, FC_G  # noqa: E402
from synth import make_problem  # noqa: E402


def main(n=1024):
    p = make_problem("C4", n=n)
    L = Library()
    ctx = L.context()
    ctx.sl_setup(n, p.a_mid, make_params(p.alpha, p.beta, p.eps, p.tol_stop))
    lam, V = ctx.sl_get_eigen(0)
    V = V.cpu().numpy()
    w, U = ctx.op_get_spectral_cp(FC_G).to_numpy()
    Wg, _ = np.linalg.qr(U[0])
    Zh = V.T @ p.b_U[0]
    K = (Wg[:, :, None] * Zh[:, None, :]).reshape(n, -1)
    nrm = np.linalg.norm(K, axis=0)
    print("K", K.shape, "col norm min %.2e max %.2e" % (nrm.min(), nrm.max()),
          "#tiny(<1e-100)", int(np.sum(np.abs(K) < 1e-300)), "denormal", int(np.sum((np.abs(K) > 0) & (np.abs(K) < 2.3e-308))))
    s = np.linalg.svd(K, compute_uv=False)
    print("sv", s[:3], "rank@1e-13 (of s_max)", int(np.sum(s > 1e-13 * s[0])))
    x = DeviceCP.from_numpy(p.b_w, p.b_U)
    os.environ["FC_TRACE"] = "1"
    y, info = ctx.fracop_apply_truncate(FC_G, x, p.eps)
    print("device tucker", list(info.tucker_rank), "basis", list(info.basis_dim), flush=True)


if __name__ == "__main__":
    main()
