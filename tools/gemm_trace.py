"""One C4 solve with every GEMM launch timed (fc_profile_gemm) and, with FC_GEMM_TRACE=1, the
time by launch shape printed on stderr."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2006_09314_b200.binding import DeviceCP, Library, make_params  # noqa: E402
from synth import make_problem  # noqa: E402

p = make_problem("C4", n=1024)
L = Library()
ctx = L.context(torch.cuda.current_stream().cuda_stream)
prm = make_params(p.alpha, p.beta, p.eps, p.tol_stop)
ctx.sl_setup(p.n, p.a_mid, prm)
b = DeviceCP.from_numpy(p.b_w, p.b_U)
ctx.pcg_solve(b, prm)
ctx.profile_gemm(True)
u, rep, rc = ctx.pcg_solve(b, prm)
print(ctx.profile_gemm(False), rep["iters"])
