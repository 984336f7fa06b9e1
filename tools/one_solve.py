"""One C4 solve (setup + pcg_solve) through the C-ABI: the short command ncu captures."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2006_09314_b200.binding import DeviceCP, Library, make_params  # noqa: E402
from synth import make_problem  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    p = make_problem("C4", n=n)
    L = Library()
    ctx = L.context(torch.cuda.current_stream().cuda_stream)
    prm = make_params(p.alpha, p.beta, p.eps, p.tol_stop)
    ctx.sl_setup(p.n, p.a_mid, prm)
    u, rep, rc = ctx.pcg_solve(DeviceCP.from_numpy(p.b_w, p.b_U), prm)
    torch.cuda.synchronize()
    print("rc", rc, "iters", rep["iters"], "rel_res", rep["rel_res"][-1], "rank", u.rank)
    assert rc == 0


if __name__ == "__main__":
    main()
