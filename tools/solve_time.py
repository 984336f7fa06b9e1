"""Event-timed warm C4 solves (setup once, 1 warm-up solve, then `reps` timed): the quick A/B
probe for environment switches.  Usage: python tools/solve_time.py [n] [eps] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2006_09314_b200.binding import DeviceCP, Library, make_params  # noqa: E402
from synth import make_problem  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    eps = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-6
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    p = make_problem("C4", n=n)
    L = Library()
    ctx = L.context(torch.cuda.current_stream().cuda_stream)
    prm = make_params(p.alpha, p.beta, eps, 10 * eps)
    ctx.sl_setup(p.n, p.a_mid, prm)
    b = DeviceCP.from_numpy(p.b_w, p.b_U)
    ctx.pcg_solve(b, prm)
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        u, rep, rc = ctx.pcg_solve(b, prm)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"n={n} eps={eps} rc={rc} iters={rep['iters']} rel_res={rep['rel_res'][-1]!r} ranks={sum(rep['rank_R'])}/{sum(rep['rank_S'])}/{sum(rep['rank_Z'])} rank={u.rank} "
          f"ms={' '.join(f'{t:.1f}' for t in ts)} env={ {k: v for k, v in os.environ.items() if k.startswith('FC_')} }")


if __name__ == "__main__":
    main()
