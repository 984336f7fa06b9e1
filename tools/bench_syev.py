"""Time fc_syev (tridiagonalisation + bisection + inverse iteration + back-transform) per size."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2006_09314_b200.binding import Library  # noqa: E402


def main():
    L = Library()
    ctx = L.context()
    out = []
    for N in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "200,300,450,600,700,840,1000").split(",")]:
        rng = np.random.default_rng(N)
        A = rng.standard_normal((N, N))
        A = 0.5 * (A + A.T)
        for nb in (1, 3):
            base = torch.tensor(A, device="cuda")
            ts = []
            for it in range(4):
                mats = [base.clone() for _ in range(nb)]
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                ctx.syev(mats, [64] * nb)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            out.append({"N": N, "nb": nb, "ms": float(np.median(ts[1:])),
                        "path": "global" if os.environ.get("FC_NO_CLUSTER") else "cluster"})
            print(json.dumps(out[-1]), flush=True)


if __name__ == "__main__":
    main()
