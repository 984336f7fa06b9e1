"""Real-run GPU timeline of one warm C4 solve (CUPTI through torch.profiler): per-kernel time,
launch counts and the GPU idle time between kernels (what the serialised ncu launch list
cannot show).  Usage: python tools/timeline.py [n] [eps] > out.txt
"""
import collections
import re
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2006_09314_b200.binding import DeviceCP, Library, make_params  # noqa: E402
from synth import make_problem  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    eps = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-6
    p = make_problem("C4", n=n)
    L = Library()
    ctx = L.context(torch.cuda.current_stream().cuda_stream)
    prm = make_params(p.alpha, p.beta, eps, 10 * eps)
    ctx.sl_setup(p.n, p.a_mid, prm)
    b = DeviceCP.from_numpy(p.b_w, p.b_U)
    for _ in range(2):   # warm
        ctx.pcg_solve(b, prm)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record()
        u, rep, rc = ctx.pcg_solve(b, prm)
        ev1.record()
        torch.cuda.synchronize()
    wall = ev0.elapsed_time(ev1)
    ks = []
    syncs = 0
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            ks.append((e.time_range.start, e.time_range.end, e.name))
        elif "Synchronize" in e.name:
            syncs += 1
    ks.sort()
    busy = 0.0
    cur_s, cur_e = None, None
    gaps = []
    for s, e, _ in ks:
        if cur_e is None:
            cur_s, cur_e = s, e
        elif s > cur_e:
            busy += cur_e - cur_s
            gaps.append(s - cur_e)
            cur_s, cur_e = s, e
        else:
            cur_e = max(cur_e, e)
    if cur_e is not None:
        busy += cur_e - cur_s
    span = (ks[-1][1] - ks[0][0]) if ks else 0
    print(f"solve rc={rc} iters={rep['iters']} event_ms={wall:.2f} kernels={len(ks)} host_syncs~{syncs}")
    print(f"timeline span {span/1e3:.2f} ms, GPU busy {busy/1e3:.2f} ms ({100*busy/max(span,1):.1f} %), "
          f"idle {(span-busy)/1e3:.2f} ms in {len(gaps)} gaps (>5us: {sum(1 for g in gaps if g > 5)}, "
          f"sum {sum(g for g in gaps if g > 5)/1e3:.2f} ms)")
    agg = collections.defaultdict(lambda: [0.0, 0])
    for s, e, nm in ks:
        key = re.sub(r"\(anonymous namespace\)::", "", nm).split("(")[0][:90]
        agg[key][0] += e - s
        agg[key][1] += 1
    tot = sum(v[0] for v in agg.values())
    print(f"sum of kernel durations {tot/1e3:.2f} ms")
    for k, (t, c) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:45]:
        print(f"{100*t/tot:6.2f}% {t/1e3:8.2f} ms {c:6d}  {t/max(c,1):8.1f} us/launch  {k}")
    # duration distribution of the GEMM launches (many skinny projections vs few long contractions)
    edges = [5, 10, 15, 20, 30, 50, 100, 200, 500, 1e9]
    dist = [[0, 0.0] for _ in edges]
    for s, e, nm in ks:
        if "dgemm_dmma_kernel" not in nm:
            continue
        d = e - s
        for i, hi in enumerate(edges):
            if d < hi:
                dist[i][0] += 1
                dist[i][1] += d
                break
    print("dgemm_dmma_kernel durations (us bucket upper edge: launches, total ms):",
          {("%g" % hi): (c, round(t / 1e3, 2)) for hi, (c, t) in zip(edges, dist)})
    hist = collections.Counter()
    for g in gaps:
        hist[min(int(g // 5) * 5, 100)] += 1
    print("gap histogram (us bucket: count):", dict(sorted(hist.items())))


if __name__ == "__main__":
    main()
