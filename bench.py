#!/usr/bin/env python
"""bench.py — rank-truncated PCG on one B200 (driver contract).

Step = one pcg_solve of BASELINE.json configs[3] (C4: 3D n = 1024, C1 coefficients,
alpha = 0.5, beta = 0.01, rank-16 Gaussian-bump right-hand side, eps = 1e-6, tol = 10 eps):
Algorithm 1 [P:1825-1872] from b (resident in HBM) to u (in HBM).  The setup (S1-S4:
eigenpairs + spectral CPs) runs once before the timed region and is reported as setup_ms.
value = PCG iterations / second over the timed steps (all ranks); time_to_eps_ms = median
per-step solve time.  L2 is flushed (a 512 MiB write) between timed steps, outside the events.

--impl reference / cpu_baseline: the oracle (oracle/, NumPy/SciPy FP64, as it stands) on the host
cores, on the same workload (C4, n = 1024): Z0 + the first PCG iteration per step, with the
device-built eigenpairs and spectral CPs injected (the oracle's own setup materialises n^3
entries); cpu_baseline also keeps the n = 64 own-setup figure as an extra key.
Multi-GPU: replicas only (independent solves per rank, no collective).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOAD = "C4: 3D n=1024, a_l as config 1, alpha=0.5, beta=0.01, rank-16 Gaussian-bump b, eps=1e-6"
METRIC = "rank-truncated PCG iters/s at 3D n=1024 (C4, eps=1e-6)"
UNIT = "iters/s"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


FP64_DMMA_TFLOPS = 37.16   # measured on this pool's B200 (tools/peak_fp64.cu, profiles/r01_peak_fp64.jsonl)


class Clocks:
    """nvidia-smi sampling during the timed region (profiling recipe's clocks line)."""

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_{os.getpid()}.csv")

    def __enter__(self):
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", os.environ.get("FC_BENCH_CLOCK_MS", "200")],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()
            self.f.close()

    def summary(self):
        out = {"sm_mhz": None, "sm_max_mhz": None, "reasons": []}
        try:
            rows = [l.split(",") for l in open(self.path).read().strip().splitlines() if l.strip()]
            sm = [float(r[1]) for r in rows]
            out["sm_mhz"] = float(np.median(sm)) if sm else None
            out["sm_max_mhz"] = float(rows[0][2]) if rows else None
            names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
            seen = set()
            for r in rows:
                for k, name in enumerate(names):
                    if r[5 + k].strip().lower() == "active":
                        seen.add(name)
            out["reasons"] = sorted(seen)
            out["samples"] = len(rows)
        except Exception:
            pass
        return out


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def aggregate_over_ranks(t_seconds: float, iters: int, world: int, device: str):
    """Whole-job totals of a replicas run: the device time is the MAX over ranks (the job ends
    when the slowest replica ends), the PCG iterations are SUMMED over ranks."""
    if world <= 1:
        return t_seconds, iters
    import torch
    import torch.distributed as dist
    t = torch.tensor([t_seconds], dtype=torch.float64, device=device)
    k = torch.tensor([float(iters)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.all_reduce(k, op=dist.ReduceOp.SUM)
    return float(t.item()), int(round(k.item()))


def oracle_sample(n=64, iters_cap=3):
    """Oracle PCG on the C4 workload at n = 64 with its own setup (bounded): (iters, loop s)."""
    from oracle import cp as cpm
    from oracle import pcg as P
    from synth import make_problem
    p = make_problem("C4", n=n)
    st = P.setup(p)
    B = cpm.normalized(p.b_w, p.b_U)
    t0 = time.perf_counter()
    _, rep = P.pcg(lambda x: cpm.apply(st.V, st.F, x), lambda x: cpm.apply(st.V, st.G, x), B, p.eps,
                   p.tol_stop, kmax=iters_cap)
    dt = time.perf_counter() - t0
    return rep["iters"], dt


def device_setup_for_oracle(ctx, p, prm):
    """The oracle's PCG needs only (lambda, V) per mode and the spectral CPs F, G; its own setup
    materialises n^3 entries of D (infeasible at n = 1024), so the device-built setup is exported
    through the C-ABI (sl_get_eigen, op_get_spectral_cp) - outside every timed region."""
    from oracle import cp as cpm
    from oracle import pcg as P
    from paper_2006_09314_b200.binding import FC_F, FC_G
    ctx.sl_setup(p.n, p.a_mid, prm)
    lams, V = [], []
    for l in range(3):
        lam, Vl = ctx.sl_get_eigen(l)
        lams.append(lam.cpu().numpy())
        V.append(Vl.cpu().numpy())
    Fw, FU = ctx.op_get_spectral_cp(FC_F).to_numpy()
    Gw, GU = ctx.op_get_spectral_cp(FC_G).to_numpy()
    return P.Setup(lams, V, cpm.CP(Fw, FU), cpm.CP(Gw, GU))


def oracle_c4_step(p, st, kmax=1):
    """One bounded step of the oracle on the headline workload (C4, n = 1024): Algorithm 1 as it
    stands (oracle/pcg.py: Z0 = trunc(G B), then kmax iterations), timed on the host cores."""
    from oracle import cp as cpm
    from oracle import pcg as P
    B = cpm.normalized(p.b_w, p.b_U)
    t0 = time.perf_counter()
    _, rep = P.pcg(lambda x: cpm.apply(st.V, st.F, x), lambda x: cpm.apply(st.V, st.G, x), B, p.eps,
                   p.tol_stop, kmax=kmax)
    return rep["iters"], time.perf_counter() - t0, rep


ORACLE_SAMPLE = ("oracle (NumPy/SciPy FP64, oracle/pcg.py as it stands) on the headline workload C4 n=1024 "
                 "eps=1e-6 with the device-built eigenpairs and spectral CPs injected: Z0 + the first PCG "
                 "iteration per step (the cheapest iteration: later ones grow with the ranks)")


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import torch
    from paper_2006_09314_b200.binding import Library, make_params
    from synth import make_problem
    torch.cuda.set_device(0)
    p = make_problem("C4", n=args.n, eps=args.eps)
    ctx = Library().context()
    st = device_setup_for_oracle(ctx, p, make_params(p.alpha, p.beta, p.eps, p.tol_stop))
    for _ in range(args.warmup):
        oracle_sample(n=16, iters_cap=1)          # the oracle has nothing to warm up: tiny runs
    per, iters_tot = [], 0
    for _ in range(args.steps):
        it, dt, _ = oracle_c4_step(p, st, kmax=1)
        iters_tot += it
        per.append(dt)
    v = iters_tot / sum(per)
    cores = os.cpu_count()
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * float(np.mean(per)),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": WORKLOAD, "n": p.n, "eps": p.eps,
                                            "sample": "Z0 + 1 PCG iteration per step"},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": ORACLE_SAMPLE},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=1024)
    ap.add_argument("--eps", type=float, default=1e-6)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2006_09314_b200.binding import DeviceCP, Library, make_params, kernel_launches
    from synth import make_problem

    p = make_problem("C4", n=args.n, eps=args.eps)
    L = Library()
    stream = torch.cuda.current_stream()
    ctx = L.context(stream.cuda_stream)
    prm = make_params(p.alpha, p.beta, p.eps, p.tol_stop)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    ctx.sl_setup(p.n, p.a_mid, prm)
    e1.record(stream)
    torch.cuda.synchronize()
    setup_ms = e0.elapsed_time(e1)
    b = DeviceCP.from_numpy(p.b_w, p.b_U)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    for _ in range(max(args.warmup, 0)):
        u, rep, rc = ctx.pcg_solve(b, prm)
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize()

    # ---- device-timed region: K solves from HBM-resident b ------------------------------
    times, iters, reps, rcs = [], 0, [], []
    ucap = 4096                                 # the solution buffer is allocated once, outside
    u = DeviceCP(p.n, ucap)                     # the timed region (pcg_solve grows it if needed)
    l0 = kernel_launches(L)
    barrier()
    with Clocks(local) as clk:
        for _ in range(args.steps):
            flush.fill_(1.0)                    # L2 flush (outside the events)
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record(stream)
            u, rep, rc = ctx.pcg_solve(b, prm, cap=u.cap, u=u)
            s1.record(stream)
            s1.synchronize()
            times.append(s0.elapsed_time(s1))
            iters += rep["iters"]
            reps.append(rep)
            rcs.append(rc)
    barrier()
    launches = (kernel_launches(L) - l0) // max(args.steps, 1)
    t_total, iters = aggregate_over_ranks(sum(times) / 1e3, iters, world, "cuda")
    value = iters / t_total

    # ---- end to end through the public API with HOST buffers ----------------------------
    hw = torch.tensor(p.b_w, dtype=torch.float64).pin_memory()
    hU = [torch.tensor(np.ascontiguousarray(p.b_U[l].T), dtype=torch.float64).pin_memory() for l in range(3)]
    cap_out = max(u.cap, max(r["rank_X"][-1] for r in reps) if reps else 1)
    hu_w = torch.empty(cap_out, dtype=torch.float64).pin_memory()
    hu_U = [torch.empty(cap_out, p.n, dtype=torch.float64).pin_memory() for _ in range(3)]
    e2e_times, e2e_iters, h2d, d2h = [], 0, 0, 0
    barrier()
    for _ in range(args.steps):
        flush.fill_(1.0)
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        bd = DeviceCP(p.n, hw.numel())
        bd.rank = hw.numel()
        bd.w[:bd.rank].copy_(hw, non_blocking=True)
        for l in range(3):
            bd.U[l][:bd.rank].copy_(hU[l], non_blocking=True)
        u, rep, rc = ctx.pcg_solve(bd, prm, cap=u.cap, u=u)
        rcs.append(rc)
        R = u.rank
        hu_w[:R].copy_(u.w[:R], non_blocking=True)
        for l in range(3):
            hu_U[l][:R].copy_(u.U[l][:R], non_blocking=True)
        s1.record(stream)
        s1.synchronize()
        e2e_times.append(s0.elapsed_time(s1))
        e2e_iters += rep["iters"]
        h2d = 8 * (hw.numel() + 3 * hw.numel() * p.n)
        d2h = 8 * (R + 3 * R * p.n)
    t_e2e, e2e_iters = aggregate_over_ranks(sum(e2e_times) / 1e3, e2e_iters, world, "cuda")
    e2e_value = e2e_iters / t_e2e

    # ---- dominant kernel class of the step: the DMMA GEMMs (one extra, untimed solve with every
    # GEMM launch bracketed by events on the library stream; algorithmic flops 2MNK) ----------
    ctx.profile_gemm(True)
    ctx.profile_kernel(1, True)
    flush.fill_(1.0)
    _, rep_p, _ = ctx.pcg_solve(b, prm)
    gp = ctx.profile_gemm(False)
    step_ms = float(np.median(times))
    ach = gp["flops"] / (gp["ms"] * 1e-3) / 1e12 if gp["ms"] > 0 else 0.0
    roof = {"kernel": "dgemm_dmma_kernel / dgemm_big_kernel (all DMMA GEMM launches of one pcg_solve)",
            "bound": "tensor", "achieved": ach, "peak": FP64_DMMA_TFLOPS, "unit": "TFLOP/s",
            "frac": ach / FP64_DMMA_TFLOPS, "traffic": gemm_class_traffic(),
            "peak_source": "measured DMMA m8n8k4 FP64 peak (tools/peak_fp64.cu); MEASURED_PEAKS.json has no FP64 entry",
            "launches_per_step": gp["launches"], "gemm_ms_per_step": gp["ms"],
            "share_of_step": gp["ms"] / step_ms if step_ms > 0 else None}
    # the HBM-class kernels: the eigen-coordinate Khatri-Rao basis over the
    # same profiled solve, and cp_dot's Hadamard-of-Grams reduction at C4-iterate ranks
    kr = ctx.profile_kernel(1, False)
    roof_hbm = hbm_roofline(ctx, p.n, kr)
    # variant (not the headline): the same solve with the preconditioner CP at rank r_G = 24
    # instead of the paper's 6 [P:990] (DESIGN.md §7 iteration counts): time-to-eps it reaches
    variant = rg_variant(L, p, stream)
    # the north-star's mode-transform kernel at a C5 cell (inverse transform + Khatri-Rao operand)
    roof_apply = apply_roofline(ctx, L, p.n)
    # the same two kernels at the largest n = 1024 cell of the C5 sweep (R = 256, r = 32: 201 MB
    # written by the K6 product, 1536 output tiles): launch latency no longer dominates the K6 time
    roof_apply_large = apply_roofline(ctx, L, p.n, R=256, r=32, reps=5)
    if rank != 0:
        return
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": float(np.mean(times)), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "n": p.n, "eps": p.eps, "tol_stop": p.tol_stop,
                   "l2": "flushed (512 MiB write) between timed steps", "parallelism": "replicas",
                   "setup_ms": setup_ms},
        # every timed solve must have converged (rc 0, A13) for a time-to-eps to exist
        "rc": sorted(set(int(r) for r in rcs)),
        "converged_all": all(r == 0 for r in rcs),
        "time_to_eps_ms": float(np.median(times)) if all(r == 0 for r in rcs) else None,
        "step_ms": [round(t, 2) for t in times],
        "slowest_step_iter_ms": [round(t, 1) for t in reps[int(np.argmax(times))]["t_iter_ms"]] if reps else [],
        "fastest_step_iter_ms": [round(t, 1) for t in reps[int(np.argmin(times))]["t_iter_ms"]] if reps else [],
        "iters_per_solve": reps[-1]["iters"] if reps else 0,
        "final_rel_res": reps[-1]["rel_res"][-1] if reps else None,
        "ranks_last_iter": {k: reps[-1][k][-1] for k in ("rank_X", "rank_R", "rank_S", "rank_Z", "rank_P")} if reps else {},
        "gpu_launches": int(launches),
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)},
        "roofline": roof,
        "roofline_apply": roof_apply,
        "roofline_apply_large": roof_apply_large,
        "roofline_hbm": roof_hbm,
        "variant_rG24": variant,
        "clocks": clk.summary(),
    }
    if not args.no_cpu_baseline and world == 1:
        st_o = device_setup_for_oracle(ctx, p, prm)
        it, dt, rep_o = oracle_c4_step(p, st_o, kmax=1)
        # same inputs, same first iteration: the oracle's residual and ranks are the device's
        same = (abs(rep_o["rel_res"][0] - reps[-1]["rel_res"][0]) <= 1e-5 * reps[-1]["rel_res"][0]
                and rep_o["rank_S"][0] == reps[-1]["rank_S"][0] and rep_o["rank_R"][0] == reps[-1]["rank_R"][0])
        it64, dt64 = oracle_sample(iters_cap=2)
        line["cpu_baseline"] = {"value": it / dt, "unit": UNIT, "cores": os.cpu_count(), "kind": "oracle",
                                "sample": ORACLE_SAMPLE, "seconds": dt, "iters": it,
                                "first_iteration_matches_device": bool(same),
                                "n64_own_setup": {"value": it64 / dt64, "unit": UNIT, "iters": it64, "seconds": dt64}}
    print(json.dumps(line), flush=True)


def rg_variant(L, p, stream, rG=24, reps=3):
    """C4 with params.precond_rank = rG (everything else as the headline): median device time of
    `reps` solves after one warm-up, iterations, iters/s, final rel_res."""
    import torch
    from paper_2006_09314_b200.binding import DeviceCP, make_params
    ctx = L.context(stream.cuda_stream)
    prm = make_params(p.alpha, p.beta, p.eps, p.tol_stop, precond_rank=rG)
    ctx.sl_setup(p.n, p.a_mid, prm)
    b = DeviceCP.from_numpy(p.b_w, p.b_U)
    u, rep, rc = ctx.pcg_solve(b, prm)
    ts, its, rcs = [], [], []
    for _ in range(reps):
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        u, rep, rc = ctx.pcg_solve(b, prm, cap=u.cap, u=u)
        s1.record(stream)
        s1.synchronize()
        ts.append(s0.elapsed_time(s1))
        its.append(rep["iters"])
        rcs.append(rc)
    t = float(np.median(ts))
    return {"precond_rank": rG, "time_to_eps_ms": t if all(r == 0 for r in rcs) else None, "iters": its[-1],
            "iters_per_s": sum(its) / (sum(ts) * 1e-3), "rel_res": rep["rel_res"][-1], "rc": sorted(set(rcs)),
            "note": "variant, not the headline: the paper fixes r_G = 6 [P:990]"}


def hbm_peak():
    pk = _peaks()
    for k in ("hbm_gbs", "hbm_copy_gbs", "hbm_GBps"):
        if isinstance(pk.get(k), (int, float)):
            return float(pk[k]), f"MEASURED_PEAKS.json {k}"
    return 6536.0, "MEASURED_PEAKS.json hbm_gbs (6536) not readable: fallback"


def hbm_roofline(ctx, n, kr, R=4096, reps=5):
    """K9 (dot_reduce: sum_{k,m} wx wy G0 G1 G2, 24 B per entry) timed inside cp_dot of two
    rank-R CPs at mode size n (C4 iterates reach R ~ 4000-6000), and K6 (Khatri-Rao basis of the
    fused apply) over one profiled C4 solve (kr).  achieved = algorithmic bytes / event time."""
    from paper_2006_09314_b200.binding import DeviceCP
    from synth import random_cp
    peak, src = hbm_peak()
    w, U = random_cp(n, R, 41)
    x = DeviceCP.from_numpy(w, U)
    w, U = random_cp(n, R, 42)
    y = DeviceCP.from_numpy(w, U)
    ctx.cp_dot(x, y)
    ctx.profile_kernel(0, True)
    for _ in range(reps):
        ctx.cp_dot(x, y)
    d = ctx.profile_kernel(0, False)
    ach = d["bytes"] / (d["ms"] * 1e-3) / 1e9 if d["ms"] > 0 else 0.0
    kra = kr["bytes"] / (kr["ms"] * 1e-3) / 1e9 if kr["ms"] > 0 else 0.0
    return {"dot_reduce": {"kernel": "dot_reduce_kernel (K9, cp_dot Hadamard-of-Grams reduction)",
                           "bound": "hbm", "cell": {"n": n, "R1": R, "R2": R}, "achieved": ach, "peak": peak,
                           "unit": "GB/s", "frac": ach / peak, "bytes_per_launch": d["bytes"] / max(d["launches"], 1),
                           "ms_per_launch": d["ms"] / max(d["launches"], 1), "traffic": None, "peak_source": src},
            "kr_basis": {"kernel": "hadamard_basis_kernel (K6, eigen-coordinate Khatri-Rao basis, one C4 solve)",
                         "bound": "hbm", "achieved": kra, "peak": peak, "unit": "GB/s", "frac": kra / peak,
                         "launches": kr["launches"], "bytes_per_launch": kr["bytes"] / max(kr["launches"], 1),
                         "ms_per_launch": kr["ms"] / max(kr["launches"], 1), "traffic": None, "peak_source": src}}


def apply_roofline(ctx, L, n, R=64, r=16, reps=10):
    """fracop_apply at the C5 cell (n, R, r): the fused Khatri-Rao inverse transform timed with
    CUDA events on the library stream (fc_last_kernel_stats), algorithmic flops 3*2n^2*rR."""
    import torch
    from paper_2006_09314_b200.binding import DeviceCP, FC_F
    from synth import random_cp
    w, U = random_cp(n, R, 5)
    x = DeviceCP.from_numpy(w, U)
    y = DeviceCP(n, r * R)
    # the context already holds C4's operator; use a fixed-rank random CP of the C5 shape
    sw, sU = random_cp(n, r, 77)
    ctx.op_set_spectral_cp(FC_F, DeviceCP.from_numpy(sw, sU))
    for _ in range(3):
        ctx.fracop_apply(FC_F, x, y)
    ms = []
    ctx.profile_kernel(2, True)
    for _ in range(reps):
        ctx.fracop_apply(FC_F, x, y)
        ms.append(ctx.last_kernel_stats()["ms"])
    kp = ctx.profile_kernel(2, False)
    st = ctx.last_kernel_stats()
    t = float(np.median(ms))
    ach = st["flops"] / (t * 1e-3) / 1e12
    peak_hbm, _ = hbm_peak()
    kr_gbs = kp["bytes"] / (kp["ms"] * 1e-3) / 1e9 if kp["ms"] > 0 else 0.0
    return {"kernel": "dgemm_big_streamk_kernel (inverse mode transform Y_l = V_l Yhat_l, S7, stream-K over the SMs; Yhat = u_F (.) V^T x by kr_product_kernel, K6)",
            "cell": {"n": n, "R": R, "r": r}, "bound": "tensor", "achieved": ach,
            "peak": FP64_DMMA_TFLOPS, "unit": "TFLOP/s", "frac": ach / FP64_DMMA_TFLOPS,
            "peak_source": "measured DMMA m8n8k4 FP64 peak (tools/peak_fp64.cu); MEASURED_PEAKS.json has no FP64 entry",
            "traffic": kr_traffic(n, R, r), "ms": t,
            "kr_product": {"kernel": "kr_product_kernel (K6, Yhat = u_F (.) V^T x, 3 modes per launch)", "bound": "hbm",
                           "achieved": kr_gbs, "peak": peak_hbm, "unit": "GB/s", "frac": kr_gbs / peak_hbm,
                           "ms_per_launch": kp["ms"] / max(kp["launches"], 1),
                           "bytes_per_launch": kp["bytes"] / max(kp["launches"], 1)}}


def gemm_class_traffic():
    """DRAM bytes (read + write) per launch of the 64 x 64 DMMA GEMM kernel averaged over one C4
    setup + solve, from the committed ncu capture (profiles/r02c_gemm_class_traffic.json), or None."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "r02c_gemm_class_traffic.json")))
        return d["dram_bytes_per_launch"]
    except (OSError, ValueError, KeyError):
        return None


def kr_traffic(n, R, r):
    """DRAM bytes (read + write) of one inverse-transform launch at this C5 cell, from the committed
    `ncu --set full` capture of the current kernel (profiles/r02c_inv_traffic.json), or None."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "r02c_inv_traffic.json")))
    except (OSError, ValueError):
        return None
    if (d.get("n"), d.get("R"), d.get("r")) != (n, R, r):
        return None
    return d["dram_bytes"]


if __name__ == "__main__":
    main()
