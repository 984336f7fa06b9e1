#!/usr/bin/env python
"""bench.py — rank-truncated PCG on one B200 (driver contract).

Step = one pcg_solve of BASELINE.json configs[3] (C4: 3D n = 1024, C1 coefficients,
alpha = 0.5, beta = 0.01, rank-16 Gaussian-bump right-hand side, eps = 1e-6, tol = 10 eps):
Algorithm 1 [P:1825-1872] from b (resident in HBM) to u (in HBM).  The setup (S1-S4:
eigenpairs + spectral CPs) runs once before the timed region and is reported as setup_ms.
value = PCG iterations / second over the timed steps (all ranks); time_to_eps_ms = median
per-step solve time.  L2 is flushed (a 512 MiB write) between timed steps, outside the events.

--impl reference: the oracle (oracle/, NumPy/SciPy FP64) on the host cores, on a bounded
sample of the same workload (C4 at n = 64: the oracle's dense setup is infeasible at n = 1024).
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


FP64_DMMA_TFLOPS = 37.16   # measured on this pool's B200 (tools/peak_fp64.cu, profiles/r01_peaks.md)


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
    """Oracle PCG on the C4 workload at n = 64 (bounded): returns (iters, loop seconds)."""
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


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    per = []
    iters_tot = 0
    for _ in range(args.warmup):
        oracle_sample(iters_cap=1)
    t_all = 0.0
    for _ in range(args.steps):
        it, dt = oracle_sample(iters_cap=2)
        iters_tot += it
        t_all += dt
        per.append(dt)
    v = iters_tot / t_all
    cores = os.cpu_count()
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * float(np.mean(per)),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": WORKLOAD, "sample": "C4 workload at n=64, 2 PCG iterations per step"},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": "oracle (NumPy/SciPy) PCG loop, C4 workload at n=64, 2 iterations per step"},
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
    times, iters, reps = [], 0, []
    l0 = kernel_launches(L)
    barrier()
    with Clocks(local) as clk:
        for _ in range(args.steps):
            flush.fill_(1.0)                    # L2 flush (outside the events)
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record(stream)
            u, rep, rc = ctx.pcg_solve(b, prm)
            s1.record(stream)
            s1.synchronize()
            times.append(s0.elapsed_time(s1))
            iters += rep["iters"]
            reps.append(rep)
    barrier()
    launches = (kernel_launches(L) - l0) // max(args.steps, 1)
    t_total, iters = aggregate_over_ranks(sum(times) / 1e3, iters, world, "cuda")
    value = iters / t_total

    # ---- end to end through the public API with HOST buffers ----------------------------
    hw = torch.tensor(p.b_w, dtype=torch.float64).pin_memory()
    hU = [torch.tensor(np.ascontiguousarray(p.b_U[l].T), dtype=torch.float64).pin_memory() for l in range(3)]
    cap_out = max(r["rank_X"][-1] for r in reps) if reps else 1
    hu_w = torch.empty(4096, dtype=torch.float64).pin_memory()
    hu_U = [torch.empty(4096, p.n, dtype=torch.float64).pin_memory() for _ in range(3)]
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
        u, rep, rc = ctx.pcg_solve(bd, prm)
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
    flush.fill_(1.0)
    _, rep_p, _ = ctx.pcg_solve(b, prm)
    gp = ctx.profile_gemm(False)
    step_ms = float(np.median(times))
    ach = gp["flops"] / (gp["ms"] * 1e-3) / 1e12 if gp["ms"] > 0 else 0.0
    roof = {"kernel": "dgemm_dmma_kernel / dgemm_big_kernel (all DMMA GEMM launches of one pcg_solve)",
            "bound": "tensor", "achieved": ach, "peak": FP64_DMMA_TFLOPS, "unit": "TFLOP/s",
            "frac": ach / FP64_DMMA_TFLOPS, "traffic": None,
            "peak_source": "measured DMMA m8n8k4 FP64 peak (tools/peak_fp64.cu); MEASURED_PEAKS.json has no FP64 entry",
            "launches_per_step": gp["launches"], "gemm_ms_per_step": gp["ms"],
            "share_of_step": gp["ms"] / step_ms if step_ms > 0 else None}
    # the north-star's mode-transform kernel at a C5 cell (fused Khatri-Rao inverse transform)
    roof_apply = apply_roofline(ctx, L, p.n)
    if rank != 0:
        return
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": float(np.mean(times)), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "n": p.n, "eps": p.eps, "tol_stop": p.tol_stop,
                   "l2": "flushed (512 MiB write) between timed steps", "parallelism": "replicas",
                   "setup_ms": setup_ms},
        "time_to_eps_ms": float(np.median(times)),
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
        "clocks": clk.summary(),
    }
    if not args.no_cpu_baseline and world == 1 or (not args.no_cpu_baseline and rank == 0):
        it, dt = oracle_sample(iters_cap=2)
        line["cpu_baseline"] = {"value": it / dt, "unit": UNIT, "cores": os.cpu_count(), "kind": "oracle",
                                "sample": "oracle PCG loop, C4 workload at n=64 (dense oracle setup infeasible at n=1024), 2 iterations"}
    print(json.dumps(line), flush=True)


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
    for _ in range(reps):
        ctx.fracop_apply(FC_F, x, y)
        ms.append(ctx.last_kernel_stats()["ms"])
    st = ctx.last_kernel_stats()
    t = float(np.median(ms))
    ach = st["flops"] / (t * 1e-3) / 1e12
    return {"kernel": "dgemm_dmma_kernel<KR> (fused Khatri-Rao inverse mode transform, S6+S7)",
            "cell": {"n": n, "R": R, "r": r}, "bound": "tensor", "achieved": ach,
            "peak": FP64_DMMA_TFLOPS, "unit": "TFLOP/s", "frac": ach / FP64_DMMA_TFLOPS,
            "peak_source": "measured DMMA m8n8k4 FP64 peak (tools/peak_fp64.cu); MEASURED_PEAKS.json has no FP64 entry",
            "traffic": kr_traffic(n, R, r), "ms": t}


def kr_traffic(n, R, r):
    """DRAM bytes (read + write) of one fused KR inverse-transform launch at this C5 cell, from the
    committed `ncu --set full` capture (profiles/r01h_kr_traffic.json), or None."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "r01h_kr_traffic.json")))
    except (OSError, ValueError):
        return None
    if (d.get("n"), d.get("R"), d.get("r")) != (n, R, r):
        return None
    return d["dram_bytes"]


if __name__ == "__main__":
    main()
