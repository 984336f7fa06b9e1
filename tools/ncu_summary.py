"""Key counters of every launch in ncu reports (`ncu -i X.ncu-rep --page raw --csv`): duration, DRAM
bytes, pipe activity, occupancy, issue utilisation, the stall reasons per issued instruction.
`python tools/ncu_summary.py a.ncu-rep [b.ncu-rep ...]`"""
import csv
import io
import subprocess
import sys

KEYS = ["launch__grid_size", "launch__block_size", "launch__cluster_dim_z", "launch__registers_per_thread",
        "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]
STALL = "smsp__average_warps_issue_stalled_"


def main(paths):
    for p in paths:
        out = subprocess.run(["ncu", "-i", p, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(out)))
        if len(rows) < 3:
            print(p, ": no launches")
            continue
        h, u = rows[0], rows[1]
        for r in rows[2:]:
            d = dict(zip(h, r))
            units = dict(zip(h, u))
            print("###", p, "|", d.get("Kernel Name", "")[:110])
            for k in KEYS:
                if k in d and d[k] != "":
                    print(f"    {k:70s} {d[k]} {units.get(k, '')}")
            st = sorted(((float(v.replace(',', '')), k[len(STALL):-len('_per_issue_active.ratio')]) for k, v in d.items()
                         if k.startswith(STALL) and k.endswith("_per_issue_active.ratio") and v not in ("", "n/a")),
                        reverse=True)
            print("    stalls per issued instruction:", ", ".join(f"{k} {v:.2f}" for v, k in st[:6]))


if __name__ == "__main__":
    main(sys.argv[1:])
