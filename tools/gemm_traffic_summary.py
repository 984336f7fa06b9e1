"""Summarise an ncu --csv capture (gpu__time_duration.sum, dram__bytes_read.sum,
dram__bytes_write.sum per launch) of the small DMMA GEMM kernel over one C4 setup + solve:
launches, total time, DRAM bytes per launch (read + write).  Prints one JSON object."""
import collections
import csv
import json
import sys

UNIT_T = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3}
UNIT_B = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main(path):
    rows = list(csv.reader(open(path)))
    h = None
    per = collections.defaultdict(dict)
    for r in rows:
        if h is None:
            if "Kernel Name" in r:
                h = r
            continue
        if len(r) < len(h):
            continue
        d = dict(zip(h, r))
        if "dgemm_dmma_kernel<0, 0>" not in d["Kernel Name"] and "dgemm_dmma_kernel<false, false>" not in d["Kernel Name"]:
            continue
        v = float(d["Metric Value"].replace(",", ""))
        m = d["Metric Name"]
        if m == "gpu__time_duration.sum":
            v *= UNIT_T.get(d["Metric Unit"], 1e-6)
        else:
            v *= UNIT_B.get(d["Metric Unit"], 1.0)
        per[d["ID"]][m] = v
    n = len(per)
    t = sum(x.get("gpu__time_duration.sum", 0.0) for x in per.values())
    rd = sum(x.get("dram__bytes_read.sum", 0.0) for x in per.values())
    wr = sum(x.get("dram__bytes_write.sum", 0.0) for x in per.values())
    print(json.dumps({"kernel": "dgemm_dmma_kernel<0, 0> (64 x 64 DMMA tiles), every launch of one C4 setup + pcg_solve",
                      "source": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                                "--clock-control none -k regex:dgemm_dmma_kernel python tools/one_solve.py 1024",
                      "launches": n, "gpu_time_ms_serialised": t, "dram_read_bytes": rd, "dram_write_bytes": wr,
                      "dram_bytes_per_launch": (rd + wr) / max(n, 1)}, indent=1))


if __name__ == "__main__":
    main(sys.argv[1])
