"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list by kernel."""
import collections
import csv
import sys


def main(path, top=20):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, mi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) <= mi:
            continue
        v = float(r[mi].replace(",", ""))
        v *= {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0,
              "second": 1e3, "s": 1e3}.get(r[ui], 1.0)
        name = r[ki].split("(")[0][:72]
        tot[name] += v
        cnt[name] += 1
    T = sum(tot.values())
    print(f"total {T:.1f} ms over {sum(cnt.values())} launches")
    for k, v in sorted(tot.items(), key=lambda x: -x[1])[:top]:
        print(f"{100 * v / T:6.2f}%  {v:10.2f} ms  {cnt[k]:5d}  {k}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 20)
