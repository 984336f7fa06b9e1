"""Summarise an ncu --csv launch list (gpu__time_duration.sum per launch) by kernel name."""
import collections
import csv
import sys

UNIT = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}


def main(path, top=24):
    rows = list(csv.reader(open(path)))
    h, agg = None, collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if h is None:
            if "Kernel Name" in r:
                h = r
            continue
        if len(r) < len(h):
            continue
        d = dict(zip(h, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", "")) * UNIT.get(d["Metric Unit"], 1e-6)
        k = d["Kernel Name"].split("(")[0].replace("fc::<unnamed>::", "")[:60]
        agg[k][0] += 1
        agg[k][1] += v
    tot = sum(v[1] for v in agg.values())
    print("total %.1f ms over %d launches" % (tot, sum(v[0] for v in agg.values())))
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        print("%6.2f%% %8.2f ms %5d %s" % (100 * v[1] / tot, v[1], v[0], k))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 24)
