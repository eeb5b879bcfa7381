"""Aggregate an ncu gpu__time_duration launch list (CSV) per kernel (profiling aid)."""
import collections
import csv
import sys


def main(path, top=20):
    hdr = None
    agg = collections.defaultdict(lambda: [0, 0.0])
    each = collections.defaultdict(list)
    for r in csv.reader(open(path)):
        if "Kernel Name" in r:
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(
            d["Metric Unit"], 1.0)
        k = d["Kernel Name"].split("(")[0][:60]
        agg[k][0] += 1
        agg[k][1] += v
        each[k].append(v)
    tot = sum(v[1] for v in agg.values())
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        med = sorted(each[k])[len(each[k]) // 2]
        print(f"{k:44s} {n:6d} {t / 1e3:9.3f} ms  mean {t / n:9.2f} us  median {med:9.2f} us {100 * t / tot:5.1f}%")
    print(f"total {tot / 1e3:.3f} ms")


if __name__ == "__main__":
    main(sys.argv[1])
