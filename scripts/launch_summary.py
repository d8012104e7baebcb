"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list:
per-kernel count, average duration and share of the profiled launches."""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hdr = next(r for r in rows if r and r[0] == "ID")
    data = [dict(zip(hdr, r)) for r in rows[rows.index(hdr) + 1:] if len(r) == len(hdr)]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in data:
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        v *= {"nsecond": 1.0, "usecond": 1e3, "msecond": 1e6}.get(d["Metric Unit"], 1.0)
        name = d["Kernel Name"].split("(")[0][:70]
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    print(f"{len(data)} launches, {tot / 1e3:.1f} us total")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{100 * t / tot:6.2f}%  n={n:4d}  avg={t / n / 1e3:8.2f} us  {k}")


if __name__ == "__main__":
    main(sys.argv[1])
