"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel.

    python tools/launch_summary.py gpurun_out/launches.csv
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if "Kernel Name" in r and "Metric Value" in r:
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = d["Kernel Name"].split("(")[0][:60]
    v = float(d["Metric Value"].replace(",", ""))
    unit = d.get("Metric Unit", "ns")
    scale = {"ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6, "nsecond": 1}.get(unit, 1)
    agg[name][0] += 1
    agg[name][1] += v * scale
tot = sum(a[1] for a in agg.values())
print(f"{'kernel':62s} {'launches':>8s} {'total_ms':>10s} {'share':>7s}")
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:62s} {n:8d} {t / 1e6:10.3f} {100 * t / tot:6.2f}%")
print(f"{'total':62s} {sum(a[0] for a in agg.values()):8d} {tot / 1e6:10.3f}")
