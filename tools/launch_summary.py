"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list:
per-kernel count and total / mean duration (us), optionally only the last
`--tail` launches.    python tools/launch_summary.py launches.csv [--tail N]"""
import argparse
import collections
import csv

ap = argparse.ArgumentParser()
ap.add_argument("csv")
ap.add_argument("--tail", type=int, default=0)
a = ap.parse_args()
rows = [r for r in csv.DictReader(line for line in open(a.csv) if line.startswith('"'))
        if r.get("Metric Name") == "gpu__time_duration.sum"]
if a.tail:
    rows = rows[-a.tail:]
agg = collections.OrderedDict()
for r in rows:
    k = r["Kernel Name"].split("(")[0][:60]
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
    v = float(r["Metric Value"].replace(",", "")) * scale.get(r["Metric Unit"], 1e-3)
    c, t = agg.get(k, (0, 0.0))
    agg[k] = (c + 1, t + v)
tot = sum(t for c, t in agg.values())
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:60s} {c:5d} {t:12.1f} us {t / c:10.1f} us/launch {100 * t / tot:5.1f}%")
print(f"total {tot:.1f} us over {len(rows)} launches")
