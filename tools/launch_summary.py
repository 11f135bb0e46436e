"""Aggregate an ncu --metrics gpu__time_duration.sum CSV launch list by kernel.
usage: python tools/launch_summary.py launches.csv [passes]"""
import collections
import csv
import sys

UNIT = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3, "nsecond": 1e-6}
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
passes = int(sys.argv[2]) if len(sys.argv) > 2 else 1
h = rows[0]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    v = float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1.0)
    k = r[ki].split("(")[0].replace("lbg::<unnamed>::", "").replace("(anonymous namespace)::", "")[:60]
    agg[k][0] += 1
    agg[k][1] += v
tot = sum(a[1] for a in agg.values())
print(f"total {tot:.3f} ms over {passes} pass(es): {tot / passes:.3f} ms/pass")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:10]:
    print(f"  {k:60s} n={n:6d} {t / passes:9.3f} ms/pass {100 * t / tot:5.1f}%")
