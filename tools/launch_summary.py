"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per-kernel totals and shares."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, mi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    v = float(r[mi].replace(",", "")) * scale.get(r[ui], 1.0)
    k = r[ki].split("(")[0]
    agg[k][0] += 1
    agg[k][1] += v
tot = sum(a[1] for a in agg.values())
n = sum(a[0] for a in agg.values())
for line in sys.argv[2:]:
    print("# " + line)
print(f"# total kernel time {tot:.1f} ms over {n} launches")
print("ms_total,share_pct,launches,kernel")
for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{a[1]:.3f},{100 * a[1] / tot:.2f},{a[0]},{k}")
