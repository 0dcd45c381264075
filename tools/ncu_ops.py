"""Per-opcode totals (instructions, shared wavefronts, global L1 tag requests, stall samples) of an ncu report."""
import collections
import csv
import io
import re
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
idx = {k: i for i, k in enumerate(h)}
data = rows[2:]


def f(r, k):
    try:
        return float(r[idx[k]].replace(",", ""))
    except (KeyError, ValueError):
        return 0.0


agg = collections.defaultdict(lambda: [0.0] * 4)
for r in data:
    s = re.sub(r"^@!?U?P\w+\s+", "", r[1].strip())
    op = s.split()[0] if s else ""
    a = agg[op]
    a[0] += f(r, "Instructions Executed")
    a[1] += f(r, "L1 Wavefronts Shared")
    a[2] += f(r, "L1 Tag Requests Global")
    a[3] += f(r, "Warp Stall Sampling (All Samples)")
tot = sum(a[0] for a in agg.values())
ts = sum(a[3] for a in agg.values()) or 1
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
for op, a in sorted(agg.items(), key=lambda x: -x[1][0])[:n]:
    print(f"{op:24s} inst={a[0]:.2e} ({100*a[0]/tot:4.1f}%) shwf={a[1]:.2e} gtag={a[2]:.2e} stall={100*a[3]/ts:4.1f}%")
