"""Per CUDA source line ncu metrics (stall samples, instructions, shared wavefronts), top lines by stalls."""
import csv
import io
import subprocess
import sys

import os
flt = ["-k", os.environ["NCU_K"]] if os.environ.get("NCU_K") else []
out = subprocess.run(["ncu", "-i", sys.argv[1], *flt, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
items = []
fname, h = "?", None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        h = r
        si, ii = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
        wi = h.index("L1 Wavefronts Shared") if "L1 Wavefronts Shared" in h else si
        continue
    if h is None or not r[0].isdigit():
        continue

    def f(i):
        try:
            return float(r[i].replace(",", ""))
        except (ValueError, IndexError):
            return 0.0
    items.append((f(si), f(ii), f(wi), fname, int(r[0]), r[1]))
ts = sum(x[0] for x in items) or 1
ti = sum(x[1] for x in items) or 1
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
key = 2 if os.environ.get("NCU_SORT") == "wf" else 0
for s, i, w, fn, ln, src in sorted(items, key=lambda x: -x[key])[:n]:
    print(f"{fn[:12]:12s}:{ln:<4d} stall={100*s/ts:5.1f}% inst={100*i/ti:5.1f}% wf={w:.2e}  {src.strip()[:80]}")
