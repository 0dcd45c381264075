"""Update profiles/r02_traffic.json's entry for one workload from an ncu --set full capture of its
dominant kernel: DRAM bytes per launch and the L1 data-pipe utilisation (the binding resource).
Usage: python tools/traffic_update.py REPORT.ncu-rep KEY KERNEL CAPTURE_TXT [OUT_JSON]"""
import csv
import io
import json
import os
import subprocess
import sys

rep, key, kernel, capture = sys.argv[1:5]
out = sys.argv[5] if len(sys.argv) > 5 else os.path.join(os.path.dirname(__file__), "..", "profiles", "r02_traffic.json")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h, units, vals = r[0], r[1], r[2]
d = dict(zip(h, vals))
u = dict(zip(h, units))


def num(name):
    v = float(d[name].replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u.get(name, "byte"), 1)
    return v * scale


rd, wr = num("dram__bytes_read.sum"), num("dram__bytes_write.sum")
l1 = None
for k in d:
    if k.startswith("l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed"):
        l1 = float(d[k])
tab = json.load(open(out)) if os.path.exists(out) else {}
ent = tab.get(key, {})
ent.update({"bytes": int(rd + wr), "kernel": kernel, "capture": capture, "read_gb": round(rd / 1e9, 2),
            "write_gb": round(wr / 1e9, 2)})
if l1 is not None:
    lim = ent.get("limiter", {})
    lim.update({"pct_of_peak": round(l1, 2), "metric": "l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed",
                "capture": capture})
    lim.setdefault("resource", "L1/shared-memory data pipe (LSU wavefronts)")
    ent["limiter"] = lim
tab[key] = ent
json.dump(tab, open(out, "w"), indent=1)
print(key, ent)
