"""Print a one-line summary of bench JSON lines (diagnostic)."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(f, "unreadable", e)
        continue
    r = d.get("roofline", {})
    st = {k: round(v, 2) for k, v in d.get("ms_per_stage", {}).items()}
    print(f, round(d["ms_per_step"], 2), "%.3g" % d["value"], "kern", round(r.get("kernel_ms", 0), 2),
          "frac", round(r.get("frac", 0), 3), st, d.get("clocks", {}).get("reasons"))
