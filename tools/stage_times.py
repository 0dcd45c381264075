"""Per-stage CUDA-event times of the hot path on one config (diagnostic, not the bench)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import scenegen  # noqa: E402
from paper_2202_12567_b200 import lmc  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 3
over = dict(a.split("=") for a in sys.argv[3:])
over = {k: (float(v) if "." in v or "e" in v else int(v)) for k, v in over.items()}
t0 = time.time()
x = scenegen.make_inputs(scenegen.preset(name, **over))
print(f"{name}: m={x.m} vpls={x.vpls['px'].size} gen {time.time()-t0:.1f}s", flush=True)
t0 = time.time()
fr = lmc.Frame(x)
torch.cuda.synchronize()
print(f"create {time.time()-t0:.2f}s", flush=True)
fr.set_timing(True)
img = torch.zeros(x.height * x.width * 3, device="cuda")
for k in range(frames):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fr.run(img)
    e1.record()
    torch.cuda.synchronize()
    st = fr.stats()
    print(f"frame {k}: {e0.elapsed_time(e1):.2f} ms | " + " ".join(f"{s}={st['ms_'+s]:.2f}" for s in
          ("slices", "pass1", "coarsen", "pass2", "complete", "resolve", "solver")), flush=True)
print({k: v for k, v in st.items() if not k.startswith("ms_")})
print("completed entries/s: %.3e" % (st["sum_completed"] / (e0.elapsed_time(e1) * 1e-3)))
print("rays/pixel: %.1f" % ((st["evals_pass1"] + st["evals_coarsen"] + st["evals_pass2"]) / st["rows"]))
