"""Run a few frames of one config (for ncu captures): python tools/one_frame.py c2 [frames] [key=val ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import scenegen  # noqa: E402
from paper_2202_12567_b200 import lmc  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 1
over = dict(a.split("=") for a in sys.argv[3:])
over = {k: (float(v) if ("." in v or "e" in v) else int(v)) for k, v in over.items()}
x = scenegen.make_inputs(scenegen.preset(name, **over))
fr = lmc.Frame(x)
img = torch.zeros(x.height * x.width * 3, device="cuda")
for _ in range(frames):
    fr.run(img)
torch.cuda.synchronize()
print("ok", fr.stats()["sum_completed"])
