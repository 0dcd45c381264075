"""Time lmc_build_light_tree (step 1 on the GPU) on a config's VPLs: python tools/lighttree_time.py c4 [reps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import scenegen  # noqa: E402
from paper_2202_12567_b200 import lmc  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
x = scenegen.make_inputs(name)
lmc.build_light_tree(x.vpls, x.cfg.cut_max)
ts = []
for _ in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    t = lmc.build_light_tree(x.vpls, x.cfg.cut_max)
    ts.append(time.perf_counter() - t0)
print(f"{name}: {x.vpls['px'].size} VPLs, cut {t['global_cut'].size}: {1e3 * min(ts):.2f} ms (best of {reps}, "
      f"incl. H2D of the VPLs and D2H of the tree)")
