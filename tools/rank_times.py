"""Per-rank stage times of a P-way partition, measured one rank at a time on one GPU (the ranks'
compute is independent until the image gather; DESIGN §8 projection).  For each P and each chosen
rank r, a context with (rank r, world P) runs slicing (its replicated top levels + its subtree),
pass 1, coarsening, pass 2 and the completion of its slices; CUDA events per stage, mean over the
timed frames.  The image gather to rank 0 (one NCCL group of P - 1 receives of packed float4 rows)
is not run here.  Usage: python tools/rank_times.py c4 [frames] [P ...]   (prints one JSON line)"""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import scenegen  # noqa: E402
from paper_2202_12567_b200 import lmc  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 3
Ps = [int(a) for a in sys.argv[3:]] or [1, 2, 4, 8]
x = scenegen.make_inputs(scenegen.preset(name))
stages = ("slices", "pass1", "coarsen", "pass2", "complete")
out = {"config": name, "frames": frames, "ranks": []}
for P in Ps:
    for r in (range(P) if os.environ.get("ALL_RANKS") else sorted({0, P - 1, P // 2})):
        fr = lmc.Frame(x, rank=r, world=P, partition=int(os.environ.get("PARTITION", "0")))
        fr.set_timing(True)
        acc = {s: [] for s in stages}
        tot = []
        for k in range(frames + 1):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fr.build_slices()
            fr.sample_pass1()
            fr.coarsen_cut()
            fr.sample_pass2()
            fr.complete()
            e1.record()
            torch.cuda.synchronize()
            if k == 0:
                continue   # warm-up
            st = fr.stats()
            for s in stages:
                acc[s].append(st["ms_" + s])
            tot.append(e0.elapsed_time(e1))
        st = fr.stats()
        out["ranks"].append({"P": P, "rank": r, "partition": int(os.environ.get("PARTITION", "0")), "slices": st["slice_end"] - st["slice_begin"], "rows": st["rows"],
                             "ms": statistics.mean(tot), "ms_per_stage": {s: statistics.mean(v) for s, v in acc.items()},
                             "ms_solver": st["ms_solver"]})
        print(json.dumps(out["ranks"][-1]), file=sys.stderr, flush=True)
        fr.close()
print(json.dumps(out))
