import sys, os
sys.path.insert(0, os.getcwd())
import dataclasses, numpy as np, torch
import scenegen, oracle
src = open('tests/test_gpu_fuzz.py').read()
a = src.index('TAU ='); b = src.index('@pytest.mark.parametrize')
ns = {'np': np, 'scenegen': scenegen, 'dataclasses': dataclasses}
exec(src[a:b], ns)
from paper_2202_12567_b200 import lmc
cfg = ns['random_config'](int(sys.argv[1]))
x = scenegen.make_inputs(cfg)
fr = lmc.Frame(x)
img = torch.zeros(x.height * x.width * 3, device="cuda")
fr.run(img); torch.cuda.synchronize()
off, rows = fr.slices()
o = oracle.Oracle(x)
for r in o.run_slices(list(range(off.size - 1)), stage=2):
    s = r["slice"]
    sm = fr.samples(s)
    g = set(zip(sm["row"].tolist(), sm["col"].tolist()))
    oo = set(zip(r["om_row"].tolist(), r["om_col"].tolist()))
    if g != oo:
        gc = {(a, b) for a, b, c in zip(sm["row"], sm["col"], sm["carried"]) if c}
        oc = {(a, b) for a, b, c in zip(r["om_row"], r["om_col"], r["om_carried"]) if c}
        print("slice", s, "m", off[s+1]-off[s], "n", len(r["cut_nodes"]), "nnz gpu", sm["nnz"], "orc", r["nnz"], "N", sm["target_N"], r["target_N"],
              "carried gpu", len(gc), "orc", len(oc), "n_new", r["n_new"], "forced", r["n_forced"], "draws", r["n_draws"])
        print(" only gpu", sorted(g - oo)[:10], "only oracle", sorted(oo - g)[:10])
        print(" carried only gpu", sorted(gc - oc)[:10], "carried only orc", sorted(oc - gc)[:10])
