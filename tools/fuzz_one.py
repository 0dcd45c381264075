import sys, os
sys.path.insert(0, os.getcwd())
import importlib, dataclasses, numpy as np, torch
import scenegen
src = open('tests/test_gpu_fuzz.py').read()
a = src.index('TAU ='); b = src.index('@pytest.mark.parametrize')
ns = {'np': np, 'scenegen': scenegen, 'dataclasses': dataclasses}
exec(src[a:b], ns)
from paper_2202_12567_b200 import lmc
k = int(sys.argv[1])
cfg = ns['random_config'](k)
over = dict(a.split('=') for a in sys.argv[2:])
cfg = dataclasses.replace(cfg, **{kk: type(getattr(cfg, kk))(v) for kk, v in over.items()})
print(cfg)
x = scenegen.make_inputs(cfg)
fr = lmc.Frame(x)
img = torch.zeros(x.height * x.width * 3, device="cuda")
for st in ("build_slices", "sample_pass1", "coarsen_cut", "sample_pass2", "complete"):
    getattr(fr, st)(); torch.cuda.synchronize(); print("ok", st, flush=True)
fr.resolve_image(img); torch.cuda.synchronize(); print("ok resolve")
