"""Randomised GPU parity: seeded random small configurations (scene kind incl. triangle meshes,
image size, VPL count, cut size, slice target, rank, rate, tau, solver, iteration count, tolerance,
the f2-f3 variants, seeds) — every slice through every stage against the oracle with the same
bars as tests/test_gpu_parity.check_slice (bit-exact cuts / Omega, completion <= 1e-4, pixels
<= 1e-3)."""
import dataclasses

import numpy as np
import pytest

import oracle
import scenegen

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no GPU", allow_module_level=True)
from paper_2202_12567_b200 import lmc  # noqa: E402
from tests.test_gpu_parity import check_slice  # noqa: E402

TAU = {"cornell": 1.0e-4, "interior": 1.0e-3, "mesh": 1.0e-3}


def random_config(k):
    rng = np.random.default_rng(91000 + k)
    kind = ["cornell", "interior", "mesh"][k % 3]
    nv = int(rng.integers(300, 6000))
    cut = int(rng.integers(16, min(nv, 200) + 1))
    solver = int(rng.random() < 0.3)
    q = int(rng.choice([4, 8, 16] + ([] if solver else [32])))
    base = scenegen.PRESETS["t_mesh" if kind == "mesh" else "t_cornell" if kind == "cornell" else "t_interior"]
    return dataclasses.replace(
        base, name=f"fuzz{k}", width=int(rng.integers(16, 73)), height=int(rng.integers(12, 61)), n_vpls=nv,
        cut_max=cut, slice_target=int(rng.integers(20, 201)), rank_q=q, rate=float(rng.uniform(0.03, 0.6)),
        tau=TAU[kind] * float(rng.choice([0.0, 0.3, 1.0, 5.0])), solver=solver,
        max_iter=int(rng.integers(1, 61)), tol=float(rng.choice([0.0, 0.0, 1e-3])),
        row_importance=int(rng.random() < 0.3), cost_mode=int(rng.random() < 0.3),
        resolve_mode=int(rng.random() < 0.3),
        coarsen_target=int(rng.integers(4, cut + 1)) if rng.random() < 0.25 else 0,
        seed=int(rng.integers(1, 2**62)), fixture_seed=int(rng.integers(1, 1000)))


@pytest.mark.parametrize("k", range(48))
def test_random_small_configs(k):
    cfg = random_config(k)
    x = scenegen.make_inputs(cfg)
    fr = lmc.Frame(x)
    img = torch.zeros(x.height * x.width * 3, device="cuda")
    fr.run(img)
    torch.cuda.synchronize()
    img = img.view(-1, 3).cpu().numpy().astype(np.float64)
    off, rows = fr.slices()
    o = oracle.Oracle(x)
    ooff, orows = o.slices()
    assert np.array_equal(off, ooff) and np.array_equal(rows, orows), cfg
    for r in o.run_slices(list(range(off.size - 1)), stage=4):
        check_slice(x, fr, img, r)
    fr.close()
