"""GPU parity at BASELINE sizes for the paths added in round 2: sampled slices through every stage
against the oracle (cuts, coarsening records and Omega bit-exact, completion <= 1e-4, pixels
<= 1e-3; tests/test_gpu_parity.check_slice), in the launch configuration bench.py uses."""
import os

import numpy as np
import pytest

import oracle
import scenegen

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no GPU", allow_module_level=True)
from paper_2202_12567_b200 import lmc  # noqa: E402
from tests.test_gpu_parity import check_slice, pick  # noqa: E402


def _frame(cfg, env=None):
    old = {k: os.environ.get(k) for k in (env or {})}
    os.environ.update(env or {})
    try:
        x = scenegen.make_inputs(cfg)
        fr = lmc.Frame(x)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    img = torch.zeros(x.height * x.width * 3, device="cuda")
    fr.run(img)
    torch.cuda.synchronize()
    return x, fr, img.view(-1, 3).cpu().numpy().astype(np.float64)


def _check(x, fr, img, k=3):
    off, _ = fr.slices()
    for r in oracle.Oracle(x).run_slices(pick(off.size - 1, k), stage=4):
        check_slice(x, fr, img, r)
    fr.close()


@pytest.mark.parametrize("name,env", [("c3", {}), ("c4", {"LMC_ADM2": "1"}), ("c5_q8_r20", {})])
def test_lane_per_segment_adm_full_size(name, env):
    """the lane-per-segment ADM at full size: C3 (its default kernel at q = 16), C4 forced onto it
    (residuals spill to global memory), rank 8 at 20% sampling"""
    _check(*_frame(scenegen.preset(name), env))


def test_mesh_scene_full_size():
    """c_mesh (512 x 512, 100k VPLs, 6656 triangles): BVH visibility inside every entry kernel"""
    _check(*_frame(scenegen.preset("c_mesh")))


def test_variants_full_size():
    """SURVEY f3 at C2 size: image-space row importance, Eq. (1) sensitivity, Z-mode image"""
    _check(*_frame(scenegen.preset("c2", row_importance=1, cost_mode=1, resolve_mode=1)))


def test_count_target_full_size():
    """SURVEY f2 count-target coarsening at C2 size (cut of 450 nodes per slice)"""
    _check(*_frame(scenegen.preset("c2", coarsen_target=450)))


def test_mals_rank32_full_size():
    """masked ALS at the configs[4] corner q = 32, 5% (1024-node cut at 512-row slices)"""
    _check(*_frame(scenegen.preset("c5_q32_r5", solver=1)))
