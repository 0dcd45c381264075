"""triangle-mesh visibility through the device BVH, bit-exact against the oracle's
brute-force fp64 Moller-Trumbore test over every triangle (R39)."""
import numpy as np
import pytest

import oracle
import scenegen
from tests._mini import mini

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no GPU", allow_module_level=True)
from paper_2202_12567_b200 import lmc  # noqa: E402
from tests.test_gpu_parity import check_slice  # noqa: E402


def _pairs(x, n, seed):
    rng = np.random.default_rng(seed)
    return (rng.integers(0, x.m, n).astype(np.int32), rng.integers(0, x.vpls["px"].size, n).astype(np.int32))


@pytest.mark.parametrize("name,n", [("t_mesh", 300_000), ("c_mesh", 40_000)])
def test_mesh_entries_bit_exact(name, n):
    x = scenegen.make_inputs(name)
    fr = lmc.Frame(x)
    rows, vp = _pairs(x, n, 39)
    got = fr.eval_entries(rows, vp)
    ref = oracle.Oracle(x).entries_T(rows, vp)
    bad = np.flatnonzero(got != ref)
    assert bad.size == 0, f"{bad.size} of {n} entries differ, first at pair {bad[:3]}"
    # the meshes matter: removing them changes some decisions
    x0 = scenegen.make_inputs(name)
    x0.prims = dict(x0.prims, tri=np.zeros((0, 9), np.float32))
    ref0 = oracle.Oracle(x0).entries_T(rows, vp)
    assert np.count_nonzero(ref0 != ref) > n // 1000
    fr.close()


def test_mesh_frame_parity():
    x = scenegen.make_inputs("t_mesh")
    fr = lmc.Frame(x)
    img = torch.zeros(x.height * x.width * 3, device="cuda")
    fr.run(img)
    torch.cuda.synchronize()
    img = img.view(-1, 3).cpu().numpy().astype(np.float64)
    off, _ = fr.slices()
    for r in oracle.Oracle(x).run_slices(list(range(off.size - 1)), stage=4):
        check_slice(x, fr, img, r)
    fr.close()


def test_mesh_degenerate_segments():
    """axis-aligned segments (the slab test's zero-slope axes), segments in a triangle's plane
    (det = 0), through shared vertices and edges of a fan, and ending on the mesh"""
    fan = []
    c = np.array([0.5, 0.5, 0.5])
    for k in range(8):
        a0, a1 = 2 * np.pi * k / 8, 2 * np.pi * (k + 1) / 8
        fan.append(np.r_[c, c + 0.25 * np.array([np.cos(a0), 0.0, np.sin(a0)]),
                         c + 0.25 * np.array([np.cos(a1), 0.0, np.sin(a1)])])
    fan.append([0.25, 0.0, 0.25, 0.75, 0.0, 0.25, 0.5, 0.5, 0.25])      # vertical, plane z = 0.25
    pts, nrm = [], []
    for xx in (0.25, 0.5, 0.5 + 0.25 * np.cos(np.pi / 4), 0.6, 0.75):
        for zz in (0.25, 0.5, 0.5 + 0.25 * np.sin(np.pi / 4), 0.1):
            pts.append([xx, 0.0, zz])
            nrm.append([0.0, 1.0, 0.0])
    pts.append([0.5, 0.25, 0.25])      # on the vertical triangle, in its plane
    nrm.append([0.0, 1.0, 0.0])
    vp = [[0.5, 1.0, 0.5], [0.25, 1.0, 0.25], [0.75, 0.9, 0.5], [0.5, 0.5, 0.5], [0.5, 1.0, 0.25], [0.3, 0.25, 0.25]]
    vn = [[0.0, -1.0, 0.0]] * 5 + [[0.0, -1.0, 0.0]]
    x = mini(pts, nrm, vp, vn, [[1.0, 1.0, 1.0]] * len(vp), tri=np.asarray(fan, np.float32), shadow_eps=1e-6)
    fr = lmc.Frame(x)
    rows = np.repeat(np.arange(len(pts), dtype=np.int32), len(vp))
    vv = np.tile(np.arange(len(vp), dtype=np.int32), len(pts))
    got = fr.eval_entries(rows, vv)
    ref = oracle.Oracle(x).entries_T(rows, vv)
    assert np.array_equal(got, ref)
    assert (ref == 0).any() and (ref > 0).any()
    fr.close()


def test_mesh_bad_triangles_rejected():
    x = scenegen.make_inputs("t_mesh")
    tri = x.prims["tri"].copy()
    tri[3, 4] = np.nan
    x.prims = dict(x.prims, tri=tri)
    with pytest.raises(lmc.LmcError):
        lmc.Frame(x)
