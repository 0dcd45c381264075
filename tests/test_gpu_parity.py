"""GPU parity: the CUDA path (through the C-ABI) against the fp64 oracle on identical seeded inputs.

Bars (BASELINE north_star):
  * bit-exact: slices, pass-1 row sets and entries (fp64), coarsening decisions / eps / cost,
    final cuts, Omega index sets, carried flags; pass-2 values == float32(oracle fp64 value)
  * <= 1e-4 relative Frobenius error of every completed slice U V
  * <= 1e-3 relative error per pixel and channel (denominator floored at 1e-3 x mean luminance)
"""
import numpy as np
import pytest

import oracle
import scenegen

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no GPU", allow_module_level=True)
from paper_2202_12567_b200 import lmc  # noqa: E402

LUMW = np.array([0.2126, 0.7152, 0.0722])
_cache = {}


def frame(name, **over):
    key = (name, tuple(sorted(over.items())))
    if key not in _cache and len(_cache) >= 6:   # the library allows 16 live contexts per process
        old = next(iter(_cache))
        _cache.pop(old)[1].close()
    if key not in _cache:
        cfg_over = {k: v for k, v in over.items() if k in ("rank_q", "rate", "solver", "tau", "max_iter")}
        x = scenegen.make_inputs(scenegen.preset(name, **cfg_over))
        fr = lmc.Frame(x)
        img = torch.zeros(x.height * x.width * 3, device="cuda")
        fr.run(img)
        torch.cuda.synchronize()
        _cache[key] = (x, fr, img.view(-1, 3).cpu().numpy().astype(np.float64))
    return _cache[key]


def oracle_slices(x, ids):
    return oracle.Oracle(x).run_slices(ids, stage=4)


def pick(nslices, k=4):
    if nslices <= k:
        return list(range(nslices))
    return sorted(set([0, nslices - 1] + list(np.linspace(1, nslices - 2, k - 2).astype(int))))


def check_slice(x, fr, img, r, frob_tol=1e-4):
    s = r["slice"]
    # cut and coarsening record
    assert np.array_equal(fr.cut(s), r["cut_nodes"]), f"slice {s}: cut differs"
    co = fr.coarsen(s)
    proc = co["node"][co["processed"] == 1]
    assert np.array_equal(np.sort(proc), np.sort(r["proc_node"])), f"slice {s}: processed candidates differ"
    idx = {n: k for k, n in enumerate(co["node"])}
    for k, f in enumerate(r["proc_node"]):
        u = idx[f]
        assert co["merged"][u] == r["proc_merged"][k], f"slice {s}: merge decision of node {f}"
        assert co["eps"][u] == r["proc_eps"][k], f"slice {s}: eps of node {f}"
        assert co["cost"][u] == r["proc_cost"][k], f"slice {s}: cost of node {f}"
    # pass 1 (base pairs)
    p1 = fr.pass1(s)
    pk = {n: k for k, n in enumerate(r["proc_node"])}
    for b, f in enumerate(p1["node"]):
        k = pk[f]
        z = r["proc_zrows"][r["proc_zoff"][k]:r["proc_zoff"][k + 1]]
        n = p1["count"][b]
        assert np.array_equal(p1["rows"][b, :n], z), f"slice {s}: pass-1 rows of pair {f}"
        assert np.array_equal(p1["Ta"][b, :n], r["proc_Va"][r["proc_zoff"][k]:r["proc_zoff"][k + 1]])
        assert np.array_equal(p1["Tb"][b, :n], r["proc_Vb"][r["proc_zoff"][k]:r["proc_zoff"][k + 1]])
    # Omega
    sm = fr.samples(s)
    assert sm["nnz"] == r["nnz"], f"slice {s}: |Omega| {sm['nnz']} vs {r['nnz']}"
    assert np.array_equal(sm["row"], r["om_row"]) and np.array_equal(sm["col"], r["om_col"]), f"slice {s}: Omega"
    assert np.array_equal(sm["carried"], r["om_carried"]), f"slice {s}: carried flags"
    assert np.array_equal(sm["val"], r["om_val"].astype(np.float32)), f"slice {s}: sample values"
    assert sm["target_N"] == r["target_N"]
    # completion
    fa = fr.factors(s)
    assert (fa["flags"] & lmc.SLICE_DIRECT) == (r["flags"] & oracle.FLAG_DIRECT)
    assert (fa["flags"] & lmc.SLICE_ZERO) == (r["flags"] & oracle.FLAG_ZERO)
    if not (r["flags"] & (oracle.FLAG_DIRECT | oracle.FLAG_ZERO)):
        A = r["U"] @ r["V"]
        B = fa["U"].astype(np.float64) @ fa["V"].astype(np.float64)
        rel = np.linalg.norm(A - B) / np.linalg.norm(A)
        assert rel <= frob_tol, f"slice {s}: completed slice rel Frobenius {rel:.3g}"
        assert np.all(fa["U"] >= 0) or x.cfg.solver == 1
    # image rows of the slice
    pix = x.gbuf["pixel"][r["rows"]]
    ref = r["rgb"]
    got = img[pix]
    floor = 1e-3 * max(float((ref @ LUMW).mean()), 1e-30)
    relp = np.abs(got - ref) / np.maximum(np.abs(ref), floor)
    assert relp.max() <= 1e-3, f"slice {s}: max pixel rel error {relp.max():.3g}"
    return relp.max()


@pytest.mark.parametrize("name", ["c1", "t_interior"])
def test_entries_bit_exact(name):
    x, fr, _ = frame(name)
    o = oracle.Oracle(x)
    rng = np.random.default_rng(5)
    n = 20000
    rows = rng.integers(0, x.m, n)
    vp = rng.integers(0, x.vpls["px"].size, n)
    got = fr.eval_entries(rows, vp)
    ref = np.array([o.entry_T(r, v) for r, v in zip(rows, vp)])
    assert np.array_equal(got, ref), f"{np.sum(got != ref)} of {n} entries differ"
    assert (ref > 0).mean() > 0.2 and (ref == 0).mean() > 0.05


def test_entries_bit_exact_interior_full_scene():
    # every primitive kind (spheres, boxes, rectangles) and glossy materials
    x = scenegen.make_inputs(scenegen.preset("t_interior", n_vpls=20000))
    fr = lmc.Frame(x)
    o = oracle.Oracle(x)
    rng = np.random.default_rng(11)
    n = 60000
    rows = rng.integers(0, x.m, n)
    vp = rng.integers(0, x.vpls["px"].size, n)
    got = fr.eval_entries(rows, vp)
    ref = np.array([o.entry_T(r, v) for r, v in zip(rows, vp)])
    assert np.array_equal(got, ref), f"{np.sum(got != ref)} of {n} entries differ"
    fr.close()


def test_entries_bit_exact_c3_scene():
    # full-size interior scene (16 spheres, 8 boxes, 8 rectangles, glossy): random pairs
    x = scenegen.make_inputs("c3")
    fr = lmc.Frame(x)
    o = oracle.Oracle(x)
    rng = np.random.default_rng(123)
    n = 200000
    rows = rng.integers(0, x.m, n)
    vp = rng.integers(0, x.vpls["px"].size, n)
    got = fr.eval_entries(rows, vp)
    ref = np.array([o.entry_T(r, v) for r, v in zip(rows, vp)])
    assert np.array_equal(got, ref), f"{np.sum(got != ref)} of {n} entries differ"
    occluded = np.sum((ref == 0))
    assert occluded > 0.3 * n
    fr.close()


@pytest.mark.parametrize("name", ["c1", "t_cornell", "t_interior"])
def test_slices_bit_exact(name):
    x, fr, _ = frame(name)
    off, rows = fr.slices()
    ooff, orows = oracle.Oracle(x).slices()
    assert np.array_equal(off, ooff)
    assert np.array_equal(rows, orows)


@pytest.mark.parametrize("name", ["c1", "t_cornell", "t_interior"])
def test_small_frames_all_slices(name):
    x, fr, img = frame(name)
    off, _ = fr.slices()
    res = oracle_slices(x, list(range(off.size - 1)))
    worst = max(check_slice(x, fr, img, r) for r in res)
    # whole image: every pixel of every slice
    assert worst <= 1e-3


@pytest.mark.parametrize("over", [dict(rank_q=4), dict(rank_q=16), dict(rank_q=32), dict(rate=0.3), dict(rate=1.0),
                                  dict(rate=0.05), dict(tau=1.0), dict(tau=0.0), dict(rank_q=8, solver=1),
                                  dict(rank_q=4, solver=1)])
def test_edge_configs(over):
    x, fr, img = frame("t_interior", **over)
    off, _ = fr.slices()
    for r in oracle_slices(x, list(range(off.size - 1))):
        check_slice(x, fr, img, r)


def test_direct_slices_when_rank_exceeds_columns():
    x, fr, img = frame("t_cornell", tau=10.0)      # everything merges: n_s <= q -> direct rendering
    off, _ = fr.slices()
    res = oracle_slices(x, list(range(off.size - 1)))
    assert any(r["flags"] & oracle.FLAG_DIRECT for r in res)
    for r in res:
        check_slice(x, fr, img, r)


@pytest.mark.parametrize("name,q", [("t_interior", 8), ("c1", 8), ("t_interior", 4), ("t_interior", 16),
                                    ("t_interior", 32)])
def test_mals_parity(name, q):
    """masked ALS at every rank (q = 32: the operand gathered from global memory)"""
    x, fr, img = frame(name, solver=1, rank_q=q)
    off, _ = fr.slices()
    for r in oracle_slices(x, pick(off.size - 1, 6)):
        check_slice(x, fr, img, r)


@pytest.mark.slow
def test_c2_full_size_sampled_slices():
    x, fr, img = frame("c2")
    off, rows = fr.slices()
    ooff, orows = oracle.Oracle(x).slices()
    assert np.array_equal(off, ooff) and np.array_equal(rows, orows)
    for r in oracle_slices(x, pick(off.size - 1, 5)):
        check_slice(x, fr, img, r)


@pytest.mark.slow
def test_c4_full_size_sampled_slices():
    """the headline workload (1920x1080, 1M VPLs, 2048 slices, q=16) in the configuration bench.py
    times: slicing of the whole frame bit-exact, three sampled slices through every stage"""
    x, fr, img = frame("c4")
    off, rows = fr.slices()
    ooff, orows = oracle.Oracle(x).slices()
    assert np.array_equal(off, ooff) and np.array_equal(rows, orows)
    for r in oracle_slices(x, pick(off.size - 1, 3)):
        check_slice(x, fr, img, r)


@pytest.mark.slow
@pytest.mark.parametrize("name", ["c5_q32_r5", "c5_q4_r20"])
def test_c5_sweep_corners_sampled_slices(name):
    """BASELINE configs[4] at full size (1024x1024, 300k VPLs, glossy): the sweep's corners -- rank 32
    at 5% (a 1024-node cut at 512-row slices: the 16-warp q = 32 kernel shape) and rank 4 at 20%"""
    x, fr, img = frame(name)
    off, rows = fr.slices()
    for r in oracle_slices(x, pick(off.size - 1, 3)):
        check_slice(x, fr, img, r)


def test_empty_gbuffer():
    """no valid pixel: zero slices, every stage is a no-op, the image is untouched"""
    import dataclasses
    x = scenegen.make_inputs("t_cornell")
    g = {k: v[:0] for k, v in x.gbuf.items()}
    x0 = dataclasses.replace(x, gbuf=g)
    fr = lmc.Frame(x0)
    img = torch.full((x.height * x.width * 3,), 7.0, device="cuda")
    fr.run(img)
    torch.cuda.synchronize()
    off, rows = fr.slices()
    assert off.tolist() == [0] and rows.size == 0
    assert torch.all(img == 7.0)
    st = fr.stats()
    assert st["n_slices"] == 0 and st["sum_completed"] == 0
    fr.close()


def test_single_slice_frame():
    """slice_target >= rows: one slice holding every row"""
    x = scenegen.make_inputs(scenegen.preset("t_cornell", slice_target=1024, width=32, height=30))
    fr = lmc.Frame(x)
    img = torch.zeros(x.height * x.width * 3, device="cuda")
    fr.run(img)
    torch.cuda.synchronize()
    off, _ = fr.slices()
    assert off.tolist() == [0, x.m]
    r = oracle_slices(x, [0])[0]
    check_slice(x, fr, img.view(-1, 3).cpu().numpy().astype(np.float64), r)
    fr.close()


def test_frame_rerun_is_deterministic():
    """re-running every stage on the same inputs reproduces the image bit for bit"""
    x, fr, img = frame("t_interior")
    img2 = torch.zeros(x.height * x.width * 3, device="cuda")
    fr.run(img2)
    torch.cuda.synchronize()
    assert np.array_equal(img2.view(-1, 3).cpu().numpy().astype(np.float64), img)


@pytest.mark.slow
def test_c2_mals_sampled_slices():
    x, fr, img = frame("c2", solver=1)
    off, _ = fr.slices()
    for r in oracle_slices(x, pick(off.size - 1, 3)):
        check_slice(x, fr, img, r)
