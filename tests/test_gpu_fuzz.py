"""Randomised GPU parity: seeded random configurations (tests/_fuzz.py: scene kind incl. triangle
meshes, image size, VPL count, cut size, slice target, rank, rate, tau, solver, iteration count,
tolerance, pass-1 counts, the f2-f3 variants, seeds; 48 small, 12 with large slices and cuts, 12 of a few pixels and 1-3 node cuts); plus the configurations that exposed bugs) — every slice through every stage against the
oracle with the same bars as tests/test_gpu_parity.check_slice (bit-exact cuts / Omega, completion <= 1e-4, pixels
<= 1e-3)."""
import numpy as np
import pytest

import oracle
import scenegen

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no GPU", allow_module_level=True)
from paper_2202_12567_b200 import lmc  # noqa: E402
from tests._fuzz import REGRESSIONS, config_large, config_small, config_tiny  # noqa: E402
from tests.test_gpu_parity import check_slice  # noqa: E402


@pytest.mark.parametrize("kind,k", [("small", k) for k in range(48)] + [("large", k) for k in range(12)] +
                         [("tiny", k) for k in range(12)] + [("regression", k) for k in range(len(REGRESSIONS))])
def test_random_configs(kind, k):
    cfg = {"small": config_small, "large": config_large, "tiny": config_tiny,
           "regression": REGRESSIONS.__getitem__}[kind](k)
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


@pytest.mark.parametrize("k", range(16))
def test_random_light_trees(k):
    """lmc_build_light_tree on random VPL sets (sizes from 1 to 40k, coordinate ties, zero and
    equal intensities, cut sizes beyond the leaf count) equals the oracle node for node (R38)"""
    rng = np.random.default_rng(330 + k)
    nv = int(rng.choice([1, 2, 3, 7, 100, 1023, 1024, 1025, 5000, 40000]))
    v = {a: rng.uniform(-2, 3, nv).astype(np.float32) for a in ("px", "py", "pz")}
    v.update({a: rng.uniform(-1, 1, nv).astype(np.float32) for a in ("nx", "ny", "nz")})
    v.update({a: rng.exponential(1.0, nv).astype(np.float32) for a in ("ir", "ig", "ib")})
    if k % 4 == 1:   # coordinate ties on every axis
        for a in ("px", "py", "pz"):
            v[a] = np.round(v[a] * 2) / 2
    if k % 4 == 2:   # zero and equal intensities
        for a in ("ir", "ig", "ib"):
            v[a][::3] = 0.0
            v[a][1::3] = 1.0
    cut_max = int(rng.choice([1, 2, 16, 256, 1024, 100000]))
    got = lmc.build_light_tree(v, cut_max)
    ref = oracle.build_light_tree(v, cut_max)
    for key in ("left", "right", "rep", "ir", "ig", "ib", "global_cut"):
        assert np.array_equal(got[key], ref[key]), (key, nv, cut_max)


@pytest.mark.parametrize("k", range(10))
def test_random_warm_start_sequences(k):
    """SURVEY f4 on random small configurations: three frames, the albedo of a random share of the
    pixels changed between frames, ADM warm-started where rows and cut are unchanged (R42); every
    frame against the oracle's same sequence"""
    import dataclasses
    rng = np.random.default_rng(4400 + k)
    cfg = dataclasses.replace(config_small(k), solver=0, warm_start=1, warm_iters=int(rng.choice([0, 5, 20])),
                              tol=0.0)
    xs = [scenegen.make_inputs(cfg)]
    for _ in range(2):
        g = dict(xs[-1].gbuf)
        sel = rng.random(g["px"].size) < rng.uniform(0.0, 0.5)
        f = np.float32(rng.uniform(0.2, 1.5))
        for key in ("rho_r", "rho_g", "rho_b"):
            g[key] = np.where(sel, g[key] * f, g[key]).astype(np.float32)
        xs.append(dataclasses.replace(xs[-1], gbuf=g))
    fr = lmc.Frame(xs[0])
    prev = None
    for i, x in enumerate(xs):
        if i:
            fr.upload_inputs(x)
        img = torch.zeros(x.height * x.width * 3, device="cuda")
        fr.run(img)
        torch.cuda.synchronize()
        img = img.view(-1, 3).cpu().numpy().astype(np.float64)
        o = oracle.Oracle(x)
        if prev is not None:
            o.set_warm(prev)
        off, _ = fr.slices()
        res = o.run_slices(list(range(off.size - 1)), stage=4)
        assert fr.stats()["n_warm"] == sum(r["warm"] for r in res)
        for r in res:
            check_slice(x, fr, img, r)
        prev = res
    fr.close()


@pytest.mark.parametrize("k", range(6))
def test_random_configs_host_buffers(k):
    """the host-buffer path (inputs and image in host memory, as bench.py's e2e uses it) gives the
    device path's image bit for bit; pixels outside the G-buffer keep their host values"""
    cfg = config_small(100 + k)
    x = scenegen.make_inputs(cfg)
    fr = lmc.Frame(x)
    img = torch.zeros(x.height * x.width * 3, device="cuda")
    fr.run(img)
    torch.cuda.synchronize()
    ref = img.cpu().numpy()
    fr.close()
    frh = lmc.Frame(x, memory=lmc.MEM_HOST)
    host = np.full(x.height * x.width * 3, 7.0, np.float32)
    for _ in range(2):   # a re-upload of the same inputs renders the same frame
        frh.upload_inputs()
        frh.run(host, lmc.MEM_HOST)
    frh.close()
    covered = np.zeros(x.height * x.width, bool)
    covered[x.gbuf["pixel"]] = True
    cov3 = np.repeat(covered, 3)
    assert np.array_equal(host[cov3], ref[cov3])
    assert np.all(host[~cov3] == 7.0)


@pytest.mark.parametrize("k", range(6))
def test_random_configs_deterministic(k):
    """two contexts on the same inputs give bit-identical images and factors (no float atomics,
    fixed reduction orders), on random configurations incl. MALS and the variants"""
    cfg = config_small(200 + k)
    x = scenegen.make_inputs(cfg)
    outs = []
    for _ in range(2):
        fr = lmc.Frame(x)
        img = torch.zeros(x.height * x.width * 3, device="cuda")
        fr.run(img)
        torch.cuda.synchronize()
        off, _ = fr.slices()
        fac = [fr.factors(s) for s in range(off.size - 1)]
        outs.append((img.cpu().numpy(), fac))
        fr.close()
    assert np.array_equal(outs[0][0], outs[1][0])
    for a, b in zip(outs[0][1], outs[1][1]):
        assert np.array_equal(a["U"], b["U"]) and np.array_equal(a["V"], b["V"]) and a["iters"] == b["iters"]
