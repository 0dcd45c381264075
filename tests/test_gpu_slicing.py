"""GPU slicing (slice.cu: per-tile radix select on 32-bit keys) against the oracle's fp64 recursive
sort (oracle.c slice_rec, R26), bit for bit, on inputs built to stress what the 32-bit
keys must get exactly right: coordinate ties (the (key, row) order decides), -0 == +0,
subnormal coordinates, normal_weight = 0 (all normal keys tie), every row identical, tiles large
enough for the chunked top levels (> 64k rows: several 4096-row chunks per tile, ties spanning
chunks), and the input checks that make the 32-bit keys exact (finite G-buffer, diag and
normal_weight ranges)."""
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

KEYS = ("px", "py", "pz", "nx", "ny", "nz")


def with_gbuf(x, f):
    g = {k: (v.copy() if k in KEYS else v) for k, v in x.gbuf.items()}
    f(g)
    return dataclasses.replace(x, gbuf=g)


def check(x):
    fr = lmc.Frame(x)
    try:
        fr.build_slices()
        torch.cuda.synchronize()
        off, rows = fr.slices()
    finally:
        fr.close()
    ooff, orows = oracle.Oracle(x).slices()
    assert np.array_equal(off, ooff), "slice offsets differ"
    assert np.array_equal(rows, orows), f"{np.sum(rows != orows)} of {rows.size} rows differ"


def quantise(step):
    def f(g):
        for k in KEYS:
            g[k][:] = (np.round(g[k] / step) * step).astype(np.float32)
    return f


@pytest.mark.parametrize("name,step", [("c2", 0.25), ("c2", 0.05), ("t_interior", 0.5)])
def test_slices_with_coordinate_ties(name, step):
    check(with_gbuf(scenegen.make_inputs(name), quantise(step)))


def test_slices_signed_zero_and_subnormals():
    rng = np.random.default_rng(11)

    def f(g):
        m = g["px"].size
        for k in KEYS:
            sel = rng.random(m) < 0.3
            g[k][sel] = np.where(rng.random(sel.sum()) < 0.5, np.float32(-0.0), np.float32(0.0))
            sub = rng.random(m) < 0.1
            g[k][sub] = (rng.integers(-50, 50, sub.sum()) * np.float32(1e-44)).astype(np.float32)
    check(with_gbuf(scenegen.make_inputs("t_interior"), f))


def test_slices_normal_weight_zero():
    check(scenegen.make_inputs(scenegen.preset("t_interior", normal_weight=0.0)))


def test_slices_all_rows_identical():
    def f(g):
        for k in KEYS:
            g[k][:] = g[k][0]
    check(with_gbuf(scenegen.make_inputs("t_cornell"), f))


@pytest.mark.slow
def test_slices_c4_size_with_ties():
    """2.07M rows: the chunked top levels with ties spanning many 4096-row chunks"""
    check(with_gbuf(scenegen.make_inputs("c4"), quantise(0.1)))


@pytest.mark.parametrize("bad", [np.nan, np.inf, -np.inf])
def test_non_finite_gbuffer_rejected(bad):
    def f(g):
        g["ny"][7] = bad
    with pytest.raises(lmc.LmcError):
        lmc.Frame(with_gbuf(scenegen.make_inputs("t_cornell"), f))


@pytest.mark.parametrize("diag", [1e31, 1e-31])
def test_diag_out_of_range_rejected(diag):
    with pytest.raises(lmc.LmcError):
        lmc.Frame(dataclasses.replace(scenegen.make_inputs("t_cornell"), diag=diag))


@pytest.mark.parametrize("wn", [-0.3, 1e-31, 1e31])
def test_normal_weight_out_of_range_rejected(wn):
    with pytest.raises(lmc.LmcError):
        lmc.Frame(scenegen.make_inputs(scenegen.preset("t_cornell", normal_weight=wn)))


@pytest.mark.parametrize("m,target", [(262144, 1000), (200001, 777), (6001, 5), (70000, 33), (8193, 1024),
                                      (65537, 1024), (4097, 9)])
def test_slices_unbalanced_trees(m, target):
    """row counts and targets whose slicing trees have leaves at several depths (leaf tiles carried
    through the later levels: the copy path of both slicing kernels), tiles just above and below the
    4096-row chunk and 8192-row round sizes, and levels switching between the chunked and one-CTA paths"""
    x = scenegen.make_inputs(scenegen.preset("c2", slice_target=target))
    g = {k: np.ascontiguousarray(v[:m]) for k, v in x.gbuf.items()}
    check(dataclasses.replace(x, gbuf=g))
