"""DESIGN R43 (the CUDA slicing orders 32-bit encodings of the fp32 coordinates): check, in numpy's
IEEE fp64, that the fp64 slicing keys of R26 (x / D and w_n * n) order and tie exactly as
the fp32 inputs do (-0 == +0) for D and w_n across [1e-30, 1e30] -- the property that makes the
32-bit radix select return the oracle's slices.  The inputs span every fp32 binade, subnormals,
signed zeros and neighbouring floats (the closest pairs that could merge)."""
import numpy as np
import pytest


def float_sample(rng, n):
    bits = rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32)
    f = bits.view(np.float32)
    f = f[np.isfinite(f)]
    # neighbours of random floats, subnormals, signed zeros, a few exact ties
    nb = np.nextafter(f[:2000], np.float32(np.inf))
    sub = (rng.integers(-1000, 1000, 2000) * np.float32(1e-45)).astype(np.float32)
    zeros = np.array([0.0, -0.0] * 50, np.float32)
    small = rng.uniform(-20, 20, 20000).astype(np.float32)
    return np.concatenate([f, nb, sub, zeros, small, small[:500]])


def order_key32(f):
    """the CUDA path's order-preserving encoding (slice.cu enc32), -0 mapped to +0"""
    u = f.view(np.uint32).copy()
    u[u == 0x80000000] = 0
    neg = (u & 0x80000000) != 0
    return np.where(neg, ~u, u | np.uint32(0x80000000)).astype(np.uint64)


@pytest.mark.parametrize("scale", [1e-30, 3.7e-12, 1e-3, 0.3, 1.0, 17.3, 4.1e9, 1e30])
@pytest.mark.parametrize("kind", ["div", "mul"])
def test_fp64_keys_order_like_fp32(scale, kind):
    rng = np.random.default_rng(int(scale * 1e3) % 1000 + (kind == "mul"))
    f = float_sample(rng, 60000)
    k64 = (f.astype(np.float64) / scale) if kind == "div" else (scale * f.astype(np.float64))
    k64 = k64 + 0.0   # canonical +0 (R26)
    k32 = order_key32(f)
    o64 = np.lexsort((np.arange(f.size), k64))
    o32 = np.lexsort((np.arange(f.size), k32))
    assert np.array_equal(o64, o32), "the (key, row) order differs"
    s = np.sort(k64)
    t = np.sort(k32)
    assert np.array_equal(np.diff(s) == 0, np.diff(t) == 0), "ties differ"
    assert np.all(np.isfinite(k64)) and np.all((k64 == 0) == (f == 0)), "a key overflowed or underflowed"


def test_extent_from_float_extremes():
    """the extent max(key) - min(key) computed from the float extremes equals the one over the fp64 keys"""
    rng = np.random.default_rng(5)
    for _ in range(200):
        f = rng.uniform(-50, 50, rng.integers(1, 300)).astype(np.float32)
        for D in (1e-30, 0.37, 17.0, 1e30):
            k = f.astype(np.float64) / D + 0.0
            ext = k.max() - k.min()
            e2 = (np.float64(f.max()) / D + 0.0) - (np.float64(f.min()) / D + 0.0)
            assert ext == e2
