"""Closed-form and statistical pins of the oracle's sampling rules (no GPU).

Each test fixes one passage of PAPER.md (or one DESIGN.md reading) on a hand-made input whose
answer is known without running the oracle's own arithmetic:

  g(j)  = max C_j - min C_j                      P:141-144 (sec. 5)
  pdf weights, unobserved columns, G = 0         Eq. (2) P:134-145 with reading R14
  CDF inversion tie-break                        P:147 with reading R29
  column frequencies follow w / W                P:147 (columns drawn by importance)
  n_f linearly proportional to I_f               P:104 (sec. 4) with reading R6
  mixed pair (one merged, one original child)    P:104-118 with reading R10

tools/mutants.py re-runs this file against deliberately broken copies of oracle.c (the plausible
mistakes listed in the round-1 review) and checks that every mutant fails at least one test.
"""
import numpy as np
import pytest
from scipy import stats

import oracle
from tests._mini import mini


# ------------------------------------------------------------------------------ g(j)

def test_importance_closed_forms():
    # column 0: constant {0.5, 0.5, 0.5} -> 0; column 1: {0, 1, 0.2} -> 1 - 0 = 1;
    # column 2: one observation -> 0; column 3: unobserved -> 0 with count 0;
    # column 4: {-0.25, 0.75} -> 1 (max - min, not max)
    col = [0, 1, 0, 1, 2, 1, 0, 4, 4]
    val = [0.5, 0.0, 0.5, 1.0, 7.0, 0.2, 0.5, -0.25, 0.75]
    g, cnt = oracle.light_importance(5, col, val)
    assert list(cnt) == [3, 3, 1, 0, 2]
    assert g[0] == 0.0
    assert g[1] == 1.0
    assert g[2] == 0.0
    assert g[3] == 0.0
    assert g[4] == 1.0


def test_importance_order_free():
    rng = np.random.default_rng(5)
    col = rng.integers(0, 7, 300)
    val = rng.uniform(0, 3, 300)
    g, cnt = oracle.light_importance(7, col, val)
    perm = rng.permutation(300)
    g2, cnt2 = oracle.light_importance(7, col[perm], val[perm])
    assert np.array_equal(g, g2) and np.array_equal(cnt, cnt2)
    for c in range(7):
        v = val[col == c]
        assert g[c] == (v.max() - v.min() if v.size else 0.0)


# ------------------------------------------------------------------------------ weights, R14

def test_weights_all_equal_importance_is_uniform():
    w = oracle.pdf_weights([0.3] * 6, [2] * 6)
    assert np.all(w == 2 ** 20)


def test_weights_hand_values():
    # G = 1: g = 1 -> 1 + (2^20 - 1) = 2^20; g = 0.5 -> 1 + floor(524287.5) = 524288;
    # g = 0 -> floor 2^16; the unobserved column gets the integer mean of the observed weights
    w = oracle.pdf_weights([1.0, 0.5, 0.0, 0.0], [4, 2, 3, 0])
    assert list(w[:3]) == [1048576, 524288, 65536]
    assert w[3] == (1048576 + 524288 + 65536) // 3 == 546133


def test_weights_degenerate():
    assert list(oracle.pdf_weights([0.0, 0.0, 0.0], [1, 2, 0])) == [1, 1, 1]     # G = 0
    w = oracle.pdf_weights([2.0, 1e-9], [3, 3])                                   # tiny g hits the floor
    assert list(w) == [1048576, 65536]


# ------------------------------------------------------------------------------ CDF, R29

def test_cdf_tie_goes_to_the_next_column():
    cdf = np.array([4, 8, 12], np.uint64)      # weights 4, 4, 4
    assert oracle.cdf_pick(cdf, 0) == 0
    assert oracle.cdf_pick(cdf, 3) == 0
    assert oracle.cdf_pick(cdf, 4) == 1        # CDF_0 = 4 is not > 4
    assert oracle.cdf_pick(cdf, 7) == 1
    assert oracle.cdf_pick(cdf, 8) == 2
    assert oracle.cdf_pick(cdf, 11) == 2
    # zero-weight columns are never picked
    cdf0 = np.array([0, 5, 5, 9], np.uint64)   # weights 0, 5, 0, 4
    picks = {oracle.cdf_pick(cdf0, x) for x in range(9)}
    assert picks == {1, 3}


def test_pass2_column_frequencies_chi2():
    # 10^6 draws: columns follow w / W, rows are uniform
    rng = np.random.default_rng(11)
    n, m, N = 64, 1000, 1_000_000
    w = rng.integers(65536, 2 ** 20 + 1, n).astype(np.uint32)
    w[7] = 1                                   # a nearly impossible column
    rows, cols = oracle.pass2_draws(w, m, N, seed=2202, slice_id=3)
    cc = np.bincount(cols, minlength=n)
    exp = N * w.astype(np.float64) / w.astype(np.float64).sum()
    keep = exp > 5
    chi = stats.chisquare(cc[keep], exp[keep] * cc[keep].sum() / exp[keep].sum())
    assert chi.pvalue > 1e-4
    assert cc[7] <= 3
    rc = np.bincount(rows, minlength=m)
    assert rows.min() >= 0 and rows.max() < m
    assert stats.chisquare(rc).pvalue > 1e-4


# ------------------------------------------------------------------------------ pass-1 counts

def _tree(nodes, nv):
    """nodes: list of (left, right, rep, I) per node id; leaves have left = right = -1."""
    nn = len(nodes)
    t = dict(left=np.array([a[0] for a in nodes], np.int32), right=np.array([a[1] for a in nodes], np.int32),
             rep=np.array([a[2] for a in nodes], np.int32),
             ir=np.array([a[3] for a in nodes], np.float32), ig=np.array([a[3] for a in nodes], np.float32),
             ib=np.array([a[3] for a in nodes], np.float32), root=0)
    t["global_cut"] = np.array([k for k in range(nn) if nodes[k][0] < 0], np.int32)
    return t


def _floor_scene(m, vpl_pos, vpl_I, tree, **over):
    rng = np.random.default_rng(4)
    pts = np.column_stack([rng.uniform(0, 1, m), np.zeros(m), rng.uniform(0, 1, m)])
    nv = len(vpl_pos)
    return mini(pts, np.tile([0, 1, 0], (m, 1)), vpl_pos, np.tile([0, -1, 0], (nv, 1)),
                np.column_stack([vpl_I] * 3), tree=tree, **over)


def test_pass1_count_linear_in_intensity():
    # three base pairs with luminances 2, 0.6, 0.01 (grey, so lum = I): n_f = min(m, max(4,
    # ceil(32 lum / l_max))) = 32, ceil(9.6) = 10, max(4, ceil(0.16)) = 4 ("linearly
    # proportional to I_f", R6)
    # tree: 0 = (1, 2), 1 = (3, 4), 2 = (5, 6); base pairs 3 = (v0, v1), 4 = (v2, v3), 5 = (v4, v5);
    # 6 = leaf v6; leaves 7..12 = v0..v5
    vp = [[0.2, 1, 0.2], [0.3, 1, 0.2], [0.7, 1, 0.7], [0.8, 1, 0.7], [0.5, 1, 0.1], [0.5, 1, 0.9],
          [0.9, 1, 0.1]]
    I = [1.0, 1.0, 0.3, 0.3, 0.005, 0.005, 0.5]
    nodes = [(1, 2, 0, 3.11), (3, 4, 0, 2.6), (5, 6, 4, 0.51),
             (7, 8, 0, 2.0), (9, 10, 2, 0.6), (11, 12, 4, 0.01), (-1, -1, 6, 0.5),
             (-1, -1, 0, 1.0), (-1, -1, 1, 1.0), (-1, -1, 2, 0.3), (-1, -1, 3, 0.3),
             (-1, -1, 4, 0.005), (-1, -1, 5, 0.005)]
    tree = _tree(nodes, 7)
    x = _floor_scene(300, vp, I, tree, tau=0.0)
    r = oracle.Oracle(x).run_slices([0], stage=1)[0]
    sizes = {int(f): int(r["proc_zoff"][k + 1] - r["proc_zoff"][k]) for k, f in enumerate(r["proc_node"])}
    assert sizes[3] == 32 and sizes[4] == 10 and sizes[5] == 4
    assert r["proc_merged"].sum() == 0


def test_pass1_count_clamped_by_slice_rows():
    vp = [[0.2, 1, 0.2], [0.3, 1, 0.2]]
    nodes = [(1, 2, 0, 2.0), (-1, -1, 0, 1.0), (-1, -1, 1, 1.0)]
    x = _floor_scene(20, vp, [1.0, 1.0], _tree(nodes, 2), tau=0.0)
    r = oracle.Oracle(x).run_slices([0], stage=1)[0]
    assert list(r["proc_zrows"]) == list(range(20))       # min(m, 32) = all 20 rows


@pytest.mark.parametrize("name", ["c1", "t_interior"])
def test_pass1_counts_every_base_pair(inputs_cache, name):
    # |zeta_f| of every base pair = min(m, max(nmin, ceil(nmax lum I_f / l_max))), l_max over the
    # base pairs of the whole tree (R6), computed here from the tree arrays
    x = inputs_cache(name)
    t = x.tree
    lum = lambda f: (0.2126 * float(t["ir"][f]) + 0.7152 * float(t["ig"][f])) + 0.0722 * float(t["ib"][f])
    g = set(t["global_cut"].tolist())
    base = [f for f in range(t["left"].size) if t["left"][f] in g and t["right"][f] in g]
    lmax = max(lum(f) for f in base)
    for r in oracle.Oracle(x).run_slices([0, 3], stage=1):
        for k, f in enumerate(r["proc_node"]):
            if f not in base:
                continue
            want = min(r["m"], max(x.cfg.p1_nmin, int(np.ceil((x.cfg.p1_nmax * lum(f)) / lmax))))
            assert r["proc_zoff"][k + 1] - r["proc_zoff"][k] == want


# ------------------------------------------------------------------------------ mixed pair, R10

def test_mixed_pair_sample_set():
    # f = (h, o): h = (v0, v1) is a base pair that merges (tau huge), o is an original leaf.
    # zeta_f = zeta_h U Floyd(m, n(I_o), key f) with n(I_o) = ceil(32 * 0.55 / 2) = 9 (R10)
    m = 200
    vp = [[0.2, 1, 0.2], [0.3, 1, 0.25], [0.8, 1, 0.7]]
    nodes = [(1, 2, 0, 2.55), (3, 4, 0, 2.0), (-1, -1, 2, 0.55), (-1, -1, 0, 1.0), (-1, -1, 1, 1.0)]
    x = _floor_scene(m, vp, [1.0, 1.0, 0.55], _tree(nodes, 3), tau=1e30)
    r = oracle.Oracle(x).run_slices([0], stage=1)[0]
    proc = list(r["proc_node"])
    assert proc == [1, 0]
    z = lambda k: r["proc_zrows"][r["proc_zoff"][k]:r["proc_zoff"][k + 1]]
    zh = z(0)
    assert zh.size == 32 and r["proc_merged"][0] == 1
    fresh = oracle.floyd(m, 9, 0, 0, x.cfg.seed)
    assert fresh.size == 9
    assert np.array_equal(z(1), np.union1d(zh, fresh))
