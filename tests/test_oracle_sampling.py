"""Pins for the oracle's RNG, slicing, pass-1/coarsening and pass-2 sampling.

PAPER.md:71-73 (slicing), P:96-122 (coarsening, Eq. 1), P:134-147 (pdf sampling, Eq. 2).
"""
import os

import numpy as np
import pytest
from scipy import stats

import oracle
import scenegen
from tests._mini import mini

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_philox_known_answers():
    n = 0
    for line in open(os.path.join(GOLDEN, "philox4x32_10_kat.txt")):
        if line.startswith("#") or not line.strip():
            continue
        w = [int(t, 16) for t in line.split()]
        out = oracle.philox(w[0:4], w[4:6])
        assert list(out) == w[6:10]
        n += 1
    assert n == 3


@pytest.mark.parametrize("m,n", [(1, 1), (10, 3), (256, 32), (1013, 4), (5, 9), (800, 800)])
def test_floyd_invariants(m, n):
    rows = oracle.floyd(m, n, 17, 3, 12567)
    assert rows.size == min(m, n)
    assert np.all(np.diff(rows) > 0)
    assert rows.min() >= 0 and rows.max() < m


def test_floyd_uniform_chi2():
    m, n = 40, 5
    counts = np.zeros(m)
    for a in range(4000):
        counts[oracle.floyd(m, n, a, 0, 99)] += 1
    chi2 = stats.chisquare(counts)
    assert chi2.pvalue > 0.01
    # pairwise inclusion is also uniform for a simple random sample: P(i, j both) = n(n-1)/(m(m-1))
    both = 0
    for a in range(4000, 8000):
        r = set(oracle.floyd(m, n, a, 0, 99).tolist())
        both += (3 in r) and (17 in r)
    p = n * (n - 1) / (m * (m - 1))
    assert abs(both / 4000 - p) < 4 * np.sqrt(p * (1 - p) / 4000)


# ---------------------------------------------------------------------------------------- slicing

def _slice_sizes(n, target):
    if n <= target:
        return [n]
    nl = (n + 1) // 2
    return _slice_sizes(nl, target) + _slice_sizes(n - nl, target)


@pytest.mark.parametrize("name", ["c1", "t_cornell", "t_interior"])
def test_slicing_partition(inputs_cache, name):
    x = inputs_cache(name)
    off, rows = oracle.Oracle(x).slices()
    m = x.m
    assert off[0] == 0 and off[-1] == m
    assert np.array_equal(np.sort(rows), np.arange(m))
    sizes = np.diff(off)
    assert list(sizes) == _slice_sizes(m, x.cfg.slice_target)
    for s in range(sizes.size):
        assert np.all(np.diff(rows[off[s]:off[s + 1]]) > 0)   # ascending local row order
    off2, rows2 = oracle.Oracle(x).slices()
    assert np.array_equal(off, off2) and np.array_equal(rows, rows2)


def test_slicing_separates_clusters():
    rng = np.random.default_rng(0)
    a = rng.normal(0, 0.01, (50, 3)) + [0.1, 0.1, 0.1]
    b = rng.normal(0, 0.01, (50, 3)) + [0.9, 0.9, 0.9]
    pts = np.concatenate([a, b])
    perm = rng.permutation(100)
    pts = pts[perm]
    x = mini(pts, np.tile([0, 1, 0], (100, 1)), [0, 1, 0], [0, -1, 0], [1, 1, 1], slice_target=50)
    off, rows = oracle.Oracle(x).slices()
    assert off.size == 3
    lab = (perm >= 50).astype(int)
    assert len(set(lab[rows[:50]])) == 1 and len(set(lab[rows[50:]])) == 1


def test_slicing_normal_dimension():
    # coincident positions, opposite normals: the split must separate by normal
    pts = np.tile([0.5, 0.5, 0.5], (40, 1)) + np.random.default_rng(1).normal(0, 1e-4, (40, 3))
    nrm = np.tile([0, 1, 0], (40, 1)).astype(float)
    nrm[::2] = [0, -1, 0]
    x = mini(pts, nrm, [0, 1, 0], [0, -1, 0], [1, 1, 1], slice_target=20)
    off, rows = oracle.Oracle(x).slices()
    assert off.size == 3
    assert len(set(nrm[rows[:20], 1])) == 1


# ---------------------------------------------------------------------------------------- coarsening

def _cover_check(tree, cut):
    """every leaf covered exactly once by the cut (antichain cover)"""
    left, right = tree["left"], tree["right"]
    nn = left.size
    cover = np.zeros(nn, int)
    stack = list(cut)
    while stack:
        f = stack.pop()
        if left[f] < 0:
            cover[f] += 1
        else:
            stack += [left[f], right[f]]
    leaves = left < 0
    return np.all(cover[leaves] == 1)


def test_coarsen_tau_zero_keeps_global_cut(inputs_cache):
    x = inputs_cache("c1")
    o = oracle.Oracle(x, tau=0.0)
    for r in o.run_slices([0, 5, 11], stage=1):
        assert np.array_equal(r["cut_nodes"], np.sort(x.tree["global_cut"]))
        assert r["proc_merged"].sum() == 0
        # only base pairs were processed (no higher candidate can appear without a merge)
        left, right = x.tree["left"], x.tree["right"]
        g = set(x.tree["global_cut"].tolist())
        for f in r["proc_node"]:
            assert left[f] in g and right[f] in g


@pytest.mark.parametrize("name", ["c1", "t_interior"])
def test_coarsen_cover_costs_and_errors(inputs_cache, name):
    x = inputs_cache(name)
    o = oracle.Oracle(x)
    t = x.tree
    lum = lambda f: (0.2126 * float(t["ir"][f]) + 0.7152 * float(t["ig"][f])) + 0.0722 * float(t["ib"][f])
    g = x.gbuf
    for r in o.run_slices([0, 3, 7], stage=1):
        assert _cover_check(t, r["cut_nodes"])
        cost = {}
        merged = set()
        for k, f in enumerate(r["proc_node"]):
            l, rr = t["left"][f], t["right"][f]
            a = l if t["rep"][l] == t["rep"][f] else rr
            b = rr if a == l else l
            z = r["proc_zrows"][r["proc_zoff"][k]:r["proc_zoff"][k + 1]]
            # eps recomputed from entries evaluated one by one
            rows = r["rows"][z]
            rr_, rg_, rb_ = (g[k][rows].astype(np.float64) for k in ("rho_r", "rho_g", "rho_b"))
            lr = (0.2126 * rr_ + 0.7152 * rg_) + 0.0722 * rb_
            Ta = np.array([o.entry_T(p, t["rep"][a]) for p in rows])
            Tb = np.array([o.entry_T(p, t["rep"][b]) for p in rows])
            assert np.array_equal(Ta, r["proc_Va"][r["proc_zoff"][k]:r["proc_zoff"][k + 1]])
            Va, Vb = lr * lum(a) * Ta, lr * lum(b) * Tb
            eps = np.max(np.abs(Vb - Va * (lum(b) / lum(a)))) if lum(a) > 0 else np.max(np.abs(Vb))
            assert r["proc_eps"][k] == pytest.approx(eps, rel=1e-12, abs=1e-300)
            # Eq. (1): cost(f) = eps(f) + cost(b), cost = 0 on g
            assert r["proc_cost"][k] == pytest.approx(eps + cost.get(b, 0.0), rel=1e-12, abs=1e-300)
            # sample-set rule: union of the children's sets when both were merged
            if l in merged and rr in merged:
                kl = list(r["proc_node"]).index(l)
                kr = list(r["proc_node"]).index(rr)
                zl = r["proc_zrows"][r["proc_zoff"][kl]:r["proc_zoff"][kl + 1]]
                zr = r["proc_zrows"][r["proc_zoff"][kr]:r["proc_zoff"][kr + 1]]
                assert np.array_equal(z, np.union1d(zl, zr))
            if r["proc_merged"][k]:
                assert r["proc_cost"][k] < x.tau
                cost[f] = r["proc_cost"][k]
                merged.add(f)
            else:
                assert r["proc_cost"][k] >= x.tau


def test_coarsen_order_independent(inputs_cache):
    x = inputs_cache("t_interior")
    base = oracle.Oracle(x).run_slices([0, 2, 5], stage=1)
    for seed in (1, 2, 3):
        shuf = oracle.Oracle(x, order_seed=seed).run_slices([0, 2, 5], stage=1)
        for a, b in zip(base, shuf):
            assert np.array_equal(a["cut_nodes"], b["cut_nodes"])
            ia, ib = np.argsort(a["proc_node"]), np.argsort(b["proc_node"])
            assert np.array_equal(a["proc_node"][ia], b["proc_node"][ib])
            assert np.array_equal(a["proc_cost"][ia], b["proc_cost"][ib])
            assert a["n_evals_coarsen"] == b["n_evals_coarsen"]


def test_coarsen_proportional_siblings_merge():
    # two VPLs at the same place/orientation: V_b = V_a I_b/I_a exactly up to rounding -> merge
    pts = np.random.default_rng(3).uniform(0, 1, (30, 3)) * [1, 0, 1]
    vp = np.array([[0.5, 1.0, 0.5], [0.5, 1.0, 0.5], [0.2, 0.8, 0.9], [0.2, 0.8, 0.9]])
    vn = np.tile([0, -1, 0], (4, 1))
    vi = np.array([[1, 1, 1], [2, 2, 2], [1, 0.5, 0.2], [3, 1.5, 0.6]])
    x = mini(pts, np.tile([0, 1, 0], (30, 1)), vp, vn, vi, tau=1e-12)
    r = oracle.Oracle(x).run_slices([0], stage=1)[0]
    assert r["n"] < 4
    assert np.all(r["proc_eps"][r["proc_merged"] == 1] < 1e-12)


# ---------------------------------------------------------------------------------------- pass 2

@pytest.mark.parametrize("name", ["c1", "t_interior"])
def test_pass2_sample_set(inputs_cache, name):
    x = inputs_cache(name)
    o = oracle.Oracle(x)
    for r in o.run_slices([0, 4], stage=2):
        m, n = r["m"], r["n"]
        cells = r["om_row"].astype(np.int64) * n + r["om_col"]
        assert np.all(np.diff(cells) > 0)                 # CSR order, no duplicates
        assert r["nnz"] == r["n_carried"] + r["n_new"] + r["n_forced"]
        assert r["nnz"] >= min(r["target_N"], r["n_carried"]) or r["n_draws"] == 64 * r["target_N"]
        if r["n_carried"] < r["target_N"]:
            assert r["n_carried"] + r["n_new"] == r["target_N"] or r["n_draws"] == 64 * r["target_N"]
        assert np.all(np.bincount(r["om_col"], minlength=n) > 0)   # forced samples (R17)
        assert r["target_N"] == int(np.ceil(float(m * n) * x.cfg.rate))
        # values are the entries at those cells ("compute the lighting results")
        t = x.tree
        g = x.gbuf
        for k in range(0, r["nnz"], max(1, r["nnz"] // 50)):
            i, c = r["om_row"][k], r["om_col"][k]
            f = r["cut_nodes"][c]
            p = r["rows"][i]
            lr = (0.2126 * float(g["rho_r"][p]) + 0.7152 * float(g["rho_g"][p])) + 0.0722 * float(g["rho_b"][p])
            li = (0.2126 * float(t["ir"][f]) + 0.7152 * float(t["ig"][f])) + 0.0722 * float(t["ib"][f])
            assert r["om_val"][k] == (lr * li) * o.entry_T(p, t["rep"][f])
        # weight rule (R14): observed columns >= 2^16 floor, max column gets 2^20
        w = r["weights"]
        assert w.max() <= 2 ** 20 and w.min() >= 1


def test_pass2_rate_one_observes_everything(inputs_cache):
    x = inputs_cache("t_cornell")
    r = oracle.Oracle(x, rate=1.0).run_slices([1], stage=2)[0]
    assert r["nnz"] == r["m"] * r["n"]


def test_pass2_importance_follows_weights():
    # many draws on a slice: new samples per column correlate with the integer weights (Eq. 2)
    import scenegen
    x = scenegen.make_inputs(scenegen.preset("t_interior", rate=0.3))
    o = oracle.Oracle(x)
    rhos = []
    for r in o.run_slices([0, 1, 2, 3], stage=2):
        newcnt = np.bincount(r["om_col"][r["om_carried"] == 0], minlength=r["n"])
        rho, _ = stats.spearmanr(r["weights"], newcnt)
        rhos.append(rho)
    assert np.mean(rhos) > 0.3


# ---------------------------------------------------------------------------------------- step 1

@pytest.mark.parametrize("name", ["c1", "t_cornell", "t_interior", "c2"])
def test_light_tree_oracle_equals_the_fixture(inputs_cache, name):
    """the oracle's light tree + global cut (R38) is the scene generator's tree, built by an
    independent numpy implementation (level-synchronous lexsort, heap-driven greedy cut)"""
    x = inputs_cache(name)
    t = oracle.build_light_tree(x.vpls, x.cfg.cut_max)
    for k in ("left", "right", "rep", "ir", "ig", "ib", "global_cut"):
        assert np.array_equal(t[k], x.tree[k]), k


def test_light_tree_invariants():
    rng = np.random.default_rng(21)
    nv = 777
    v = {k: rng.uniform(0, 1, nv).astype(np.float32) for k in ("px", "py", "pz", "ir", "ig", "ib")}
    v["px"][::7] = v["px"][3]                      # coordinate ties (broken by VPL index)
    for cut_max in (1, 2, 50, 776, 777, 5000):
        t = oracle.build_light_tree(v, cut_max)
        left, right = t["left"], t["right"]
        nn = 2 * nv - 1
        assert left.size == nn and np.sum(left < 0) == nv
        for f in np.flatnonzero(left >= 0):
            l, r = left[f], right[f]
            assert t["rep"][f] in (t["rep"][l], t["rep"][r])
            for k in ("ir", "ig", "ib"):
                assert t[k][f] == np.float32(np.float64(t[k][l]) + np.float64(t[k][r])) or \
                    abs(t[k][f] - (t[k][l] + t[k][r])) <= 1e-6 * t[k][f]
        assert sorted(t["rep"][left < 0]) == list(range(nv))
        assert _cover_check(t, t["global_cut"])
        assert t["global_cut"].size == min(cut_max, nv)
