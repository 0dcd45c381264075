"""Pins of the SURVEY §8(f3) sampling / resolve variants in the oracle (no GPU):

  row importance f(i) (P:145 sets f = 1, P:246 names image-space guidance as future work; R36)
  Eq. (1) sensitivity: cost(L_f) = (eps + cost(L_b)) + cost(L_a)
  Z-mode image: factored part + the residuals of the observed entries (A24)
"""
import numpy as np
import pytest
from scipy import stats

import oracle
import scenegen


def test_row_draw_with_equal_row_weights_is_the_uniform_draw():
    # equal integer row weights w: row = floor(((u1 m w) >> 32) / w) = (u1 m) >> 32 exactly
    rng = np.random.default_rng(3)
    w = rng.integers(65536, 2 ** 20, 37)
    for m in (1, 7, 512, 1013):
        for t in range(0, 4000, 37):
            r_f, c_f = oracle.pass2_draw_f(t, w, [524288] * m, seed=99, slice_id=5)
            rows, cols = oracle.pass2_draws(w, m, 1, seed=99, slice_id=5, t0=t)
            assert (r_f, c_f) == (int(rows[0]), int(cols[0]))


def test_row_importance_sampling_follows_row_weights(inputs_cache):
    x = scenegen.make_inputs(scenegen.preset("t_interior", rate=0.3, row_importance=1))
    base = oracle.Oracle(scenegen.make_inputs(scenegen.preset("t_interior", rate=0.3)))
    rhos, differs = [], 0
    for r, r0 in zip(oracle.Oracle(x).run_slices([0, 1, 2, 3], stage=2), base.run_slices([0, 1, 2, 3], stage=2)):
        m, n = r["m"], r["n"]
        cells = r["om_row"].astype(np.int64) * n + r["om_col"]
        assert np.all(np.diff(cells) > 0)
        assert r["nnz"] == r["n_carried"] + r["n_new"] + r["n_forced"]
        assert np.all(np.bincount(r["om_col"], minlength=n) > 0)
        car = r["om_carried"] == 1
        assert np.array_equal(cells[car], (r0["om_row"].astype(np.int64) * n + r0["om_col"])[r0["om_carried"] == 1])
        # f(i) = max - min of row i's carried observations (the same rule as g(j), R14)
        f, cnt = oracle.light_importance(m, r["om_row"][car], r["om_val"][car])
        wr = oracle.pdf_weights(f, cnt)
        newcnt = np.bincount(r["om_row"][~car], minlength=m)
        rhos.append(stats.spearmanr(wr, newcnt)[0])
        differs += not np.array_equal(r["om_row"], r0["om_row"])
    assert np.mean(rhos) > 0.3 and differs > 0


def test_eq1_sensitivity_cost_recursion(inputs_cache):
    x = scenegen.make_inputs(scenegen.preset("t_interior", cost_mode=1))
    t = x.tree
    for r in oracle.Oracle(x).run_slices([0, 3], stage=1):
        cost = {}
        for k, f in enumerate(r["proc_node"]):
            l, rr = t["left"][f], t["right"][f]
            a = l if t["rep"][l] == t["rep"][f] else rr
            b = rr if a == l else l
            want = (r["proc_eps"][k] + cost.get(b, 0.0)) + cost.get(a, 0.0)
            assert r["proc_cost"][k] == want
            if r["proc_merged"][k]:
                cost[f] = r["proc_cost"][k]
    # the accumulated cost of L_a can only make merging harder: never more merges than Eq. (1)
    lit = oracle.Oracle(scenegen.make_inputs("t_interior")).run_slices(range(8), stage=1)
    sen = oracle.Oracle(x).run_slices(range(8), stage=1)
    assert all(b["n"] >= a["n"] for a, b in zip(lit, sen))
    assert any(b["n"] > a["n"] for a, b in zip(lit, sen))


@pytest.mark.parametrize("name", ["t_cornell", "t_interior"])
def test_z_mode_at_full_rate_is_the_full_cut_rendering(name):
    # every entry observed: U V + (M~ - U V) = M~, so the image is the exact column sums
    x = scenegen.make_inputs(scenegen.preset(name, rate=1.0, resolve_mode=1))
    o = oracle.Oracle(x)
    for r in o.run_slices([0, 2, 5], stage=4):
        assert r["nnz"] == r["m"] * r["n"]
        ref = o.fullcut_slice(r["rows"], r["cut_nodes"])
        np.testing.assert_allclose(r["rgb"], ref, rtol=1e-9, atol=1e-12 * np.abs(ref).max())


def test_z_mode_adds_the_observed_residuals():
    x0 = scenegen.make_inputs(scenegen.preset("t_interior"))
    x1 = scenegen.make_inputs(scenegen.preset("t_interior", resolve_mode=1))
    for a, b in zip(oracle.Oracle(x0).run_slices([1, 4], stage=4), oracle.Oracle(x1).run_slices([1, 4], stage=4)):
        assert np.array_equal(a["U"], b["U"]) and np.array_equal(a["V"], b["V"])   # same factors
        M = np.zeros((a["m"], a["n"]))
        M[a["om_row"], a["om_col"]] = a["om_val"] - (a["U"] @ a["V"])[a["om_row"], a["om_col"]]
        t = x0.tree
        cols = a["cut_nodes"]
        I = np.stack([t["ir"][cols], t["ig"][cols], t["ib"][cols]], 1).astype(np.float64)
        lI = (0.2126 * I[:, 0] + 0.7152 * I[:, 1]) + 0.0722 * I[:, 2]
        wk = I / lI[:, None]
        g = x0.gbuf
        rho = np.stack([g["rho_r"], g["rho_g"], g["rho_b"]], 1).astype(np.float64)[a["rows"]]
        lr = (0.2126 * rho[:, 0] + 0.7152 * rho[:, 1]) + 0.0722 * rho[:, 2]
        extra = (rho / lr[:, None]) * (M @ wk)
        np.testing.assert_allclose(b["rgb"] - a["rgb"], extra, rtol=1e-9, atol=1e-12 * np.abs(a["rgb"]).max())


# ------------------------------------------------------------------------------ warm start

def test_exact_nonnegative_factors_are_an_adm_fixed_point():
    # fully observed M = X* Y* >= 0: Z = M, U = X*, Lambda = 0 give X_1 = (M Y*^T + a X*)(Y* Y*^T + a I)^-1 = X*
    # and then Y_1 = Y*, so a warm start from the exact factors stays there (App. A updates)
    rng = np.random.default_rng(8)
    m, n, q = 60, 40, 4
    Xs = rng.uniform(0.1, 1.0, (m, q))
    Ys = rng.uniform(0.1, 1.0, (q, n))
    M = Xs @ Ys
    row, col = np.nonzero(np.ones((m, n)))
    val = M[row, col]
    sg = val.max()
    w = oracle.adm_warm(m, n, row, col, val, q, Xs, Ys / sg, K=50)
    assert w["iters"] == 50
    np.testing.assert_allclose(w["U"] @ w["V"], M, rtol=1e-11, atol=1e-12)
    c = oracle.adm(m, n, row, col, val, q, K=50)          # the cold start is not there after 50 steps
    assert np.linalg.norm(c["U"] @ c["V"] - M) / np.linalg.norm(M) > 1e-6


def test_warm_start_frame_sequence():
    x = scenegen.make_inputs(scenegen.preset("t_interior", warm_start=1, warm_iters=20))
    o = oracle.Oracle(x)
    off, _ = o.slices()
    ids = list(range(off.size - 1))
    f1 = o.run_slices(ids, stage=4)
    assert not any(r["warm"] for r in f1)
    o.set_warm(f1)
    f2 = o.run_slices(ids, stage=4)       # same inputs: every regular ADM slice starts warm
    for a, b in zip(f1, f2):
        assert np.array_equal(a["cut_nodes"], b["cut_nodes"])
        if a["flags"] == 0:
            assert b["warm"] == 1 and b["iters"] == 20
            # the multipliers restart at 0, so ADM leaves the previous point but stays near its fit
            assert b["resid"] < 2.0 * a["resid"] and not np.array_equal(a["U"], b["U"])
        else:
            assert b["warm"] == 0
    # a changed row set (other slice id) never matches: cold start
    o2 = oracle.Oracle(x)
    o2.set_warm([dict(f1[0], slice=1)])
    assert o2.run_slices([1], stage=3)[0]["warm"] == 0


# ------------------------------------------------------------------------------ count target

@pytest.mark.parametrize("tau", [3e-6, 1e-5, 4e-5])
def test_count_target_reproduces_the_threshold_cut(tau):
    # least-cost-first merging stopped at the size of the threshold cut merges the
    # same nodes: while a candidate of cost < tau is open the least cost is below tau, and the
    # threshold rule merges exactly the candidates below tau (costs depend on subtrees only)
    base = scenegen.make_inputs(scenegen.preset("t_interior", tau=tau))
    thr = oracle.Oracle(base).run_slices([0, 2, 5], stage=1)
    for r in thr:
        K = r["n"]
        x = scenegen.make_inputs(scenegen.preset("t_interior", tau=tau, coarsen_target=K))
        c = oracle.Oracle(x).run_slices([r["slice"]], stage=1)[0]
        assert np.array_equal(c["cut_nodes"], r["cut_nodes"])
        mc = {f: k for k, f in enumerate(c["proc_node"])}
        for k, f in enumerate(r["proc_node"]):
            if r["proc_merged"][k]:
                assert c["proc_merged"][mc[f]] == 1 and c["proc_cost"][mc[f]] == r["proc_cost"][k]


def test_count_target_sizes_and_order():
    x = scenegen.make_inputs(scenegen.preset("t_interior", coarsen_target=40))
    t = x.tree
    g = t["global_cut"].size
    for r in oracle.Oracle(x).run_slices(range(8), stage=1):
        assert r["n"] == 40 or r["proc_merged"].sum() == len(r["proc_node"])   # reached, or nothing left
        assert g - r["proc_merged"].sum() == r["n"]
    big = scenegen.make_inputs(scenegen.preset("t_interior", coarsen_target=10 ** 6))
    for r in oracle.Oracle(big).run_slices([0, 1], stage=1):
        assert r["proc_merged"].sum() == 0 and r["n"] == g
