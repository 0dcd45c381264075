"""Pins for the oracle's completion (ADM, PAPER.md:149 and App. A; masked ALS,
BASELINE north_star) and rendering I(s) = X (Y e).

Each pin is fixed by something other than the oracle itself: an independent re-derivation
(implicit-Z ADM written here in numpy), closed forms, planted recovery, Eckart-Young (LAPACK
SVD), brute force over all VPLs.
"""
import numpy as np
import pytest

import oracle
import scenegen
from tests._mini import mini


def _planted(m, n, r, frac, seed):
    rng = np.random.default_rng(seed)
    A = rng.uniform(0, 1, (m, r)) @ rng.uniform(0, 1, (r, n))
    mask = rng.uniform(size=(m, n)) < frac
    rows, cols = np.nonzero(mask)
    return A, rows.astype(np.int32), cols.astype(np.int32), A[rows, cols], mask


def _philox_unif(a, b, s, tag, seed):
    u = oracle.philox([a, b, s, tag], [seed & 0xFFFFFFFF, seed >> 32])[0]
    return (int(u) >> 8) * 2.0 ** -24


def _adm_implicit_numpy(m, n, rows, cols, vals, q, K, alpha, beta, gamma, seed, s):
    """Independent re-derivation of App. A with Z never formed: Z = XY + S, S sparse on Omega
    (so Z Y^T = X (Y Y^T) + S Y^T and X_new^T Z = (X_new^T X) Y + X_new^T S)."""
    sg = vals.max()
    Mh = vals / sg
    mu = Mh.sum() / Mh.size
    c0 = 2.0 * np.sqrt(mu / q)
    X = np.array([[c0 * _philox_unif(i, l, s, 4, seed) for l in range(q)] for i in range(m)])
    Y = np.array([[c0 * _philox_unif(l, j, s, 5, seed) for j in range(n)] for l in range(q)])
    U, V = X.copy(), Y.copy()
    Lam, Pi = np.zeros_like(X), np.zeros_like(Y)
    S = np.zeros((m, n))
    S[rows, cols] = Mh          # Z_0 = P_Omega(M): X_0 Y_0 is not part of Z_0
    XY0 = np.zeros((m, n))
    I = np.eye(q)
    first = True
    for _ in range(K):
        ZYt = S @ Y.T + (0 if first else X @ (Y @ Y.T))
        Xn = np.linalg.solve((Y @ Y.T + alpha * I).T, (ZYt + alpha * U - Lam).T).T
        XtZ = Xn.T @ S + (0 if first else (Xn.T @ X) @ Y)
        Yn = np.linalg.solve(Xn.T @ Xn + beta * I, XtZ + beta * V - Pi)
        X, Y = Xn, Yn
        first = False
        S = np.zeros((m, n))
        S[rows, cols] = Mh - np.einsum("ij,ji->i", X[rows], Y[:, cols])
        U = np.maximum(0, X + Lam / alpha)
        V = np.maximum(0, Y + Pi / beta)
        Lam = Lam + gamma * alpha * (X - U)
        Pi = Pi + gamma * beta * (Y - V)
    return U, sg * V


def test_adm_literal_equals_implicit_form():
    A, rows, cols, vals, _ = _planted(60, 40, 3, 0.3, 1)
    q, K = 5, 30
    o = oracle.adm(60, 40, rows, cols, vals, q, K=K, seed=77, slice_id=3)
    U, V = _adm_implicit_numpy(60, 40, rows, cols, vals, q, K, 1.0, 1.0, 1.6, 77, 3)
    assert np.linalg.norm(o["U"] - U) / np.linalg.norm(U) < 1e-10
    assert np.linalg.norm(o["V"] - V) / np.linalg.norm(V) < 1e-10


def test_adm_nonnegative_outputs():
    A, rows, cols, vals, _ = _planted(80, 50, 4, 0.2, 2)
    o = oracle.adm(80, 50, rows, cols, vals, 8, K=50)
    assert np.all(o["U"] >= 0) and np.all(o["V"] >= 0)
    assert o["iters"] == 50


def test_adm_rank1_fully_observed():
    rng = np.random.default_rng(3)
    a, b = rng.uniform(0.1, 1, 30), rng.uniform(0.1, 1, 20)
    A = np.outer(a, b)
    rows, cols = np.nonzero(np.ones_like(A, bool))
    o = oracle.adm(30, 20, rows, cols, A[rows, cols], 1, K=100)
    rel = np.linalg.norm(o["U"] @ o["V"] - A) / np.linalg.norm(A)
    assert rel <= 1e-3


def test_adm_zero_matrix():
    rows = np.array([0, 1, 2], np.int32)
    cols = np.array([0, 1, 2], np.int32)
    o = oracle.adm(5, 4, rows, cols, np.zeros(3), 2, K=10)
    assert o["flags"] & oracle.FLAG_ZERO
    assert not o["U"].any() and not o["V"].any()


def test_adm_planted_recovery():
    # N >= 5 dof, q = r, alpha = beta = 0.1: held-out error -> 0 (SURVEY 8(c) pin; [calib] 3e-6)
    m, n, r = 200, 100, 4
    A, rows, cols, vals, mask = _planted(m, n, r, 0.3, 5)
    assert rows.size >= 5 * r * (m + n - r)
    o = oracle.adm(m, n, rows, cols, vals, r, K=3000, alpha=0.1, beta=0.1)
    R = o["U"] @ o["V"]
    held = np.linalg.norm((R - A)[~mask]) / np.linalg.norm(A[~mask])
    assert held <= 1e-5


def test_adm_tolerance_stop():
    A, rows, cols, vals, _ = _planted(60, 40, 2, 0.5, 9)
    o = oracle.adm(60, 40, rows, cols, vals, 2, K=5000, tol=1e-3, alpha=0.1, beta=0.1)
    assert o["iters"] < 5000 and o["resid"] < 1e-3


def test_mals_monotone_objective():
    A, rows, cols, vals, _ = _planted(80, 60, 5, 0.15, 4)
    A2 = A + np.random.default_rng(1).uniform(0, 0.3, A.shape)   # not exactly low rank
    o = oracle.mals(80, 60, rows, cols, A2[rows, cols], 6, K=40, lam=1e-3)
    f = o["obj"]
    assert np.all(np.diff(f) <= 1e-12 * np.abs(f[:-1]))


def test_mals_planted_recovery():
    m, n, r = 200, 100, 4
    A, rows, cols, vals, mask = _planted(m, n, r, 0.3, 6)
    o = oracle.mals(m, n, rows, cols, vals, r, K=60, lam=1e-9)
    R = o["X"] @ o["Y"]
    held = np.linalg.norm((R - A)[~mask]) / np.linalg.norm(A[~mask])
    assert held <= 1e-8


def test_mals_fully_observed_eckart_young():
    rng = np.random.default_rng(8)
    m, n, q = 40, 30, 3
    A = rng.uniform(0, 1, (m, n))
    rows, cols = np.nonzero(np.ones((m, n), bool))
    o = oracle.mals(m, n, rows, cols, A[rows, cols], q, K=500, lam=1e-12)
    s = np.linalg.svd(A / A.max(), compute_uv=False)
    best = (s[q:] ** 2).sum()
    assert o["obj"][-1] == pytest.approx(best, rel=1e-6)


# ---------------------------------------------------------------------------------------- resolve

def test_resolve_is_factored_column_sum(inputs_cache):
    x = inputs_cache("c1")
    o = oracle.Oracle(x)
    t = x.tree
    g = x.gbuf
    for r in o.run_slices([2, 9], stage=4):
        if r["flags"] & oracle.FLAG_DIRECT:
            continue
        M = r["U"] @ r["V"]                       # (U V) materialised only here, in the test
        f = r["cut_nodes"]
        I = np.stack([t["ir"][f], t["ig"][f], t["ib"][f]], 1).astype(np.float64)
        lI = I @ np.array([0.2126, 0.7152, 0.0722])
        w = I / lI[:, None]
        p = r["rows"]
        rho = np.stack([g["rho_r"][p], g["rho_g"][p], g["rho_b"][p]], 1).astype(np.float64)
        tint = rho / (rho @ np.array([0.2126, 0.7152, 0.0722]))[:, None]
        img = tint * (M @ w)
        assert np.allclose(r["rgb"], img, rtol=1e-9, atol=1e-14)


def test_single_vpl_equals_brute_force():
    # one VPL: n = 1 <= q so the slice is rendered directly, which must equal brute force
    rng = np.random.default_rng(2)
    pts = rng.uniform(0, 1, (64, 3)) * [1, 0, 1]
    x = mini(pts, np.tile([0, 1, 0], (64, 1)), [0.4, 0.7, 0.6], [0, -1, 0], [0.5, 0.7, 0.9],
             rho=rng.uniform(0.2, 0.9, (64, 3)), sph=[[0.5, 0.3, 0.5, 0.1]], slice_target=32)
    o = oracle.Oracle(x)
    img, res = o.render()
    bf = o.bruteforce_rows(np.arange(64))
    assert all(r["flags"] & oracle.FLAG_DIRECT for r in res)
    assert np.allclose(img, bf, rtol=1e-12, atol=1e-300)


def test_all_leaves_direct_equals_brute_force():
    # global cut = all leaves, tau = 0 (no merge), q >= n -> direct: image = sum over all VPLs
    rng = np.random.default_rng(4)
    npt, nv = 50, 6
    pts = rng.uniform(0, 1, (npt, 3)) * [1, 0, 1]
    vp = rng.uniform(0.1, 0.9, (nv, 3)) * [1, 0, 1] + [0, 0.8, 0]
    x = mini(pts, np.tile([0, 1, 0], (npt, 1)), vp, np.tile([0, -1, 0], (nv, 1)), rng.uniform(0.2, 1, (nv, 3)),
             rho=rng.uniform(0.2, 0.9, (npt, 3)), box=[[0.4, 0.2, 0.4, 0.6, 0.4, 0.6]], tau=0.0, rank_q=8,
             slice_target=25)
    o = oracle.Oracle(x)
    img, res = o.render()
    bf = o.bruteforce_rows(np.arange(npt))
    assert np.allclose(img, bf, rtol=1e-12, atol=1e-300)


def test_pipeline_sanity_against_brute_force(inputs_cache):
    # loose quality bound (not a parity target): the completed image is near brute force
    x = inputs_cache("c1")
    o = oracle.Oracle(x)
    img, res = o.render()
    sel = np.arange(0, x.m, 5)
    bf = o.bruteforce_rows(sel)
    lumw = np.array([0.2126, 0.7152, 0.0722])
    a, b = img[x.gbuf["pixel"][sel]] @ lumw, bf @ lumw
    assert np.sqrt(np.mean((a - b) ** 2)) / np.sqrt(np.mean(b ** 2)) < 0.35
    assert np.all(img >= 0)
