"""Python face of the fp64 CPU oracle (oracle.c).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this module.  It shares no code with the CUDA path
(paper_2202_12567_b200/) and neither imports the other; both consume inputs from scenegen/.

Functions return numpy arrays; every stage follows PAPER.md as cited in oracle.c.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared", "-Wall"]

FLAG_DIRECT, FLAG_DIVERGED, FLAG_ZERO = 1, 2, 4


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "oracle.c")
    hdr = os.path.join(_HERE, "oracle.h")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(os.path.getmtime(src), os.path.getmtime(hdr)):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, src, "-lm"])
        os.replace(tmp, _SO)
    return _SO


class _Inputs(C.Structure):
    _fields_ = [
        ("m", C.c_int64),
        *[(k, C.c_void_p) for k in ("px", "py", "pz", "nx", "ny", "nz", "vx", "vy", "vz", "rr", "rg", "rb", "spec")],
        ("expo", C.c_void_p),
        ("nv", C.c_int64),
        *[(k, C.c_void_p) for k in ("lx", "ly", "lz", "lnx", "lny", "lnz", "lir", "lig", "lib")],
        ("nn", C.c_int64),
        ("left", C.c_void_p), ("right", C.c_void_p), ("rep", C.c_void_p),
        ("tir", C.c_void_p), ("tig", C.c_void_p), ("tib", C.c_void_p),
        ("ncut", C.c_int64), ("cut", C.c_void_p),
        ("nsph", C.c_int32), ("nbox", C.c_int32), ("nrect", C.c_int32),
        ("sph", C.c_void_p), ("box", C.c_void_p), ("rect", C.c_void_p),
        ("clamp_dist", C.c_double), ("shadow_eps", C.c_double), ("diag", C.c_double),
        ("wn", C.c_double), ("target", C.c_int32), ("seed", C.c_uint64),
        ("nmax", C.c_int32), ("nmin", C.c_int32), ("tau", C.c_double), ("rate", C.c_double),
        ("q", C.c_int32), ("solver", C.c_int32), ("K", C.c_int32),
        ("tol", C.c_double), ("alpha", C.c_double), ("beta", C.c_double), ("gamma", C.c_double), ("lam", C.c_double),
        ("order_seed", C.c_uint64),
        ("row_importance", C.c_int32), ("cost_mode", C.c_int32), ("resolve_mode", C.c_int32),
        ("warm_iters", C.c_int32), ("nwarm", C.c_int32), ("coarsen_target", C.c_int32), ("warm", C.c_void_p),
        ("ntri", C.c_int64), ("tri", C.c_void_p),
    ]


class _Warm(C.Structure):
    _fields_ = [("slice", C.c_int32), ("m", C.c_int32), ("n", C.c_int32), ("flags", C.c_int32),
                ("rows", C.c_void_p), ("cut", C.c_void_p), ("U", C.c_void_p), ("V", C.c_void_p)]


class _Result(C.Structure):
    _fields_ = [
        ("slice", C.c_int32), ("m", C.c_int32), ("n", C.c_int32),
        ("rows", C.POINTER(C.c_int32)), ("cut_nodes", C.POINTER(C.c_int32)),
        ("n_proc", C.c_int32),
        ("proc_node", C.POINTER(C.c_int32)), ("proc_merged", C.POINTER(C.c_int32)), ("proc_zoff", C.POINTER(C.c_int32)),
        ("proc_eps", C.POINTER(C.c_double)), ("proc_cost", C.POINTER(C.c_double)),
        ("proc_zrows", C.POINTER(C.c_int32)),
        ("proc_Va", C.POINTER(C.c_double)), ("proc_Vb", C.POINTER(C.c_double)),
        ("n_evals_coarsen", C.c_int64),
        ("nnz", C.c_int64), ("n_carried", C.c_int64), ("n_new", C.c_int64), ("n_forced", C.c_int64),
        ("n_draws", C.c_int64), ("target_N", C.c_int64),
        ("om_row", C.POINTER(C.c_int32)), ("om_col", C.POINTER(C.c_int32)),
        ("om_val", C.POINTER(C.c_double)), ("om_carried", C.POINTER(C.c_int32)),
        ("weights", C.POINTER(C.c_uint32)),
        ("q", C.c_int32), ("iters", C.c_int32), ("flags", C.c_int32),
        ("sigma", C.c_double), ("resid", C.c_double),
        ("U", C.POINTER(C.c_double)), ("V", C.POINTER(C.c_double)),
        ("obj", C.POINTER(C.c_double)), ("n_obj", C.c_int32),
        ("full", C.POINTER(C.c_double)),
        ("rgb", C.POINTER(C.c_double)),
        ("warm", C.c_int32),
    ]


def lib():
    global _lib
    with _lock:
        if _lib is None:
            # ORACLE_LIB: a prebuilt alternative (tools/mutants.py loads deliberately broken copies)
            L = C.CDLL(os.environ.get("ORACLE_LIB") or build())
            P = C.c_void_p
            L.orc_philox.argtypes = [P, P, P]
            L.orc_floyd.argtypes = [C.c_int32, C.c_int32, C.c_uint32, C.c_int32, C.c_uint64, C.c_uint32, P]
            L.orc_floyd.restype = C.c_int32
            L.orc_entry_T.argtypes = [C.POINTER(_Inputs), C.c_int64, C.c_int64]
            L.orc_entry_T.restype = C.c_double
            L.orc_entry_T_many.argtypes = [C.POINTER(_Inputs), C.c_int64, P, P, P]
            L.orc_entry_flops.argtypes = [C.POINTER(_Inputs), C.c_int64, P, P]
            L.orc_entry_flops.restype = C.c_int64
            L.orc_visible.argtypes = [C.POINTER(_Inputs), P, P]
            L.orc_visible.restype = C.c_int32
            L.orc_build_slices.argtypes = [C.POINTER(_Inputs), P, P, P]
            L.orc_run_slice.argtypes = [C.POINTER(_Inputs), P, C.c_int32, C.c_int32, C.c_int32]
            L.orc_run_slice.restype = C.POINTER(_Result)
            L.orc_run_slices.argtypes = [C.POINTER(_Inputs), P, P, C.c_int32, P, C.c_int32, P]
            L.orc_free_result.argtypes = [C.POINTER(_Result)]
            L.orc_adm.argtypes = [C.c_int32, C.c_int32, C.c_int64, P, P, P, C.c_int32, C.c_int32, C.c_double,
                                  C.c_double, C.c_double, C.c_double, C.c_uint64, C.c_int32, P, P, P, P, P]
            L.orc_adm.restype = C.c_int32
            L.orc_adm_warm.argtypes = [C.c_int32, C.c_int32, C.c_int64, P, P, P, C.c_int32, C.c_int32, C.c_double,
                                       C.c_double, C.c_double, C.c_double, P, P, P, P, P, P, P]
            L.orc_adm_warm.restype = C.c_int32
            L.orc_mals.argtypes = [C.c_int32, C.c_int32, C.c_int64, P, P, P, C.c_int32, C.c_int32, C.c_double,
                                   C.c_uint64, C.c_int32, P, P, P, P]
            L.orc_mals.restype = C.c_int32
            L.orc_fullcut_slice.argtypes = [C.POINTER(_Inputs), P, C.c_int32, P, C.c_int32, P]
            L.orc_bruteforce_rows.argtypes = [C.POINTER(_Inputs), P, C.c_int32, P]
            L.orc_build_light_tree.argtypes = [C.c_int64, P, P, P, P, P, P, C.c_int32, P, P, P, P, P, P, P, P]
            L.orc_build_light_tree.restype = C.c_int32
            L.orc_light_importance.argtypes = [C.c_int32, C.c_int64, P, P, P, P]
            L.orc_pdf_weights.argtypes = [C.c_int32, P, P, P]
            L.orc_cdf_pick.argtypes = [C.c_int32, P, C.c_uint64]
            L.orc_cdf_pick.restype = C.c_int32
            L.orc_pass2_draw_f.argtypes = [C.c_uint64, C.c_int32, C.c_uint32, C.c_uint64, P, C.c_int32, C.c_uint64, P,
                                           C.c_int32, P, P]
            L.orc_pass2_draws.argtypes = [C.c_uint64, C.c_int32, C.c_uint32, C.c_int64, P, C.c_int32, C.c_int32, P, P]
            _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


class Oracle:
    """Binds one scenegen.Inputs (arrays kept alive here) to the C oracle."""

    def __init__(self, x, **override):
        self.x = x
        prm = x.params()
        prm.update(override)
        self.prm = prm
        g, v, t, pr = x.gbuf, x.vpls, x.tree, x.prims
        keep = []

        def arr(a, dt):
            a = np.ascontiguousarray(a, dt)
            keep.append(a)
            return _p(a)

        s = _Inputs()
        s.m = g["px"].shape[0]
        for k, src in (("px", "px"), ("py", "py"), ("pz", "pz"), ("nx", "nx"), ("ny", "ny"), ("nz", "nz"),
                       ("vx", "vx"), ("vy", "vy"), ("vz", "vz"), ("rr", "rho_r"), ("rg", "rho_g"),
                       ("rb", "rho_b"), ("spec", "spec")):
            setattr(s, k, arr(g[src], np.float32))
        s.expo = arr(g["exponent"], np.int32)
        s.nv = v["px"].shape[0]
        for k, src in (("lx", "px"), ("ly", "py"), ("lz", "pz"), ("lnx", "nx"), ("lny", "ny"), ("lnz", "nz"),
                       ("lir", "ir"), ("lig", "ig"), ("lib", "ib")):
            setattr(s, k, arr(v[src], np.float32))
        s.nn = t["left"].shape[0]
        s.left = arr(t["left"], np.int32)
        s.right = arr(t["right"], np.int32)
        s.rep = arr(t["rep"], np.int32)
        s.tir = arr(t["ir"], np.float32)
        s.tig = arr(t["ig"], np.float32)
        s.tib = arr(t["ib"], np.float32)
        s.ncut = t["global_cut"].shape[0]
        s.cut = arr(t["global_cut"], np.int32)
        s.nsph, s.nbox, s.nrect = pr["sph"].shape[0], pr["box"].shape[0], pr["rect"].shape[0]
        s.sph = arr(pr["sph"], np.float32)
        s.box = arr(pr["box"], np.float32)
        s.rect = arr(pr["rect"], np.float32)
        tri = pr.get("tri", np.zeros((0, 9), np.float32))
        s.ntri = tri.shape[0]
        s.tri = arr(tri, np.float32)
        s.clamp_dist, s.shadow_eps, s.diag = x.clamp_dist, x.shadow_eps, x.diag
        s.wn = prm["normal_weight"]
        s.target = prm["slice_target"]
        s.seed = prm["seed"]
        s.nmax, s.nmin = prm["p1_nmax"], prm["p1_nmin"]
        s.tau, s.rate = prm["tau"], prm["rate"]
        s.q, s.solver, s.K = prm["rank_q"], prm["solver"], prm["max_iter"]
        s.tol, s.alpha, s.beta, s.gamma, s.lam = prm["tol"], prm["alpha"], prm["beta"], prm["gamma"], prm["lam"]
        s.order_seed = prm.get("order_seed", 0)
        s.row_importance = prm.get("row_importance", 0)
        s.cost_mode = prm.get("cost_mode", 0)
        s.resolve_mode = prm.get("resolve_mode", 0)
        s.warm_iters = prm.get("warm_iters", 0)
        s.coarsen_target = prm.get("coarsen_target", 0)
        s.nwarm = 0
        s.warm = None
        self._keep = keep
        self.s = s
        self._slices = None

    # -- primitives -------------------------------------------------------------------------
    def entry_T(self, row: int, vpl: int) -> float:
        return lib().orc_entry_T(C.byref(self.s), int(row), int(vpl))

    def entries_T(self, rows, vpls):
        rows = np.ascontiguousarray(rows, np.int32)
        vpls = np.ascontiguousarray(vpls, np.int32)
        out = np.zeros(rows.size)
        lib().orc_entry_T_many(C.byref(self.s), rows.size, _p(rows), _p(vpls), _p(out))
        return out

    def entry_flops(self, rows, vpls) -> int:
        """fp64 operations (+ - * / sqrt) the oracle's entry function executes over these pairs"""
        rows = np.ascontiguousarray(rows, np.int32)
        vpls = np.ascontiguousarray(vpls, np.int32)
        return int(lib().orc_entry_flops(C.byref(self.s), rows.size, _p(rows), _p(vpls)))

    def visible(self, x, y) -> bool:
        a = np.ascontiguousarray(x, np.float64)
        b = np.ascontiguousarray(y, np.float64)
        return bool(lib().orc_visible(C.byref(self.s), _p(a), _p(b)))

    def slices(self):
        if self._slices is None:
            m = int(self.s.m)
            off = np.zeros(m + 2, np.int32)
            rows = np.zeros(max(m, 1), np.int32)
            ns = np.zeros(1, np.int64)
            lib().orc_build_slices(C.byref(self.s), _p(off), _p(rows), _p(ns))
            n = int(ns[0])
            self._slices = (off[: n + 1].copy(), rows[:m].copy())
        return self._slices

    def set_warm(self, prev_results):
        """warm start from the results of the previous frame (dicts of run_slices, stage >= 3)"""
        keep = []
        arr = (_Warm * max(len(prev_results), 1))()
        for k, r in enumerate(prev_results):
            cols = [np.ascontiguousarray(r["rows"], np.int32), np.ascontiguousarray(r["cut_nodes"], np.int32),
                    np.ascontiguousarray(r["U"], np.float64), np.ascontiguousarray(r["V"], np.float64)]
            keep += cols
            arr[k] = _Warm(r["slice"], r["m"], r["n"], r["flags"], *[_p(a).value for a in cols])
        self._warm_keep = (keep, arr)
        self.s.nwarm = len(prev_results)
        self.s.warm = C.cast(arr, C.c_void_p)

    def run_slices(self, slice_ids, stage: int = 4):
        off, rows = self.slices()
        ids = np.ascontiguousarray(slice_ids, np.int32)
        out = (C.POINTER(_Result) * max(len(ids), 1))()
        lib().orc_run_slices(C.byref(self.s), _p(off), _p(rows), len(ids), _p(ids), stage, C.cast(out, C.c_void_p))
        res = []
        for k in range(len(ids)):
            res.append(_convert(out[k].contents, stage))
            lib().orc_free_result(out[k])
        return res

    def fullcut_slice(self, rows, cut_nodes):
        rows = np.ascontiguousarray(rows, np.int32)
        cut = np.ascontiguousarray(cut_nodes, np.int32)
        out = np.zeros((rows.size, 3))
        lib().orc_fullcut_slice(C.byref(self.s), _p(rows), rows.size, _p(cut), cut.size, _p(out))
        return out

    def bruteforce_rows(self, rows):
        rows = np.ascontiguousarray(rows, np.int32)
        out = np.zeros((rows.size, 3))
        lib().orc_bruteforce_rows(C.byref(self.s), _p(rows), rows.size, _p(out))
        return out

    def render(self, slice_ids=None, stage: int = 4):
        """Full pipeline; returns (image H*W*3 float64, per-slice results)."""
        off, rows = self.slices()
        if slice_ids is None:
            slice_ids = np.arange(off.size - 1)
        res = self.run_slices(slice_ids, stage)
        img = np.zeros((self.x.height * self.x.width, 3))
        pix = self.x.gbuf["pixel"]
        for r in res:
            if r.get("rgb") is not None:
                img[pix[r["rows"]]] = r["rgb"]
        return img, res


def _arr(ptr, n, dt):
    if n <= 0 or not ptr:
        return np.zeros(0, dt)
    return np.ctypeslib.as_array(ptr, shape=(n,)).astype(dt, copy=True)


def _convert(r: _Result, stage: int) -> dict:
    m, n, q = r.m, r.n, r.q
    d = dict(slice=r.slice, m=m, n=n, rows=_arr(r.rows, m, np.int32), cut_nodes=_arr(r.cut_nodes, n, np.int32))
    npr = r.n_proc
    zoff = _arr(r.proc_zoff, npr + 1, np.int32)
    nz = int(zoff[-1]) if npr else 0
    d.update(proc_node=_arr(r.proc_node, npr, np.int32), proc_merged=_arr(r.proc_merged, npr, np.int32),
             proc_eps=_arr(r.proc_eps, npr, np.float64), proc_cost=_arr(r.proc_cost, npr, np.float64),
             proc_zoff=zoff, proc_zrows=_arr(r.proc_zrows, nz, np.int32),
             proc_Va=_arr(r.proc_Va, nz, np.float64), proc_Vb=_arr(r.proc_Vb, nz, np.float64),
             n_evals_coarsen=r.n_evals_coarsen)
    if stage >= 2:
        k = r.nnz
        d.update(nnz=k, n_carried=r.n_carried, n_new=r.n_new, n_forced=r.n_forced, n_draws=r.n_draws,
                 target_N=r.target_N, om_row=_arr(r.om_row, k, np.int32), om_col=_arr(r.om_col, k, np.int32),
                 om_val=_arr(r.om_val, k, np.float64), om_carried=_arr(r.om_carried, k, np.int32),
                 weights=_arr(r.weights, n, np.uint32))
    if stage >= 3:
        d.update(q=q, iters=r.iters, flags=r.flags, sigma=r.sigma, resid=r.resid, warm=r.warm,
                 U=_arr(r.U, m * q, np.float64).reshape(m, q), V=_arr(r.V, q * n, np.float64).reshape(q, n),
                 obj=_arr(r.obj, r.n_obj, np.float64),
                 full=_arr(r.full, m * n, np.float64).reshape(m, n) if r.full else None)
    if stage >= 4:
        d["rgb"] = _arr(r.rgb, m * 3, np.float64).reshape(m, 3)
    return d


def philox(ctr, key):
    c = np.ascontiguousarray(ctr, np.uint32)
    k = np.ascontiguousarray(key, np.uint32)
    o = np.zeros(4, np.uint32)
    lib().orc_philox(_p(c), _p(k), _p(o))
    return o


def floyd(m, n, a, slice_id, seed, tag=1):
    out = np.zeros(max(min(n, m), 1), np.int32)
    cnt = lib().orc_floyd(m, n, a, slice_id, seed, tag, _p(out))
    return out[:cnt].copy()


def adm(m, n, row, col, val, q, K=100, tol=0.0, alpha=1.0, beta=1.0, gamma=1.6, seed=12567, slice_id=0):
    row = np.ascontiguousarray(row, np.int32)
    col = np.ascontiguousarray(col, np.int32)
    val = np.ascontiguousarray(val, np.float64)
    U = np.zeros((m, q))
    V = np.zeros((q, n))
    it = np.zeros(1, np.int32)
    res = np.zeros(1)
    sg = np.zeros(1)
    flags = lib().orc_adm(m, n, row.size, _p(row), _p(col), _p(val), q, K, tol, alpha, beta, gamma, seed,
                          slice_id, _p(U), _p(V), _p(it), _p(res), _p(sg))
    return dict(U=U, V=V, iters=int(it[0]), resid=float(res[0]), sigma=float(sg[0]), flags=flags)


def mals(m, n, row, col, val, q, K=100, lam=1e-3, seed=12567, slice_id=0):
    row = np.ascontiguousarray(row, np.int32)
    col = np.ascontiguousarray(col, np.int32)
    val = np.ascontiguousarray(val, np.float64)
    X = np.zeros((m, q))
    Y = np.zeros((q, n))
    obj = np.zeros(2 * K)
    sg = np.zeros(1)
    flags = lib().orc_mals(m, n, row.size, _p(row), _p(col), _p(val), q, K, lam, seed, slice_id, _p(X), _p(Y),
                           _p(obj), _p(sg))
    return dict(X=X, Y=Y, obj=obj, sigma=float(sg[0]), flags=flags)


def light_importance(n, col, val):
    """g(c) = max - min of column c's observations and the observation counts."""
    col = np.ascontiguousarray(col, np.int32)
    val = np.ascontiguousarray(val, np.float64)
    g = np.zeros(max(n, 1))
    cnt = np.zeros(max(n, 1), np.int32)
    lib().orc_light_importance(n, col.size, _p(col), _p(val), _p(g), _p(cnt))
    return g[:n], cnt[:n]


def pdf_weights(g, cnt):
    g = np.ascontiguousarray(g, np.float64)
    cnt = np.ascontiguousarray(cnt, np.int32)
    w = np.zeros(max(g.size, 1), np.uint32)
    lib().orc_pdf_weights(g.size, _p(g), _p(cnt), _p(w))
    return w[:g.size]


def cdf_pick(cdf, x):
    cdf = np.ascontiguousarray(cdf, np.uint64)
    return int(lib().orc_cdf_pick(cdf.size, _p(cdf), int(x)))


def pass2_draws(w, m, count, seed=12567, slice_id=0, t0=0):
    w = np.ascontiguousarray(w, np.uint32)
    rows = np.zeros(count, np.int32)
    cols = np.zeros(count, np.int32)
    lib().orc_pass2_draws(seed, slice_id, t0, count, _p(w), w.size, m, _p(rows), _p(cols))
    return rows, cols


def pass2_draw_f(t, w, wr, seed=12567, slice_id=0):
    """one pass-2 draw with row importance (column CDF from w, row CDF from wr) -> (row, col)"""
    cdf = np.cumsum(np.asarray(w, np.uint64)).astype(np.uint64)
    rcdf = np.cumsum(np.asarray(wr, np.uint64)).astype(np.uint64)
    r = np.zeros(1, np.int32)
    c = np.zeros(1, np.int32)
    lib().orc_pass2_draw_f(seed, slice_id, t, int(cdf[-1]), _p(cdf), cdf.size, int(rcdf[-1]), _p(rcdf), rcdf.size,
                           _p(r), _p(c))
    return int(r[0]), int(c[0])


def adm_warm(m, n, row, col, val, q, X0, Y0, K=100, tol=0.0, alpha=1.0, beta=1.0, gamma=1.6):
    row = np.ascontiguousarray(row, np.int32)
    col = np.ascontiguousarray(col, np.int32)
    val = np.ascontiguousarray(val, np.float64)
    X0 = np.ascontiguousarray(X0, np.float64)
    Y0 = np.ascontiguousarray(Y0, np.float64)
    U = np.zeros((m, q))
    V = np.zeros((q, n))
    it = np.zeros(1, np.int32)
    res = np.zeros(1)
    sg = np.zeros(1)
    flags = lib().orc_adm_warm(m, n, row.size, _p(row), _p(col), _p(val), q, K, tol, alpha, beta, gamma, _p(X0), _p(Y0),
                               _p(U), _p(V), _p(it), _p(res), _p(sg))
    return dict(U=U, V=V, iters=int(it[0]), resid=float(res[0]), sigma=float(sg[0]), flags=flags)


def build_light_tree(vpls, cut_max):
    """light tree + global cut (R38) from VPL SoA arrays -> dict like scenegen's tree"""
    v = {k: np.ascontiguousarray(vpls[k], np.float32) for k in ("px", "py", "pz", "ir", "ig", "ib")}
    nv = v["px"].size
    nn = 2 * nv - 1
    left, right, rep = (np.zeros(nn, np.int32) for _ in range(3))
    ir, ig, ib = (np.zeros(nn, np.float32) for _ in range(3))
    cut = np.zeros(max(nn, 1), np.int32)
    nc = np.zeros(1, np.int64)
    st = lib().orc_build_light_tree(nv, *[_p(v[k]) for k in ("px", "py", "pz", "ir", "ig", "ib")], cut_max, _p(left),
                                    _p(right), _p(rep), _p(ir), _p(ig), _p(ib), _p(cut), _p(nc))
    assert st == 0
    return dict(left=left, right=right, rep=rep, ir=ir, ig=ig, ib=ib, global_cut=cut[: int(nc[0])].copy(), root=0)
