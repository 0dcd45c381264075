"""ctypes binding of liblmc.so (include/lmc.h) — argument marshalling only.

Every stage of the hot path runs in the library's CUDA kernels; this module only converts
numpy arrays / torch tensors into the C structs and pointers the ABI takes.  There is no CPU
fallback: if the library cannot be loaded, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np
import torch  # noqa: F401  -- before liblmc.so: one libnccl.so.2 (torch's) serves both

_HERE = os.path.dirname(os.path.abspath(__file__))
# LMC_LIB: alternative build of the same library (diagnostic builds); default in-tree
LIB_PATH = os.environ.get("LMC_LIB") or os.path.join(_HERE, "liblmc.so")

LMC_OK, LMC_EINVAL, LMC_ESTATE, LMC_ENOMEM, LMC_ECUDA, LMC_EOVERFLOW, LMC_ENCCL = range(7)
SOLVER_ADM, SOLVER_MALS = 0, 1
MEM_DEVICE, MEM_HOST = 0, 1
SLICE_DIRECT, SLICE_DIVERGED, SLICE_ZERO = 1, 2, 4

_P = C.c_void_p


class Gbuffer(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("count", C.c_int64), ("pixel", _P),
                *[(k, _P) for k in ("px", "py", "pz", "nx", "ny", "nz", "vx", "vy", "vz", "rho_r", "rho_g", "rho_b",
                                    "spec")],
                ("exponent", _P)]


class Vpls(C.Structure):
    _fields_ = [("count", C.c_int64), *[(k, _P) for k in ("px", "py", "pz", "nx", "ny", "nz", "ir", "ig", "ib")]]


class LightTree(C.Structure):
    _fields_ = [("num_nodes", C.c_int64), ("root", C.c_int32), ("left", _P), ("right", _P), ("rep", _P),
                ("ir", _P), ("ig", _P), ("ib", _P), ("cut_size", C.c_int64), ("global_cut", _P)]


class Scene(C.Structure):
    _fields_ = [("n_sph", C.c_int32), ("n_box", C.c_int32), ("n_rect", C.c_int32), ("sph", _P), ("box", _P),
                ("rect", _P), ("clamp_dist", C.c_double), ("shadow_eps", C.c_double), ("diag", C.c_double),
                ("n_tri", C.c_int32), ("tri", _P)]


class Config(C.Structure):
    _fields_ = [("slice_target", C.c_int32), ("normal_weight", C.c_double), ("seed", C.c_uint64),
                ("p1_nmax", C.c_int32), ("p1_nmin", C.c_int32), ("coarsen_tau", C.c_double), ("rate", C.c_double),
                ("rank_q", C.c_int32), ("solver", C.c_int32), ("max_iter", C.c_int32), ("tol", C.c_double),
                ("alpha", C.c_double), ("beta", C.c_double), ("gamma", C.c_double), ("lambda_", C.c_double),
                ("rank", C.c_int32), ("world", C.c_int32), ("input_memory", C.c_int32), ("stream", _P),
                ("nccl_id", C.c_uint8 * 128), ("row_importance", C.c_int32), ("cost_mode", C.c_int32),
                ("resolve_mode", C.c_int32), ("warm_start", C.c_int32), ("warm_iters", C.c_int32),
                ("coarsen_target", C.c_int32), ("partition", C.c_int32)]


class Stats(C.Structure):
    _fields_ = [(k, C.c_int64) for k in ("n_slices", "slice_begin", "slice_end", "rows", "sum_cols", "sum_samples",
                                         "sum_completed", "evals_pass1", "evals_coarsen", "evals_pass2", "n_direct",
                                         "n_zero", "n_diverged", "pool_used_max", "pool_cap", "launches")] + \
              [(k, C.c_float) for k in ("ms_slices", "ms_pass1", "ms_coarsen", "ms_pass2", "ms_complete",
                                        "ms_resolve", "ms_solver")] + \
              [(k, C.c_int64) for k in ("layout_row_slots", "layout_col_slots")] + [("ms_eval2", C.c_float), ("n_warm", C.c_int64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


EXPORTS = ["lmc_create", "lmc_upload_inputs", "lmc_build_slices", "lmc_sample_pass1", "lmc_coarsen_cut",
           "lmc_sample_pass2", "lmc_complete", "lmc_resolve_image", "lmc_resolve_rows", "lmc_scatter_rows",
           "lmc_destroy", "lmc_last_error", "lmc_status_str", "lmc_get_slices", "lmc_get_pass1", "lmc_get_coarsen",
           "lmc_get_cut", "lmc_get_samples", "lmc_get_factors", "lmc_get_stats", "lmc_set_timing",
           "lmc_eval_entries", "lmc_nccl_unique_id", "lmc_get_partition", "lmc_plan_partition", "lmc_sizeof_struct",
           "lmc_build_light_tree", "lmc_plan_bvh"]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with paper_2202_12567_b200/build.py (no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    ST = C.c_int
    L.lmc_create.argtypes = [C.POINTER(Gbuffer), C.POINTER(Vpls), C.POINTER(LightTree), C.POINTER(Scene),
                             C.POINTER(Config), C.POINTER(_P)]
    L.lmc_create.restype = ST
    L.lmc_upload_inputs.argtypes = [_P, C.POINTER(Gbuffer), C.POINTER(Vpls), C.POINTER(LightTree)]
    for f in ("lmc_build_slices", "lmc_sample_pass1", "lmc_coarsen_cut", "lmc_sample_pass2", "lmc_complete"):
        getattr(L, f).argtypes = [_P]
        getattr(L, f).restype = ST
    L.lmc_resolve_image.argtypes = [_P, _P, C.c_int32]
    L.lmc_resolve_rows.argtypes = [_P, _P]
    L.lmc_scatter_rows.argtypes = [_P, _P, C.c_int64, _P]
    L.lmc_nccl_unique_id.argtypes = [_P]
    L.lmc_get_partition.argtypes = [_P, _P, _P]
    L.lmc_build_light_tree.argtypes = [C.POINTER(Vpls), C.c_int32, C.c_int32, _P, _P, _P, _P, _P, _P, _P, _P, _P]
    L.lmc_sizeof_struct.argtypes = [C.c_int32]
    L.lmc_sizeof_struct.restype = C.c_int64
    L.lmc_plan_partition.argtypes = [C.c_int64, C.c_int32, C.c_int32, _P, _P, _P]
    L.lmc_plan_bvh.argtypes = [_P, C.c_int32, _P, _P, _P, _P]
    L.lmc_destroy.argtypes = [_P]
    L.lmc_destroy.restype = None
    L.lmc_last_error.argtypes = [_P]
    L.lmc_last_error.restype = C.c_char_p
    L.lmc_status_str.argtypes = [C.c_int]
    L.lmc_status_str.restype = C.c_char_p
    L.lmc_get_slices.argtypes = [_P, _P, _P, _P]
    L.lmc_get_pass1.argtypes = [_P, C.c_int32, _P, _P, _P, _P, _P, _P, _P]
    L.lmc_get_coarsen.argtypes = [_P, C.c_int32, _P, _P, _P, _P, _P, _P]
    L.lmc_get_cut.argtypes = [_P, C.c_int32, _P, _P]
    L.lmc_get_samples.argtypes = [_P, C.c_int32, _P, _P, _P, _P, _P, _P]
    L.lmc_get_factors.argtypes = [_P, C.c_int32, _P, _P, _P, _P, _P, _P, _P, _P]
    L.lmc_get_stats.argtypes = [_P, C.POINTER(Stats)]
    L.lmc_set_timing.argtypes = [_P, C.c_int32]
    L.lmc_eval_entries.argtypes = [_P, C.c_int64, _P, _P, _P]
    return L


lib = _load()


class LmcError(RuntimeError):
    pass


def _ptr(a):
    """device pointer of a torch tensor or host pointer of a numpy array"""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data_as(_P)
    return _P(a.data_ptr())


class Frame:
    """One lmc context: inputs resident on the GPU, the seven stage calls, getters.

    ``inputs`` is a scenegen.Inputs; ``memory`` chooses whether the arrays handed to
    lmc_create are device tensors (MEM_DEVICE, via torch) or pinned host arrays (MEM_HOST).
    """

    def __init__(self, inputs, memory=MEM_DEVICE, rank=0, world=1, stream=None, device="cuda", nccl_id=None,
                 **override):
        import torch
        self.x = inputs
        self.memory = memory
        prm = inputs.params()
        prm.update(override)
        self.prm = prm
        self._keep = []
        self._torch = torch
        self.device = device

        def arr(a, dt):
            a = np.ascontiguousarray(a, dt)
            if memory == MEM_DEVICE:
                t = torch.from_numpy(a).to(device)
            else:
                t = torch.from_numpy(a).pin_memory()
            self._keep.append(t)
            return _P(t.data_ptr())

        self.arr = arr
        g, v, t = inputs.gbuf, inputs.vpls, inputs.tree
        self.gb = Gbuffer(inputs.width, inputs.height, g["px"].shape[0], arr(g["pixel"], np.int32),
                          *[arr(g[k], np.float32) for k in ("px", "py", "pz", "nx", "ny", "nz", "vx", "vy", "vz",
                                                            "rho_r", "rho_g", "rho_b", "spec")],
                          arr(g["exponent"], np.int32))
        self.vp = Vpls(v["px"].shape[0], *[arr(v[k], np.float32) for k in ("px", "py", "pz", "nx", "ny", "nz", "ir",
                                                                           "ig", "ib")])
        self.tr = LightTree(t["left"].shape[0], int(t["root"]), arr(t["left"], np.int32), arr(t["right"], np.int32),
                            arr(t["rep"], np.int32), arr(t["ir"], np.float32), arr(t["ig"], np.float32),
                            arr(t["ib"], np.float32), t["global_cut"].shape[0], arr(t["global_cut"], np.int32))
        pr = inputs.prims
        tri = pr.get("tri", np.zeros((0, 9), np.float32))
        self._prims = [np.ascontiguousarray(pr[k], np.float32) for k in ("sph", "box", "rect")] + \
            [np.ascontiguousarray(tri, np.float32)]
        self.sc = Scene(pr["sph"].shape[0], pr["box"].shape[0], pr["rect"].shape[0], *[_ptr(a) for a in self._prims[:3]],
                        inputs.clamp_dist, inputs.shadow_eps, inputs.diag, tri.shape[0], _ptr(self._prims[3]))
        if stream is None:
            stream = torch.cuda.current_stream(device)
        self.stream = stream
        self.cfg = Config(prm["slice_target"], prm["normal_weight"], prm["seed"], prm["p1_nmax"], prm["p1_nmin"],
                          prm["tau"], prm["rate"], prm["rank_q"], prm["solver"], prm["max_iter"], prm["tol"],
                          prm["alpha"], prm["beta"], prm["gamma"], prm["lam"], rank, world, memory,
                          _P(stream.cuda_stream))
        if nccl_id is not None:
            self.cfg.nccl_id = (C.c_uint8 * 128)(*bytes(nccl_id))
        self.cfg.row_importance = int(prm.get("row_importance", 0))
        self.cfg.cost_mode = int(prm.get("cost_mode", 0))
        self.cfg.resolve_mode = int(prm.get("resolve_mode", 0))
        self.cfg.warm_start = int(prm.get("warm_start", 0))
        self.cfg.warm_iters = int(prm.get("warm_iters", 0))
        self.cfg.coarsen_target = int(prm.get("coarsen_target", 0))
        self.cfg.partition = int(prm.get("partition", 0))   # world > 1: 0 subtrees / ranges, 1 interleaved
        h = _P()
        st = lib.lmc_create(C.byref(self.gb), C.byref(self.vp), C.byref(self.tr), C.byref(self.sc),
                            C.byref(self.cfg), C.byref(h))
        if st != LMC_OK:
            raise LmcError(f"lmc_create failed: {lib.lmc_status_str(st).decode()}")
        self.h = h

    # -- lifecycle ---------------------------------------------------------------------------
    def close(self):
        if getattr(self, "h", None):
            lib.lmc_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _ck(self, st, what):
        if st != LMC_OK:
            msg = lib.lmc_last_error(self.h).decode(errors="replace")
            raise LmcError(f"{what}: {lib.lmc_status_str(st).decode()}: {msg}")

    # -- the seven calls -------------------------------------------------------------------------
    def upload_inputs(self, inputs=None):
        """re-upload the per-frame inputs (G-buffer, VPLs) -- of `inputs` (same sizes) if given; the light
        tree and global cut stay those of lmc_create"""
        if inputs is not None:
            g, v = inputs.gbuf, inputs.vpls
            arr = self.arr
            self.gb = Gbuffer(inputs.width, inputs.height, g["px"].shape[0], arr(g["pixel"], np.int32),
                              *[arr(g[k], np.float32) for k in ("px", "py", "pz", "nx", "ny", "nz", "vx", "vy", "vz",
                                                                "rho_r", "rho_g", "rho_b", "spec")],
                              arr(g["exponent"], np.int32))
            self.vp = Vpls(v["px"].shape[0], *[arr(v[k], np.float32) for k in ("px", "py", "pz", "nx", "ny", "nz",
                                                                               "ir", "ig", "ib")])
        self._ck(lib.lmc_upload_inputs(self.h, C.byref(self.gb), C.byref(self.vp), C.byref(self.tr)), "upload_inputs")

    def build_slices(self):
        self._ck(lib.lmc_build_slices(self.h), "build_slices")

    def sample_pass1(self):
        self._ck(lib.lmc_sample_pass1(self.h), "sample_pass1")

    def coarsen_cut(self):
        self._ck(lib.lmc_coarsen_cut(self.h), "coarsen_cut")

    def sample_pass2(self):
        self._ck(lib.lmc_sample_pass2(self.h), "sample_pass2")

    def complete(self):
        self._ck(lib.lmc_complete(self.h), "complete")

    def resolve_image(self, image, memory=MEM_DEVICE):
        self._ck(lib.lmc_resolve_image(self.h, _ptr(image), memory), "resolve_image")

    def resolve_rows(self, tile):
        """this rank's rows packed as (r, g, b, pixel bits) float32 x 4 into a device tensor"""
        self._ck(lib.lmc_resolve_rows(self.h, _ptr(tile)), "resolve_rows")

    def scatter_rows(self, tiles, image):
        """packed rows (n x 4 float32, any order) into a device image"""
        n = tiles.numel() // 4
        self._ck(lib.lmc_scatter_rows(self.h, _ptr(tiles), n, _ptr(image)), "scatter_rows")

    def partition(self):
        """(slice_first, row_first): every rank's first slice / slice-ordered row, world + 1 entries"""
        w = int(self.cfg.world)
        s = np.zeros(w + 1, np.int32)
        r = np.zeros(w + 1, np.int64)
        self._ck(lib.lmc_get_partition(self.h, _ptr(s), _ptr(r)), "get_partition")
        return s, r

    def run(self, image, memory=MEM_DEVICE):
        self.build_slices()
        self.sample_pass1()
        self.coarsen_cut()
        self.sample_pass2()
        self.complete()
        self.resolve_image(image, memory)

    def set_timing(self, on=True):
        self._ck(lib.lmc_set_timing(self.h, 1 if on else 0), "set_timing")

    # -- getters ------------------------------------------------------------------------------
    def slices(self):
        ns = np.zeros(1, np.int64)
        self._ck(lib.lmc_get_slices(self.h, None, None, _ptr(ns)), "get_slices")
        off = np.zeros(int(ns[0]) + 1, np.int32)
        rows = np.zeros(max(int(self.gb.count), 1), np.int32)
        self._ck(lib.lmc_get_slices(self.h, _ptr(off), _ptr(rows), _ptr(ns)), "get_slices")
        return off, rows[: int(self.gb.count)]

    def pass1(self, s):
        nb = np.zeros(1, np.int32)
        nm = np.zeros(1, np.int32)
        self._ck(lib.lmc_get_pass1(self.h, s, None, None, None, None, None, _ptr(nb), _ptr(nm)), "get_pass1")
        B, K = int(nb[0]), int(nm[0])
        node = np.zeros(max(B, 1), np.int32)
        cnt = np.zeros(max(B, 1), np.int32)
        rows = np.zeros(max(B * K, 1), np.int32)
        Ta = np.zeros(max(B * K, 1))
        Tb = np.zeros(max(B * K, 1))
        self._ck(lib.lmc_get_pass1(self.h, s, _ptr(node), _ptr(cnt), _ptr(rows), _ptr(Ta), _ptr(Tb), _ptr(nb),
                                   _ptr(nm)), "get_pass1")
        return dict(node=node[:B], count=cnt[:B], rows=rows[:B * K].reshape(B, K), Ta=Ta[:B * K].reshape(B, K),
                    Tb=Tb[:B * K].reshape(B, K))

    def coarsen(self, s):
        nn = np.zeros(1, np.int32)
        self._ck(lib.lmc_get_coarsen(self.h, s, None, None, None, None, None, _ptr(nn)), "get_coarsen")
        U = int(nn[0])
        node, proc, merged = (np.zeros(U, np.int32) for _ in range(3))
        eps, cost = np.zeros(U), np.zeros(U)
        self._ck(lib.lmc_get_coarsen(self.h, s, _ptr(node), _ptr(proc), _ptr(merged), _ptr(eps), _ptr(cost),
                                     _ptr(nn)), "get_coarsen")
        return dict(node=node, processed=proc, merged=merged, eps=eps, cost=cost)

    def cut(self, s):
        n = np.zeros(1, np.int32)
        self._ck(lib.lmc_get_cut(self.h, s, None, _ptr(n)), "get_cut")
        nodes = np.zeros(max(int(n[0]), 1), np.int32)
        self._ck(lib.lmc_get_cut(self.h, s, _ptr(nodes), _ptr(n)), "get_cut")
        return nodes[: int(n[0])]

    def samples(self, s):
        n = np.zeros(1, np.int64)
        tn = np.zeros(1, np.int64)
        self._ck(lib.lmc_get_samples(self.h, s, None, None, None, None, _ptr(n), _ptr(tn)), "get_samples")
        k = int(n[0])
        row, col, car = (np.zeros(max(k, 1), np.int32) for _ in range(3))
        val = np.zeros(max(k, 1), np.float32)
        self._ck(lib.lmc_get_samples(self.h, s, _ptr(row), _ptr(col), _ptr(val), _ptr(car), _ptr(n), _ptr(tn)),
                 "get_samples")
        return dict(row=row[:k], col=col[:k], val=val[:k], carried=car[:k], nnz=k, target_N=int(tn[0]))

    def factors(self, s):
        m, n, q, fl, it = (np.zeros(1, np.int32) for _ in range(5))
        res = np.zeros(1, np.float32)
        self._ck(lib.lmc_get_factors(self.h, s, None, None, _ptr(m), _ptr(n), _ptr(q), _ptr(fl), _ptr(it),
                                     _ptr(res)), "get_factors")
        U = np.zeros((int(m[0]), int(q[0])), np.float32)
        V = np.zeros((int(q[0]), int(n[0])), np.float32)
        self._ck(lib.lmc_get_factors(self.h, s, _ptr(U), _ptr(V), _ptr(m), _ptr(n), _ptr(q), _ptr(fl), _ptr(it),
                                     _ptr(res)), "get_factors")
        return dict(U=U, V=V, flags=int(fl[0]), iters=int(it[0]), resid=float(res[0]))

    def stats(self):
        st = Stats()
        self._ck(lib.lmc_get_stats(self.h, C.byref(st)), "get_stats")
        return st.as_dict()

    def eval_entries(self, rows, vpls):
        rows = np.ascontiguousarray(rows, np.int32)
        vpls = np.ascontiguousarray(vpls, np.int32)
        out = np.zeros(rows.size)
        self._ck(lib.lmc_eval_entries(self.h, rows.size, _ptr(rows), _ptr(vpls), _ptr(out)), "eval_entries")
        return out


def nccl_unique_id() -> bytes:
    """128-byte ncclUniqueId for Frame(nccl_id=...) (rank 0 creates it, the caller broadcasts it)"""
    buf = (C.c_uint8 * 128)()
    st = lib.lmc_nccl_unique_id(C.cast(buf, _P))
    if st != LMC_OK:
        raise LmcError(f"lmc_nccl_unique_id: {lib.lmc_status_str(st).decode()}")
    return bytes(buf)


def plan_partition(rows: int, slice_target: int, world: int):
    """(slice_first, row_first, n_slices) of the ranks' shares -- host planning only, no GPU needed"""
    s = np.zeros(world + 1, np.int32)
    r = np.zeros(world + 1, np.int64)
    n = np.zeros(1, np.int64)
    st = lib.lmc_plan_partition(rows, slice_target, world, _ptr(s), _ptr(r), _ptr(n))
    if st != LMC_OK:
        raise LmcError(f"lmc_plan_partition: {lib.lmc_status_str(st).decode()}")
    return s, r, int(n[0])


def plan_bvh(tri):
    """the triangle BVH lmc_create builds (host only, no GPU): (nodes (N, 8) float32 with int32
    first / count in columns 3 / 7, reordered triangles (n, 12), order (n,))"""
    tri = np.ascontiguousarray(tri, np.float32).reshape(-1, 9)
    n = tri.shape[0]
    nodes = np.zeros((max(2 * n - 1, 1), 8), np.float32)
    tris = np.zeros((n, 12), np.float32)
    order = np.zeros(n, np.int32)
    nn = np.zeros(1, np.int32)
    st = lib.lmc_plan_bvh(_ptr(tri), n, _ptr(nodes), _ptr(nn), _ptr(tris), _ptr(order))
    if st != LMC_OK:
        raise LmcError(f"lmc_plan_bvh: {lib.lmc_status_str(st).decode()}")
    return nodes[:int(nn[0])], tris, order


def build_light_tree(vpls, cut_max: int, device="cuda"):
    """Step 1 on the GPU (lmc_build_light_tree): light tree + global cut of the VPL SoA arrays, returned
    as numpy arrays (dict like scenegen's tree)"""
    import torch
    t = {k: torch.from_numpy(np.ascontiguousarray(vpls[k], np.float32)).to(device)
         for k in ("px", "py", "pz", "nx", "ny", "nz", "ir", "ig", "ib")}
    nv = t["px"].numel()
    nn = 2 * nv - 1
    out = {k: torch.zeros(nn, dtype=torch.int32, device=device) for k in ("left", "right", "rep")}
    out.update({k: torch.zeros(nn, dtype=torch.float32, device=device) for k in ("ir", "ig", "ib")})
    cut = torch.zeros(max(cut_max, 1), dtype=torch.int32, device=device)
    v = Vpls(nv, *[_P(t[k].data_ptr()) for k in ("px", "py", "pz", "nx", "ny", "nz", "ir", "ig", "ib")])
    n = np.zeros(1, np.int64)
    st = lib.lmc_build_light_tree(C.byref(v), cut_max, MEM_DEVICE, _P(torch.cuda.current_stream().cuda_stream),
                                  *[_P(out[k].data_ptr()) for k in ("left", "right", "rep", "ir", "ig", "ib")],
                                  _P(cut.data_ptr()), _ptr(n))
    if st != LMC_OK:
        raise LmcError(f"lmc_build_light_tree: {lib.lmc_status_str(st).decode()}")
    res = {k: a.cpu().numpy() for k, a in out.items()}
    res["global_cut"] = cut[: int(n[0])].cpu().numpy()
    res["root"] = 0
    return res
