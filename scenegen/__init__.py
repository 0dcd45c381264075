"""Seeded synthetic inputs for the lighting-matrix hot path (shared by tests, oracle harness, bench).

This module produces the *inputs* of the method — an analytic procedural scene, a G-buffer
(one surface point per pixel, "m surface points each of which corresponds to a
pixel"), a VPL set from instant radiosity, a binary light tree with node
intensities I_f = I_a + I_b and a global cut 𝔤 of it.
It holds none of the method's arithmetic: no lighting-matrix entry, no slicing, no
sampling, no coarsening, no completion.  Both the CUDA path (through the C-ABI) and the
oracle consume exactly the float32/int32 arrays built here.

Recipe (DESIGN.md §"Input recipe"):
  * C1/C2 "cornell": closed unit box, red/green side walls, ceiling area light, two AABB
    occluders, camera inside (every pixel hits), diffuse.
  * C3/C4/C5 "interior": room [0,4]x[0,3]x[0,6] with 16 spheres, 8 AABBs, 8 rectangles,
    24 ceiling area lights (cf. Tearoom's 24 area lights), glossy materials
    s in {0,0.25,0.5}, e in {8,32,64}.
  * VPLs: emitter samples + 3 cosine bounces (4 VPLs per light path), closest-hit tracing.
  * Light tree: median split on the longest bbox axis, node ids in BFS order,
    rep(f) = rep of the brighter child (so rep(f) in {rep(l), rep(r)}).
  * Global cut: greedy split of the node with the largest lum(I)·bbox-diagonal bound until
    |𝔤| = cut_max ("about 800~900 nodes"; we use 1024, 256 for C1).
"""
from __future__ import annotations

import dataclasses
import heapq
import math

import numpy as np

__all__ = ["Config", "PRESETS", "Inputs", "make_inputs", "preset"]


@dataclasses.dataclass
class Config:
    name: str
    scene: str            # "cornell" | "interior" | "mesh" (interior + triangle meshes)
    width: int
    height: int
    n_vpls: int
    cut_max: int
    slice_target: int
    rank_q: int
    rate: float
    tau: float            # coarsening error bound in lighting-matrix units, calibrated (R11)
    solver: int = 0       # 0 = ADM (paper, App. A), 1 = MALS (north_star)
    max_iter: int = 100   # PAPER.md:149 "We set the maximum iteration as 100"
    tol: float = 0.0
    alpha: float = 1.0
    beta: float = 1.0
    gamma: float = 1.6    # PAPER.md:277 gamma in (0, 1.618)
    lam: float = 1e-2     # MALS ridge on max-normalised data (R34)
    normal_weight: float = 0.3
    seed: int = 12567
    p1_nmax: int = 32
    p1_nmin: int = 4
    fixture_seed: int = 1
    # SURVEY §8(f3) variants (0 = the paper's method): rows drawn by image-space importance f(i)
    # (R36), Eq. (1) sensitivity cost(L_f) = eps + cost(L_b) + cost(L_a), Z-mode image (A24)
    row_importance: int = 0
    cost_mode: int = 0
    resolve_mode: int = 0
    # warm start of the completion from the previous frame's factors
    warm_start: int = 0
    warm_iters: int = 0
    # count-target coarsening, 0 = threshold rule
    coarsen_target: int = 0
    # tessellation level of the triangle meshes of the "mesh" scene
    mesh_level: int = 0


PRESETS = {
    "c1": Config("c1", "cornell", 64, 64, 4096, 256, 256, 8, 0.10, 1.0e-4),
    "c2": Config("c2", "cornell", 512, 512, 100_000, 1024, 800, 16, 0.10, 3.0e-6),
    "c3": Config("c3", "interior", 1024, 1024, 300_000, 1024, 800, 16, 0.10, 3.0e-6),
    "c4": Config("c4", "interior", 1920, 1080, 1_000_000, 1024, 1024, 16, 0.10, 3.0e-6),
    # small variants used by parity tests (a few slices, ragged sizes)
    "t_cornell": Config("t_cornell", "cornell", 40, 37, 2048, 128, 200, 8, 0.10, 1.0e-4),
    "t_interior": Config("t_interior", "interior", 48, 40, 4096, 256, 256, 8, 0.15, 1.0e-3),
    # the interior plus three triangle meshes (416 / 6656 triangles)
    "t_mesh": Config("t_mesh", "mesh", 48, 40, 4096, 256, 256, 8, 0.15, 1.0e-3, mesh_level=1),
    "c_mesh": Config("c_mesh", "mesh", 512, 512, 100_000, 1024, 800, 16, 0.10, 3.0e-6, mesh_level=3),
}


def preset(name: str, **over) -> Config:
    if name.startswith("c5"):
        # c5_q{4,8,16,32}_r{5,10,20}: the C3 shape with rank/rate swept (BASELINE.json configs[4])
        parts = name.split("_")
        q = int(parts[1][1:])
        r = int(parts[2][1:]) / 100.0
        base = dataclasses.replace(PRESETS["c3"], name=name, rank_q=q, rate=r)
        return dataclasses.replace(base, **over)
    return dataclasses.replace(PRESETS[name], **over)


# ----------------------------------------------------------------------------------------
# Scene description (analytic primitives)
# ----------------------------------------------------------------------------------------

@dataclasses.dataclass
class Scene:
    lo: np.ndarray            # room box (walls are its inner faces)
    hi: np.ndarray
    wall_mat: list            # 6 material ids: -x, +x, -y (floor), +y (ceiling), -z, +z
    spheres: np.ndarray       # (ns, 4) cx, cy, cz, r
    sph_mat: list
    boxes: np.ndarray         # (nb, 6) lo3, hi3
    box_mat: list
    rects: np.ndarray         # (nr, 12) p0, e1, e2, nrm
    rect_mat: list
    materials: np.ndarray     # (nm, 5) rho_r, rho_g, rho_b, spec s, exponent e
    lights: np.ndarray        # (nl, 4) ceiling patches x0, x1, z0, z1 (at y = hi.y)
    light_power: np.ndarray   # (3,) total RGB power
    cam_pos: np.ndarray
    cam_look: np.ndarray
    vfov_deg: float
    tris: np.ndarray = dataclasses.field(default_factory=lambda: np.zeros((0, 9)))  # (nt, 9) v0, v1, v2
    tri_mat: np.ndarray = dataclasses.field(default_factory=lambda: np.zeros(0, np.int64))

    @property
    def diag(self) -> float:
        d = self.hi - self.lo
        return float(math.sqrt(float(d[0] * d[0] + d[1] * d[1] + d[2] * d[2])))


def _rect(p0, e1, e2):
    p0 = np.asarray(p0, np.float64)
    e1 = np.asarray(e1, np.float64)
    e2 = np.asarray(e2, np.float64)
    n = np.cross(e1, e2)
    return np.concatenate([p0, e1, e2, n])


def _cornell() -> Scene:
    mats = np.array([
        [0.725, 0.71, 0.68, 0.0, 1],   # 0 white
        [0.63, 0.065, 0.05, 0.0, 1],   # 1 red
        [0.14, 0.45, 0.091, 0.0, 1],   # 2 green
    ], np.float64)
    boxes = np.array([
        [0.13, 0.0, 0.37, 0.43, 0.30, 0.67],
        [0.53, 0.0, 0.20, 0.83, 0.60, 0.50],
    ], np.float64)
    return Scene(
        lo=np.zeros(3), hi=np.ones(3), wall_mat=[1, 2, 0, 0, 0, 0],
        spheres=np.zeros((0, 4)), sph_mat=[], boxes=boxes, box_mat=[0, 0],
        rects=np.zeros((0, 12)), rect_mat=[], materials=mats,
        lights=np.array([[0.4, 0.6, 0.4, 0.6]]), light_power=np.array([2.4, 2.0, 1.5]),
        cam_pos=np.array([0.5, 0.5, 0.02]), cam_look=np.array([0.5, 0.5, 1.0]), vfov_deg=70.0)


def _interior(seed: int = 3) -> Scene:
    rng = np.random.default_rng(seed)
    lo = np.array([0.0, 0.0, 0.0])
    hi = np.array([4.0, 3.0, 6.0])
    spec_choices = [0.0, 0.25, 0.5]
    exp_choices = [8, 32, 64]
    mats = [
        [0.75, 0.74, 0.72, 0.0, 1],   # 0 ceiling, white diffuse
        [0.55, 0.45, 0.35, 0.25, 32],  # 1 glossy wood floor
        [0.70, 0.62, 0.55, 0.0, 1],   # 2 warm wall
        [0.45, 0.55, 0.70, 0.0, 1],   # 3 blue wall
        [0.65, 0.65, 0.60, 0.25, 8],  # 4 back wall, slightly glossy
    ]
    nbase = len(mats)
    for _ in range(12):
        c = rng.uniform(0.15, 0.85, 3)
        mats.append([c[0], c[1], c[2], spec_choices[rng.integers(0, 3)], exp_choices[rng.integers(0, 3)]])
    mats = np.array(mats, np.float64)

    def rmat():
        return int(nbase + rng.integers(0, 12))

    cam = np.array([2.0, 1.6, 0.35])
    spheres, sph_mat = [], []
    while len(spheres) < 16:
        r = rng.uniform(0.1, 0.4)
        c = np.array([rng.uniform(0.2 + r, 3.8 - r), rng.uniform(r, 2.4 - r), rng.uniform(1.2 + r, 5.8 - r)])
        if np.linalg.norm(c - cam) < r + 0.5:
            continue
        if any(np.linalg.norm(c - s[:3]) < r + s[3] + 0.05 for s in spheres):
            continue
        spheres.append(np.r_[c, r])
        sph_mat.append(rmat())
    boxes, box_mat = [], []
    for k in range(4):   # tables: thin slabs
        x0 = rng.uniform(0.3, 2.7)
        z0 = rng.uniform(1.5, 5.0)
        y0 = rng.uniform(0.7, 0.9)
        boxes.append([x0, y0, z0, x0 + rng.uniform(0.6, 1.0), y0 + 0.05, z0 + rng.uniform(0.4, 0.7)])
        box_mat.append(rmat())
    for k in range(4):   # pillars
        x0 = rng.uniform(0.3, 3.4)
        z0 = rng.uniform(1.5, 5.5)
        boxes.append([x0, 0.0, z0, x0 + 0.3, rng.uniform(1.5, 2.4), z0 + 0.3])
        box_mat.append(rmat())
    rects, rect_mat = [], []
    for k in range(4):   # vertical partition panels
        x0 = rng.uniform(0.3, 3.0)
        z0 = rng.uniform(2.0, 5.5)
        w = rng.uniform(0.5, 1.0)
        h = rng.uniform(0.8, 1.8)
        rects.append(_rect([x0, 0.1, z0], [w, 0.0, rng.uniform(-0.3, 0.3)], [0.0, h, 0.0]))
        rect_mat.append(rmat())
    for k in range(4):   # horizontal shelves
        x0 = rng.uniform(0.2, 3.0)
        z0 = rng.uniform(1.5, 5.0)
        y = rng.uniform(1.2, 2.3)
        rects.append(_rect([x0, y, z0], [rng.uniform(0.5, 0.9), 0.0, 0.0], [0.0, 0.0, rng.uniform(0.3, 0.6)]))
        rect_mat.append(rmat())
    lights = []
    for ix in range(4):
        for iz in range(6):
            cx = 0.5 + ix * 1.0
            cz = 0.5 + iz * 1.0
            lights.append([cx - 0.15, cx + 0.15, cz - 0.15, cz + 0.15])
    return Scene(lo=lo, hi=hi, wall_mat=[2, 3, 1, 0, 2, 4],
                 spheres=np.array(spheres), sph_mat=sph_mat, boxes=np.array(boxes), box_mat=box_mat,
                 rects=np.array(rects), rect_mat=rect_mat, materials=mats,
                 lights=np.array(lights), light_power=np.array([60.0, 55.0, 48.0]),
                 cam_pos=cam, cam_look=np.array([2.0, 1.25, 6.0]), vfov_deg=62.0)


def _icosphere(level: int):
    """Unit icosphere: the icosahedron with every face split in 4, `level` times (20 * 4^level faces)."""
    t = (1.0 + math.sqrt(5.0)) / 2.0
    V = [[-1, t, 0], [1, t, 0], [-1, -t, 0], [1, -t, 0], [0, -1, t], [0, 1, t], [0, -1, -t], [0, 1, -t],
         [t, 0, -1], [t, 0, 1], [-t, 0, -1], [-t, 0, 1]]
    V = [list(np.array(v, np.float64) / math.sqrt(1.0 + t * t)) for v in V]
    F = [[0, 11, 5], [0, 5, 1], [0, 1, 7], [0, 7, 10], [0, 10, 11], [1, 5, 9], [5, 11, 4], [11, 10, 2],
         [10, 7, 6], [7, 1, 8], [3, 9, 4], [3, 4, 2], [3, 2, 6], [3, 6, 8], [3, 8, 9], [4, 9, 5], [2, 4, 11],
         [6, 2, 10], [8, 6, 7], [9, 8, 1]]
    for _ in range(level):
        mid = {}

        def m(a, b):
            k = (min(a, b), max(a, b))
            if k not in mid:
                p = np.array(V[a]) + np.array(V[b])
                V.append(list(p / np.linalg.norm(p)))
                mid[k] = len(V) - 1
            return mid[k]

        F2 = []
        for a, b, c in F:
            ab, bc, ca = m(a, b), m(b, c), m(c, a)
            F2 += [[a, ab, ca], [b, bc, ab], [c, ca, bc], [ab, bc, ca]]
        F = F2
    V = np.array(V)
    F = np.array(F)
    return np.concatenate([V[F[:, 0]], V[F[:, 1]], V[F[:, 2]]], 1)


def _torus(R: float, r: float, nu: int, nv: int):
    """Torus around the y axis, nu x nv quads, each split in two triangles."""
    u = np.arange(nu) * (2.0 * math.pi / nu)
    v = np.arange(nv) * (2.0 * math.pi / nv)

    def P(i, j):
        a, b = u[i % nu], v[j % nv]
        return np.array([(R + r * math.cos(b)) * math.cos(a), r * math.sin(b), (R + r * math.cos(b)) * math.sin(a)])

    T = []
    for i in range(nu):
        for j in range(nv):
            p00, p10, p01, p11 = P(i, j), P(i + 1, j), P(i, j + 1), P(i + 1, j + 1)
            T.append(np.r_[p00, p10, p11])
            T.append(np.r_[p00, p11, p01])
    return np.array(T)


def _mesh_scene(level: int) -> Scene:
    """The interior with three triangle meshes (DESIGN.md input recipe): an
    icosphere, a tilted torus and a bumpy icosphere (radius modulated by a smooth function of the
    vertex direction), 416 triangles at level 1, 6656 at level 3."""
    sc = _interior()
    tris, mats = [], []
    ico = _icosphere(level) * 0.42 + np.tile([1.0, 0.55, 3.2], 3)
    tris.append(ico)
    mats.append(np.full(ico.shape[0], 5 + 1))
    tor = _torus(0.42, 0.14, 8 << level, 4 << level)
    ca, sa = math.cos(0.6), math.sin(0.6)
    rot = np.array([[1.0, 0.0, 0.0], [0.0, ca, -sa], [0.0, sa, ca]])
    tor = np.concatenate([tor[:, 3 * k:3 * k + 3] @ rot.T + np.array([2.9, 1.3, 3.9]) for k in range(3)], 1)
    tris.append(tor)
    mats.append(np.full(tor.shape[0], 5 + 7))
    bump = _icosphere(level)
    for k in range(3):
        d = bump[:, 3 * k:3 * k + 3]
        rad = 0.34 * (1.0 + 0.15 * np.sin(5.0 * d[:, 0]) * np.cos(4.0 * d[:, 1] + 3.0 * d[:, 2]))
        bump[:, 3 * k:3 * k + 3] = d * rad[:, None] + np.array([2.1, 1.9, 4.9])
    tris.append(bump)
    mats.append(np.full(bump.shape[0], 5 + 3))
    # the arrays handed to both sides are float32: cast the vertices so the fixture rays see them too
    sc.tris = np.concatenate(tris).astype(np.float32).astype(np.float64)
    sc.tri_mat = np.concatenate(mats).astype(np.int64)
    return sc


# ----------------------------------------------------------------------------------------
# Closest-hit ray casting (fixture-only: camera rays and light paths; never a shadow test)
# ----------------------------------------------------------------------------------------

def _closest_hit(sc: Scene, O: np.ndarray, D: np.ndarray, tmin: float):
    """Vectorised closest hit of rays O + t D (t > tmin) against walls and occluders.

    Returns t, normal (facing the incoming ray), material id.
    """
    n = O.shape[0]
    best_t = np.full(n, np.inf)
    best_n = np.zeros((n, 3))
    best_m = np.full(n, -1, np.int64)

    def take(t, nrm, mat):
        better = (t > tmin) & (t < best_t)
        if not np.any(better):
            return
        best_t[better] = t[better]
        if nrm.ndim == 1:
            best_n[better] = nrm
        else:
            best_n[better] = nrm[better]
        if np.ndim(mat) == 0:
            best_m[better] = mat
        else:
            best_m[better] = mat[better]

    with np.errstate(divide="ignore", invalid="ignore"):
        # walls: inner faces of the room box
        for axis in range(3):
            for side, plane in ((0, sc.lo[axis]), (1, sc.hi[axis])):
                t = (plane - O[:, axis]) / D[:, axis]
                nrm = np.zeros(3)
                nrm[axis] = 1.0 if side == 0 else -1.0
                take(np.where(np.isfinite(t), t, np.inf), nrm, sc.wall_mat[2 * axis + side])
        for k in range(sc.spheres.shape[0]):
            c = sc.spheres[k, :3]
            r = sc.spheres[k, 3]
            oc = O - c
            b = np.einsum("ij,ij->i", oc, D)
            cc = np.einsum("ij,ij->i", oc, oc) - r * r
            disc = b * b - cc
            sq = np.sqrt(np.maximum(disc, 0.0))
            t0 = -b - sq
            t1 = -b + sq
            t = np.where(t0 > tmin, t0, t1)
            t = np.where(disc >= 0, t, np.inf)
            P = O + t[:, None] * D
            nrm = (P - c) / r
            take(t, nrm, sc.sph_mat[k])
        for k in range(sc.boxes.shape[0]):
            lo = sc.boxes[k, :3]
            hi = sc.boxes[k, 3:]
            inv = 1.0 / D
            t1 = (lo - O) * inv
            t2 = (hi - O) * inv
            tn = np.nanmax(np.minimum(t1, t2), axis=1)
            tf = np.nanmin(np.maximum(t1, t2), axis=1)
            hit = (tn <= tf) & (tn > tmin)
            t = np.where(hit, tn, np.inf)
            ax = np.argmax(np.minimum(t1, t2), axis=1)
            nrm = np.zeros((n, 3))
            nrm[np.arange(n), ax] = -np.sign(D[np.arange(n), ax])
            take(t, nrm, sc.box_mat[k])
        for k in range(sc.rects.shape[0]):
            p0 = sc.rects[k, 0:3]
            e1 = sc.rects[k, 3:6]
            e2 = sc.rects[k, 6:9]
            nr = sc.rects[k, 9:12]
            den = D @ nr
            t = ((p0 - O) @ nr) / den
            P = O + t[:, None] * D
            hp = P - p0
            a = (hp @ e1) / (e1 @ e1)
            b = (hp @ e2) / (e2 @ e2)
            ok = (den != 0) & (a >= 0) & (a <= 1) & (b >= 0) & (b <= 1)
            t = np.where(ok, t, np.inf)
            nn = nr / np.linalg.norm(nr)
            nrm = np.where((den < 0)[:, None], nn[None, :], -nn[None, :])
            take(t, nrm, sc.rect_mat[k])
        if sc.tris.shape[0]:
            _hit_tris(sc, O, D, tmin, take)
    nl = np.linalg.norm(best_n, axis=1, keepdims=True)
    best_n = best_n / np.where(nl > 0, nl, 1.0)
    return best_t, best_n, best_m


def _hit_tris(sc: Scene, O, D, tmin, take):
    """Closest triangle hits (Moller-Trumbore) by clusters of 64 consecutive triangles (spatially
    coherent by construction): rays that miss a cluster's bounding sphere skip it."""
    T = sc.tris
    nt = T.shape[0]
    n = O.shape[0]
    for c0 in range(0, nt, 64):
        Tm = T[c0:c0 + 64]
        mat = sc.tri_mat[c0:c0 + 64]
        V = Tm.reshape(-1, 3)
        c = V.mean(0)
        rad = np.sqrt(((V - c) ** 2).sum(1).max()) * 1.001
        oc = O - c
        b = np.einsum("ij,ij->i", oc, D)
        cc = np.einsum("ij,ij->i", oc, oc) - rad * rad
        idx = np.nonzero((b * b - cc >= 0) & (-b + np.sqrt(np.maximum(b * b - cc, 0.0)) > tmin))[0]
        if idx.size == 0:
            continue
        v0, e1, e2 = Tm[:, 0:3], Tm[:, 3:6] - Tm[:, 0:3], Tm[:, 6:9] - Tm[:, 0:3]
        fn = np.cross(e1, e2)
        fn /= np.linalg.norm(fn, axis=1, keepdims=True)
        o = O[idx][:, None, :]
        d = D[idx][:, None, :]
        p = np.cross(d, e2[None])
        det = (e1[None] * p).sum(2)
        inv = 1.0 / np.where(det == 0, 1.0, det)
        sv = o - v0[None]
        u = (sv * p).sum(2) * inv
        qv = np.cross(sv, e1[None])
        v = (d * qv).sum(2) * inv
        t = (e2[None] * qv).sum(2) * inv
        ok = (det != 0) & (u >= 0) & (u <= 1) & (v >= 0) & (u + v <= 1) & (t > tmin)
        t = np.where(ok, t, np.inf)
        j = np.argmin(t, 1)
        tb = t[np.arange(idx.size), j]
        nrm = fn[j]
        nrm = np.where(((nrm * D[idx]).sum(1) > 0)[:, None], -nrm, nrm)
        tt = np.full(n, np.inf)
        tt[idx] = tb
        nn = np.zeros((n, 3))
        nn[idx] = nrm
        mm = np.full(n, -1, np.int64)
        mm[idx] = mat[j]
        take(tt, nn, mm)


def _cosine_dirs(nrm: np.ndarray, u1: np.ndarray, u2: np.ndarray) -> np.ndarray:
    r = np.sqrt(u1)
    phi = 2.0 * np.pi * u2
    lx = r * np.cos(phi)
    lz = r * np.sin(phi)
    ly = np.sqrt(np.maximum(0.0, 1.0 - u1))
    # orthonormal basis around nrm
    a = np.where(np.abs(nrm[:, :1]) > 0.9, np.array([[0.0, 1.0, 0.0]]), np.array([[1.0, 0.0, 0.0]]))
    t = np.cross(a, nrm)
    t /= np.linalg.norm(t, axis=1, keepdims=True)
    b = np.cross(nrm, t)
    d = lx[:, None] * t + ly[:, None] * nrm + lz[:, None] * b
    return d / np.linalg.norm(d, axis=1, keepdims=True)


# ----------------------------------------------------------------------------------------
# Inputs
# ----------------------------------------------------------------------------------------

@dataclasses.dataclass
class Inputs:
    cfg: Config
    scene: Scene
    width: int
    height: int
    gbuf: dict          # SoA float32 arrays + "pixel" int32 + "exponent" int32
    vpls: dict          # SoA float32 arrays
    tree: dict          # left/right/rep int32, ir/ig/ib float32, global_cut int32, root int
    prims: dict         # analytic occluders for visibility: sph (ns,4) box (nb,6) rect (nr,12), float32
    diag: float
    clamp_dist: float
    shadow_eps: float
    tau: float

    @property
    def m(self) -> int:
        return int(self.gbuf["px"].shape[0])

    def params(self) -> dict:
        c = self.cfg
        return dict(slice_target=c.slice_target, normal_weight=c.normal_weight, seed=c.seed,
                    p1_nmax=c.p1_nmax, p1_nmin=c.p1_nmin, tau=self.tau, rate=c.rate, rank_q=c.rank_q,
                    solver=c.solver, max_iter=c.max_iter, tol=c.tol, alpha=c.alpha, beta=c.beta,
                    gamma=c.gamma, lam=c.lam, row_importance=c.row_importance, cost_mode=c.cost_mode,
                    resolve_mode=c.resolve_mode, warm_start=c.warm_start, warm_iters=c.warm_iters,
                    coarsen_target=c.coarsen_target)


def _gbuffer(sc: Scene, W: int, H: int):
    fwd = sc.cam_look - sc.cam_pos
    fwd /= np.linalg.norm(fwd)
    right = np.cross(fwd, np.array([0.0, 1.0, 0.0]))
    right /= np.linalg.norm(right)
    up = np.cross(right, fwd)
    th = math.tan(math.radians(sc.vfov_deg) * 0.5)
    aspect = W / H
    py, px = np.mgrid[0:H, 0:W]
    sx = ((px.ravel() + 0.5) / W * 2.0 - 1.0) * th * aspect
    sy = (1.0 - (py.ravel() + 0.5) / H * 2.0) * th
    D = fwd[None, :] + sx[:, None] * right[None, :] + sy[:, None] * up[None, :]
    D /= np.linalg.norm(D, axis=1, keepdims=True)
    O = np.broadcast_to(sc.cam_pos, D.shape).copy()
    t, nrm, mat = _closest_hit(sc, O, D, 1e-6)
    hit = np.isfinite(t) & (mat >= 0)
    pix = np.nonzero(hit)[0].astype(np.int32)
    P = O[hit] + t[hit, None] * D[hit]
    N = nrm[hit]
    V = -D[hit]
    M = sc.materials[mat[hit]]
    f32 = np.float32
    g = dict(pixel=pix,
             px=P[:, 0].astype(f32), py=P[:, 1].astype(f32), pz=P[:, 2].astype(f32),
             nx=N[:, 0].astype(f32), ny=N[:, 1].astype(f32), nz=N[:, 2].astype(f32),
             vx=V[:, 0].astype(f32), vy=V[:, 1].astype(f32), vz=V[:, 2].astype(f32),
             rho_r=M[:, 0].astype(f32), rho_g=M[:, 1].astype(f32), rho_b=M[:, 2].astype(f32),
             spec=M[:, 3].astype(f32), exponent=M[:, 4].astype(np.int32))
    return g


def _vpls(sc: Scene, n_vpls: int, rng: np.random.Generator):
    bounces = 3
    per_path = bounces + 1
    n_paths = (n_vpls + per_path - 1) // per_path
    L = sc.lights
    li = rng.integers(0, L.shape[0], n_paths)
    u = rng.uniform(size=(n_paths, 2))
    P = np.stack([L[li, 0] + u[:, 0] * (L[li, 1] - L[li, 0]),
                  np.full(n_paths, sc.hi[1]),
                  L[li, 2] + u[:, 1] * (L[li, 3] - L[li, 2])], axis=1)
    N = np.tile(np.array([0.0, -1.0, 0.0]), (n_paths, 1))
    # VPL intensity: power / (pi * paths) so that sum_v I_v cos/d^2 has the radiometric scale
    I = np.tile(sc.light_power / (math.pi * n_paths), (n_paths, 1))
    pos, nrm, inten = [P], [N], [I]
    for b in range(bounces):
        d = _cosine_dirs(N, rng.uniform(size=n_paths), rng.uniform(size=n_paths))
        t, nh, mat = _closest_hit(sc, P + 1e-6 * N, d, 1e-6)
        ok = np.isfinite(t)
        t = np.where(ok, t, 0.0)
        P = P + t[:, None] * d
        N = np.where(ok[:, None], nh, N)
        rho = sc.materials[np.maximum(mat, 0), :3]
        I = I * np.where(ok[:, None], rho, 0.0)
        pos.append(P)
        nrm.append(N)
        inten.append(I)
    # interleave so that truncation keeps whole early paths
    Pa = np.stack(pos, 1).reshape(-1, 3)[:n_vpls]
    Na = np.stack(nrm, 1).reshape(-1, 3)[:n_vpls]
    Ia = np.stack(inten, 1).reshape(-1, 3)[:n_vpls]
    Na = Na / np.linalg.norm(Na, axis=1, keepdims=True)
    f32 = np.float32
    return dict(px=Pa[:, 0].astype(f32), py=Pa[:, 1].astype(f32), pz=Pa[:, 2].astype(f32),
                nx=Na[:, 0].astype(f32), ny=Na[:, 1].astype(f32), nz=Na[:, 2].astype(f32),
                ir=Ia[:, 0].astype(f32), ig=Ia[:, 1].astype(f32), ib=Ia[:, 2].astype(f32))


def _lum(r, g, b):
    return (0.2126 * r + 0.7152 * g) + 0.0722 * b


def _light_tree(v: dict, cut_max: int):
    """Binary light tree by level-synchronous median split; BFS node ids."""
    pos = np.stack([v["px"], v["py"], v["pz"]], 1).astype(np.float64)
    nv = pos.shape[0]
    nn = 2 * nv - 1
    left = np.full(nn, -1, np.int64)
    right = np.full(nn, -1, np.int64)
    leaf_vpl = np.full(nn, -1, np.int64)
    blo = np.zeros((nn, 3))
    bhi = np.zeros((nn, 3))
    order = np.arange(nv)
    starts = np.array([0], np.int64)
    lens = np.array([nv], np.int64)
    nodes = np.array([0], np.int64)
    nxt = 1
    level_nodes = []
    while starts.size:
        level_nodes.append(nodes)
        P = pos[order]
        seg_id = np.repeat(np.arange(starts.size), lens)
        lo = np.minimum.reduceat(P, starts, axis=0)
        hi = np.maximum.reduceat(P, starts, axis=0)
        blo[nodes] = lo
        bhi[nodes] = hi
        is_leaf = lens == 1
        leaf_vpl[nodes[is_leaf]] = order[starts[is_leaf]]
        axis = np.argmax(hi - lo, axis=1)
        key = P[np.arange(nv), axis[seg_id]]
        key = np.where(is_leaf[seg_id], 0.0, key)
        perm = np.lexsort((order, key, seg_id))
        order = order[perm]
        internal = ~is_leaf
        s_i = starts[internal]
        l_i = lens[internal]
        n_i = nodes[internal]
        nl = (l_i + 1) // 2
        k = n_i.size
        lid = nxt + 2 * np.arange(k)
        rid = lid + 1
        nxt += 2 * k
        left[n_i] = lid
        right[n_i] = rid
        # children segments, in BFS order (left, right interleaved per parent)
        starts = np.stack([s_i, s_i + nl], 1).ravel()
        lens = np.stack([nl, l_i - nl], 1).ravel()
        nodes = np.stack([lid, rid], 1).ravel()
        # the next level tiles only the elements of the new (child) segments: finished leaves
        # drop out, so gather those ranges and re-base the segment starts onto the sub-array
        if starts.size:
            order = order[_ranges(starts, lens)]
            starts = np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(np.int64)
            nv = order.size
    assert nxt == nn
    ir = np.zeros(nn)
    ig = np.zeros(nn)
    ib = np.zeros(nn)
    rep = np.full(nn, -1, np.int64)
    lf = leaf_vpl >= 0
    rep[lf] = leaf_vpl[lf]
    ir[lf] = v["ir"][leaf_vpl[lf]]
    ig[lf] = v["ig"][leaf_vpl[lf]]
    ib[lf] = v["ib"][leaf_vpl[lf]]
    for nodes in reversed(level_nodes):
        inn = nodes[left[nodes] >= 0]
        if inn.size == 0:
            continue
        l = left[inn]
        r = right[inn]
        ir[inn] = ir[l] + ir[r]
        ig[inn] = ig[l] + ig[r]
        ib[inn] = ib[l] + ib[r]
        ll = _lum(ir[l], ig[l], ib[l])
        lr = _lum(ir[r], ig[r], ib[r])
        rep[inn] = np.where(ll >= lr, rep[l], rep[r])
    # global cut: greedy split by a lightcut-style bound lum(I_f) * bbox diagonal
    diag = np.linalg.norm(bhi - blo, axis=1)
    bound = _lum(ir, ig, ib) * diag
    heap = [(-bound[0], 0)]
    cut = []
    while heap and len(heap) + len(cut) < cut_max:
        b, f = heapq.heappop(heap)
        if left[f] < 0:
            cut.append(f)
            continue
        heapq.heappush(heap, (-bound[left[f]], int(left[f])))
        heapq.heappush(heap, (-bound[right[f]], int(right[f])))
    cut.extend(f for _, f in heap)
    cut = np.sort(np.array(cut, np.int64))
    f32 = np.float32
    return dict(left=left.astype(np.int32), right=right.astype(np.int32), rep=rep.astype(np.int32),
                ir=ir.astype(f32), ig=ig.astype(f32), ib=ib.astype(f32),
                global_cut=cut.astype(np.int32), root=0)


def _ranges(starts, lens):
    total = int(lens.sum())
    if total == 0:
        return np.zeros(0, np.int64)
    rep_start = np.repeat(starts, lens)
    off = np.arange(total) - np.repeat(np.cumsum(lens) - lens, lens)
    return rep_start + off


def make_inputs(cfg: Config | str) -> Inputs:
    if isinstance(cfg, str):
        cfg = preset(cfg)
    rng = np.random.default_rng(cfg.fixture_seed)
    sc = _cornell() if cfg.scene == "cornell" else _mesh_scene(cfg.mesh_level) if cfg.scene == "mesh" else _interior()
    g = _gbuffer(sc, cfg.width, cfg.height)
    v = _vpls(sc, cfg.n_vpls, rng)
    t = _light_tree(v, cfg.cut_max)
    f32 = np.float32
    prims = dict(sph=np.ascontiguousarray(sc.spheres, f32).reshape(-1, 4),
                 box=np.ascontiguousarray(sc.boxes, f32).reshape(-1, 6),
                 rect=np.ascontiguousarray(sc.rects, f32).reshape(-1, 12),
                 tri=np.ascontiguousarray(sc.tris, f32).reshape(-1, 9))
    D = sc.diag
    return Inputs(cfg=cfg, scene=sc, width=cfg.width, height=cfg.height, gbuf=g, vpls=v, tree=t,
                  prims=prims, diag=D, clamp_dist=0.01 * D, shadow_eps=1e-4 * D, tau=cfg.tau)
