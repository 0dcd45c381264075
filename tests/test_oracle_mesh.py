"""Pins for the oracle's triangle occluders (reading R39).

The segment-vs-triangle test is checked against geometry it must reproduce, not against its own
formula: the barycentric closed form of a unit right triangle, the tmin/tmax segment shrink, both
windings, a rectangle split into two triangles against the rectangle primitive, and a closed
icosphere against the ball it contains and the ball containing it.
"""
import math

import numpy as np
import pytest

import oracle
import scenegen
from tests._mini import mini, rect_prim


def _orc(**prims):
    x = mini([0, 0, 0], [0, 1, 0], [0, 2, 0], [0, -1, 0], [1, 1, 1], shadow_eps=1e-6, **prims)
    return oracle.Oracle(x)


TRI = [0, 0, 0, 1, 0, 0, 0, 1, 0]          # z = 0 plane, legs on the x and y axes


def test_unit_triangle_barycentric_closed_form():
    rng = np.random.default_rng(11)
    for tri in (TRI, [0, 0, 0, 0, 1, 0, 1, 0, 0]):   # both windings (det of either sign)
        o = _orc(tri=[tri])
        n_hit = 0
        for _ in range(3000):
            a, b = rng.uniform(-0.5, 1.5, 2)
            d = rng.uniform(-0.3, 0.3, 2)
            # segment (a+d, b+d', 1) -> (a-d, b-d', -1) crosses z = 0 at (a, b)
            x = [a + d[0], b + d[1], 1.0]
            y = [a - d[0], b - d[1], -1.0]
            inside = a > 1e-9 and b > 1e-9 and a + b < 1 - 1e-9
            outside = a < -1e-9 or b < -1e-9 or a + b > 1 + 1e-9
            if not (inside or outside):
                continue
            vis = o.visible(x, y)
            assert vis == outside, (tri, a, b)
            assert o.visible(y, x) == vis   # direction does not matter
            n_hit += inside
        assert 250 < n_hit < 500   # area 1/2 of the 2 x 2 square


def test_segment_shrink_tmin_tmax():
    o = _orc(tri=[TRI])
    assert not o.visible([0.2, 0.2, 1.0], [0.2, 0.2, -1.0])
    assert o.visible([0.2, 0.2, 1.0], [0.2, 0.2, 1e-3])      # stops short of the plane
    assert o.visible([0.2, 0.2, 1.0], [0.2, 0.2, 0.0])       # ends on it: t = dist >= tmax
    assert o.visible([0.2, 0.2, 0.0], [0.2, 0.2, 1.0])       # starts on it: t = 0 <= tmin
    assert o.visible([0.2, 0.2, -1e-3], [0.2, 0.2, -1.0])    # both below
    assert o.visible([0.2, 0.2, 1.0], [3.2, 0.2, 1.0])       # parallel to the plane (det = 0)


def test_rectangle_as_two_triangles():
    rng = np.random.default_rng(5)
    # a rectangle (orthogonal edges, the rect primitive's definition) with dyadic coordinates:
    # vertices, edges and the normal e1 x e2 are exact in float32
    v00 = np.array([0.125, 0.25, 0.375])
    e1 = np.array([0.5, 0.0, 0.25])
    e2 = np.array([-0.125, 0.75, 0.25])
    assert e1 @ e2 == 0.0
    v10, v01, v11 = v00 + e1, v00 + e2, v00 + e1 + e2
    o_rect = _orc(rect=[rect_prim(v00, e1, e2)])
    o_tri = _orc(tri=[np.r_[v00, v10, v11], np.r_[v00, v11, v01]])
    n_occ = 0
    for _ in range(4000):
        a, b = rng.uniform(-0.5, 1.5, 3), rng.uniform(-0.5, 1.5, 3)
        v = o_rect.visible(a, b)
        assert o_tri.visible(a, b) == v, (a, b)
        n_occ += not v
    assert n_occ > 300


def test_icosphere_between_inscribed_and_circumscribed_balls():
    ico = scenegen._icosphere(2)           # unit circumscribed radius, 320 faces
    c = np.array([0.3, -0.2, 0.5])
    tris = (ico + np.tile(c, 3)).astype(np.float32)
    v0 = tris[:, 0:3].astype(np.float64) - c
    nrm = np.cross(tris[:, 3:6] - tris[:, 0:3], tris[:, 6:9] - tris[:, 0:3]).astype(np.float64)
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    r_in = float(np.min(np.abs((v0 * nrm).sum(1))))     # every face plane is at least this far
    r_out = float(np.max(np.linalg.norm(tris.reshape(-1, 3).astype(np.float64) - c, axis=1)))
    assert 0.9 < r_in < r_out < 1.0 + 1e-6
    o = _orc(tri=tris)
    rng = np.random.default_rng(3)
    for _ in range(400):
        dirn = rng.normal(size=3)
        dirn /= np.linalg.norm(dirn)
        perp = np.cross(dirn, rng.normal(size=3))
        perp /= np.linalg.norm(perp)
        d = rng.uniform(0.0, 1.3)
        if abs(d - r_in) < 1e-3 or (r_in < d < r_out + 1e-3):
            continue
        mid = c + d * perp
        x, y = mid - 3.0 * dirn, mid + 2.5 * dirn
        # a line closer to the centre than every face plane crosses the closed convex mesh
        assert o.visible(x, y) == (d > r_out), d


def test_mesh_scene_fixture_shape():
    x = scenegen.make_inputs("t_mesh")
    assert x.prims["tri"].shape == (416, 9) and x.prims["tri"].dtype == np.float32
    assert scenegen._icosphere(3).shape == (1280, 9)
    assert x.m == 48 * 40
    # some G-buffer points lie on the meshes: within 1e-4 of a triangle's plane and inside its bbox
    T = x.prims["tri"].astype(np.float64)
    P = np.stack([x.gbuf["px"], x.gbuf["py"], x.gbuf["pz"]], 1).astype(np.float64)
    nrm = np.cross(T[:, 3:6] - T[:, 0:3], T[:, 6:9] - T[:, 0:3])
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    dist = np.abs(((P[:, None, :] - T[None, :, 0:3]) * nrm[None]).sum(2))
    lo = np.minimum(np.minimum(T[:, 0:3], T[:, 3:6]), T[:, 6:9]) - 1e-4
    hi = np.maximum(np.maximum(T[:, 0:3], T[:, 3:6]), T[:, 6:9]) + 1e-4
    inb = np.all((P[:, None, :] >= lo[None]) & (P[:, None, :] <= hi[None]), axis=2)
    on_mesh = np.any((dist < 1e-4) & inb, axis=1)
    assert 50 < on_mesh.sum() < x.m // 2
