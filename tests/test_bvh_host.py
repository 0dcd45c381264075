"""CPU checks of the triangle BVH the library builds at lmc_create (host logic, no
GPU): the leaves partition the triangles, every node box is exactly the float min / max of the
vertices below it, children are adjacent, leaves hold at most 4 triangles, the depth fits the
32-entry traversal stack.  The GPU walk that relies on these is checked bit-exact against the
oracle's brute force in tests/test_gpu_mesh.py."""
import numpy as np
import pytest

import scenegen
from paper_2202_12567_b200 import lmc


def _walk(nodes):
    first = nodes[:, 3].view(np.int32)
    count = nodes[:, 7].view(np.int32)
    leaves, depth = [], 0
    stack = [(0, 1)]
    seen = set()
    while stack:
        k, d = stack.pop()
        assert k not in seen
        seen.add(k)
        depth = max(depth, d)
        if count[k] == 0:
            stack += [(first[k], d + 1), (first[k] + 1, d + 1)]
        else:
            assert 1 <= count[k] <= 4
            leaves.append((k, first[k], count[k]))
    assert len(seen) == nodes.shape[0]              # every node reachable exactly once
    return leaves, depth


def _boxes_exact(nodes, tris):
    first = nodes[:, 3].view(np.int32)
    count = nodes[:, 7].view(np.int32)
    V = tris[:, :9].reshape(-1, 3, 3)

    def span(k):
        if count[k] > 0:
            return first[k], first[k] + count[k]
        a, _ = span(first[k])
        _, b = span(first[k] + 1)
        return a, b

    for k in range(nodes.shape[0]):
        a, b = span(k)
        P = V[a:b].reshape(-1, 3)
        assert np.array_equal(nodes[k, 0:3], P.min(0)) and np.array_equal(nodes[k, 4:7], P.max(0)), k


@pytest.mark.parametrize("kind", ["icosphere", "mesh_scene", "soup", "one", "coplanar"])
def test_bvh_structure(kind):
    rng = np.random.default_rng(4)
    if kind == "icosphere":
        tri = scenegen._icosphere(3).astype(np.float32)
    elif kind == "mesh_scene":
        tri = scenegen.make_inputs("t_mesh").prims["tri"]
    elif kind == "soup":
        c = rng.uniform(-5, 5, (3001, 1, 3))
        tri = (c + rng.normal(0, 0.1, (3001, 3, 3))).reshape(-1, 9).astype(np.float32)
    elif kind == "one":
        tri = np.array([[0, 0, 0, 1, 0, 0, 0, 1, 0]], np.float32)
    else:   # identical centroids: ties broken by index
        tri = np.tile(np.array([[0, 0, 0, 1, 0, 0, 0, 1, 0]], np.float32), (37, 1))
    nodes, tris, order = lmc.plan_bvh(tri)
    n = tri.shape[0]
    assert np.array_equal(np.sort(order), np.arange(n))              # a permutation
    assert np.array_equal(tris[:, :9], tri[order])                   # reordered triangles
    leaves, depth = _walk(nodes)
    covered = np.zeros(n, np.int32)
    for _, f, c in leaves:
        covered[f:f + c] += 1
    assert np.all(covered == 1)                                       # leaves partition the list
    assert depth <= 32
    _boxes_exact(nodes, tris)


def test_bvh_rejects_bad_input():
    tri = np.zeros((2, 9), np.float32)
    tri[1, 4] = np.inf
    with pytest.raises(lmc.LmcError):
        lmc.plan_bvh(tri)
    with pytest.raises(lmc.LmcError):
        lmc.plan_bvh(np.zeros((0, 9), np.float32))
