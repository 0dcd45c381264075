"""Pins for the oracle's lighting-matrix entry A(i,j) (reading R1-R3, R32).

Closed forms, special cases and invariants — independent of the oracle's own code path.
"""
import math

import numpy as np
import pytest

import oracle
from tests._mini import mini, rect_prim

LUMW = np.array([0.2126, 0.7152, 0.0722])


def T(x, i=0, j=0):
    return oracle.Oracle(x).entry_T(i, j)


def test_closed_form_unit_configuration():
    # d = 1, both cosines 1, diffuse albedo 1, I = pi  ->  A = rho/pi * I * 1 * 1 / 1 = 1
    x = mini([0, 0, 0], [0, 1, 0], [0, 1, 0], [0, -1, 0], [math.pi] * 3)
    t = T(x)
    assert t == pytest.approx(1.0 / math.pi, rel=1e-15)
    assert (1.0 * math.pi) * t == pytest.approx(1.0, rel=1e-15)


def test_inverse_square_and_cosines():
    # d = 2 along the normal: 1/(pi d^2); tilted VPL normal by 60 deg: times cos 60
    x = mini([0, 0, 0], [0, 1, 0], [0, 2, 0], [0, -1, 0], [1, 1, 1])
    assert T(x) == pytest.approx(1.0 / (math.pi * 4.0), rel=1e-7)
    c, s = math.cos(math.radians(60)), math.sin(math.radians(60))
    x = mini([0, 0, 0], [0, 1, 0], [0, 2, 0], [s, -c, 0], [1, 1, 1])
    assert T(x) == pytest.approx(c / (math.pi * 4.0), rel=1e-6)
    # receiver tilted: point normal at 60 deg
    x = mini([0, 0, 0], [s, c, 0], [0, 2, 0], [0, -1, 0], [1, 1, 1])
    assert T(x) == pytest.approx(c / (math.pi * 4.0), rel=1e-6)


def test_back_facing_is_zero():
    assert T(mini([0, 0, 0], [0, -1, 0], [0, 1, 0], [0, -1, 0], [1, 1, 1])) == 0.0   # receiver faces away
    assert T(mini([0, 0, 0], [0, 1, 0], [0, 1, 0], [0, 1, 0], [1, 1, 1])) == 0.0    # VPL faces away
    assert T(mini([0, 0, 0], [0, 1, 0], [0, 0, 0], [0, -1, 0], [1, 1, 1])) == 0.0    # coincident


def test_clamp_saturates():
    # for d < d_c the denominator is d_c^2: value independent of d (P:50 clamping; R2)
    vals = [T(mini([0, 0, 0], [0, 1, 0], [0, d, 0], [0, -1, 0], [1, 1, 1], clamp_dist=0.5)) for d in (0.1, 0.2, 0.4)]
    assert vals[0] == vals[1] == vals[2] == pytest.approx(1.0 / (math.pi * 0.25))
    far = T(mini([0, 0, 0], [0, 1, 0], [0, 1, 0], [0, -1, 0], [1, 1, 1], clamp_dist=0.5))
    assert far == pytest.approx(1.0 / math.pi, rel=1e-7)


def test_occluders_each_kind():
    base = dict(points=[0, 0, 0], normals=[0, 1, 0], vpl_pos=[0, 2, 0], vpl_nrm=[0, -1, 0], vpl_I=[1, 1, 1])
    assert T(mini(**base, sph=[[0, 1, 0, 0.2]])) == 0.0
    assert T(mini(**base, sph=[[0.5, 1, 0, 0.2]])) > 0.0          # misses
    assert T(mini(**base, sph=[[0, 3, 0, 0.2]])) > 0.0            # beyond the light
    assert T(mini(**base, box=[[-0.1, 0.9, -0.1, 0.1, 1.1, 0.1]])) == 0.0
    assert T(mini(**base, box=[[0.2, 0.9, -0.1, 0.4, 1.1, 0.1]])) > 0.0
    r = rect_prim([-0.5, 1.0, -0.5], [1, 0, 0], [0, 0, 1])
    assert T(mini(**base, rect=[r])) == 0.0
    r2 = rect_prim([0.1, 1.0, -0.5], [1, 0, 0], [0, 0, 1])         # shifted off the segment
    assert T(mini(**base, rect=[r2])) > 0.0


def test_visibility_symmetric_and_hand_cases():
    rng = np.random.default_rng(7)
    sph = [[0.5, 0.5, 0.5, 0.2], [0.2, 0.7, 0.3, 0.1]]
    box = [[0.6, 0.1, 0.1, 0.8, 0.4, 0.3]]
    rect = [rect_prim([0.1, 0.2, 0.6], [0.5, 0, 0], [0, 0.5, 0.1])]
    x = mini([0, 0, 0], [0, 1, 0], [0, 1, 0], [0, -1, 0], [1, 1, 1], sph=sph, box=box, rect=rect)
    o = oracle.Oracle(x)
    n_occ = 0
    for _ in range(2000):
        a, b = rng.uniform(-0.2, 1.2, 3), rng.uniform(-0.2, 1.2, 3)
        # skip endpoints inside a sphere or box (never surface points)
        inside = any(np.linalg.norm(p - np.array(s[:3])) < s[3] for s in sph for p in (a, b))
        inside |= any(np.all((p > np.array(bx[:3])) & (p < np.array(bx[3:]))) for bx in box for p in (a, b))
        if inside:
            continue
        vab, vba = o.visible(a, b), o.visible(b, a)
        assert vab == vba
        n_occ += not vab
        # independent analytic check against the sphere: segment-sphere distance test
        for s in sph:
            c, r = np.array(s[:3]), s[3]
            d = b - a
            t = np.clip(np.dot(c - a, d) / np.dot(d, d), 0, 1)
            if np.linalg.norm(a + t * d - c) < r * 0.999:
                assert not vab
    assert n_occ > 50


def test_linear_in_intensity():
    # T does not depend on I; the matrix entry M~ = (lum rho lum I) T is linear in I
    x1 = mini([0, 0, 0], [0, 1, 0], [0.3, 1, 0.1], [0, -1, 0], [1, 1, 1])
    x2 = mini([0, 0, 0], [0, 1, 0], [0.3, 1, 0.1], [0, -1, 0], [3, 3, 3])
    assert T(x1) == T(x2)


def test_glossy_lobe_normalisation():
    # s = 1, e = 0: phi = (0 + 2) / (2 pi) * 1 = 1/pi, the diffuse value
    kw = dict(points=[0, 0, 0], normals=[0, 1, 0], vpl_pos=[0.3, 1, 0.2], vpl_nrm=[0, -1, 0], vpl_I=[1, 1, 1])
    d = T(mini(**kw))
    g = T(mini(**kw, spec=[1.0], expo=[0], views=[[0, 1, 0]]))
    assert g == pytest.approx(d, rel=1e-15)


def test_glossy_energy_bound_and_peak():
    # integral over the hemisphere of phi(l, o) cos(theta_l) d omega <= 1 (energy conservation of
    # the normalised Phong lobe), by quadrature over VPL directions at distance 1 facing the point
    o = np.array([math.sin(0.5), math.cos(0.5), 0.0])
    for s, e in ((0.5, 8), (1.0, 32), (0.25, 64)):
        nth, nph = 96, 192
        total = 0.0
        best, best_dir = -1, None
        pts, nrm = [], []
        for it in range(nth):
            th = (it + 0.5) / nth * (math.pi / 2)
            for ip in range(nph):
                ph = (ip + 0.5) / nph * 2 * math.pi
                l = np.array([math.sin(th) * math.cos(ph), math.cos(th), math.sin(th) * math.sin(ph)])
                pts.append(l)
                nrm.append(-l)
        x = mini([0, 0, 0], [0, 1, 0], np.array(pts), np.array(nrm), np.ones((len(pts), 3)),
                 views=[o], spec=[s], expo=[e], clamp_dist=1e-6)
        orc = oracle.Oracle(x)
        k = 0
        for it in range(nth):
            th = (it + 0.5) / nth * (math.pi / 2)
            dw = math.sin(th) * (math.pi / 2 / nth) * (2 * math.pi / nph)
            for ip in range(nph):
                t = orc.entry_T(0, k)          # = phi * cos(theta) * 1 * 1 / 1
                total += t * dw
                if t > best:
                    best, best_dir = t, pts[k]
                k += 1
        assert total <= 1.0 + 2e-3
        assert total > 0.5
        # mirror direction of o about n maximises the glossy part
        refl = np.array([-o[0], o[1], -o[2]])
        assert np.dot(best_dir, refl) > 0.99


def test_entry_flop_count_hand_cases():
    """the measurement counter of the entry evaluation (bench.py's entry roofline) on hand cases:
    d (3) + d.d (5) + sqrt and l = d/|d| (4) + two cosines (10) = 22 up to the back-facing exit;
    + d_c^2, G (3) + segment end (1) + phi G (1) = 27 for a lit diffuse pair with no occluder;
    a box costs 15 (3 axes x (1 / l_a, two slab distances)); a sphere 17 to the disc < 0 exit,
    20 when the roots are formed (a hit skips the final product)"""
    from tests._mini import mini
    pts = [[0.5, 0.0, 0.5]]
    lit = dict(points=pts, normals=[[0, 1, 0]], vpl_pos=[[0.5, 1.0, 0.5]], vpl_nrm=[[0, -1, 0]], vpl_I=[[1, 1, 1]])
    x = mini(**lit)
    o = oracle.Oracle(x)
    assert o.entry_flops([0], [0]) == 27
    xb = mini(**{**lit, "normals": [[0, -1, 0]]})           # back-facing point
    assert oracle.Oracle(xb).entry_flops([0], [0]) == 22
    xbox = mini(**lit, box=[[2.0, 2.0, 2.0, 3.0, 3.0, 3.0]])   # a box off the segment
    assert oracle.Oracle(xbox).entry_flops([0], [0]) == 27 + 15
    xs_miss = mini(**lit, sph=[[3.0, 0.5, 0.5, 0.1]])        # disc < 0
    assert oracle.Oracle(xs_miss).entry_flops([0], [0]) == 27 + 17
    xs_hit = mini(**lit, sph=[[0.5, 0.5, 0.5, 0.1]])         # on the segment: occluded
    oh = oracle.Oracle(xs_hit)
    assert oh.entry_T(0, 0) == 0.0
    assert oh.entry_flops([0], [0]) == 22 + 3 + 1 + 20
    assert o.entry_flops([0, 0, 0], [0, 0, 0]) == 3 * 27     # additive over pairs
