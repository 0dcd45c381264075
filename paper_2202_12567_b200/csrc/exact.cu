// exact.cu — decision-precision kernels of the lighting-matrix hot path (sm_100a).
//
// Everything that takes a discrete decision (slice splits, pass-1 rows, merge decisions,
// pass-2 weights/draws) or produces an entry value runs here in IEEE binary64 with NO
// contraction (this translation unit is compiled with -fmad=false), in the operation order
// fixed by DESIGN.md §"Entry formula" (readings R1-R3, R30) — so index sets and cuts are
// bit-identical to an fp64 reference by construction.
//
//   slicing      PAPER.md:71-73, P:172   (R26)
//   pass 1       P:104                   (R6, R7)
//   coarsening   P:96-122, Eq. (1)       (R5, R8-R11)
//   pass 2       P:129-147, Eq. (2)      (R13-R17, R27)
//   entry A(i,j) P:61, P:48, P:50        (R1-R3, R32)
#include <cub/cub.cuh>

#include <mutex>

#include "lmc_internal.h"
#include "philox.cuh"

namespace lmc {

// one scene per live context (slot acquired in lmc_create): uniform reads hit the constant cache
__constant__ SceneConst c_scenes[SCENE_SLOTS];

#define LMC_INV_PI 0.31830988618379067
#define LMC_INV_2PI 0.15915494309189535
#define FULL_MASK 0xffffffffu

// ------------------------------------------------------------------------------------------
// Entry T(p, v): cosine VPL emitter x clamped geometry x normalised Phong x visibility.
// Packed row (4 x float4): (px,py,pz,nx) (ny,nz,vx,vy) (vz,spec,rr,rg) (rb,expo,0,0)
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ double dot3d(double a0, double a1, double a2, double b0, double b1, double b2)
{
    return (a0 * b0 + a1 * b1) + a2 * b2;
}

__device__ __forceinline__ double powi_d(double base, int e)
{
    double r = 1.0;
    while (e > 0) {
        if (e & 1) r = r * base;
        base = base * base;
        e >>= 1;
    }
    return r;
}

// Segment vs triangle (R39): Moller-Trumbore in the oracle's operation
// order — e1 = v1 - v0, e2 = v2 - v0, p = l x e2, det = e1 . p, inv = 1 / det, s = x - v0,
// u = (s . p) inv, qv = s x e1, v = (l . qv) inv, t = (e2 . qv) inv.
__device__ __forceinline__ bool tri_hit(const float4 *__restrict__ t4, double x0, double x1, double x2, double l0,
                                        double l1, double l2, double tmin, double tmax)
{
    const float4 A = t4[0], B = t4[1], C = t4[2];
    const double v00 = A.x, v01 = A.y, v02 = A.z;
    const double e10 = (double)A.w - v00, e11 = (double)B.x - v01, e12 = (double)B.y - v02;
    const double e20 = (double)B.z - v00, e21 = (double)B.w - v01, e22 = (double)C.x - v02;
    const double p0 = l1 * e22 - l2 * e21, p1 = l2 * e20 - l0 * e22, p2 = l0 * e21 - l1 * e20;
    const double det = dot3d(e10, e11, e12, p0, p1, p2);
    if (det == 0.0) return false;
    const double inv = 1.0 / det;
    const double s0 = x0 - v00, s1 = x1 - v01, s2 = x2 - v02;
    const double u = dot3d(s0, s1, s2, p0, p1, p2) * inv;
    if (u < 0.0 || u > 1.0) return false;
    const double q0 = s1 * e12 - s2 * e11, q1 = s2 * e10 - s0 * e12, q2 = s0 * e11 - s1 * e10;
    const double v = dot3d(l0, l1, l2, q0, q1, q2) * inv;
    if (v < 0.0 || u + v > 1.0) return false;
    const double t = dot3d(e20, e21, e22, q0, q1, q2) * inv;
    return t > tmin && t < tmax;
}

constexpr int BVH_STACK = 32;   // > depth of the median-split BVH of 2^26 triangles (lmc_create checks)

// 1 iff some triangle is hit by the open segment.  The BVH is walked with fp32 slab tests of the
// segment [x, y] (parameter s in [0, 1] over w = y - x) against node boxes widened by the margin
// (1e-3 D, far above fp32 rounding of the coordinates): a node is skipped only when no point of
// the segment lies within the margin of its box, so every triangle the exact test could report is
// reached and the decision equals the brute-force OR over all triangles.
__device__ bool bvh_hit(const SceneConst *sc, double x0, double x1, double x2, double l0, double l1, double l2,
                        double tmin, double tmax, float x0f, float x1f, float x2f, float y0f, float y1f, float y2f)
{
    const float mg = sc->margin;
    float w0 = y0f - x0f, w1 = y1f - x1f, w2 = y2f - x2f;
    // an axis the segment does not move along: a tiny slope keeps the slab test finite and exact in sign
    if (fabsf(w0) < 1e-20f) w0 = copysignf(1e-20f, w0);
    if (fabsf(w1) < 1e-20f) w1 = copysignf(1e-20f, w1);
    if (fabsf(w2) < 1e-20f) w2 = copysignf(1e-20f, w2);
    const float i0 = 1.f / w0, i1 = 1.f / w1, i2 = 1.f / w2;
    const float4 *__restrict__ bv = sc->bvh;
    const float4 *__restrict__ tr = sc->tri4;
    int stack[BVH_STACK];
    int sp = 0, node = 0;
    while (true) {
        const float4 A = bv[2 * node], B = bv[2 * node + 1];
        float ta = (A.x - mg - x0f) * i0, tb = (B.x + mg - x0f) * i0;
        float tn = fminf(ta, tb), tf = fmaxf(ta, tb);
        ta = (A.y - mg - x1f) * i1;
        tb = (B.y + mg - x1f) * i1;
        tn = fmaxf(tn, fminf(ta, tb));
        tf = fminf(tf, fmaxf(ta, tb));
        ta = (A.z - mg - x2f) * i2;
        tb = (B.z + mg - x2f) * i2;
        tn = fmaxf(tn, fminf(ta, tb));
        tf = fminf(tf, fmaxf(ta, tb));
        if (fmaxf(tn, 0.f) <= fminf(tf, 1.f)) {
            const int first = __float_as_int(A.w), cnt = __float_as_int(B.w);
            if (cnt == 0) {
                stack[sp++] = first + 1;
                node = first;
                continue;
            }
            for (int k = 0; k < cnt; ++k)
                if (tri_hit(tr + 3 * (first + k), x0, x1, x2, l0, l1, l2, tmin, tmax)) return true;
        }
        if (sp == 0) return false;
        node = stack[--sp];
    }
}

// 1 iff the open segment x + t l, t in (eps, dist - eps), misses every occluder.
// Each primitive is first screened by a conservative fp32 test on the segment [x, y] (y = VPL
// position) with a margin of 1e-3 D, orders of magnitude above fp32 rounding: a primitive is
// skipped only when the exact fp64 test below cannot report a hit, so the visibility decision is
// exactly the reference's (an OR over primitives does not depend on which misses are skipped).
__device__ bool visible_d(int slot, double x0, double x1, double x2, double l0, double l1,
                          double l2, double dist, float y0f, float y1f, float y2f)
{
    const SceneConst *sc = &c_scenes[slot];
    const double tmin = sc->eps, tmax = dist - sc->eps;
    const float x0f = (float)x0, x1f = (float)x1, x2f = (float)x2;   // exact: the inputs are float32
    const float mg = sc->margin;
    const float lo0 = fminf(x0f, y0f), lo1 = fminf(x1f, y1f), lo2 = fminf(x2f, y2f);
    const float hi0 = fmaxf(x0f, y0f), hi1 = fmaxf(x1f, y1f), hi2 = fmaxf(x2f, y2f);
    const float w0 = y0f - x0f, w1 = y1f - x1f, w2 = y2f - x2f;
    const float ww = w0 * w0 + w1 * w1 + w2 * w2;
    for (int k = 0; k < sc->nsph; ++k) {
        const float *s = sc->sph + 4 * k;
        {   // screen: distance from the segment to the centre against r + margin
            const float v0 = s[0] - x0f, v1 = s[1] - x1f, v2 = s[2] - x2f;
            const float tt = fminf(fmaxf((v0 * w0 + v1 * w1 + v2 * w2) / ww, 0.f), 1.f);
            const float d0 = v0 - tt * w0, d1 = v1 - tt * w1, d2 = v2 - tt * w2;
            const float rr = s[3] + mg;
            if (d0 * d0 + d1 * d1 + d2 * d2 > rr * rr) continue;
        }
        double o0 = x0 - (double)s[0], o1 = x1 - (double)s[1], o2 = x2 - (double)s[2];
        double r = s[3];
        double b = dot3d(o0, o1, o2, l0, l1, l2);
        double cc = dot3d(o0, o1, o2, o0, o1, o2) - r * r;
        double disc = b * b - cc;
        if (disc < 0.0) continue;
        double sq = sqrt(disc);
        double t0 = -b - sq, t1 = -b + sq;
        if ((t0 > tmin && t0 < tmax) || (t1 > tmin && t1 < tmax)) return false;
    }
    if (sc->nbox > 0) {
        double i0 = 0.0, i1 = 0.0, i2 = 0.0;
        bool inv = false;
        for (int k = 0; k < sc->nbox; ++k) {
            const float *bx = sc->box + 6 * k;
            // screen: segment bounding box against the box grown by the margin
            if (hi0 < bx[0] - mg || lo0 > bx[3] + mg || hi1 < bx[1] - mg || lo1 > bx[4] + mg || hi2 < bx[2] - mg ||
                lo2 > bx[5] + mg)
                continue;
            if (!inv) { i0 = 1.0 / l0; i1 = 1.0 / l1; i2 = 1.0 / l2; inv = true; }
            double a1 = ((double)bx[0] - x0) * i0, a2 = ((double)bx[3] - x0) * i0;
            double b1 = ((double)bx[1] - x1) * i1, b2 = ((double)bx[4] - x1) * i1;
            double e1 = ((double)bx[2] - x2) * i2, e2 = ((double)bx[5] - x2) * i2;
            double tnear = fmax(fmax(fmin(a1, a2), fmin(b1, b2)), fmin(e1, e2));
            double tfar = fmin(fmin(fmax(a1, a2), fmax(b1, b2)), fmax(e1, e2));
            if (tnear <= tfar && tfar > tmin && tnear < tmax) return false;
        }
    }
    for (int k = 0; k < sc->nrect; ++k) {
        const float *rc = sc->rect + 12 * k;
        {   // screen: bounding boxes, then both end points strictly on one side of the plane
            const float *rb = sc->rbox + 6 * k;
            if (hi0 < rb[0] - mg || lo0 > rb[3] + mg || hi1 < rb[1] - mg || lo1 > rb[4] + mg || hi2 < rb[2] - mg ||
                lo2 > rb[5] + mg)
                continue;
            const float sx = (x0f - rc[0]) * rc[9] + (x1f - rc[1]) * rc[10] + (x2f - rc[2]) * rc[11];
            const float sy = (y0f - rc[0]) * rc[9] + (y1f - rc[1]) * rc[10] + (y2f - rc[2]) * rc[11];
            const float dl = mg * sc->rnorm[k];
            if ((sx > dl && sy > dl) || (sx < -dl && sy < -dl)) continue;
        }
        double p0 = rc[0], p1 = rc[1], p2 = rc[2];
        double e10 = rc[3], e11 = rc[4], e12 = rc[5];
        double e20 = rc[6], e21 = rc[7], e22 = rc[8];
        double n0 = rc[9], n1 = rc[10], n2 = rc[11];
        double den = dot3d(n0, n1, n2, l0, l1, l2);
        if (den == 0.0) continue;
        double t = dot3d(p0 - x0, p1 - x1, p2 - x2, n0, n1, n2) / den;
        if (!(t > tmin && t < tmax)) continue;
        double h0 = x0 + t * l0, h1 = x1 + t * l1, h2 = x2 + t * l2;
        double q0 = h0 - p0, q1 = h1 - p1, q2 = h2 - p2;
        double a = dot3d(q0, q1, q2, e10, e11, e12) / dot3d(e10, e11, e12, e10, e11, e12);
        double b = dot3d(q0, q1, q2, e20, e21, e22) / dot3d(e20, e21, e22, e20, e21, e22);
        if (a >= 0.0 && a <= 1.0 && b >= 0.0 && b <= 1.0) return false;
    }
    if (sc->ntri > 0 && bvh_hit(sc, x0, x1, x2, l0, l1, l2, tmin, tmax, x0f, x1f, x2f, y0f, y1f, y2f)) return false;
    return true;
}

// Visibility with the scene staged in shared memory and the exact tests batched per warp: every
// lane first runs the fp32 screens of all primitives (uniform loop) and keeps a bitmask of the
// primitives that need the exact fp64 test; the warp then runs those tests type by type, each lane
// on its own next primitive, until every lane has a hit or no candidate left.  The decision is the
// same OR over primitives as visible_d (only the order of the exact tests differs), but the exact
// tests run with most lanes busy instead of with the few lanes whose screen passed for the
// primitive of the moment.
__device__ __forceinline__ bool sphere_hit(const float *s, double x0, double x1, double x2, double l0, double l1, double l2,
                                           double tmin, double tmax)
{
    double o0 = x0 - (double)s[0], o1 = x1 - (double)s[1], o2 = x2 - (double)s[2];
    double r = s[3];
    double b = dot3d(o0, o1, o2, l0, l1, l2);
    double cc = dot3d(o0, o1, o2, o0, o1, o2) - r * r;
    double disc = b * b - cc;
    if (disc < 0.0) return false;
    double sq = sqrt(disc);
    double t0 = -b - sq, t1 = -b + sq;
    return (t0 > tmin && t0 < tmax) || (t1 > tmin && t1 < tmax);
}

__device__ __forceinline__ bool box_hit(const float *bx, double x0, double x1, double x2, double i0, double i1, double i2,
                                        double tmin, double tmax)
{
    double a1 = ((double)bx[0] - x0) * i0, a2 = ((double)bx[3] - x0) * i0;
    double b1 = ((double)bx[1] - x1) * i1, b2 = ((double)bx[4] - x1) * i1;
    double e1 = ((double)bx[2] - x2) * i2, e2 = ((double)bx[5] - x2) * i2;
    double tnear = fmax(fmax(fmin(a1, a2), fmin(b1, b2)), fmin(e1, e2));
    double tfar = fmin(fmin(fmax(a1, a2), fmax(b1, b2)), fmax(e1, e2));
    return tnear <= tfar && tfar > tmin && tnear < tmax;
}

__device__ __forceinline__ bool rect_hit(const float *rc, double x0, double x1, double x2, double l0, double l1, double l2,
                                         double tmin, double tmax)
{
    double p0 = rc[0], p1 = rc[1], p2 = rc[2];
    double e10 = rc[3], e11 = rc[4], e12 = rc[5];
    double e20 = rc[6], e21 = rc[7], e22 = rc[8];
    double n0 = rc[9], n1 = rc[10], n2 = rc[11];
    double den = dot3d(n0, n1, n2, l0, l1, l2);
    if (den == 0.0) return false;
    double t = dot3d(p0 - x0, p1 - x1, p2 - x2, n0, n1, n2) / den;
    if (!(t > tmin && t < tmax)) return false;
    double h0 = x0 + t * l0, h1 = x1 + t * l1, h2 = x2 + t * l2;
    double q0 = h0 - p0, q1 = h1 - p1, q2 = h2 - p2;
    double a = dot3d(q0, q1, q2, e10, e11, e12) / dot3d(e10, e11, e12, e10, e11, e12);
    double b = dot3d(q0, q1, q2, e20, e21, e22) / dot3d(e20, e21, e22, e20, e21, e22);
    return a >= 0.0 && a <= 1.0 && b >= 0.0 && b <= 1.0;
}

// copy the context's scene into shared memory (all threads of the block; barrier inside)
__device__ __forceinline__ void stage_scene(SceneConst *dst, int slot)
{
    const int4 *src = reinterpret_cast<const int4 *>(&c_scenes[slot]);
    int4 *d = reinterpret_cast<int4 *>(dst);
    for (int k = threadIdx.x; k < (int)(sizeof(SceneConst) / 16); k += blockDim.x) d[k] = src[k];
    __syncthreads();
}

// Candidate occluders of every segment from a point of a slice (box bx = lo3, hi3) to the VPL
// position y: a primitive is a candidate when (1) its bounds meet the box of the slice and y, and
// (2) its bounding sphere (S, r) comes within R + r of the segment [C, y], (C, R) the sphere around
// the slice's box — both widened by the screening margin.  Each segment [x, y] of the slice lies
// in that box and within distance R of [C, y] (|x - C| <= R), and an exact hit lies on the
// primitive, so a primitive left out cannot hit.  Warp-collective (lane k tests primitive k of
// each kind); fp32 with the margin far above its rounding.
struct Cand {
    uint32_t s, b, r;
};
__device__ __forceinline__ bool near_seg(float S0, float S1, float S2, float rad, float C0, float C1, float C2, float w0,
                                         float w1, float w2, float ww, float reach)
{
    // distance from S to the segment C + t w, t in [0, 1], against reach + rad
    const float v0 = S0 - C0, v1 = S1 - C1, v2 = S2 - C2;
    const float t = ww > 0.f ? fminf(fmaxf((v0 * w0 + v1 * w1 + v2 * w2) / ww, 0.f), 1.f) : 0.f;
    const float d0 = v0 - t * w0, d1 = v1 - t * w1, d2 = v2 - t * w2;
    const float lim = reach + rad;
    return d0 * d0 + d1 * d1 + d2 * d2 <= lim * lim;
}
__device__ __forceinline__ Cand col_candidates(const SceneConst *sc, const float *bx, float y0, float y1, float y2)
{
    const int lane = threadIdx.x & 31;
    const float mg = sc->margin;
    const float L0 = fminf(bx[0], y0) - mg, L1 = fminf(bx[1], y1) - mg, L2 = fminf(bx[2], y2) - mg;
    const float H0 = fmaxf(bx[3], y0) + mg, H1 = fmaxf(bx[4], y1) + mg, H2 = fmaxf(bx[5], y2) + mg;
    // sphere around the slice's box, and the segment from its centre to the VPL
    const float C0 = 0.5f * (bx[0] + bx[3]), C1 = 0.5f * (bx[1] + bx[4]), C2 = 0.5f * (bx[2] + bx[5]);
    const float e0 = bx[3] - bx[0], e1 = bx[4] - bx[1], e2 = bx[5] - bx[2];
    const float reach = 0.5f * sqrtf(e0 * e0 + e1 * e1 + e2 * e2) + 2.f * mg;
    const float w0 = y0 - C0, w1 = y1 - C1, w2 = y2 - C2;
    const float ww = w0 * w0 + w1 * w1 + w2 * w2;
    bool ps = false, pb = false, pr = false;
    if (lane < sc->nsph) {
        const float *q = sc->sph + 4 * lane;
        const float r = q[3];
        ps = q[0] - r <= H0 && q[0] + r >= L0 && q[1] - r <= H1 && q[1] + r >= L1 && q[2] - r <= H2 && q[2] + r >= L2 &&
             near_seg(q[0], q[1], q[2], r, C0, C1, C2, w0, w1, w2, ww, reach);
    }
    if (lane < sc->nbox) {
        const float *q = sc->box + 6 * lane;
        const float f0 = q[3] - q[0], f1 = q[4] - q[1], f2 = q[5] - q[2];
        pb = q[0] <= H0 && q[3] >= L0 && q[1] <= H1 && q[4] >= L1 && q[2] <= H2 && q[5] >= L2 &&
             near_seg(0.5f * (q[0] + q[3]), 0.5f * (q[1] + q[4]), 0.5f * (q[2] + q[5]),
                      0.5f * sqrtf(f0 * f0 + f1 * f1 + f2 * f2), C0, C1, C2, w0, w1, w2, ww, reach);
    }
    if (lane < sc->nrect) {
        const float *q = sc->rbox + 6 * lane;
        const float f0 = q[3] - q[0], f1 = q[4] - q[1], f2 = q[5] - q[2];
        pr = q[0] <= H0 && q[3] >= L0 && q[1] <= H1 && q[4] >= L1 && q[2] <= H2 && q[5] >= L2 &&
             near_seg(0.5f * (q[0] + q[3]), 0.5f * (q[1] + q[4]), 0.5f * (q[2] + q[5]),
                      0.5f * sqrtf(f0 * f0 + f1 * f1 + f2 * f2), C0, C1, C2, w0, w1, w2, ww, reach);
    }
    Cand c;
    c.s = __ballot_sync(FULL_MASK, ps);
    c.b = __ballot_sync(FULL_MASK, pb);
    c.r = __ballot_sync(FULL_MASK, pr);
    return c;
}

__device__ bool visible_w(const SceneConst *sc, double x0, double x1, double x2, double l0, double l1, double l2,
                          double dist, float y0f, float y1f, float y2f, uint32_t cs = ~0u, uint32_t cb = ~0u,
                          uint32_t cr = ~0u)
{
    // cs / cb / cr: candidate spheres / boxes / rectangles (all by default); a primitive left out
    // must be unable to meet the segment (see col_candidates)
    const double tmin = sc->eps, tmax = dist - sc->eps;
    const float x0f = (float)x0, x1f = (float)x1, x2f = (float)x2;   // exact: the inputs are float32
    const float mg = sc->margin;
    const float lo0 = fminf(x0f, y0f), lo1 = fminf(x1f, y1f), lo2 = fminf(x2f, y2f);
    const float hi0 = fmaxf(x0f, y0f), hi1 = fmaxf(x1f, y1f), hi2 = fmaxf(x2f, y2f);
    const float w0 = y0f - x0f, w1 = y1f - x1f, w2 = y2f - x2f;
    const float ww = w0 * w0 + w1 * w1 + w2 * w2;
    // screens (identical arithmetic to visible_d)
    uint32_t ms = 0u, mb = 0u, mr = 0u;
    cs &= sc->nsph >= 32 ? ~0u : (1u << sc->nsph) - 1u;
    cb &= sc->nbox >= 32 ? ~0u : (1u << sc->nbox) - 1u;
    cr &= sc->nrect >= 32 ? ~0u : (1u << sc->nrect) - 1u;
    for (uint32_t cm = cs; cm; cm &= cm - 1u) {
        const int k = __ffs(cm) - 1;
        const float *s = sc->sph + 4 * k;
        const float v0 = s[0] - x0f, v1 = s[1] - x1f, v2 = s[2] - x2f;
        const float tt = fminf(fmaxf((v0 * w0 + v1 * w1 + v2 * w2) / ww, 0.f), 1.f);
        const float d0 = v0 - tt * w0, d1 = v1 - tt * w1, d2 = v2 - tt * w2;
        const float rr = s[3] + mg;
        if (!(d0 * d0 + d1 * d1 + d2 * d2 > rr * rr)) ms |= 1u << k;
    }
    for (uint32_t cm = cb; cm; cm &= cm - 1u) {
        const int k = __ffs(cm) - 1;
        const float *bx = sc->box + 6 * k;
        if (!(hi0 < bx[0] - mg || lo0 > bx[3] + mg || hi1 < bx[1] - mg || lo1 > bx[4] + mg || hi2 < bx[2] - mg ||
              lo2 > bx[5] + mg))
            mb |= 1u << k;
    }
    for (uint32_t cm = cr; cm; cm &= cm - 1u) {
        const int k = __ffs(cm) - 1;
        const float *rc = sc->rect + 12 * k;
        const float *rb = sc->rbox + 6 * k;
        if (hi0 < rb[0] - mg || lo0 > rb[3] + mg || hi1 < rb[1] - mg || lo1 > rb[4] + mg || hi2 < rb[2] - mg ||
            lo2 > rb[5] + mg)
            continue;
        const float sx = (x0f - rc[0]) * rc[9] + (x1f - rc[1]) * rc[10] + (x2f - rc[2]) * rc[11];
        const float sy = (y0f - rc[0]) * rc[9] + (y1f - rc[1]) * rc[10] + (y2f - rc[2]) * rc[11];
        const float dl = mg * sc->rnorm[k];
        if ((sx > dl && sy > dl) || (sx < -dl && sy < -dl)) continue;
        mr |= 1u << k;
    }
    // exact tests, batched across the active lanes
    const unsigned act = __activemask();
    bool hit = false;
    while (__any_sync(act, ms != 0u)) {
        if (ms) {
            const int k = __ffs(ms) - 1;
            ms &= ms - 1u;
            if (sphere_hit(sc->sph + 4 * k, x0, x1, x2, l0, l1, l2, tmin, tmax)) { hit = true; ms = mb = mr = 0u; }
        }
    }
    if (__any_sync(act, mb != 0u)) {
        const double i0 = 1.0 / l0, i1 = 1.0 / l1, i2 = 1.0 / l2;
        while (__any_sync(act, mb != 0u)) {
            if (mb) {
                const int k = __ffs(mb) - 1;
                mb &= mb - 1u;
                if (box_hit(sc->box + 6 * k, x0, x1, x2, i0, i1, i2, tmin, tmax)) { hit = true; mb = mr = 0u; }
            }
        }
    }
    while (__any_sync(act, mr != 0u)) {
        if (mr) {
            const int k = __ffs(mr) - 1;
            mr &= mr - 1u;
            if (rect_hit(sc->rect + 12 * k, x0, x1, x2, l0, l1, l2, tmin, tmax)) { hit = true; mr = 0u; }
        }
    }
    if (!hit && sc->ntri > 0) hit = bvh_hit(sc, x0, x1, x2, l0, l1, l2, tmin, tmax, x0f, x1f, x2f, y0f, y1f, y2f);
    return !hit;
}

// entry T with the warp-batched visibility (sc: the scene staged in shared memory)
__device__ __forceinline__ double entry_T_w(const SceneConst *sc, int slot, const float4 *__restrict__ prow, int64_t li,
                                            const float4 *__restrict__ vpl, int32_t v, uint32_t cs = ~0u,
                                            uint32_t cb = ~0u, uint32_t cr = ~0u);

// Shading part of T: phi * G, or 0 when the entry is zero without a visibility test; the
// segment (unit direction l, length dist) the visibility test needs is returned through g.
struct Seg {
    double l0, l1, l2, dist;
};
__device__ __forceinline__ double entry_shade(int slot, const float4 *__restrict__ prow, int64_t li,
                                              const float4 *__restrict__ vpl, int32_t v, Seg &g)
{
    const float4 A = prow[4 * li], B = prow[4 * li + 1], C = prow[4 * li + 2], D = prow[4 * li + 3];
    const float4 P = vpl[2 * (int64_t)v], Q = vpl[2 * (int64_t)v + 1];
    double x0 = A.x, x1 = A.y, x2 = A.z;
    double n0 = A.w, n1 = B.x, n2 = B.y;
    double d0 = (double)P.x - x0, d1 = (double)P.y - x1, d2 = (double)P.z - x2;
    double dd = dot3d(d0, d1, d2, d0, d1, d2);
    if (dd == 0.0) return 0.0;
    double dist = sqrt(dd);
    double l0 = d0 / dist, l1 = d1 / dist, l2 = d2 / dist;
    double ci = dot3d(n0, n1, n2, l0, l1, l2);
    double cj = -dot3d((double)P.w, (double)Q.x, (double)Q.y, l0, l1, l2);
    if (ci <= 0.0 || cj <= 0.0) return 0.0;
    double G = (ci * cj) / fmax(dd, c_scenes[slot].dc2);
    double s = C.y;
    double phi;
    if (s == 0.0) {
        phi = LMC_INV_PI;
    } else {
        int e = __float_as_int(D.y);
        double o0 = B.z, o1 = B.w, o2 = C.x;
        double rv = (2.0 * ci) * dot3d(n0, n1, n2, o0, o1, o2) - dot3d(l0, l1, l2, o0, o1, o2);
        double lobe = rv > 0.0 ? powi_d(rv, e) : 0.0;
        phi = (1.0 - s) * LMC_INV_PI + (s * (((double)(e + 2)) * LMC_INV_2PI)) * lobe;
    }
    g.l0 = l0;
    g.l1 = l1;
    g.l2 = l2;
    g.dist = dist;
    return phi * G;
}

__device__ __forceinline__ bool entry_visible(int slot, const float4 *__restrict__ prow, int64_t li,
                                              const float4 *__restrict__ vpl, int32_t v, const Seg &g)
{
    const float4 A = prow[4 * li];
    const float4 P = vpl[2 * (int64_t)v];
    return visible_d(slot, A.x, A.y, A.z, g.l0, g.l1, g.l2, g.dist, P.x, P.y, P.z);
}

__device__ double entry_T(int slot, const float4 *__restrict__ prow, int64_t li,
                          const float4 *__restrict__ vpl, int32_t v)
{
    Seg g;
    const double pg = entry_shade(slot, prow, li, vpl, v, g);
    if (pg == 0.0) return 0.0;
    return entry_visible(slot, prow, li, vpl, v, g) ? pg : 0.0;
}

__device__ __forceinline__ double entry_T_w(const SceneConst *sc, int slot, const float4 *__restrict__ prow, int64_t li,
                                            const float4 *__restrict__ vpl, int32_t v, uint32_t cs, uint32_t cb,
                                            uint32_t cr)
{
    Seg g;
    const double pg = entry_shade(slot, prow, li, vpl, v, g);
    bool vis = false;
    // every lane takes part in the batched test (a lane with pg == 0 brings no candidates)
    const float4 A = prow[4 * li];
    const float4 P = vpl[2 * (int64_t)v];
    if (pg != 0.0) vis = visible_w(sc, A.x, A.y, A.z, g.l0, g.l1, g.l2, g.dist, P.x, P.y, P.z, cs, cb, cr);
    return vis ? pg : 0.0;
}

__device__ __forceinline__ double lum_rho_d(const float4 *__restrict__ prow, int64_t li)
{
    const float4 C = prow[4 * li + 2], D = prow[4 * li + 3];
    return (0.2126 * (double)C.z + 0.7152 * (double)C.w) + 0.0722 * (double)D.x;
}

// ------------------------------------------------------------------------------------------
// Row packing in slice order (slicing itself: slice.cu)
// ------------------------------------------------------------------------------------------
struct GView {
    const float *px, *py, *pz, *nx, *ny, *nz;
};

__global__ void k_pack_rows(const int32_t *__restrict__ rows, int64_t row0, int64_t ML, GView g,
                            const float *__restrict__ vx, const float *__restrict__ vy, const float *__restrict__ vz,
                            const float *__restrict__ rr, const float *__restrict__ rg, const float *__restrict__ rb,
                            const float *__restrict__ spec, const int32_t *__restrict__ expo, float4 *prow)
{
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= ML) return;
    int r = rows[row0 + k];
    prow[4 * k + 0] = make_float4(g.px[r], g.py[r], g.pz[r], g.nx[r]);
    prow[4 * k + 1] = make_float4(g.ny[r], g.nz[r], vx[r], vy[r]);
    prow[4 * k + 2] = make_float4(vz[r], spec[r], rr[r], rg[r]);
    prow[4 * k + 3] = make_float4(rb[r], __int_as_float(expo[r]), 0.f, 0.f);
}

__global__ void k_pack_vpls(const float *__restrict__ soa, int64_t nv, float4 *vpl)
{
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= nv) return;
    vpl[2 * k] = make_float4(soa[k], soa[nv + k], soa[2 * nv + k], soa[3 * nv + k]);
    vpl[2 * k + 1] = make_float4(soa[4 * nv + k], soa[5 * nv + k], 0.f, 0.f);
}

static std::mutex g_slot_mu;
static bool g_slot_used[SCENE_SLOTS];

int acquire_scene_slot()
{
    std::lock_guard<std::mutex> lk(g_slot_mu);
    for (int k = 0; k < SCENE_SLOTS; ++k)
        if (!g_slot_used[k]) { g_slot_used[k] = true; return k; }
    return -1;
}

void release_scene_slot(int slot)
{
    std::lock_guard<std::mutex> lk(g_slot_mu);
    if (slot >= 0 && slot < SCENE_SLOTS) g_slot_used[slot] = false;
}

cudaError_t upload_scene(int slot, const SceneConst &sc)
{
    return cudaMemcpyToSymbol(c_scenes, &sc, sizeof(SceneConst), (size_t)slot * sizeof(SceneConst));
}

cudaError_t run_pack_vpls(lmc_ctx *c)
{
    if (c->NV == 0) return cudaSuccess;
    k_pack_vpls<<<(unsigned)((c->NV + 255) / 256), 256, 0, c->stream>>>(c->d.vpl_soa, c->NV, c->d.vpl);
    return cudaGetLastError();
}



static GView gview(lmc_ctx *c)
{
    GView g;
    g.px = c->d.g[0]; g.py = c->d.g[1]; g.pz = c->d.g[2];
    g.nx = c->d.g[3]; g.ny = c->d.g[4]; g.nz = c->d.g[5];
    return g;
}

cudaError_t run_pack_rows(lmc_ctx *c)
{
    if (c->ML == 0) return cudaSuccess;
    GView g = gview(c);
    k_pack_rows<<<(unsigned)((c->ML + 255) / 256), 256, 0, c->stream>>>(
        c->rows_k, c->row0_k, c->ML, g, c->d.g[6], c->d.g[7], c->d.g[8], c->d.g[9], c->d.g[10], c->d.g[11], c->d.g[12],
        c->d.expo, c->d.prow);
    return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------
// Pass 1: Floyd sampling of n_f distinct rows per base pair, one warp per (slice, pair)
// ------------------------------------------------------------------------------------------
// lane k < n returns the k-th smallest of Floyd(m, n) keyed by (a, j, slice, tag)
__device__ int warp_floyd(int m, int n, uint32_t a, int s, uint64_t seed, int lane)
{
    int j = m - n + lane;
    int t = -1;
    if (lane < n) {
        uint4 u = philox4(a, (uint32_t)j, (uint32_t)s, TAG_P1, seed);
        t = (int)randint_u(u.x, (uint32_t)(j + 1));
    }
    int elem = -1;
    for (int k = 0; k < n; ++k) {
        int tk = __shfl_sync(FULL_MASK, t, k);
        bool mem = __ballot_sync(FULL_MASK, lane < k && elem == tk) != 0u;
        if (lane == k) elem = mem ? (m - n + k) : tk;
    }
    int rank = 0;
    for (int k = 0; k < n; ++k) {
        int ek = __shfl_sync(FULL_MASK, elem, k);
        rank += (lane < n && ek < elem) ? 1 : 0;
    }
    int out = -1;
    for (int k = 0; k < n; ++k) {
        int ek = __shfl_sync(FULL_MASK, elem, k);
        int rk = __shfl_sync(FULL_MASK, rank, k);
        if (rk == lane) out = ek;
    }
    return out;
}

// Floyd sampling of n distinct rows of [0, m) (any n <= m <= 1024) into the bitmap fb (zeroed by
// the caller): step k (j = m - n + k) draws t = randint(j + 1) with the same Philox counter as
// warp_floyd and inserts t, or j when t is already in the set.  Rounds of 32 steps: lane k draws
// t_k, then the round's inserts are applied in step order with the bitmap as the set.
__device__ void warp_floyd_bm(int m, int n, uint32_t a, int s, uint64_t seed, int lane, uint32_t *fb)
{
    for (int k0 = 0; k0 < n; k0 += 32) {
        const int k = k0 + lane, j = m - n + k;
        int t = 0;
        if (k < n) {
            uint4 u = philox4(a, (uint32_t)j, (uint32_t)s, TAG_P1, seed);
            t = (int)randint_u(u.x, (uint32_t)(j + 1));
        }
        const int kn = min(32, n - k0);
        for (int q = 0; q < kn; ++q) {
            if (lane == q) {
                const int e = ((fb[t >> 5] >> (t & 31)) & 1u) ? j : t;
                fb[e >> 5] |= 1u << (e & 31);
            }
            __syncwarp();
        }
    }
}

// bounding box (lo3, hi3) of each slice's points: exact fp32 min / max (order-free)
__global__ void __launch_bounds__(256) k_slice_bbox(const int32_t *__restrict__ slice_off, int32_t s0, int32_t lbase,
                                                    const float4 *__restrict__ prow, float *sbox)
{
    __shared__ float red[8][6];
    const int ls = blockIdx.x, s = s0 + ls, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int m = slice_off[s + 1] - slice_off[s];
    const int64_t lrow0 = slice_off[s] - lbase;
    float v[6] = {INFINITY, INFINITY, INFINITY, -INFINITY, -INFINITY, -INFINITY};
    for (int i = threadIdx.x; i < m; i += blockDim.x) {
        const float4 A = prow[4 * (lrow0 + i)];
        v[0] = fminf(v[0], A.x); v[1] = fminf(v[1], A.y); v[2] = fminf(v[2], A.z);
        v[3] = fmaxf(v[3], A.x); v[4] = fmaxf(v[4], A.y); v[5] = fmaxf(v[5], A.z);
    }
#pragma unroll
    for (int k = 0; k < 6; ++k)
        for (int o = 16; o > 0; o >>= 1) {
            const float t = __shfl_xor_sync(FULL_MASK, v[k], o);
            v[k] = k < 3 ? fminf(v[k], t) : fmaxf(v[k], t);
        }
    if (lane == 0)
        for (int k = 0; k < 6; ++k) red[w][k] = v[k];
    __syncthreads();
    if (threadIdx.x < 6) {
        const int k = threadIdx.x;
        float r = red[0][k];
        for (int q = 1; q < (int)(blockDim.x >> 5); ++q) r = k < 3 ? fminf(r, red[q][k]) : fmaxf(r, red[q][k]);
        sbox[6 * ls + k] = r;
    }
}

#ifndef P1_MINB
#define P1_MINB 4   // 64 registers, 4 CTAs per SM: pass 1 3.27 -> 2.12 ms at C4 (despite spills)
#endif
#ifndef CO_MINB
#define CO_MINB 3   // 80 registers: coarsening 3.5 -> 3.35 ms at C4 (4: 3.6 ms)
#endif
__global__ void __launch_bounds__(256, P1_MINB) k_pass1(int slot, Upper up, const int32_t *__restrict__ slice_off, int32_t s0, int32_t SL,
                                               int32_t lbase, const float4 *__restrict__ prow,
                                               const float4 *__restrict__ vpl, uint64_t seed, int nmax,
                                               uint16_t *p1_rows, double *p1_Ta, double *p1_Tb, int32_t *p1_cnt,
                                               const float *__restrict__ sbox, unsigned long long *counters)
{
    __shared__ __align__(16) SceneConst sc;
    stage_scene(&sc, slot);   // once per CTA: the CTAs stride over the (slice, pair) warps
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)SL * up.nB, wstride = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; gw < nw; gw += wstride) {
    const int ls = (int)(gw / up.nB), b = (int)(gw % up.nB);
    const int s = s0 + ls;
    const int m = slice_off[s + 1] - slice_off[s];
    const int64_t lrow0 = slice_off[s] - lbase;
    const int f = up.base_list[b];
    const int l = up.left[f], r = up.right[f];
    const int a = (up.rep[l] == up.rep[f]) ? l : r;
    const int bb = (a == l) ? r : l;
    int n = up.nunc[f] < m ? up.nunc[f] : m;
    int row = warp_floyd(m, n, (uint32_t)up.node[f], up.rs0 + ls * up.rss, seed, lane);
    const int va = up.rep[a], vb = up.rep[bb];
    const float4 Pa = vpl[2 * (int64_t)va], Pb = vpl[2 * (int64_t)vb];
    const Cand ca = col_candidates(&sc, sbox + 6 * ls, Pa.x, Pa.y, Pa.z);
    const Cand cb = col_candidates(&sc, sbox + 6 * ls, Pb.x, Pb.y, Pb.z);
    const int64_t o = gw * nmax;
    if (lane < n) p1_rows[o + lane] = (uint16_t)row;
    // the 2n evaluations T(row_j, rep a), T(row_j, rep b) spread over the warp's lanes
    for (int base = 0; base < 2 * n; base += 32) {
        const int j = base + lane;
        const int jr = j < n ? j : j - n;
        const int rj = __shfl_sync(FULL_MASK, row, jr & 31);
        if (j < 2 * n) {
            const Cand &cd = j < n ? ca : cb;
            const double T = entry_T_w(&sc, slot, prow, lrow0 + rj, vpl, j < n ? va : vb, cd.s, cd.b, cd.r);
            if (j < n) p1_Ta[o + j] = T;
            else p1_Tb[o + jr] = T;
        }
    }
    if (lane == 0) {
        p1_cnt[gw] = n;
        atomicAdd(&counters[0], (unsigned long long)(2 * n));
    }
    }
}

cudaError_t run_pass1(lmc_ctx *c)
{
    if (c->SL == 0) return cudaSuccess;
    k_slice_bbox<<<c->SL, 256, 0, c->stream>>>(c->soff_k, c->s0k, c->lbase_k, c->d.prow, c->d.sbox);
    if (c->up.nB == 0) return cudaGetLastError();
    int64_t warps = (int64_t)c->SL * c->up.nB;
    // persistent: P1_MINB resident CTAs per SM stride over the warps (the scene is staged once per CTA)
    unsigned blocks = (unsigned)std::min<int64_t>((warps * 32 + 255) / 256, (int64_t)c->nsm * P1_MINB);
    k_pass1<<<blocks, 256, 0, c->stream>>>(c->scene_slot, c->up, c->soff_k, c->s0k, c->SL, c->lbase_k, c->d.prow,
                                           c->d.vpl, c->cfg.seed, c->nmax, c->d.p1_rows, c->d.p1_Ta, c->d.p1_Tb,
                                           c->d.p1_cnt, c->d.sbox, c->d.counters);
    return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------
// Coarsening: one CTA per slice, level-synchronous over node heights.  A node's
// outcome depends only on its own subtree (fresh rows keyed by node id), so any order over
// candidates of one height gives the reference's cut.
// ------------------------------------------------------------------------------------------
enum { F_INCUT = 1, F_MERGED = 2, F_PROC = 4 };
constexpr int CO_THREADS = 256;
constexpr int CO_WARPS = CO_THREADS / 32;

__device__ __forceinline__ double warp_max_d(double v)
{
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(FULL_MASK, v, o));
    return v;
}

__global__ void __launch_bounds__(CO_THREADS, CO_MINB) k_coarsen(
    int slot, Upper up, const int32_t *__restrict__ slice_off, int32_t s0, int32_t lbase, const float4 *__restrict__ prow,
    const float4 *__restrict__ vpl, uint64_t seed, int nmax, double tau, const uint16_t *__restrict__ p1_rows,
    const double *__restrict__ p1_Ta, const double *__restrict__ p1_Tb, const int32_t *__restrict__ p1_cnt,
    uint16_t *pool_rows, double *pool_Ta, double *pool_Tb, int32_t *pool_used, int64_t pool_cap, uint8_t *cs_flags,
    double *cs_eps, double *cs_cost, int32_t *cs_zoff, int32_t *cs_zlen, int32_t *cut_n, int32_t *cut_cols,
    int32_t *src_off, int32_t *src_len, int32_t *src_side, int G, unsigned long long *counters, int cost_mode,
    int count_target)
{
    extern __shared__ __align__(16) unsigned char smem[];
    const int U = up.U;
    double *sh_cost = (double *)smem;
    double *sh_eps = sh_cost + U;
    int32_t *sh_zoff = (int32_t *)(sh_eps + U);
    int32_t *sh_zlen = sh_zoff + U;
    uint32_t *sh_bm = (uint32_t *)(sh_zlen + U);           // CO_WARPS x 32 words
    uint8_t *sh_flag = (uint8_t *)(sh_bm + CO_WARPS * 32);
    __shared__ int sh_pool;
    __shared__ int sh_scan[CO_THREADS];
    __shared__ uint32_t sh_fbm[CO_WARPS][32];   // per-warp Floyd set of a mixed pair with n > 32

    const int ls = blockIdx.x, s = s0 + ls;
    const int m = slice_off[s + 1] - slice_off[s];
    const int64_t lrow0 = slice_off[s] - lbase;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t pbase = (int64_t)ls * pool_cap;
    for (int u = threadIdx.x; u < U; u += CO_THREADS) {
        sh_flag[u] = up.left[u] < 0 ? F_INCUT : 0;
        sh_cost[u] = 0.0;
        sh_eps[u] = 0.0;
        sh_zoff[u] = 0;
        sh_zlen[u] = 0;
    }
    if (threadIdx.x == 0) sh_pool = 0;
    __syncthreads();
    unsigned long long evals = 0;
    bool overflow = false;
    uint32_t *bm = sh_bm + w * 32;
    // one warp evaluates candidate f (both children in the cut): zeta_f, the entries, eps and
    // cost; `decide` applies the threshold rule right away
    auto eval_cand = [&](const int f, const bool decide) {
        const int l = up.left[f], r = up.right[f];
        if (!((sh_flag[l] & F_INCUT) && (sh_flag[r] & F_INCUT))) return;   // not a candidate
        const int a = (up.rep[l] == up.rep[f]) ? l : r;
        const int b = (a == l) ? r : l;
        const int va = up.rep[a], vb = up.rep[b];
        const double la = up.lum[a], lb = up.lum[b];
        const double ratio = la > 0.0 ? lb / la : 0.0;
        const bool ml = (sh_flag[l] & F_MERGED) != 0, mr = (sh_flag[r] & F_MERGED) != 0;
        int total, off = 0;
        double eps = 0.0;
        if (!ml && !mr) {
            // base pair: rows and entries from pass 1
            const int bi = up.base_of[f];
            const int64_t pi = ((int64_t)ls * up.nB + bi);
            total = p1_cnt[pi];
            if (lane == 0) off = atomicAdd(&sh_pool, total);
            off = __shfl_sync(FULL_MASK, off, 0);
            if (off + total > pool_cap) { overflow = true; return; }
            if (lane < total) {
                int i = p1_rows[pi * nmax + lane];
                double Ta = p1_Ta[pi * nmax + lane], Tb = p1_Tb[pi * nmax + lane];
                pool_rows[pbase + off + lane] = (uint16_t)i;
                pool_Ta[pbase + off + lane] = Ta;
                pool_Tb[pbase + off + lane] = Tb;
                double lr = lum_rho_d(prow, lrow0 + i);
                double Va = (lr * la) * Ta, Vb = (lr * lb) * Tb;
                eps = la > 0.0 ? fabs(Vb - Va * ratio) : fabs(Vb);
            }
        } else {
            // zeta_f = zeta_a U zeta_b (both merged) or zeta_h U Floyd(n(o)) (mixed), R10
            bm[lane] = 0u;
            __syncwarp();
            const int h1 = ml ? l : r;
            {
                int o1 = sh_zoff[h1], n1 = sh_zlen[h1];
                for (int k = lane; k < n1; k += 32) {
                    int i = pool_rows[pbase + o1 + k];
                    atomicOr(&bm[i >> 5], 1u << (i & 31));
                }
            }
            if (ml && mr) {
                int o2 = sh_zoff[r], n2 = sh_zlen[r];
                for (int k = lane; k < n2; k += 32) {
                    int i = pool_rows[pbase + o2 + k];
                    atomicOr(&bm[i >> 5], 1u << (i & 31));
                }
            } else {
                const int o = ml ? r : l;
                int n = up.nunc[o] < m ? up.nunc[o] : m;
                if (n <= 32) {
                    int i = warp_floyd(m, n, (uint32_t)up.node[f], up.rs0 + ls * up.rss, seed, lane);
                    if (lane < n) atomicOr(&bm[i >> 5], 1u << (i & 31));
                } else {   // n(I_o) > 32: an original node brighter than every base pair (P:104 sets no cap)
                    uint32_t *fb = sh_fbm[w];
                    fb[lane] = 0u;
                    __syncwarp();
                    warp_floyd_bm(m, n, (uint32_t)up.node[f], up.rs0 + ls * up.rss, seed, lane, fb);
                    atomicOr(&bm[lane], fb[lane]);
                }
            }
            __syncwarp();
            uint32_t word = bm[lane];
            int cnt = __popc(word), incl = cnt;
            for (int o = 1; o < 32; o <<= 1) {
                int t = __shfl_up_sync(FULL_MASK, incl, o);
                if (lane >= o) incl += t;
            }
            total = __shfl_sync(FULL_MASK, incl, 31);
            if (lane == 0) off = atomicAdd(&sh_pool, total);
            off = __shfl_sync(FULL_MASK, off, 0);
            if (off + total > pool_cap) { overflow = true; return; }
            int pos = off + incl - cnt;
            while (word) {
                int bit = __ffs(word) - 1;
                word &= word - 1;
                pool_rows[pbase + pos++] = (uint16_t)(lane * 32 + bit);
            }
            __syncwarp();
            for (int k = lane; k < total; k += 32) {
                int i = pool_rows[pbase + off + k];
                double Ta = entry_T(slot, prow, lrow0 + i, vpl, va);
                double Tb = entry_T(slot, prow, lrow0 + i, vpl, vb);
                pool_Ta[pbase + off + k] = Ta;
                pool_Tb[pbase + off + k] = Tb;
                double lr = lum_rho_d(prow, lrow0 + i);
                double Va = (lr * la) * Ta, Vb = (lr * lb) * Tb;
                double e = la > 0.0 ? fabs(Vb - Va * ratio) : fabs(Vb);
                eps = fmax(eps, e);
            }
            evals += (lane == 0) ? 2ull * total : 0ull;
        }
        eps = warp_max_d(eps);
        // Eq. (1): cost(L_f) = eps(L_f) + cost(L_b); merge iff below the bound.
        // cost_mode 1 (SURVEY f3 sensitivity): (eps + cost(L_b)) + cost(L_a)
        double cf = eps + sh_cost[b];
        if (cost_mode) cf = cf + sh_cost[a];
        if (lane == 0) {
            sh_eps[f] = eps;
            sh_cost[f] = cf;
            sh_zoff[f] = off;
            sh_zlen[f] = total;
            uint8_t fl = F_PROC;
            if (decide && cf < tau) {
                fl |= F_INCUT | F_MERGED;
                sh_flag[l] &= (uint8_t)~F_INCUT;
                sh_flag[r] &= (uint8_t)~F_INCUT;
            }
            sh_flag[f] = fl;
        }
        __syncwarp();
    };
    if (count_target <= 0) {
        // threshold rule: candidates height by height (a node's outcome depends on its subtree only);
        // the warps take the nodes of a height from a shared counter (merged candidates cost far
        // more than base pairs), counters alternate between heights so one barrier per height stays
        __shared__ int sh_next[2];
        if (threadIdx.x == 0 && up.H >= 1) sh_next[1] = up.hoff[1];
        __syncthreads();
        for (int h = 1; h <= up.H; ++h) {
            if (threadIdx.x == 0 && h < up.H) sh_next[(h + 1) & 1] = up.hoff[h + 1];
            const int hend = up.hoff[h + 1];
            for (;;) {
                int idx = 0;
                if (lane == 0) idx = atomicAdd(&sh_next[h & 1], 1);
                idx = __shfl_sync(FULL_MASK, idx, 0);
                if (idx >= hend) break;
                const int f = up.hlist[idx];
                const int l = up.left[f], r = up.right[f];
                if (!((sh_flag[l] & F_INCUT) && (sh_flag[r] & F_INCUT))) continue;   // not a candidate
                eval_cand(f, true);
            }
            __syncthreads();
        }
    } else {
        // count target (R37): every base pair is evaluated, then the least-cost candidate
        // (ties: smallest node id) merges until the cut has count_target nodes; a merge may make
        // the parent a candidate, evaluated before the next choice
        if (up.H >= 1)
            for (int idx = up.hoff[1] + w; idx < up.hoff[2]; idx += CO_WARPS) eval_cand(up.hlist[idx], false);
        __syncthreads();
        __shared__ int sh_best, sh_pend, sh_cut;
        __shared__ double sh_bc[CO_WARPS];
        __shared__ int sh_bu[CO_WARPS];
        if (threadIdx.x == 0) sh_cut = G;
        __syncthreads();
        for (;;) {
            if (sh_cut <= count_target) break;
            double bc = 0.0;
            int bu = -1;
            for (int u = threadIdx.x; u < U; u += CO_THREADS) {
                const uint8_t fl = sh_flag[u];
                if (!(fl & F_PROC) || (fl & F_MERGED)) continue;
                if (!((sh_flag[up.left[u]] & F_INCUT) && (sh_flag[up.right[u]] & F_INCUT))) continue;
                if (bu < 0 || sh_cost[u] < bc) { bc = sh_cost[u]; bu = u; }   // u ascending: first = smallest id
            }
            for (int o = 16; o > 0; o >>= 1) {
                const double oc = __shfl_xor_sync(FULL_MASK, bc, o);
                const int ou = __shfl_xor_sync(FULL_MASK, bu, o);
                if (ou >= 0 && (bu < 0 || oc < bc || (oc == bc && ou < bu))) { bc = oc; bu = ou; }
            }
            if (lane == 0) { sh_bc[w] = bc; sh_bu[w] = bu; }
            __syncthreads();
            if (threadIdx.x == 0) {
                double c2 = 0.0;
                int u2 = -1;
                for (int k = 0; k < CO_WARPS; ++k) {
                    const int ou = sh_bu[k];
                    if (ou >= 0 && (u2 < 0 || sh_bc[k] < c2 || (sh_bc[k] == c2 && ou < u2))) { c2 = sh_bc[k]; u2 = ou; }
                }
                sh_best = u2;
                sh_pend = -1;
                if (u2 >= 0) {
                    sh_flag[up.left[u2]] &= (uint8_t)~F_INCUT;
                    sh_flag[up.right[u2]] &= (uint8_t)~F_INCUT;
                    sh_flag[u2] |= F_INCUT | F_MERGED;
                    sh_cut -= 1;
                    const int p = up.parent[u2];
                    if (p >= 0) {
                        const int sib = up.left[p] == u2 ? up.right[p] : up.left[p];
                        if (sh_flag[sib] & F_INCUT) sh_pend = p;
                    }
                }
            }
            __syncthreads();
            if (sh_best < 0) break;
            if (sh_pend >= 0 && w == 0) eval_cand(sh_pend, false);
            __syncthreads();
        }
    }
    if (lane == 0 && evals) atomicAdd(&counters[1], evals);
    if (overflow) atomicOr(&counters[3], 1ull);
    // write the per-node record
    const int64_t nb = (int64_t)ls * U;
    for (int u = threadIdx.x; u < U; u += CO_THREADS) {
        cs_flags[nb + u] = sh_flag[u];
        cs_eps[nb + u] = sh_eps[u];
        cs_cost[nb + u] = sh_cost[u];
        cs_zoff[nb + u] = sh_zoff[u];
        cs_zlen[nb + u] = sh_zlen[u];
    }
    // final cut in ascending node id (= local id) order, with each column's carried-sample source
    const int per = (U + CO_THREADS - 1) / CO_THREADS;
    const int u0 = threadIdx.x * per;
    int mine = 0;
    for (int u = u0; u < u0 + per && u < U; ++u) mine += (sh_flag[u] & F_INCUT) ? 1 : 0;
    sh_scan[threadIdx.x] = mine;
    __syncthreads();
    for (int o = 1; o < CO_THREADS; o <<= 1) {
        int t = threadIdx.x >= o ? sh_scan[threadIdx.x - o] : 0;
        __syncthreads();
        sh_scan[threadIdx.x] += t;
        __syncthreads();
    }
    int col = sh_scan[threadIdx.x] - mine;
    if (threadIdx.x == CO_THREADS - 1) {
        cut_n[ls] = sh_scan[threadIdx.x];
        atomicMax(&counters[5], (unsigned long long)sh_scan[threadIdx.x]);
    }
    const int64_t cb = (int64_t)ls * G;
    for (int u = u0; u < u0 + per && u < U; ++u) {
        if (!(sh_flag[u] & F_INCUT)) continue;
        cut_cols[cb + col] = u;
        int p = up.parent[u];
        int so = 0, sl = 0, sd = 0;
        if (p >= 0 && (sh_flag[p] & F_PROC)) {
            int ap = (up.rep[up.left[p]] == up.rep[p]) ? up.left[p] : up.right[p];
            so = sh_zoff[p];
            sl = sh_zlen[p];
            sd = (u == ap) ? 0 : 1;
        } else if (sh_flag[u] & F_MERGED) {
            so = sh_zoff[u];
            sl = sh_zlen[u];
            sd = 0;
        }
        src_off[cb + col] = so;
        src_len[cb + col] = sl;
        src_side[cb + col] = sd;
        ++col;
    }
    if (threadIdx.x == 0) {
        pool_used[ls] = sh_pool;
        atomicMax(&counters[4], (unsigned long long)sh_pool);
    }
}

static size_t coarsen_smem(int U) { return (size_t)U * (8 + 8 + 4 + 4) + CO_WARPS * 32 * 4 + (size_t)U + 16; }

cudaError_t run_coarsen(lmc_ctx *c)
{
    if (c->SL == 0) return cudaSuccess;
    size_t sm = coarsen_smem(c->up.U);
    cudaError_t e = cudaFuncSetAttribute(k_coarsen, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    k_coarsen<<<c->SL, CO_THREADS, sm, c->stream>>>(
        c->scene_slot, c->up, c->soff_k, c->s0k, c->lbase_k, c->d.prow, c->d.vpl, c->cfg.seed, c->nmax,
        c->cfg.coarsen_tau, c->d.p1_rows, c->d.p1_Ta, c->d.p1_Tb, c->d.p1_cnt, c->d.pool_rows, c->d.pool_Ta,
        c->d.pool_Tb, c->d.pool_used, c->pool_cap, c->d.cs_flags, c->d.cs_eps, c->d.cs_cost, c->d.cs_zoff,
        c->d.cs_zlen, c->d.cut_n, c->d.cut_cols, c->d.src_off, c->d.src_len, c->d.src_side, c->G, c->d.counters,
        c->cfg.cost_mode, c->cfg.coarsen_target);
    return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------
// Pass 2: one CTA (1024 threads) per slice; the observed-cell bitmap lives in
// shared memory (m x n <= 2^20 bits).
// ------------------------------------------------------------------------------------------
constexpr int P2_THREADS = 1024;
constexpr unsigned P2_INVALID = 0xFFFFFFFFu; // empty hash slot / no candidate (cells < 2^21)
constexpr int P2_HBITS = 11;
constexpr int P2_HSLOTS = 1 << P2_HBITS;     // 2 x P2_THREADS hash slots
#ifndef P2_FAST_DRAWS
#define P2_FAST_DRAWS 4
#endif
constexpr int P2_FAST = P2_FAST_DRAWS;       // draws per thread in a fast (uncut) batch

struct P2Args {
    Upper up;
    const int32_t *slice_off;
    int32_t s0, lbase, G;
    const float4 *prow;
    uint64_t seed;
    double rate;
    const int32_t *cut_n, *cut_cols, *src_off, *src_len, *src_side;
    const uint16_t *pool_rows;
    const double *pool_Ta, *pool_Tb;
    int64_t pool_cap, ncap;
    int mmax;
    int32_t *rowptr;
    uint16_t *col;
    float *val;
    double *val64;                 // fp64 copy of the values (masked ALS only), else null
    uint8_t *carried;
    int32_t *colptr;
    uint16_t *csc_row;
    int32_t *csc_src;
    int32_t *nnz, *target_n, *n_new;
    unsigned long long *counters;
    int row_importance;            // rows drawn by f(i) = max - min of their carried entries
};

// smallest i with rcdf[i] > y (R29)
__device__ __forceinline__ int row_pick(const unsigned long long *rcdf, int m, unsigned long long y)
{
    int lo = 0, hi = m - 1;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (rcdf[mid] > y) hi = mid; else lo = mid + 1;
    }
    return lo;
}

__device__ __forceinline__ int csr_pos(const uint32_t *bm, int Wb, const uint16_t *P, const int32_t *rp, int W, int i, int c)
{
    const int wi = c >> 5;
    return rp[i] + P[i * (W + 1) + wi] + __popc(bm[i * Wb + wi] & ((1u << (c & 31)) - 1u));
}

// P2_PROF (diagnostic build): block-cycles per phase of k_pass2, printed by run_pass2
#ifdef P2_PROF
#define P2T(k) do { __syncthreads(); if (threadIdx.x == 0) { long long t_ = clock64(); if (k > 0) atomicAdd(&A.counters[8 + (k) - 1], (unsigned long long)(t_ - p2t0)); p2t0 = t_; } } while (0)
#else
#define P2T(k) do { } while (0)
#endif
__global__ void __launch_bounds__(P2_THREADS, 1) k_pass2(P2Args A)
{
#ifdef P2_PROF
    long long p2t0 = 0;
#endif
    extern __shared__ __align__(16) unsigned char smem[];
    typedef cub::BlockScan<int32_t, P2_THREADS> ScanI;
    typedef cub::BlockScan<unsigned long long, P2_THREADS> ScanU;
    const int ls = blockIdx.x, s = A.s0 + ls, tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const uint32_t srng = (uint32_t)(A.up.rs0 + ls * A.up.rss);   // global slice id: the draws' key
    const int m = A.slice_off[s + 1] - A.slice_off[s];
    const int n = A.cut_n[ls];
    const int64_t lrow0 = A.slice_off[s] - A.lbase;
    const int W = (n + 31) >> 5;
    const int Wb = W | 1;   // bitmap row stride in words: odd, so a warp reading one word of 32 rows is conflict-free
    const int64_t cb = (int64_t)ls * A.G, pb = (int64_t)ls * A.pool_cap, ob = (int64_t)ls * A.ncap;
    // shared memory carve-up
    uint32_t *bm = (uint32_t *)smem;                                    // m * Wb
    int32_t *colcnt = (int32_t *)(bm + (size_t)A.mmax * 33);            // G
    unsigned char *phase = smem + ((((size_t)A.mmax * 33 + A.G) * 4 + 15) & ~(size_t)15);   // 16-byte aligned (odd G)
    // phase A
    unsigned long long *cdf = (unsigned long long *)phase;              // G (also holds g as double)
    uint32_t *hkey = (uint32_t *)(cdf + A.G);                           // P2_HSLOTS
    uint32_t *hmin = hkey + P2_HSLOTS;                                  // P2_HSLOTS
    // row importance (A.row_importance): per row max (bits, then the row CDF), min (bits), count
    unsigned long long *rcdf = (unsigned long long *)(hmin + P2_HSLOTS);   // mmax
    unsigned long long *rlo = rcdf + A.mmax;                            // mmax
    int32_t *rcnt = (int32_t *)(rlo + A.mmax);                          // mmax
    __shared__ typename ScanI::TempStorage scani_tmp;
    __shared__ typename ScanU::TempStorage scanu_tmp;
    // phase B
    uint16_t *P = (uint16_t *)phase;                                    // m*(W+1)
    int32_t *rp = (int32_t *)(P + (((size_t)A.mmax * 33 + 7) & ~(size_t)7));  // m+1
    __shared__ double sh_dred[32];
    __shared__ unsigned long long sh_ured[32];
    __shared__ int sh_ired[32];
    __shared__ int sh_count, sh_obs, sh_nnew, sh_draws, sh_bacc;
    __shared__ int sh_cpre[P2_THREADS];   // per-column prefix offsets (carried entries, CSC)
    __shared__ int sh_guide[257];         // CDF guide table of the draws

    for (int k = tid; k < m * Wb; k += P2_THREADS) bm[k] = 0u;
    for (int c = tid; c < n; c += P2_THREADS) colcnt[c] = 0;
    if (A.row_importance)
        for (int i = tid; i < m; i += P2_THREADS) { rcdf[i] = 0ull; rlo[i] = 0x7FF0000000000000ull; rcnt[i] = 0; }
    __syncthreads();
    P2T(0);
    // carried observations (R13) and light importance g(c) = max C_c - min C_c.
    // The carried entries of all columns form one flat list (prefix of the per-column counts), so
    // all threads work on them at once; values are >= +0, so their bit patterns order like the
    // values and the per-column max / min are integer atomics (order-free: exact).
    double *gcol = (double *)cdf;
    unsigned long long *chi = (unsigned long long *)cdf;   // per column max (bits), then g
    unsigned long long *clo = (unsigned long long *)hkey;  // per column min (bits); hash area is free
    int obs_local = 0;
    {
        const int sl_t = tid < n ? A.src_len[cb + tid] : 0;
        int pre, tot;
        ScanI(scani_tmp).ExclusiveSum(sl_t, pre, tot);
        if (tid < n) {
            sh_cpre[tid] = pre;
            colcnt[tid] = sl_t;
            chi[tid] = 0ull;
            clo[tid] = 0x7FF0000000000000ull;   // +inf
        }
        if (tid == 0) obs_local = tot;
        __syncthreads();
        for (int e = tid; e < tot; e += P2_THREADS) {
            int lo = 0, hi = n - 1;   // last column whose entries start at or before e
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (sh_cpre[mid] <= e) lo = mid; else hi = mid - 1;
            }
            const int c = lo, k = e - sh_cpre[c];
            const int so = A.src_off[cb + c], sd = A.src_side[cb + c];
            const double lI = A.up.lum[A.cut_cols[cb + c]];
            const double *Tv = sd ? A.pool_Tb : A.pool_Ta;
            const int i = A.pool_rows[pb + so + k];
            const double v = (lum_rho_d(A.prow, lrow0 + i) * lI) * Tv[pb + so + k];
            const unsigned long long vb = (unsigned long long)__double_as_longlong(v);
            atomicMax(&chi[c], vb);
            atomicMin(&clo[c], vb);
            atomicOr(&bm[i * Wb + (c >> 5)], 1u << (c & 31));
            if (A.row_importance) {
                atomicMax(&rcdf[i], vb);
                atomicMin(&rlo[i], vb);
                atomicAdd(&rcnt[i], 1);
            }
        }
        __syncthreads();
        if (tid < n) {
            const int sl = colcnt[tid];
            const double hv = __longlong_as_double((long long)chi[tid]), lv = __longlong_as_double((long long)clo[tid]);
            gcol[tid] = sl > 0 ? hv - lv : -1.0;
        }
    }
    __syncthreads();
    P2T(1);
    // G = max g; integer weights (R14)
    double gmax = 0.0;
    for (int c = tid; c < n; c += P2_THREADS) gmax = fmax(gmax, gcol[c]);
    gmax = warp_max_d(gmax);
    if (lane == 0) sh_dred[w] = gmax;
    int obs_w = obs_local;
    for (int o = 16; o > 0; o >>= 1) obs_w += __shfl_xor_sync(FULL_MASK, obs_w, o);
    if (lane == 0) sh_ired[w] = obs_w;
    __syncthreads();
    if (tid == 0) {
        double gm = 0.0;
        int ob = 0;
        for (int k = 0; k < 32; ++k) { gm = fmax(gm, sh_dred[k]); ob += sh_ired[k]; }
        sh_dred[0] = gm;
        sh_obs = ob;
    }
    __syncthreads();
    const double Gm = sh_dred[0];
    unsigned long long wc = 0ull;
    int observed = 0;
    if (tid < n) {
        double gc = gcol[tid];
        observed = gc >= 0.0;
        if (Gm > 0.0) {
            if (observed) {
                double x = floor(1048575.0 * (gc / Gm));
                uint32_t ww = 1u + (uint32_t)x;
                wc = ww > 65536u ? ww : 65536u;
            }
        } else {
            wc = 1ull;
        }
    }
    __syncthreads();   // gcol (aliases cdf) fully read
    unsigned long long sumw = observed ? wc : 0ull;
    for (int o = 16; o > 0; o >>= 1) sumw += __shfl_xor_sync(FULL_MASK, sumw, o);
    int nobs = observed;
    for (int o = 16; o > 0; o >>= 1) nobs += __shfl_xor_sync(FULL_MASK, nobs, o);
    if (lane == 0) { sh_ured[w] = sumw; sh_ired[w] = nobs; }
    __syncthreads();
    if (tid < n && Gm > 0.0 && !observed) {
        unsigned long long sw = 0ull;
        int no = 0;
        for (int k = 0; k < 32; ++k) { sw += sh_ured[k]; no += sh_ired[k]; }
        wc = no ? (unsigned long long)(uint32_t)(sw / (unsigned long long)no) : 524288ull;
    }
    unsigned long long incl;
    ScanU(scanu_tmp).InclusiveSum(wc, incl);
    __syncthreads();
    if (tid < n) cdf[tid] = incl;
    __syncthreads();
    const unsigned long long Wsum = n > 0 ? cdf[n - 1] : 0ull;
    // guide table of the CDF inversion: for the draws whose u has top byte j, x = (u W) >> 32 lies
    // in [(j W) >> 8, ((j + 1) W) >> 8], so the column is in [guide[j], guide[j + 1]] with guide[j] =
    // the smallest c with CDF_c > (j W) >> 8 (guide[256] = n - 1): the same smallest c with CDF_c > x
    // (R29) after a search over a few columns instead of all n
    if (tid <= 256 && n > 0) {
        int c = n - 1;
        if (tid < 256) {
            const unsigned long long xl = ((unsigned long long)tid * Wsum) >> 8;
            int lo = 0, hi = n - 1;
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (cdf[mid] > xl) hi = mid; else lo = mid + 1;
            }
            c = lo;
        }
        sh_guide[tid] = c;
    }
    __syncthreads();
    // row weights by the rule of the column weights (R14) on f(i) = max - min of row i's carried
    // entries, and the row CDF (DESIGN R36); m <= 1024 = one row per thread
    unsigned long long Wr = 0ull;
    if (A.row_importance) {
        double fi = -1.0;
        if (tid < m && rcnt[tid] > 0)
            fi = __longlong_as_double((long long)rcdf[tid]) - __longlong_as_double((long long)rlo[tid]);
        double fm = warp_max_d(fmax(fi, 0.0));
        if (lane == 0) sh_dred[w] = fm;
        __syncthreads();
        if (tid == 0) {
            double v = 0.0;
            for (int k = 0; k < 32; ++k) v = fmax(v, sh_dred[k]);
            sh_dred[0] = v;
        }
        __syncthreads();
        const double Fm = sh_dred[0];
        const int robs = fi >= 0.0;
        unsigned long long wr = 0ull;
        if (tid < m) {
            if (Fm > 0.0) {
                if (robs) {
                    double xx = floor(1048575.0 * (fi / Fm));
                    uint32_t ww = 1u + (uint32_t)xx;
                    wr = ww > 65536u ? ww : 65536u;
                }
            } else {
                wr = 1ull;
            }
        }
        unsigned long long sw = robs ? wr : 0ull;
        for (int o = 16; o > 0; o >>= 1) sw += __shfl_xor_sync(FULL_MASK, sw, o);
        int no = robs;
        for (int o = 16; o > 0; o >>= 1) no += __shfl_xor_sync(FULL_MASK, no, o);
        __syncthreads();
        if (lane == 0) { sh_ured[w] = sw; sh_ired[w] = no; }
        __syncthreads();
        if (tid < m && Fm > 0.0 && !robs) {
            unsigned long long s2 = 0ull;
            int n2 = 0;
            for (int k = 0; k < 32; ++k) { s2 += sh_ured[k]; n2 += sh_ired[k]; }
            wr = n2 ? (unsigned long long)(uint32_t)(s2 / (unsigned long long)n2) : 524288ull;
        }
        unsigned long long rincl;
        ScanU(scanu_tmp).InclusiveSum(wr, rincl);
        __syncthreads();
        if (tid < m) rcdf[tid] = rincl;
        __syncthreads();
        Wr = m > 0 ? rcdf[m - 1] : 0ull;
    }
    P2T(2);
    const int64_t N = (int64_t)ceil(((double)((int64_t)m * (int64_t)n)) * A.rate);
    const int64_t cap = 64 * N;
    if (tid == 0) { sh_count = sh_obs; sh_nnew = 0; sh_draws = 0; sh_bacc = 0; }
    for (int e = tid; e < P2_HSLOTS; e += P2_THREADS) { hkey[e] = P2_INVALID; hmin[e] = 0xFFFFFFFFu; }
    __syncthreads();
    // draws: column by the CDF, row uniformly; skip observed entries (R15, R16).  The
    // accepted set is the first N - |carried| distinct unobserved cells in draw order.  While the
    // budget left is at least a whole fast batch (P2_FAST draws per thread), no draw of the batch can
    // be cut off, so every new cell of the batch is accepted and duplicates resolve by atomicOr on
    // the bitmap in any order (same set).  The last batches take the
    // exact path: first occurrence per cell by smallest draw index, cut off at the budget.
    for (int64_t t0 = 0; t0 < cap;) {
        const int count = sh_count;
        if (count >= N) break;
        if (N - count >= (int64_t)P2_FAST * P2_THREADS) {
#pragma unroll
            for (int u = 0; u < P2_FAST; ++u) {
                const int64_t t = t0 + (int64_t)u * P2_THREADS + tid;
                bool isnew = false;
                int cc = 0;
                if (t < cap && n > 0) {
                    uint4 uu = philox4((uint32_t)t, 0u, srng, TAG_P2, A.seed);
                    unsigned long long x = ((unsigned long long)uu.x * Wsum) >> 32;
                    int lo = sh_guide[uu.x >> 24], hi = sh_guide[(uu.x >> 24) + 1];
                    while (lo < hi) {
                        int mid = (lo + hi) >> 1;
                        if (cdf[mid] > x) hi = mid; else lo = mid + 1;
                    }
                    cc = lo;
                    const int i = A.row_importance ? row_pick(rcdf, m, ((unsigned long long)uu.y * Wr) >> 32)
                                                   : (int)randint_u(uu.y, (uint32_t)m);
                    const uint32_t bit = 1u << (cc & 31);
                    isnew = !(atomicOr(&bm[i * Wb + (cc >> 5)], bit) & bit);
                }
                const unsigned bal = __ballot_sync(FULL_MASK, isnew);
                if (lane == 0 && bal) atomicAdd(&sh_bacc, __popc(bal));
                if (isnew) atomicAdd(&colcnt[cc], 1);
            }
            __syncthreads();
            if (tid == 0) { sh_count = count + sh_bacc; sh_bacc = 0; }
            __syncthreads();
            t0 += (int64_t)P2_FAST * P2_THREADS;
            continue;
        }
        const int64_t t = t0 + tid;
        t0 += P2_THREADS;
        uint32_t key = P2_INVALID;
        int cell = 0, cc = 0;
        if (t < cap && n > 0) {
            uint4 u = philox4((uint32_t)t, 0u, srng, TAG_P2, A.seed);
            unsigned long long x = ((unsigned long long)u.x * Wsum) >> 32;
            int lo = sh_guide[u.x >> 24], hi = sh_guide[(u.x >> 24) + 1];
            while (lo < hi) {
                int mid = (lo + hi) >> 1;
                if (cdf[mid] > x) hi = mid; else lo = mid + 1;
            }
            cc = lo;
            int i = A.row_importance ? row_pick(rcdf, m, ((unsigned long long)u.y * Wr) >> 32) : (int)randint_u(u.y, (uint32_t)m);
            cell = (i << 11) | cc;   // i < 1024, cc < 2048
            if (!(bm[i * Wb + (cc >> 5)] & (1u << (cc & 31)))) key = (uint32_t)cell;
        }
        // first occurrence of each new cell within the batch: a shared hash table keeps the
        // smallest draw index per cell (linear probing, 2 x P2_THREADS slots)
        int slot = -1;
        if (key != P2_INVALID) {
            uint32_t h = (key * 2654435761u) >> (32 - P2_HBITS);
            for (;;) {
                const uint32_t old = atomicCAS(&hkey[h], P2_INVALID, key);
                if (old == P2_INVALID || old == key) break;
                h = (h + 1) & (P2_HSLOTS - 1);
            }
            atomicMin(&hmin[h], (uint32_t)tid);
            slot = (int)h;
        }
        __syncthreads();
        const int acc = (slot >= 0 && hmin[slot] == (uint32_t)tid) ? 1 : 0;
        int pre, tot;
        ScanI(scani_tmp).ExclusiveSum(acc, pre, tot);
        for (int e = tid; e < P2_HSLOTS; e += P2_THREADS) { hkey[e] = P2_INVALID; hmin[e] = 0xFFFFFFFFu; }
        const int64_t remaining = N - count;
        const bool accept = acc && pre < remaining;
        if (accept) {
            atomicOr(&bm[(cell >> 11) * Wb + (cc >> 5)], 1u << (cc & 31));
            atomicAdd(&colcnt[cc], 1);
            if (pre == remaining - 1) sh_draws = (int)(t + 1);
        }
        __syncthreads();
        if (tid == 0) sh_count = count + (int)(tot < remaining ? tot : remaining);
        __syncthreads();
    }
    P2T(3);
    // one forced entry per still-empty column (R17)
    int nd = sh_count - sh_obs;
    {
        int need = 0, cell = 0;
        if (tid < n && colcnt[tid] == 0) {
            uint4 u = philox4((uint32_t)tid, 0u, srng, TAG_FORCE, A.seed);
            int i = (int)randint_u(u.x, (uint32_t)m);
            cell = (i << 11) | tid;
            need = 1;
        }
        int pre, tot;
        ScanI(scani_tmp).ExclusiveSum(need, pre, tot);
        if (need) {
            int c = cell & 2047;
            atomicOr(&bm[(cell >> 11) * Wb + (c >> 5)], 1u << (c & 31));
            colcnt[c] = 1;
        }
        __syncthreads();
        if (tid == 0) {
            sh_nnew = nd + tot;
            if (sh_draws == 0) sh_draws = (int)(sh_count >= N ? 0 : cap);
        }
        __syncthreads();
    }
    const int nnew = sh_nnew;
    const int nnz = sh_obs + nnew;
    P2T(4);
    // phase B: CSR row pointers from per-row word prefix counts.  A warp per row: lane wi takes
    // bitmap word wi (W <= 32), the word prefix is a warp scan, so the row's column indices are
    // then written by all lanes at once in ascending order (consecutive lanes, consecutive ranges).
    for (int i = w; i < m; i += P2_THREADS / 32) {
        const uint32_t word = lane < W ? bm[i * Wb + lane] : 0u;
        const int cnt = __popc(word);
        int incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(FULL_MASK, incl, o);
            if (lane >= o) incl += t;
        }
        if (lane < W) P[i * (W + 1) + lane] = (uint16_t)(incl - cnt);
        if (lane == 31) {
            P[i * (W + 1) + W] = (uint16_t)incl;
            rp[i] = incl;   // row total (the row pointers replace it below)
        }
    }
    __syncthreads();
    const int rowtot = tid < m ? rp[tid] : 0;
    __syncthreads();
    int rpre, rtot;
    ScanI(scani_tmp).ExclusiveSum(rowtot, rpre, rtot);
    if (tid < m) rp[tid] = rpre;
    if (tid == 0) rp[m] = rtot;
    __syncthreads();
    int32_t *grp = A.rowptr + (int64_t)ls * (A.mmax + 1);
    for (int i = tid; i <= m; i += P2_THREADS) grp[i] = rp[i];
    for (int i = w; i < m; i += P2_THREADS / 32) {   // column indices, ascending within the row
        if (lane < W) {
            uint32_t word = bm[i * Wb + lane];
            int pos = rp[i] + P[i * (W + 1) + lane];
            while (word) {
                const int bit = __ffs(word) - 1;
                word &= word - 1;
                A.carried[ob + pos] = 0;   // the carried pass below sets the carried entries' flags
                A.col[ob + pos++] = (uint16_t)(lane * 32 + bit);
            }
        }
    }
    P2T(5);
    // CSC: column pointers, rows ascending within a column, CSR index of each entry
    int cpre, ctot;
    int cc0 = tid < n ? colcnt[tid] : 0;
    ScanI(scani_tmp).ExclusiveSum(cc0, cpre, ctot);
    int32_t *gcp = A.colptr + (int64_t)ls * (A.G + 1);
    if (tid < n) gcp[tid] = cpre;
    if (tid == 0) gcp[n] = ctot;
    sh_cpre[tid] = cpre;
    __syncthreads();
    // a warp per column: the lanes test bit c of 32 rows at a time, and the set rows are written in
    // ascending order by consecutive lanes (coalesced stores of csc_row / csc_src)
    for (int c = w; c < n; c += P2_THREADS / 32) {
        const int wi = c >> 5;
        const uint32_t bit = 1u << (c & 31);
        int k = sh_cpre[c];
        for (int r0 = 0; r0 < m; r0 += 128) {   // 4 blocks of 32 rows: their loads in flight together
            uint32_t wd[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int i = r0 + 32 * u + lane;
                wd[u] = i < m ? bm[i * Wb + wi] : 0u;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int i = r0 + 32 * u + lane;
                const bool set = (wd[u] & bit) != 0u;
                const unsigned bal = __ballot_sync(FULL_MASK, set);
                if (set) {
                    const int kk = k + __popc(bal & ((1u << lane) - 1u));
                    A.csc_row[ob + kk] = (uint16_t)i;
                    A.csc_src[ob + kk] = rp[i] + P[i * (W + 1) + wi] + __popc(wd[u] & (bit - 1u));
                }
                k += __popc(bal);
            }
        }
    }
    P2T(6);
    // carried values at their CSR positions (flat list over all columns, as above)
    {
        const int sl_t = tid < n ? A.src_len[cb + tid] : 0;
        int pre, tot;
        __syncthreads();   // sh_cpre of the CSC pass fully read
        ScanI(scani_tmp).ExclusiveSum(sl_t, pre, tot);
        if (tid < n) sh_cpre[tid] = pre;
        __syncthreads();
        for (int e = tid; e < tot; e += P2_THREADS) {
            int lo = 0, hi = n - 1;
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (sh_cpre[mid] <= e) lo = mid; else hi = mid - 1;
            }
            const int c = lo, k = e - sh_cpre[c];
            const int so = A.src_off[cb + c], sd = A.src_side[cb + c];
            const double lI = A.up.lum[A.cut_cols[cb + c]];
            const double *Tv = sd ? A.pool_Tb : A.pool_Ta;
            const int i = A.pool_rows[pb + so + k];
            const double v = (lum_rho_d(A.prow, lrow0 + i) * lI) * Tv[pb + so + k];
            const int pos = csr_pos(bm, Wb, P, rp, W, i, c);
            A.val[ob + pos] = (float)v;
            if (A.val64) A.val64[ob + pos] = v;
            A.carried[ob + pos] = 1;
        }
    }
    P2T(7);
    // new entries: their values are evaluated by k_eval_new in CSC order (carried flag 0)
    P2T(8);
    if (tid == 0) {
        A.nnz[ls] = nnz;
        A.target_n[ls] = (int32_t)N;
        A.n_new[ls] = nnew;
        if (nnz > A.ncap) atomicOr(&A.counters[3], 2ull);
    }
}

// Pass-2 entry values, column by column (a warp per column of a slice, lanes over the column's
// entries in CSC order, carried entries skipped): every lane of a warp shares the column's VPL,
// so the visibility screens run over the column's candidate primitives only, uniformly across the
// warp.  Candidates: primitives whose bounds meet the box of the slice's points and the VPL,
// widened by the screening margin.  Every segment from a point of the slice to the VPL lies in
// that box, and an exact hit lies on the primitive, so a primitive left out cannot hit: the
// decision is the same OR over primitives as before.
#ifndef EV_WARPS_PER_BLOCK
#define EV_WARPS_PER_BLOCK 8
#endif
constexpr int EV_WARPS = EV_WARPS_PER_BLOCK;
#ifndef EV_MINB
#define EV_MINB 4   // 64 registers: 4 blocks per SM (measured 7.6 -> 5.5 ms at C4 against 1)
#endif
__global__ void __launch_bounds__(EV_WARPS * 32, EV_MINB) k_eval_new(int slot, Upper up, const int32_t *__restrict__ slice_off, int32_t s0,
                                                  int32_t lbase, int G, const float4 *__restrict__ prow,
                                                  const float4 *__restrict__ vpl, const int32_t *__restrict__ cut_n,
                                                  const int32_t *__restrict__ cut_cols, const int32_t *__restrict__ colptr,
                                                  const uint16_t *__restrict__ csc_row, const int32_t *__restrict__ csc_src,
                                                  const uint8_t *__restrict__ carried, const int32_t *__restrict__ n_new,
                                                  const float *__restrict__ sbox,
                                                  float *val, double *val64, int64_t ncap, unsigned long long *counters)
{
    __shared__ __align__(16) SceneConst sc;
    stage_scene(&sc, slot);
    const int ls = blockIdx.y, s = s0 + ls, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int n = cut_n[ls];
    const int64_t lrow0 = slice_off[s] - lbase;
    const int64_t ob = (int64_t)ls * ncap, cb = (int64_t)ls * G;
    const int32_t *cp = colptr + (int64_t)ls * (G + 1);
    const float *bx = sbox + 6 * ls;
    for (int c = blockIdx.x * EV_WARPS + w; c < n; c += gridDim.x * EV_WARPS) {
        const int u = cut_cols[cb + c];
        const int v = up.rep[u];
        const float4 P = vpl[2 * (int64_t)v];
        const Cand cd = col_candidates(&sc, bx, P.x, P.y, P.z);
        const double lu = up.lum[u];
        const int k1 = cp[c + 1];
        // the CSR position and row of the next 32 entries are loaded one batch ahead, so only
        // the carried-flag load is exposed before the evaluation
        int k0 = cp[c];
        int pos_n = 0, row_n = 0;
        if (k0 + lane < k1) { pos_n = csc_src[ob + k0 + lane]; row_n = csc_row[ob + k0 + lane]; }
        for (; k0 < k1; k0 += 32) {
            const bool in = k0 + lane < k1;
            const int pos = pos_n, i = row_n;
            const bool todo = in && !carried[ob + pos];
            if (k0 + 32 + lane < k1) { pos_n = csc_src[ob + k0 + 32 + lane]; row_n = csc_row[ob + k0 + 32 + lane]; }
            if (!__any_sync(FULL_MASK, todo)) continue;
            if (todo) {
                const double T = entry_T_w(&sc, slot, prow, lrow0 + i, vpl, v, cd.s, cd.b, cd.r);
                const double val_d = (lum_rho_d(prow, lrow0 + i) * lu) * T;
                val[ob + pos] = (float)val_d;
                if (val64) val64[ob + pos] = val_d;
            }
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(&counters[2], (unsigned long long)n_new[ls]);
}

static size_t pass2_smem(int mmax, int G)
{
    size_t phaseA = (size_t)G * 8 + (size_t)P2_HSLOTS * 4 * 2 + (size_t)mmax * 20;   // + row importance
    size_t phaseB = ((((size_t)mmax * 33 + 7) & ~(size_t)7) * 2) + ((size_t)mmax + 1) * 4;
    size_t base = (((size_t)mmax * 33 + G) * 4 + 15) & ~(size_t)15;
    return base + (phaseA > phaseB ? phaseA : phaseB) + 64;
}

cudaError_t run_pass2(lmc_ctx *c)
{
    if (c->SL == 0) return cudaSuccess;
    P2Args A;
    A.up = c->up;
    A.slice_off = c->soff_k;
    A.s0 = c->s0k;
    A.lbase = c->lbase_k;
    A.G = c->G;
    A.prow = c->d.prow;
    A.seed = c->cfg.seed;
    A.rate = c->cfg.rate;
    A.cut_n = c->d.cut_n;
    A.cut_cols = c->d.cut_cols;
    A.src_off = c->d.src_off;
    A.src_len = c->d.src_len;
    A.src_side = c->d.src_side;
    A.pool_rows = c->d.pool_rows;
    A.pool_Ta = c->d.pool_Ta;
    A.pool_Tb = c->d.pool_Tb;
    A.pool_cap = c->pool_cap;
    A.ncap = c->ncap;
    A.mmax = c->mmax;
    A.rowptr = c->d.rowptr;
    A.col = c->d.col;
    A.val = c->d.val;
    A.val64 = c->d.val64;
    A.carried = c->d.carried;
    A.colptr = c->d.colptr;
    A.csc_row = c->d.csc_row;
    A.csc_src = c->d.csc_src;
    A.nnz = c->d.nnz;
    A.target_n = c->d.target_n;
    A.n_new = c->d.n_new;
    A.counters = c->d.counters;
    A.row_importance = c->cfg.row_importance;
    size_t sm = pass2_smem(c->mmax, c->G);
    cudaError_t e = cudaFuncSetAttribute(k_pass2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) {
        cudaFuncAttributes fa;
        cudaFuncGetAttributes(&fa, k_pass2);
        fprintf(stderr, "lmc: k_pass2 needs %zu + %zu bytes of shared memory (limit %d)\n", sm, (size_t)fa.sharedSizeBytes,
                fa.maxDynamicSharedSizeBytes);
        return e;
    }
    k_pass2<<<c->SL, P2_THREADS, sm, c->stream>>>(A);
#ifdef P2_PROF
    {
        cudaStreamSynchronize(c->stream);
        unsigned long long h[8];
        cudaMemcpy(h, c->d.counters + 8, sizeof h, cudaMemcpyDeviceToHost);
        double tot = 0;
        for (int k = 0; k < 8; ++k) tot += (double)h[k];
        fprintf(stderr, "k_pass2 phase shares: carried %.3f weights %.3f draws %.3f forced %.3f csr %.3f csc %.3f "
                "carried-values %.3f tail %.3f\n", h[0] / tot, h[1] / tot, h[2] / tot, h[3] / tot, h[4] / tot, h[5] / tot,
                h[6] / tot, h[7] / tot);
        cudaMemsetAsync(c->d.counters + 8, 0, sizeof h, c->stream);
    }
#endif
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    dim3 grid(64 / EV_WARPS, c->SL);   // 64 warps per slice
    if (c->timing && c->ev_ok) cudaEventRecord(c->ev[10], c->stream);   // pass-2 entry kernel alone (stats.ms_eval2)
    k_eval_new<<<grid, EV_WARPS * 32, 0, c->stream>>>(c->scene_slot, c->up, c->soff_k, c->s0k, A.lbase, c->G, c->d.prow,
                                                      c->d.vpl, c->d.cut_n, c->d.cut_cols, c->d.colptr, c->d.csc_row,
                                                      c->d.csc_src, c->d.carried, c->d.n_new, c->d.sbox, c->d.val, c->d.val64,
                                                      c->ncap, c->d.counters);
    e = cudaGetLastError();
    if (c->timing && c->ev_ok) cudaEventRecord(c->ev[11], c->stream);
    return e;
}

// ------------------------------------------------------------------------------------------
// Direct rendering of flagged slices (R25 / non-finite fallback): every entry, fp64 sums
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_direct(int slot, Upper up, const int32_t *__restrict__ slice_off, int32_t s0,
                                                int32_t lbase, int G, const float4 *__restrict__ prow,
                                                const float4 *__restrict__ vpl, const int32_t *__restrict__ cut_n,
                                                const int32_t *__restrict__ cut_cols, const int32_t *__restrict__ flags,
                                                float *direct_rgb)
{
    const int ls = blockIdx.x, s = s0 + ls;
    if (!(flags[ls] & LMC_SLICE_DIRECT)) return;   // uniform per block
    const int m = slice_off[s + 1] - slice_off[s], n = cut_n[ls];
    const int64_t lrow0 = slice_off[s] - lbase, cb = (int64_t)ls * G;
    for (int i = threadIdx.x; i < m; i += blockDim.x) {
        double lr = lum_rho_d(prow, lrow0 + i);
        double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0;
        for (int c = 0; c < n; ++c) {
            int u = cut_cols[cb + c];
            double lI = up.lum[u];
            double T = entry_T(slot, prow, lrow0 + i, vpl, up.rep[u]);
            double v = (lr * lI) * T;
            double w0 = lI != 0.0 ? (double)up.I[3 * u + 0] / lI : 0.0;
            double w1 = lI != 0.0 ? (double)up.I[3 * u + 1] / lI : 0.0;
            double w2 = lI != 0.0 ? (double)up.I[3 * u + 2] / lI : 0.0;
            acc0 += v * w0;
            acc1 += v * w1;
            acc2 += v * w2;
        }
        const float4 C = prow[4 * (lrow0 + i) + 2], D = prow[4 * (lrow0 + i) + 3];
        double t0 = lr != 0.0 ? (double)C.z / lr : 0.0;
        double t1 = lr != 0.0 ? (double)C.w / lr : 0.0;
        double t2 = lr != 0.0 ? (double)D.x / lr : 0.0;
        direct_rgb[3 * (lrow0 + i) + 0] = (float)(t0 * acc0);
        direct_rgb[3 * (lrow0 + i) + 1] = (float)(t1 * acc1);
        direct_rgb[3 * (lrow0 + i) + 2] = (float)(t2 * acc2);
    }
}

cudaError_t run_direct(lmc_ctx *c)
{
    if (c->SL == 0) return cudaSuccess;
    k_direct<<<c->SL, 256, 0, c->stream>>>(c->scene_slot, c->up, c->soff_k, c->s0k, c->lbase_k, c->G, c->d.prow,
                                            c->d.vpl, c->d.cut_n, c->d.cut_cols, c->d.flags, c->d.direct_rgb);
    return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------
// Test hook: T on arbitrary (row, vpl) pairs through the same entry function
// ------------------------------------------------------------------------------------------
__global__ void k_eval_pairs(int slot, int64_t n, const int32_t *rows, const int32_t *vpls, GView g, const float *vx,
                             const float *vy, const float *vz, const float *rr, const float *rg, const float *rb,
                             const float *spec, const int32_t *expo, float4 *tmp, const float4 *vpl, double *out)
{
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    int r = rows[k];
    tmp[4 * k + 0] = make_float4(g.px[r], g.py[r], g.pz[r], g.nx[r]);
    tmp[4 * k + 1] = make_float4(g.ny[r], g.nz[r], vx[r], vy[r]);
    tmp[4 * k + 2] = make_float4(vz[r], spec[r], rr[r], rg[r]);
    tmp[4 * k + 3] = make_float4(rb[r], __int_as_float(expo[r]), 0.f, 0.f);
    out[k] = entry_T(slot, tmp, k, vpl, vpls[k]);
}

cudaError_t run_eval_entries(lmc_ctx *c, int64_t n, const int32_t *d_rows, const int32_t *d_vpls, double *d_out,
                             float4 *d_tmp_rows)
{
    if (n == 0) return cudaSuccess;
    GView g = gview(c);
    k_eval_pairs<<<(unsigned)((n + 255) / 256), 256, 0, c->stream>>>(
        c->scene_slot, n, d_rows, d_vpls, g, c->d.g[6], c->d.g[7], c->d.g[8], c->d.g[9], c->d.g[10], c->d.g[11], c->d.g[12],
        c->d.expo, d_tmp_rows, c->d.vpl, d_out);
    return cudaGetLastError();
}

}  // namespace lmc
