/*
 * oracle.c — plain, slow, fp64 CPU oracle of arXiv 2202.12567's hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h).  Shares no code with the CUDA path.
 * Compile: gcc -O2 -ffp-contract=off -fno-fast-math -fopenmp -fPIC -shared.
 *
 * Citations: P:<line> = /root/reference/PAPER.md line; R<k> = DESIGN.md reading k (where the
 * paper is silent, ambiguous or garbled).  Each stage is written in the paper's order and
 * notation; no blocking, fusion or reordering beyond the stated algorithm.
 *
 * parity pins: see tests/test_oracle_*.py; the whole-pipeline error vs. the paper's own scenes
 * and the free constants (R2, R3, R6, R11, R14, R19, R20) are "parity unpinned".
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define INV_PI 0.31830988618379067
#define INV_2PI 0.15915494309189535

enum { TAG_P1 = 1, TAG_P2 = 2, TAG_FORCE = 3, TAG_X0 = 4, TAG_Y0 = 5 };

/* ------------------------------------------------------------------------------------------
 * Philox4x32-10 (R7/O3): counter-based RNG, Salmon et al. SC'11 (Random123 constants).
 * ---------------------------------------------------------------------------------------- */
void orc_philox(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4])
{
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    uint32_t k0 = key[0], k1 = key[1];
    for (int r = 0; r < 10; ++r) {
        uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
        if (r < 9) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

static void philox_draw(uint64_t seed, uint32_t a, uint32_t b, uint32_t s, uint32_t tag, uint32_t out[4])
{
    uint32_t ctr[4] = {a, b, s, tag};
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    orc_philox(ctr, key, out);
}

/* uniform integer in [0, n): (u * n) >> 32 */
static uint32_t randint(uint32_t u, uint32_t n) { return (uint32_t)(((uint64_t)u * (uint64_t)n) >> 32); }
/* uniform real in [0,1): (u >> 8) * 2^-24, exact */
static double unif(uint32_t u) { return (double)(u >> 8) * (1.0 / 16777216.0); }

static int cmp_i32(const void *a, const void *b)
{
    int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
    return (x > y) - (x < y);
}

/* Floyd's algorithm: n distinct uniformly random rows of [0,m) ("uniformly distributed
 * inside the image block", R7 without replacement), keyed by (a, j, slice, tag). */
int32_t orc_floyd(int32_t m, int32_t n, uint32_t a, int32_t slice, uint64_t seed, uint32_t tag, int32_t *out)
{
    if (n > m) n = m;
    int32_t cnt = 0;
    for (int32_t j = m - n; j < m; ++j) {
        uint32_t u[4];
        philox_draw(seed, a, (uint32_t)j, (uint32_t)slice, tag, u);
        int32_t t = (int32_t)randint(u[0], (uint32_t)(j + 1));
        int in = 0;
        for (int32_t k = 0; k < cnt; ++k)
            if (out[k] == t) { in = 1; break; }
        out[cnt++] = in ? j : t;
    }
    qsort(out, (size_t)cnt, sizeof(int32_t), cmp_i32);
    return cnt;
}

/* ------------------------------------------------------------------------------------------
 * Entry A(i,j) ("illumination contribution from light j to surface point i"; never
 * stated — reading R1): cosine-weighted VPL emitter (R32), d^2 clamp (R2),
 * normalised-Phong BRDF (R1), visibility against the analytic occluders (R3).
 * ---------------------------------------------------------------------------------------- */
/* Floating-point operation counter of the entry evaluation (measurement only: bench.py's roofline
 * of the entry kernels).  FL(k) adds k for every +, -, *, / and sqrt the code below executes
 * (comparisons, fmin / fmax and negations count 0); it does not change any arithmetic. */
static _Thread_local int64_t orc_fl;
#define FL(k) (orc_fl += (k))

static double dot3(const double a[3], const double b[3]) { FL(5); return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2]; }

static double lum3(double r, double g, double b) { return (0.2126 * r + 0.7152 * g) + 0.0722 * b; }

static int seg_hits_sphere(const float *s, const double x[3], const double l[3], double tmin, double tmax)
{
    double c[3] = {s[0], s[1], s[2]};
    double r = s[3];
    double oc[3] = {x[0] - c[0], x[1] - c[1], x[2] - c[2]};
    FL(3);
    double b = dot3(oc, l);
    double cc = dot3(oc, oc) - r * r;
    double disc = b * b - cc;
    FL(4);
    if (disc < 0.0) return 0;
    double sq = sqrt(disc);
    double t0 = -b - sq, t1 = -b + sq;
    FL(3);
    return (t0 > tmin && t0 < tmax) || (t1 > tmin && t1 < tmax);
}

static int seg_hits_box(const float *bx, const double x[3], const double l[3], double tmin, double tmax)
{
    double tn[3], tf[3];
    for (int a = 0; a < 3; ++a) {
        double inv = 1.0 / l[a];
        double t1 = ((double)bx[a] - x[a]) * inv;
        double t2 = ((double)bx[3 + a] - x[a]) * inv;
        FL(5);
        tn[a] = fmin(t1, t2);
        tf[a] = fmax(t1, t2);
    }
    double tnear = fmax(fmax(tn[0], tn[1]), tn[2]);
    double tfar = fmin(fmin(tf[0], tf[1]), tf[2]);
    return tnear <= tfar && tfar > tmin && tnear < tmax;
}

static int seg_hits_rect(const float *rc, const double x[3], const double l[3], double tmin, double tmax)
{
    double p0[3] = {rc[0], rc[1], rc[2]};
    double e1[3] = {rc[3], rc[4], rc[5]};
    double e2[3] = {rc[6], rc[7], rc[8]};
    double nr[3] = {rc[9], rc[10], rc[11]};
    double den = dot3(nr, l);
    if (den == 0.0) return 0;
    double pd[3] = {p0[0] - x[0], p0[1] - x[1], p0[2] - x[2]};
    double t = dot3(pd, nr) / den;
    FL(4);
    if (!(t > tmin && t < tmax)) return 0;
    double h[3] = {x[0] + t * l[0], x[1] + t * l[1], x[2] + t * l[2]};
    double hp[3] = {h[0] - p0[0], h[1] - p0[1], h[2] - p0[2]};
    FL(9);
    double a = dot3(hp, e1) / dot3(e1, e1);
    double b = dot3(hp, e2) / dot3(e2, e2);
    FL(2);
    return a >= 0.0 && a <= 1.0 && b >= 0.0 && b <= 1.0;
}

/* Segment vs triangle (v0, v1, v2) — SURVEY §8(f1), reading R39: the Moller-Trumbore test
 * (Moller & Trumbore 1997) in this exact operation order, written out once here and once in the
 * CUDA path.  e1 = v1 - v0, e2 = v2 - v0, p = l x e2, det = e1 . p (0: parallel, miss),
 * s = x - v0, u = (s . p) / det in [0, 1], qv = s x e1, v = (l . qv) / det >= 0, u + v <= 1,
 * t = (e2 . qv) / det in (tmin, tmax).  Each "/ det" is a multiplication by inv = 1 / det. */
static void cross3(const double a[3], const double b[3], double c[3])
{
    c[0] = a[1] * b[2] - a[2] * b[1];
    c[1] = a[2] * b[0] - a[0] * b[2];
    c[2] = a[0] * b[1] - a[1] * b[0];
    FL(9);
}

static int seg_hits_tri(const float *tr, const double x[3], const double l[3], double tmin, double tmax)
{
    double v0[3] = {tr[0], tr[1], tr[2]};
    double e1[3] = {(double)tr[3] - v0[0], (double)tr[4] - v0[1], (double)tr[5] - v0[2]};
    double e2[3] = {(double)tr[6] - v0[0], (double)tr[7] - v0[1], (double)tr[8] - v0[2]};
    FL(6);
    double p[3];
    cross3(l, e2, p);
    double det = dot3(e1, p);
    if (det == 0.0) return 0;
    double inv = 1.0 / det;
    double sv[3] = {x[0] - v0[0], x[1] - v0[1], x[2] - v0[2]};
    FL(4);
    double u = dot3(sv, p) * inv;
    FL(1);
    if (u < 0.0 || u > 1.0) return 0;
    double qv[3];
    cross3(sv, e1, qv);
    double v = dot3(l, qv) * inv;
    FL(2);
    if (v < 0.0 || u + v > 1.0) return 0;
    double t = dot3(e2, qv) * inv;
    FL(1);
    return t > tmin && t < tmax;
}

/* V(x, y): 1 iff no occluder is hit with t in (eps, dist - eps) along the segment. */
static int visible_dir(const orc_inputs *in, const double x[3], const double l[3], double dist)
{
    double tmin = in->shadow_eps, tmax = dist - in->shadow_eps;
    FL(1);
    for (int k = 0; k < in->nsph; ++k)
        if (seg_hits_sphere(in->sph + 4 * k, x, l, tmin, tmax)) return 0;
    for (int k = 0; k < in->nbox; ++k)
        if (seg_hits_box(in->box + 6 * k, x, l, tmin, tmax)) return 0;
    for (int k = 0; k < in->nrect; ++k)
        if (seg_hits_rect(in->rect + 12 * k, x, l, tmin, tmax)) return 0;
    for (int64_t k = 0; k < in->ntri; ++k)   /* brute force: every triangle (no BVH) */
        if (seg_hits_tri(in->tri + 9 * k, x, l, tmin, tmax)) return 0;
    return 1;
}

int32_t orc_visible(const orc_inputs *in, const double x[3], const double y[3])
{
    double d[3] = {y[0] - x[0], y[1] - x[1], y[2] - x[2]};
    double d2 = dot3(d, d);
    if (d2 == 0.0) return 1;
    double dist = sqrt(d2);
    double l[3] = {d[0] / dist, d[1] / dist, d[2] / dist};
    return visible_dir(in, x, l, dist);
}

static double powi(double base, int32_t e)
{
    double r = 1.0;
    while (e > 0) {
        if (e & 1) { r = r * base; FL(1); }
        base = base * base;
        FL(1);
        e >>= 1;
    }
    return r;
}

double orc_entry_T(const orc_inputs *in, int64_t p, int64_t v)
{
    double x[3] = {in->px[p], in->py[p], in->pz[p]};
    double np_[3] = {in->nx[p], in->ny[p], in->nz[p]};
    double o[3] = {in->vx[p], in->vy[p], in->vz[p]};
    double y[3] = {in->lx[v], in->ly[v], in->lz[v]};
    double nv[3] = {in->lnx[v], in->lny[v], in->lnz[v]};
    double d[3] = {y[0] - x[0], y[1] - x[1], y[2] - x[2]};
    FL(3);
    double d2 = dot3(d, d);
    if (d2 == 0.0) return 0.0;
    double dist = sqrt(d2);
    double l[3] = {d[0] / dist, d[1] / dist, d[2] / dist};
    FL(4);
    double ci = dot3(np_, l);
    double cj = -dot3(nv, l);
    if (ci <= 0.0 || cj <= 0.0) return 0.0;
    double dc2 = in->clamp_dist * in->clamp_dist;
    double G = (ci * cj) / fmax(d2, dc2);
    FL(3);
    double s = in->spec[p];
    double phi;
    if (s == 0.0) {
        phi = INV_PI;
    } else {
        int32_t e = in->expo[p];
        double rv = (2.0 * ci) * dot3(np_, o) - dot3(l, o);
        FL(3);
        double lobe = rv > 0.0 ? powi(rv, e) : 0.0;
        phi = (1.0 - s) * INV_PI + (s * (((double)(e + 2)) * INV_2PI)) * lobe;
        FL(6);
    }
    if (!visible_dir(in, x, l, dist)) return 0.0;
    FL(1);
    return phi * G;
}

/* struct sizes for the binding's layout check */
int64_t orc_sizeof_inputs(void) { return (int64_t)sizeof(orc_inputs); }
int64_t orc_sizeof_result(void) { return (int64_t)sizeof(orc_slice_result); }

/* T for n (row, vpl) pairs, one orc_entry_T call each (test convenience, no new arithmetic) */
void orc_entry_T_many(const orc_inputs *in, int64_t n, const int32_t *rows, const int32_t *vpls, double *out)
{
    for (int64_t k = 0; k < n; ++k) out[k] = orc_entry_T(in, rows[k], vpls[k]);
}

/* floating-point operations executed by orc_entry_T over n pairs (FL counter above) */
int64_t orc_entry_flops(const orc_inputs *in, int64_t n, const int32_t *rows, const int32_t *vpls)
{
    orc_fl = 0;
    for (int64_t k = 0; k < n; ++k) (void)orc_entry_T(in, rows[k], vpls[k]);
    return orc_fl;
}

static double lum_rho(const orc_inputs *in, int64_t p) { return lum3(in->rr[p], in->rg[p], in->rb[p]); }
static double lum_node(const orc_inputs *in, int32_t f) { return lum3(in->tir[f], in->tig[f], in->tib[f]); }

/* ------------------------------------------------------------------------------------------
 * Matrix slicing (R26): rows as 6D points (x/D, w_n n), recursive binary
 * split on the dimension of largest extent, lower median by (key, row), left gets ceil(n/2).
 * ---------------------------------------------------------------------------------------- */
typedef struct { double k; int32_t r; } keyrow;

static int cmp_keyrow(const void *a, const void *b)
{
    const keyrow *x = a, *y = b;
    if (x->k < y->k) return -1;
    if (x->k > y->k) return 1;
    return (x->r > y->r) - (x->r < y->r);
}

static double slice_key(const orc_inputs *in, int32_t r, int d)
{
    switch (d) {
    case 0: return (double)in->px[r] / in->diag;
    case 1: return (double)in->py[r] / in->diag;
    case 2: return (double)in->pz[r] / in->diag;
    case 3: return in->wn * (double)in->nx[r];
    case 4: return in->wn * (double)in->ny[r];
    default: return in->wn * (double)in->nz[r];
    }
}

static void slice_rec(const orc_inputs *in, int32_t *rows, int32_t n, int32_t *off, int32_t *rows_out,
                      int64_t *ns, int32_t *pos)
{
    if (n <= in->target) {
        memcpy(rows_out + *pos, rows, (size_t)n * sizeof(int32_t));
        *pos += n;
        off[++(*ns)] = *pos;
        return;
    }
    int best = 0;
    double bext = -1.0;
    for (int d = 0; d < 6; ++d) {
        double lo = slice_key(in, rows[0], d), hi = lo;
        for (int32_t i = 1; i < n; ++i) {
            double k = slice_key(in, rows[i], d);
            lo = fmin(lo, k);
            hi = fmax(hi, k);
        }
        double ext = hi - lo;
        if (ext > bext) { bext = ext; best = d; }
    }
    keyrow *kr = malloc((size_t)n * sizeof(keyrow));
    for (int32_t i = 0; i < n; ++i) { kr[i].k = slice_key(in, rows[i], best); kr[i].r = rows[i]; }
    qsort(kr, (size_t)n, sizeof(keyrow), cmp_keyrow);
    for (int32_t i = 0; i < n; ++i) rows[i] = kr[i].r;
    free(kr);
    int32_t nl = (n + 1) / 2;
    qsort(rows, (size_t)nl, sizeof(int32_t), cmp_i32);
    qsort(rows + nl, (size_t)(n - nl), sizeof(int32_t), cmp_i32);
    slice_rec(in, rows, nl, off, rows_out, ns, pos);
    slice_rec(in, rows + nl, n - nl, off, rows_out, ns, pos);
}

int32_t orc_build_slices(const orc_inputs *in, int32_t *off, int32_t *rows, int64_t *nslices)
{
    int32_t m = (int32_t)in->m;
    int32_t *work = malloc((size_t)(m > 0 ? m : 1) * sizeof(int32_t));
    for (int32_t i = 0; i < m; ++i) work[i] = i;
    int64_t ns = 0;
    int32_t pos = 0;
    off[0] = 0;
    if (m > 0) slice_rec(in, work, m, off, rows, &ns, &pos);
    free(work);
    *nslices = ns;
    return 0;
}

/* ------------------------------------------------------------------------------------------
 * Small containers (hash map u64 -> double, dynamic arrays)
 * ---------------------------------------------------------------------------------------- */
typedef struct { uint64_t *key; double *val; int64_t cap, cnt; } hmap;

static void hm_init(hmap *h, int64_t cap)
{
    int64_t c = 64;
    while (c < 2 * cap) c <<= 1;
    h->cap = c;
    h->cnt = 0;
    h->key = malloc((size_t)c * sizeof(uint64_t));
    h->val = malloc((size_t)c * sizeof(double));
    for (int64_t i = 0; i < c; ++i) h->key[i] = UINT64_MAX;
}
static void hm_free(hmap *h) { free(h->key); free(h->val); }
static uint64_t hm_hash(uint64_t k) { k ^= k >> 33; k *= 0xff51afd7ed558ccdULL; k ^= k >> 33; return k; }
static int hm_get(const hmap *h, uint64_t k, double *v)
{
    uint64_t i = hm_hash(k) & (uint64_t)(h->cap - 1);
    while (h->key[i] != UINT64_MAX) {
        if (h->key[i] == k) { *v = h->val[i]; return 1; }
        i = (i + 1) & (uint64_t)(h->cap - 1);
    }
    return 0;
}
static void hm_put(hmap *h, uint64_t k, double v);
static void hm_grow(hmap *h)
{
    hmap n;
    hm_init(&n, h->cap);
    for (int64_t i = 0; i < h->cap; ++i)
        if (h->key[i] != UINT64_MAX) hm_put(&n, h->key[i], h->val[i]);
    hm_free(h);
    *h = n;
}
static void hm_put(hmap *h, uint64_t k, double v)
{
    if (2 * (h->cnt + 1) > h->cap) hm_grow(h);
    uint64_t i = hm_hash(k) & (uint64_t)(h->cap - 1);
    while (h->key[i] != UINT64_MAX) {
        if (h->key[i] == k) { h->val[i] = v; return; }
        i = (i + 1) & (uint64_t)(h->cap - 1);
    }
    h->key[i] = k;
    h->val[i] = v;
    h->cnt++;
}

typedef struct { int32_t *a; int64_t n, cap; } ivec;
static void iv_push(ivec *v, int32_t x)
{
    if (v->n == v->cap) { v->cap = v->cap ? 2 * v->cap : 64; v->a = realloc(v->a, (size_t)v->cap * sizeof(int32_t)); }
    v->a[v->n++] = x;
}
typedef struct { double *a; int64_t n, cap; } dvec;
static void dv_push(dvec *v, double x)
{
    if (v->n == v->cap) { v->cap = v->cap ? 2 * v->cap : 64; v->a = realloc(v->a, (size_t)v->cap * sizeof(double)); }
    v->a[v->n++] = x;
}

/* ------------------------------------------------------------------------------------------
 * Per-slice state
 * ---------------------------------------------------------------------------------------- */
typedef struct {
    const orc_inputs *in;
    const int32_t *rows;
    int32_t m, s;
    hmap Tcache;                /* key (vpl << 16 | local row) -> T */
    int64_t evals;
} slice_ctx;

static double T_cached(slice_ctx *c, int32_t i, int32_t vpl)
{
    uint64_t k = ((uint64_t)(uint32_t)vpl << 16) | (uint64_t)(uint32_t)i;
    double v;
    if (hm_get(&c->Tcache, k, &v)) return v;
    v = orc_entry_T(c->in, c->rows[i], vpl);
    hm_put(&c->Tcache, k, v);
    c->evals++;
    return v;
}

/* Pass-1 count n_f, linearly proportional to lum(I_f) (reading R6) */
static int32_t n_of(const orc_inputs *in, int32_t m, double lum, double lmax)
{
    int32_t n;
    if (lmax > 0.0) {
        double x = ceil(((double)in->nmax * lum) / lmax);
        n = x > (double)in->nmin ? (int32_t)x : in->nmin;
    } else {
        n = in->nmin;
    }
    return n < m ? n : m;
}

static uint64_t splitmix(uint64_t *s)
{
    uint64_t z = (*s += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* ------------------------------------------------------------------------------------------
 * Light coarsening (Eq. (1); readings R5, R8-R11).
 * ---------------------------------------------------------------------------------------- */
static void coarsen(slice_ctx *c, orc_slice_result *res, const int32_t *parent)
{
    const orc_inputs *in = c->in;
    int64_t nn = in->nn;
    uint8_t *in_cut = calloc((size_t)nn, 1);
    uint8_t *merged = calloc((size_t)nn, 1);
    double *cost = calloc((size_t)nn, sizeof(double));
    int32_t *zidx = malloc((size_t)nn * sizeof(int32_t)); /* processed-record index of merged nodes */
    for (int64_t k = 0; k < in->ncut; ++k) in_cut[in->cut[k]] = 1; /* cost = 0 on g */

    /* base pairs B = parents with both children in g; l_max over B (global, R6) */
    ivec work = {0};
    double lmax = 0.0;
    for (int64_t k = 0; k < in->ncut; ++k) {
        int32_t g = in->cut[k];
        int32_t f = parent[g];
        if (f < 0 || in->left[f] != g) continue; /* visit each parent once, via its left child */
        if (in_cut[in->right[f]]) {
            iv_push(&work, f);
            double lf = lum_node(in, f);
            if (lf > lmax) lmax = lf;
        }
    }
    qsort(work.a, (size_t)work.n, sizeof(int32_t), cmp_i32);

    ivec pnode = {0}, pmerged = {0}, zoff = {0}, zrows = {0};
    dvec peps = {0}, pcost = {0}, pva = {0}, pvb = {0};
    iv_push(&zoff, 0);
    int32_t *buf = malloc((size_t)(2 * c->m + 2) * sizeof(int32_t));
    int32_t *fresh = malloc((size_t)(c->m + 1) * sizeof(int32_t));
    uint64_t rs = in->order_seed;
    int64_t head = 0;
    /* count-target mode (reading R37): candidates are evaluated when they appear, merges
     * follow the least cost (ties: smallest node id) until the cut has coarsen_target nodes */
    const int count_mode = in->coarsen_target > 0;
    int64_t cut_size = in->ncut;
    ivec cands = {0};
    for (;;) {
    while (head < work.n) {
        int32_t f;
        if (in->order_seed) { /* order-independence pin: process a random pending candidate */
            int64_t pick = head + (int64_t)(splitmix(&rs) % (uint64_t)(work.n - head));
            f = work.a[pick];
            work.a[pick] = work.a[head];
            work.a[head] = f;
        } else {
            f = work.a[head];
        }
        head++;
        int32_t l = in->left[f], r = in->right[f];
        /* "L_f is the same as L_a except intensity": a shares rep(f) (R5) */
        int32_t a = (in->rep[l] == in->rep[f]) ? l : r;
        int32_t b = (a == l) ? r : l;
        /* zeta_f (R10) */
        int32_t nz = 0;
        if (!merged[l] && !merged[r]) {
            nz = orc_floyd(c->m, n_of(in, c->m, lum_node(in, f), lmax), (uint32_t)f, c->s, in->seed, TAG_P1, buf);
        } else {
            const int32_t *A, *Bv;
            int32_t na, nb;
            if (merged[l] && merged[r]) {
                A = zrows.a + zoff.a[zidx[l]]; na = zoff.a[zidx[l] + 1] - zoff.a[zidx[l]];
                Bv = zrows.a + zoff.a[zidx[r]]; nb = zoff.a[zidx[r] + 1] - zoff.a[zidx[r]];
            } else {
                int32_t h = merged[l] ? l : r, o = merged[l] ? r : l;
                A = zrows.a + zoff.a[zidx[h]]; na = zoff.a[zidx[h] + 1] - zoff.a[zidx[h]];
                nb = orc_floyd(c->m, n_of(in, c->m, lum_node(in, o), lmax), (uint32_t)f, c->s, in->seed, TAG_P1, fresh);
                Bv = fresh;
            }
            /* sorted set union */
            int32_t i = 0, j = 0;
            while (i < na || j < nb) {
                if (j >= nb || (i < na && A[i] < Bv[j])) buf[nz++] = A[i++];
                else if (i >= na || Bv[j] < A[i]) buf[nz++] = Bv[j++];
                else { buf[nz++] = A[i++]; j++; }
            }
        }
        /* V_a, V_b on zeta_f and the merge error (R8) */
        double la = lum_node(in, a), lb = lum_node(in, b);
        double eps = 0.0;
        double ratio = la > 0.0 ? lb / la : 0.0;
        for (int32_t k = 0; k < nz; ++k) {
            int32_t i = buf[k];
            double Ta = T_cached(c, i, in->rep[a]);
            double Tb = T_cached(c, i, in->rep[b]);
            double lr = lum_rho(in, c->rows[i]);
            double Va = (lr * la) * Ta;
            double Vb = (lr * lb) * Tb;
            double e = la > 0.0 ? fabs(Vb - Va * ratio) : fabs(Vb);
            if (e > eps) eps = e;
            iv_push(&zrows, i);
            dv_push(&pva, Ta);
            dv_push(&pvb, Tb);
        }
        /* Eq. (1): cost(L_f) = eps(L_f) + cost(L_b) (R9); the sensitivity variant also adds
         * the accumulated error of L_a (cost_mode 1): (eps + cost(L_b)) + cost(L_a) */
        double cf = eps + cost[b];
        if (in->cost_mode) cf = cf + cost[a];
        int do_merge = !count_mode && cf < in->tau; /* P:116 "less than a prespecified error bound" (R11) */
        zidx[f] = (int32_t)pnode.n;
        iv_push(&pnode, f);
        iv_push(&pmerged, do_merge);
        dv_push(&peps, eps);
        dv_push(&pcost, cf);
        iv_push(&zoff, (int32_t)zrows.n);
        cost[f] = cf;
        if (count_mode) iv_push(&cands, f);
        if (do_merge) {
            in_cut[l] = 0;
            in_cut[r] = 0;
            in_cut[f] = 1;
            merged[f] = 1;
            cut_size--;
            int32_t p = parent[f];
            if (p >= 0) {
                int32_t sib = in->left[p] == f ? in->right[p] : in->left[p];
                if (in_cut[sib]) iv_push(&work, p);
            }
        }
    }
    if (!count_mode || cut_size <= in->coarsen_target) break;
    /* the least-cost pair of sibling cut nodes */
    int64_t bk = -1;
    for (int64_t k = 0; k < cands.n; ++k) {
        int32_t g = cands.a[k];
        if (merged[g]) continue;
        if (bk < 0 || cost[g] < cost[cands.a[bk]] || (cost[g] == cost[cands.a[bk]] && g < cands.a[bk])) bk = k;
    }
    if (bk < 0) break;
    {
        int32_t f = cands.a[bk];
        in_cut[in->left[f]] = 0;
        in_cut[in->right[f]] = 0;
        in_cut[f] = 1;
        merged[f] = 1;
        pmerged.a[zidx[f]] = 1;
        cut_size--;
        int32_t p = parent[f];
        if (p >= 0) {
            int32_t sib = in->left[p] == f ? in->right[p] : in->left[p];
            if (in_cut[sib]) iv_push(&work, p);
        }
    }
    }
    free(cands.a);
    /* final cut, sorted by node id = column order (R29) */
    int32_t n = 0;
    ivec cutv = {0};
    for (int64_t k = 0; k < in->ncut; ++k) {
        /* walk up from every g node to its topmost cut ancestor-or-self */
        int32_t g = in->cut[k];
        int32_t t = g;
        while (!in_cut[t]) t = parent[t];
        iv_push(&cutv, t);
    }
    qsort(cutv.a, (size_t)cutv.n, sizeof(int32_t), cmp_i32);
    for (int64_t k = 0; k < cutv.n; ++k)
        if (k == 0 || cutv.a[k] != cutv.a[k - 1]) cutv.a[n++] = cutv.a[k];
    res->n = n;
    res->cut_nodes = malloc((size_t)(n > 0 ? n : 1) * sizeof(int32_t));
    memcpy(res->cut_nodes, cutv.a, (size_t)n * sizeof(int32_t));
    res->n_proc = (int32_t)pnode.n;
    res->proc_node = pnode.a;
    res->proc_merged = pmerged.a;
    res->proc_eps = peps.a;
    res->proc_cost = pcost.a;
    res->proc_zoff = zoff.a;
    res->proc_zrows = zrows.a;
    res->proc_Va = pva.a;
    res->proc_Vb = pvb.a;
    free(cutv.a);
    free(work.a);
    free(buf);
    free(fresh);
    free(in_cut);
    free(merged);
    free(cost);
    free(zidx);
}

/* ------------------------------------------------------------------------------------------
 * Pass-2 building blocks (public so that tests can pin them on hand-made inputs).
 * ---------------------------------------------------------------------------------------- */
/* g(c) = max(C_c) - min(C_c) over the observations of column c ("the maximal value
 * minus the minimal value of the sampled elements of C_j"); cnt[c] = observations of c, g = 0
 * when cnt[c] <= 1 (R14).  Order-free, exact. */
void orc_light_importance(int32_t n, int64_t nobs, const int32_t *col, const double *val, double *g, int32_t *cnt)
{
    double *lo = malloc((size_t)(n > 0 ? n : 1) * sizeof(double));
    double *hi = malloc((size_t)(n > 0 ? n : 1) * sizeof(double));
    for (int32_t c = 0; c < n; ++c) { cnt[c] = 0; lo[c] = INFINITY; hi[c] = -INFINITY; g[c] = 0.0; }
    for (int64_t k = 0; k < nobs; ++k) {
        int32_t c = col[k];
        lo[c] = fmin(lo[c], val[k]);
        hi[c] = fmax(hi[c], val[k]);
        cnt[c]++;
    }
    for (int32_t c = 0; c < n; ++c)
        if (cnt[c]) g[c] = hi[c] - lo[c];
    free(lo);
    free(hi);
}

/* Integer pdf weights of the columns (Eq. 2 with f(i) = 1, reading R14): with G = max_c g(c) > 0,
 * an observed column gets max(2^16, 1 + floor((2^20 - 1) g(c) / G)), an unobserved one the mean
 * (integer division) of the observed weights (2^19 if none is observed); G = 0 gives 1 everywhere. */
void orc_pdf_weights(int32_t n, const double *g, const int32_t *cnt, uint32_t *w)
{
    double G = 0.0;
    for (int32_t c = 0; c < n; ++c)
        if (cnt[c] && g[c] > G) G = g[c];
    if (G > 0.0) {
        uint64_t sumw = 0;
        int32_t nobsc = 0;
        for (int32_t c = 0; c < n; ++c) {
            if (!cnt[c]) continue;
            double x = floor(1048575.0 * (g[c] / G));
            uint32_t wc = 1u + (uint32_t)x;
            w[c] = wc > 65536u ? wc : 65536u;
            sumw += w[c];
            nobsc++;
        }
        uint32_t wu = nobsc ? (uint32_t)(sumw / (uint64_t)nobsc) : 524288u;
        for (int32_t c = 0; c < n; ++c)
            if (!cnt[c]) w[c] = wu;
    } else {
        for (int32_t c = 0; c < n; ++c) w[c] = 1u;
    }
}

/* CDF inversion (R29): the smallest c with cdf[c] > x (cdf inclusive prefix sums of the weights) */
int32_t orc_cdf_pick(int32_t n, const uint64_t *cdf, uint64_t x)
{
    int32_t lo = 0, hi = n - 1;
    while (lo < hi) {
        int32_t mid = (lo + hi) / 2;
        if (cdf[mid] > x) hi = mid; else lo = mid + 1;
    }
    return lo;
}

/* Draw t of pass 2 ("select a column by its importance, then a row uniformly", O7):
 * u = Philox(t, 0, slice, P2); column = CDF^-1((u0 W) >> 32); row = (u1 m) >> 32. */
void orc_pass2_draw(uint64_t seed, int32_t slice, uint32_t t, uint64_t W, const uint64_t *cdf, int32_t n, int32_t m,
                    int32_t *row, int32_t *col)
{
    uint32_t u[4];
    philox_draw(seed, t, 0u, (uint32_t)slice, TAG_P2, u);
    uint64_t x = ((uint64_t)u[0] * W) >> 32;
    *col = orc_cdf_pick(n, cdf, x);
    *row = (int32_t)randint(u[1], (uint32_t)m);
}

/* Draw t with an image-space row importance f(i) (P:145 sets f(i) = 1, P:246 names
 * image-space guidance as future work): the row is CDF_r^-1((u1 W_r) >> 32) over integer row
 * weights built like the column weights (R14) from the rows' carried observations (reading R36). */
void orc_pass2_draw_f(uint64_t seed, int32_t slice, uint32_t t, uint64_t W, const uint64_t *cdf, int32_t n, uint64_t Wr,
                      const uint64_t *rcdf, int32_t m, int32_t *row, int32_t *col)
{
    uint32_t u[4];
    philox_draw(seed, t, 0u, (uint32_t)slice, TAG_P2, u);
    uint64_t x = ((uint64_t)u[0] * W) >> 32;
    *col = orc_cdf_pick(n, cdf, x);
    uint64_t y = ((uint64_t)u[1] * Wr) >> 32;
    *row = orc_cdf_pick(m, rcdf, y);
}

/* draws t0 .. t0+count-1 of pass 2 without the observed-cell test (statistical pins) */
void orc_pass2_draws(uint64_t seed, int32_t slice, uint32_t t0, int64_t count, const uint32_t *w, int32_t n, int32_t m,
                     int32_t *rows, int32_t *cols)
{
    uint64_t *cdf = malloc((size_t)(n > 0 ? n : 1) * sizeof(uint64_t));
    uint64_t W = 0;
    for (int32_t c = 0; c < n; ++c) { W += w[c]; cdf[c] = W; }
    for (int64_t k = 0; k < count; ++k) orc_pass2_draw(seed, slice, t0 + (uint32_t)k, W, cdf, n, m, rows + k, cols + k);
    free(cdf);
}

/* ------------------------------------------------------------------------------------------
 * Sampling pass 2 (Eq. (2); readings R13-R17, R27).
 * ---------------------------------------------------------------------------------------- */
static void pass2(slice_ctx *c, orc_slice_result *res)
{
    const orc_inputs *in = c->in;
    int32_t m = c->m, n = res->n;
    uint8_t *obs = calloc((size_t)m * (size_t)(n > 0 ? n : 1), 1);
    uint8_t *carried = calloc((size_t)m * (size_t)(n > 0 ? n : 1), 1);
    double *val = calloc((size_t)m * (size_t)(n > 0 ? n : 1), sizeof(double));
    int32_t *colcnt = calloc((size_t)(n > 0 ? n : 1), sizeof(int32_t));
    /* carried observations ("we have actually sparsely sampled the lighting matrices", R13) */
    int64_t n_obs = 0;
    for (int32_t cc = 0; cc < n; ++cc) {
        int32_t node = res->cut_nodes[cc];
        int32_t v = in->rep[node];
        double lI = lum_node(in, node);
        for (int32_t i = 0; i < m; ++i) {
            double T;
            uint64_t k = ((uint64_t)(uint32_t)v << 16) | (uint64_t)(uint32_t)i;
            if (hm_get(&c->Tcache, k, &T)) {
                size_t at = (size_t)i * (size_t)n + (size_t)cc;
                obs[at] = 1;
                carried[at] = 1;
                val[at] = (lum_rho(in, c->rows[i]) * lI) * T;
                colcnt[cc]++;
                n_obs++;
            }
        }
    }
    res->n_carried = n_obs;
    /* light importance g(j) = max(C_j) - min(C_j) over the observed entries (R14) */
    int32_t *ocol = malloc((size_t)(n_obs > 0 ? n_obs : 1) * sizeof(int32_t));
    double *oval = malloc((size_t)(n_obs > 0 ? n_obs : 1) * sizeof(double));
    int64_t no = 0;
    for (int32_t cc = 0; cc < n; ++cc)
        for (int32_t i = 0; i < m; ++i) {
            size_t at = (size_t)i * (size_t)n + (size_t)cc;
            if (obs[at]) { ocol[no] = cc; oval[no] = val[at]; no++; }
        }
    uint32_t *w = malloc((size_t)(n > 0 ? n : 1) * sizeof(uint32_t));
    double *g = calloc((size_t)(n > 0 ? n : 1), sizeof(double));
    int32_t *gcnt = calloc((size_t)(n > 0 ? n : 1), sizeof(int32_t));
    orc_light_importance(n, no, ocol, oval, g, gcnt);
    /* pixel importance f(i) = 1; pdf(i,j) ∝ f(i) g(j) (Eq. 2) as integer weights (R14) */
    orc_pdf_weights(n, g, gcnt, w);
    /* variant (reading R36): f(i) = max - min of row i's carried observations, row
     * weights by the same rule, rows drawn from their CDF */
    uint64_t *rcdf = NULL, Wr = 0;
    if (in->row_importance) {
        int32_t *orow = malloc((size_t)(no > 0 ? no : 1) * sizeof(int32_t));
        int64_t kk = 0;
        for (int32_t cc = 0; cc < n; ++cc)
            for (int32_t i = 0; i < m; ++i)
                if (obs[(size_t)i * (size_t)n + (size_t)cc]) orow[kk++] = i;
        double *fr = calloc((size_t)(m > 0 ? m : 1), sizeof(double));
        int32_t *fcnt = calloc((size_t)(m > 0 ? m : 1), sizeof(int32_t));
        uint32_t *wr = malloc((size_t)(m > 0 ? m : 1) * sizeof(uint32_t));
        orc_light_importance(m, no, orow, oval, fr, fcnt);
        orc_pdf_weights(m, fr, fcnt, wr);
        rcdf = malloc((size_t)(m > 0 ? m : 1) * sizeof(uint64_t));
        for (int32_t i = 0; i < m; ++i) { Wr += wr[i]; rcdf[i] = Wr; }
        free(orow);
        free(fr);
        free(fcnt);
        free(wr);
    }
    free(ocol);
    free(oval);
    free(gcnt);
    uint64_t *cdf = malloc((size_t)(n > 0 ? n : 1) * sizeof(uint64_t));
    uint64_t W = 0;
    for (int32_t cc = 0; cc < n; ++cc) { W += w[cc]; cdf[cc] = W; }
    /* draw: column by g, then row uniformly; skip already-sampled entries (R15, R16) */
    int64_t N = (int64_t)ceil(((double)((int64_t)m * (int64_t)n)) * in->rate);
    res->target_N = N;
    int64_t n_new = 0, t = 0;
    for (t = 0; t < 64 * N && n_obs < N; ++t) {
        int32_t i, cc;
        if (rcdf) orc_pass2_draw_f(in->seed, c->s, (uint32_t)t, W, cdf, n, Wr, rcdf, m, &i, &cc);
        else orc_pass2_draw(in->seed, c->s, (uint32_t)t, W, cdf, n, m, &i, &cc);
        size_t at = (size_t)i * (size_t)n + (size_t)cc;
        if (!obs[at]) {
            obs[at] = 1;
            double T = T_cached(c, i, in->rep[res->cut_nodes[cc]]);
            val[at] = (lum_rho(in, c->rows[i]) * lum_node(in, res->cut_nodes[cc])) * T;
            colcnt[cc]++;
            n_obs++;
            n_new++;
        }
    }
    res->n_draws = t;
    res->n_new = n_new;
    free(rcdf);
    /* forced sample for every still-empty column (R17) */
    int64_t n_forced = 0;
    for (int32_t cc = 0; cc < n; ++cc) {
        if (colcnt[cc]) continue;
        uint32_t u[4];
        philox_draw(in->seed, (uint32_t)cc, 0u, (uint32_t)c->s, TAG_FORCE, u);
        int32_t i = (int32_t)randint(u[0], (uint32_t)m);
        size_t at = (size_t)i * (size_t)n + (size_t)cc;
        obs[at] = 1;
        double T = T_cached(c, i, in->rep[res->cut_nodes[cc]]);
        val[at] = (lum_rho(in, c->rows[i]) * lum_node(in, res->cut_nodes[cc])) * T;
        colcnt[cc]++;
        n_obs++;
        n_forced++;
    }
    res->n_forced = n_forced;
    /* Omega in CSR order */
    res->nnz = n_obs;
    res->om_row = malloc((size_t)(n_obs > 0 ? n_obs : 1) * sizeof(int32_t));
    res->om_col = malloc((size_t)(n_obs > 0 ? n_obs : 1) * sizeof(int32_t));
    res->om_val = malloc((size_t)(n_obs > 0 ? n_obs : 1) * sizeof(double));
    res->om_carried = malloc((size_t)(n_obs > 0 ? n_obs : 1) * sizeof(int32_t));
    int64_t k = 0;
    for (int32_t i = 0; i < m; ++i)
        for (int32_t cc = 0; cc < n; ++cc) {
            size_t at = (size_t)i * (size_t)n + (size_t)cc;
            if (!obs[at]) continue;
            res->om_row[k] = i;
            res->om_col[k] = cc;
            res->om_val[k] = val[at];
            res->om_carried[k] = carried[at];
            k++;
        }
    res->weights = w;
    free(cdf);
    free(g);
    free(obs);
    free(carried);
    free(val);
    free(colcnt);
}

/* ------------------------------------------------------------------------------------------
 * Dense helpers for the completion (fp64, plain loops)
 * ---------------------------------------------------------------------------------------- */
/* unpivoted Cholesky A = L L^T in place (lower), A is q x q SPD; returns 0 on failure */
static int chol(double *A, int q)
{
    for (int j = 0; j < q; ++j) {
        double d = A[j * q + j];
        for (int k = 0; k < j; ++k) d -= A[j * q + k] * A[j * q + k];
        if (!(d > 0.0)) return 0;
        d = sqrt(d);
        A[j * q + j] = d;
        for (int i = j + 1; i < q; ++i) {
            double s = A[i * q + j];
            for (int k = 0; k < j; ++k) s -= A[i * q + k] * A[j * q + k];
            A[i * q + j] = s / d;
        }
    }
    return 1;
}
/* solve L L^T x = b in place */
static void chol_solve(const double *L, int q, double *b)
{
    for (int i = 0; i < q; ++i) {
        double s = b[i];
        for (int k = 0; k < i; ++k) s -= L[i * q + k] * b[k];
        b[i] = s / L[i * q + i];
    }
    for (int i = q - 1; i >= 0; --i) {
        double s = b[i];
        for (int k = i + 1; k < q; ++k) s -= L[k * q + i] * b[k];
        b[i] = s / L[i * q + i];
    }
}

static double max_omega(int64_t nnz, const double *val)
{
    double s = 0.0;
    for (int64_t k = 0; k < nnz; ++k) s = fmax(s, val[k]);
    return s;
}

/* R20: X_0, Y_0 Philox-uniform scaled so that E[X_0 Y_0] = mean_Omega(M^) */
static void init_factors(int32_t m, int32_t n, int32_t q, double c0, uint64_t seed, int32_t s, double *X, double *Y)
{
    for (int32_t i = 0; i < m; ++i)
        for (int32_t l = 0; l < q; ++l) {
            uint32_t u[4];
            philox_draw(seed, (uint32_t)i, (uint32_t)l, (uint32_t)s, TAG_X0, u);
            X[(size_t)i * q + l] = c0 * unif(u[0]);
        }
    for (int32_t l = 0; l < q; ++l)
        for (int32_t j = 0; j < n; ++j) {
            uint32_t u[4];
            philox_draw(seed, (uint32_t)l, (uint32_t)j, (uint32_t)s, TAG_Y0, u);
            Y[(size_t)l * n + j] = c0 * unif(u[0]);
        }
}

/* ------------------------------------------------------------------------------------------
 * ADM nonnegative factorisation (Appendix A; typo readings R18).
 * Literal: Z is kept dense (m x n), every product is formed as written.
 * ---------------------------------------------------------------------------------------- */
/* ADM of App. A with the initial factors X_0 = Xw, Y_0 = Yw when given (warm start, SURVEY f4:
 * the previous frame's factors of the same slice), else the Philox initialisation (R20) */
static int32_t adm_core(int32_t m, int32_t n, int64_t nnz, const int32_t *row, const int32_t *col, const double *val,
                        int32_t q, int32_t K, double tol, double alpha, double beta, double gamma, uint64_t seed,
                        int32_t slice, const double *Xw, const double *Yw, double *U, double *V, int32_t *iters,
                        double *resid, double *sigma);

int32_t orc_adm_warm(int32_t m, int32_t n, int64_t nnz, const int32_t *row, const int32_t *col, const double *val,
                     int32_t q, int32_t K, double tol, double alpha, double beta, double gamma, const double *X0,
                     const double *Y0, double *U, double *V, int32_t *iters, double *resid, double *sigma)
{
    return adm_core(m, n, nnz, row, col, val, q, K, tol, alpha, beta, gamma, 0, 0, X0, Y0, U, V, iters, resid, sigma);
}

int32_t orc_adm(int32_t m, int32_t n, int64_t nnz, const int32_t *row, const int32_t *col, const double *val,
                int32_t q, int32_t K, double tol, double alpha, double beta, double gamma, uint64_t seed,
                int32_t slice, double *U, double *V, int32_t *iters, double *resid, double *sigma)
{
    return adm_core(m, n, nnz, row, col, val, q, K, tol, alpha, beta, gamma, seed, slice, NULL, NULL, U, V, iters, resid,
                    sigma);
}

static int32_t adm_core(int32_t m, int32_t n, int64_t nnz, const int32_t *row, const int32_t *col, const double *val,
                        int32_t q, int32_t K, double tol, double alpha, double beta, double gamma, uint64_t seed,
                        int32_t slice, const double *Xw, const double *Yw, double *U, double *V, int32_t *iters,
                        double *resid, double *sigma)
{
    size_t mq = (size_t)m * q, qn = (size_t)q * n, mn = (size_t)m * n;
    double sg = max_omega(nnz, val); /* R23 */
    *sigma = sg;
    *iters = 0;
    *resid = 0.0;
    if (sg == 0.0) {
        memset(U, 0, mq * sizeof(double));
        memset(V, 0, qn * sizeof(double));
        return ORC_FLAG_ZERO;
    }
    double *Mh = malloc((size_t)nnz * sizeof(double));
    double mu = 0.0, nrmM = 0.0;
    for (int64_t k = 0; k < nnz; ++k) { Mh[k] = val[k] / sg; mu += Mh[k]; nrmM += Mh[k] * Mh[k]; }
    mu = mu / (double)nnz;
    nrmM = sqrt(nrmM);
    double c0 = 2.0 * sqrt(mu / (double)q);
    double *X = malloc(mq * sizeof(double)), *Y = malloc(qn * sizeof(double));
    double *Lam = calloc(mq, sizeof(double)), *Pi = calloc(qn, sizeof(double));
    double *Z = calloc(mn, sizeof(double)), *W = malloc(mn * sizeof(double));
    double *A = malloc((size_t)q * q * sizeof(double));
    double *rhs = malloc((size_t)(q > 0 ? q : 1) * sizeof(double));
    if (Xw && Yw) {
        /* warm start: the previous frame's U and V (already divided by this frame's sigma) */
        memcpy(X, Xw, mq * sizeof(double));
        memcpy(Y, Yw, qn * sizeof(double));
    } else {
        init_factors(m, n, q, c0, seed, slice, X, Y);
    }
    memcpy(U, X, mq * sizeof(double));
    memcpy(V, Y, qn * sizeof(double));
    for (int64_t k = 0; k < nnz; ++k) Z[(size_t)row[k] * n + col[k]] = Mh[k]; /* Z_0 = P_Omega(M) */
    int32_t flags = 0;
    int32_t it;
    for (it = 0; it < K; ++it) {
        /* X_{k+1} = (Z_k Y_k^T + alpha U_k - Lambda_k)(Y_k Y_k^T + alpha I)^{-1} */
        for (int a = 0; a < q; ++a)
            for (int b = 0; b < q; ++b) {
                double s = 0.0;
                for (int32_t j = 0; j < n; ++j) s += Y[(size_t)a * n + j] * Y[(size_t)b * n + j];
                A[a * q + b] = s + (a == b ? alpha : 0.0);
            }
        if (!chol(A, q)) { flags |= ORC_FLAG_DIVERGED; break; }
        for (int32_t i = 0; i < m; ++i) {
            for (int a = 0; a < q; ++a) {
                double s = 0.0;
                for (int32_t j = 0; j < n; ++j) s += Z[(size_t)i * n + j] * Y[(size_t)a * n + j];
                rhs[a] = s + alpha * U[(size_t)i * q + a] - Lam[(size_t)i * q + a];
            }
            chol_solve(A, q, rhs); /* (G + aI) symmetric: x (G + aI) = r  <=>  (G + aI) x^T = r^T */
            for (int a = 0; a < q; ++a) X[(size_t)i * q + a] = rhs[a];
        }
        /* Y_{k+1} = (X_{k+1}^T X_{k+1} + beta I)^{-1}(X_{k+1}^T Z_k + beta V_k - Pi_k)   (R18: X^T Z) */
        for (int a = 0; a < q; ++a)
            for (int b = 0; b < q; ++b) {
                double s = 0.0;
                for (int32_t i = 0; i < m; ++i) s += X[(size_t)i * q + a] * X[(size_t)i * q + b];
                A[a * q + b] = s + (a == b ? beta : 0.0);
            }
        if (!chol(A, q)) { flags |= ORC_FLAG_DIVERGED; break; }
        for (int32_t j = 0; j < n; ++j) {
            for (int a = 0; a < q; ++a) {
                double s = 0.0;
                for (int32_t i = 0; i < m; ++i) s += X[(size_t)i * q + a] * Z[(size_t)i * n + j];
                rhs[a] = s + beta * V[(size_t)a * n + j] - Pi[(size_t)a * n + j];
            }
            chol_solve(A, q, rhs);
            for (int a = 0; a < q; ++a) Y[(size_t)a * n + j] = rhs[a];
        }
        /* Z_{k+1} = X_{k+1} Y_{k+1} + P_Omega(M - X_{k+1} Y_{k+1})   (R18: P_Omega keeps Omega) */
        for (int32_t i = 0; i < m; ++i)
            for (int32_t j = 0; j < n; ++j) {
                double s = 0.0;
                for (int a = 0; a < q; ++a) s += X[(size_t)i * q + a] * Y[(size_t)a * n + j];
                W[(size_t)i * n + j] = s;
            }
        memcpy(Z, W, mn * sizeof(double));
        double r2 = 0.0;
        for (int64_t k = 0; k < nnz; ++k) {
            size_t at = (size_t)row[k] * n + col[k];
            double d = Mh[k] - W[at];
            r2 += d * d;
            Z[at] = Mh[k];
        }
        /* U_{k+1} = P_+(X_{k+1} + Lambda_k/alpha);  V_{k+1} = P_+(Y_{k+1} + Pi_k/beta) */
        for (size_t e = 0; e < mq; ++e) U[e] = fmax(0.0, X[e] + Lam[e] / alpha);
        for (size_t e = 0; e < qn; ++e) V[e] = fmax(0.0, Y[e] + Pi[e] / beta);
        /* Lambda_{k+1} = Lambda_k + gamma alpha (X_{k+1} - U_{k+1})   (R18: Lambda_k on the right) */
        for (size_t e = 0; e < mq; ++e) Lam[e] = Lam[e] + gamma * alpha * (X[e] - U[e]);
        for (size_t e = 0; e < qn; ++e) Pi[e] = Pi[e] + gamma * beta * (Y[e] - V[e]);
        double r = sqrt(r2) / nrmM;
        *resid = r;
        if (!isfinite(r)) { flags |= ORC_FLAG_DIVERGED; it++; break; }
        if (r < tol) { it++; break; } /* P:149 "stop ... when the error is below a tolerance" (R21) */
    }
    *iters = it;
    for (size_t e = 0; e < qn; ++e) V[e] = sg * V[e]; /* R22: output (U, sigma V) */
    free(Mh); free(X); free(Y); free(Lam); free(Pi); free(Z); free(W); free(A); free(rhs);
    return flags;
}

/* ------------------------------------------------------------------------------------------
 * Masked ALS (BASELINE north_star): per-row / per-column ridge normal equations over Omega.
 * ---------------------------------------------------------------------------------------- */
static double mals_objective(int32_t m, int32_t n, int32_t q, int64_t nnz, const int32_t *row, const int32_t *col,
                             const double *Mh, const double *X, const double *Y, double lam)
{
    double f = 0.0;
    for (int64_t k = 0; k < nnz; ++k) {
        double s = 0.0;
        for (int a = 0; a < q; ++a) s += X[(size_t)row[k] * q + a] * Y[(size_t)a * n + col[k]];
        double d = s - Mh[k];
        f += d * d;
    }
    double rx = 0.0, ry = 0.0;
    for (size_t e = 0; e < (size_t)m * q; ++e) rx += X[e] * X[e];
    for (size_t e = 0; e < (size_t)q * n; ++e) ry += Y[e] * Y[e];
    return f + lam * (rx + ry);
}

int32_t orc_mals(int32_t m, int32_t n, int64_t nnz, const int32_t *row, const int32_t *col, const double *val,
                 int32_t q, int32_t K, double lam, uint64_t seed, int32_t slice, double *X, double *Y,
                 double *obj, double *sigma)
{
    size_t mq = (size_t)m * q, qn = (size_t)q * n;
    double sg = max_omega(nnz, val);
    *sigma = sg;
    if (sg == 0.0) {
        memset(X, 0, mq * sizeof(double));
        memset(Y, 0, qn * sizeof(double));
        return ORC_FLAG_ZERO;
    }
    double *Mh = malloc((size_t)nnz * sizeof(double));
    double mu = 0.0;
    for (int64_t k = 0; k < nnz; ++k) { Mh[k] = val[k] / sg; mu += Mh[k]; }
    mu = mu / (double)nnz;
    double c0 = 2.0 * sqrt(mu / (double)q);
    init_factors(m, n, q, c0, seed, slice, X, Y);
    /* CSC order: column-major listing of Omega (ascending row within a column) */
    int64_t *cptr = calloc((size_t)n + 1, sizeof(int64_t));
    int64_t *cidx = malloc((size_t)(nnz > 0 ? nnz : 1) * sizeof(int64_t));
    for (int64_t k = 0; k < nnz; ++k) cptr[col[k] + 1]++;
    for (int32_t j = 0; j < n; ++j) cptr[j + 1] += cptr[j];
    int64_t *fill = malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
    for (int32_t j = 0; j < n; ++j) fill[j] = cptr[j];
    for (int64_t k = 0; k < nnz; ++k) cidx[fill[col[k]]++] = k;
    int64_t *rptr = calloc((size_t)m + 1, sizeof(int64_t));
    for (int64_t k = 0; k < nnz; ++k) rptr[row[k] + 1]++;
    for (int32_t i = 0; i < m; ++i) rptr[i + 1] += rptr[i];
    double *A = malloc((size_t)q * q * sizeof(double)), *b = malloc((size_t)q * sizeof(double));
    int32_t flags = 0;
    for (int32_t it = 0; it < K; ++it) {
        /* X half: x_i = (sum_{j in Omega_i} y_j y_j^T + lam I)^{-1} sum_j M_ij y_j */
        for (int32_t i = 0; i < m; ++i) {
            for (int e = 0; e < q * q; ++e) A[e] = 0.0;
            for (int a = 0; a < q; ++a) b[a] = 0.0;
            for (int64_t k = rptr[i]; k < rptr[i + 1]; ++k) {
                int32_t j = col[k];
                for (int a = 0; a < q; ++a) {
                    for (int c = 0; c < q; ++c) A[a * q + c] += Y[(size_t)a * n + j] * Y[(size_t)c * n + j];
                    b[a] += Mh[k] * Y[(size_t)a * n + j];
                }
            }
            for (int a = 0; a < q; ++a) A[a * q + a] += lam;
            if (!chol(A, q)) { flags |= ORC_FLAG_DIVERGED; goto done; }
            chol_solve(A, q, b);
            for (int a = 0; a < q; ++a) X[(size_t)i * q + a] = b[a];
        }
        if (obj) obj[2 * it] = mals_objective(m, n, q, nnz, row, col, Mh, X, Y, lam);
        /* Y half: y_j = (sum_{i in Omega^j} x_i x_i^T + lam I)^{-1} sum_i M_ij x_i */
        for (int32_t j = 0; j < n; ++j) {
            for (int e = 0; e < q * q; ++e) A[e] = 0.0;
            for (int a = 0; a < q; ++a) b[a] = 0.0;
            for (int64_t t = cptr[j]; t < cptr[j + 1]; ++t) {
                int64_t k = cidx[t];
                int32_t i = row[k];
                for (int a = 0; a < q; ++a) {
                    for (int c = 0; c < q; ++c) A[a * q + c] += X[(size_t)i * q + a] * X[(size_t)i * q + c];
                    b[a] += Mh[k] * X[(size_t)i * q + a];
                }
            }
            for (int a = 0; a < q; ++a) A[a * q + a] += lam;
            if (!chol(A, q)) { flags |= ORC_FLAG_DIVERGED; goto done; }
            chol_solve(A, q, b);
            for (int a = 0; a < q; ++a) Y[(size_t)a * n + j] = b[a];
        }
        if (obj) obj[2 * it + 1] = mals_objective(m, n, q, nnz, row, col, Mh, X, Y, lam);
    }
    for (size_t e = 0; e < qn; ++e)
        if (!isfinite(Y[e])) flags |= ORC_FLAG_DIVERGED;
done:
    for (size_t e = 0; e < qn; ++e) Y[e] = sg * Y[e];
    free(Mh); free(cptr); free(cidx); free(fill); free(rptr); free(A); free(b);
    return flags;
}

/* ------------------------------------------------------------------------------------------
 * Image rendering of a slice: I(s) = X (Y e) with RGB weights (R4, O9).
 * ---------------------------------------------------------------------------------------- */
static void resolve(const orc_inputs *in, orc_slice_result *res)
{
    int32_t m = res->m, n = res->n, q = res->q;
    res->rgb = calloc((size_t)m * 3, sizeof(double));
    double *w = malloc((size_t)3 * (size_t)(n > 0 ? n : 1) * sizeof(double));
    for (int32_t c = 0; c < n; ++c) {
        int32_t f = res->cut_nodes[c];
        double lI = lum_node(in, f);
        w[0 * n + c] = lI != 0.0 ? (double)in->tir[f] / lI : 0.0;
        w[1 * n + c] = lI != 0.0 ? (double)in->tig[f] / lI : 0.0;
        w[2 * n + c] = lI != 0.0 ? (double)in->tib[f] / lI : 0.0;
    }
    if (res->flags & ORC_FLAG_ZERO) { free(w); return; }
    int64_t *rowptr = calloc((size_t)m + 1, sizeof(int64_t));   /* CSR row pointers of Omega */
    for (int64_t e = 0; e < res->nnz; ++e) rowptr[res->om_row[e] + 1]++;
    for (int32_t i = 0; i < m; ++i) rowptr[i + 1] += rowptr[i];
    for (int32_t i = 0; i < m; ++i) {
        int32_t p = res->rows[i];
        double lr = lum_rho(in, p);
        double tint[3] = {lr != 0.0 ? (double)in->rr[p] / lr : 0.0, lr != 0.0 ? (double)in->rg[p] / lr : 0.0,
                          lr != 0.0 ? (double)in->rb[p] / lr : 0.0};
        for (int k = 0; k < 3; ++k) {
            double s = 0.0;
            if (res->flags & ORC_FLAG_DIRECT) {
                for (int32_t c = 0; c < n; ++c) s += res->full[(size_t)i * n + c] * w[k * n + c];
            } else {
                for (int a = 0; a < q; ++a) {
                    double t = 0.0; /* t^k = V w^k */
                    for (int32_t c = 0; c < n; ++c) t += res->V[(size_t)a * n + c] * w[k * n + c];
                    s += res->U[(size_t)i * q + a] * t;
                }
                if (in->resolve_mode) {
                    /* Z-mode (A24): the observed entries enter as themselves,
                     * + sum_{j in Omega_i} (M~_ij - <U_i, V_j>) w^k_j (row i's samples in CSR order) */
                    for (int64_t e = rowptr[i]; e < rowptr[i + 1]; ++e) {
                        int32_t c = res->om_col[e];
                        double uv = 0.0;
                        for (int a = 0; a < q; ++a) uv += res->U[(size_t)i * q + a] * res->V[(size_t)a * n + c];
                        s += (res->om_val[e] - uv) * w[k * n + c];
                    }
                }
            }
            res->rgb[(size_t)i * 3 + k] = tint[k] * s;
        }
    }
    free(rowptr);
    free(w);
}

static void direct_full(slice_ctx *c, orc_slice_result *res)
{
    const orc_inputs *in = c->in;
    int32_t m = res->m, n = res->n;
    res->full = malloc((size_t)m * (size_t)(n > 0 ? n : 1) * sizeof(double));
    for (int32_t i = 0; i < m; ++i)
        for (int32_t cc = 0; cc < n; ++cc) {
            int32_t f = res->cut_nodes[cc];
            double T = T_cached(c, i, in->rep[f]);
            res->full[(size_t)i * n + cc] = (lum_rho(in, c->rows[i]) * lum_node(in, f)) * T;
        }
}

static int32_t *make_parent(const orc_inputs *in)
{
    int32_t *parent = malloc((size_t)in->nn * sizeof(int32_t));
    for (int64_t f = 0; f < in->nn; ++f) parent[f] = -1;
    for (int64_t f = 0; f < in->nn; ++f)
        if (in->left[f] >= 0) { parent[in->left[f]] = (int32_t)f; parent[in->right[f]] = (int32_t)f; }
    return parent;
}

static orc_slice_result *run_slice(const orc_inputs *in, const int32_t *parent, const int32_t *rows, int32_t m,
                                   int32_t s, int32_t stage)
{
    orc_slice_result *res = calloc(1, sizeof(orc_slice_result));
    res->slice = s;
    res->m = m;
    res->q = in->q;
    res->rows = malloc((size_t)(m > 0 ? m : 1) * sizeof(int32_t));
    memcpy(res->rows, rows, (size_t)m * sizeof(int32_t));
    slice_ctx c;
    c.in = in;
    c.rows = rows;
    c.m = m;
    c.s = s;
    c.evals = 0;
    hm_init(&c.Tcache, 4096);
    coarsen(&c, res, parent);
    res->n_evals_coarsen = c.evals;
    if (stage >= 2) pass2(&c, res);
    if (stage >= 3) {
        int32_t q = in->q, n = res->n;
        res->U = calloc((size_t)m * q + 1, sizeof(double));
        res->V = calloc((size_t)q * n + 1, sizeof(double));
        if (m <= q || n <= q) { /* R25: rank not below the slice dimensions -> direct */
            res->flags = ORC_FLAG_DIRECT;
        } else if (in->solver == 0) {
            /* warm start: the same slice of the previous frame with the same rows, the same
             * cut and a regular ADM result starts from that result's factors, for warm_iters iterations */
            const orc_warm *wp = NULL;
            for (int32_t k = 0; k < in->nwarm && !wp; ++k) {
                const orc_warm *e = &in->warm[k];
                if (e->slice == s && e->m == m && e->n == n && e->flags == 0 &&
                    !memcmp(e->rows, rows, (size_t)m * sizeof(int32_t)) &&
                    !memcmp(e->cut, res->cut_nodes, (size_t)n * sizeof(int32_t)))
                    wp = e;
            }
            if (wp) {
                double sg = max_omega(res->nnz, res->om_val);
                double *Yw = malloc((size_t)q * n * sizeof(double) + 8);
                for (size_t k = 0; k < (size_t)q * n; ++k) Yw[k] = sg > 0.0 ? wp->V[k] / sg : 0.0;
                res->flags = adm_core(m, n, res->nnz, res->om_row, res->om_col, res->om_val, q,
                                      in->warm_iters > 0 ? in->warm_iters : in->K, in->tol, in->alpha, in->beta, in->gamma,
                                      in->seed, s, wp->U, Yw, res->U, res->V, &res->iters, &res->resid, &res->sigma);
                res->warm = 1;
                free(Yw);
            } else {
                res->flags = orc_adm(m, n, res->nnz, res->om_row, res->om_col, res->om_val, q, in->K, in->tol,
                                     in->alpha, in->beta, in->gamma, in->seed, s, res->U, res->V, &res->iters,
                                     &res->resid, &res->sigma);
            }
        } else {
            res->obj = malloc((size_t)2 * (size_t)(in->K > 0 ? in->K : 1) * sizeof(double));
            res->n_obj = 2 * in->K;
            res->flags = orc_mals(m, n, res->nnz, res->om_row, res->om_col, res->om_val, q, in->K, in->lam,
                                  in->seed, s, res->U, res->V, res->obj, &res->sigma);
            res->iters = in->K;
        }
        if (res->flags & ORC_FLAG_DIVERGED) res->flags |= ORC_FLAG_DIRECT; /* S:396 fallback */
        if (res->flags & ORC_FLAG_DIRECT) direct_full(&c, res);
    }
    if (stage >= 4) resolve(in, res);
    hm_free(&c.Tcache);
    return res;
}

orc_slice_result *orc_run_slice(const orc_inputs *in, const int32_t *rows, int32_t m, int32_t slice, int32_t stage)
{
    int32_t *parent = make_parent(in);
    orc_slice_result *r = run_slice(in, parent, rows, m, slice, stage);
    free(parent);
    return r;
}

void orc_run_slices(const orc_inputs *in, const int32_t *off, const int32_t *rows, int32_t nsel,
                    const int32_t *slice_ids, int32_t stage, orc_slice_result **out)
{
    int32_t *parent = make_parent(in);
#pragma omp parallel for schedule(dynamic, 1)
    for (int32_t k = 0; k < nsel; ++k) {
        int32_t s = slice_ids[k];
        out[k] = run_slice(in, parent, rows + off[s], off[s + 1] - off[s], s, stage);
    }
    free(parent);
}

void orc_free_result(orc_slice_result *r)
{
    if (!r) return;
    free(r->rows); free(r->cut_nodes);
    free(r->proc_node); free(r->proc_merged); free(r->proc_zoff); free(r->proc_eps); free(r->proc_cost);
    free(r->proc_zrows); free(r->proc_Va); free(r->proc_Vb);
    free(r->om_row); free(r->om_col); free(r->om_val); free(r->om_carried); free(r->weights);
    free(r->U); free(r->V); free(r->obj); free(r->full); free(r->rgb);
    free(r);
}

void orc_fullcut_slice(const orc_inputs *in, const int32_t *rows, int32_t m, const int32_t *cut_nodes,
                       int32_t n, double *out)
{
    for (int32_t i = 0; i < m; ++i) {
        int32_t p = rows[i];
        double acc[3] = {0.0, 0.0, 0.0};
        for (int32_t c = 0; c < n; ++c) {
            int32_t f = cut_nodes[c];
            double T = orc_entry_T(in, p, in->rep[f]);
            acc[0] += ((double)in->rr[p] * (double)in->tir[f]) * T;
            acc[1] += ((double)in->rg[p] * (double)in->tig[f]) * T;
            acc[2] += ((double)in->rb[p] * (double)in->tib[f]) * T;
        }
        out[3 * i + 0] = acc[0];
        out[3 * i + 1] = acc[1];
        out[3 * i + 2] = acc[2];
    }
}

void orc_bruteforce_rows(const orc_inputs *in, const int32_t *rows, int32_t nrows, double *out)
{
#pragma omp parallel for schedule(dynamic, 16)
    for (int32_t i = 0; i < nrows; ++i) {
        int32_t p = rows[i];
        double acc[3] = {0.0, 0.0, 0.0};
        for (int64_t v = 0; v < in->nv; ++v) {
            double T = orc_entry_T(in, p, v);
            acc[0] += ((double)in->rr[p] * (double)in->lir[v]) * T;
            acc[1] += ((double)in->rg[p] * (double)in->lig[v]) * T;
            acc[2] += ((double)in->rb[p] * (double)in->lib[v]) * T;
        }
        out[3 * i + 0] = acc[0];
        out[3 * i + 1] = acc[1];
        out[3 * i + 2] = acc[2];
    }
}

/* ------------------------------------------------------------------------------------------
 * Light tree and conservative global lightcut (step 1, reading R38).
 * Binary tree by median split: a node's VPLs split on the axis of largest bounding-box extent
 * (first maximum), ordered by (coordinate, VPL index), the left child taking ceil(n/2); node ids
 * breadth-first (children of a level's internal nodes in level order, left then right).  I_f =
 * I_l + I_r (fp64), rep(f) = rep of the brighter child (lum, ties: left).  Global cut: the
 * internal nodes with the largest bounds lum(I_f) * |bbox diagonal| (ties: smaller id) are split
 * while the cut has fewer than cut_max nodes -- a lightcut-style greedy refinement, which with
 * bounds non-increasing down the tree is the same as a threshold on the bound (split test per node).
 * ---------------------------------------------------------------------------------------- */
static const float *lt_pos[3];
static int lt_axis;
static int cmp_vpl_axis(const void *a, const void *b)
{
    int32_t i = *(const int32_t *)a, j = *(const int32_t *)b;
    double ki = lt_pos[lt_axis][i], kj = lt_pos[lt_axis][j];
    if (ki < kj) return -1;
    if (ki > kj) return 1;
    return (i > j) - (i < j);
}

int32_t orc_build_light_tree(int64_t nv, const float *px, const float *py, const float *pz, const float *ir,
                             const float *ig, const float *ib, int32_t cut_max, int32_t *left, int32_t *right,
                             int32_t *rep, float *tir, float *tig, float *tib, int32_t *cut, int64_t *ncut)
{
    if (nv < 1 || cut_max < 1) return -1;
    int64_t nn = 2 * nv - 1;
    int32_t *idx = malloc((size_t)nv * sizeof(int32_t));
    for (int64_t k = 0; k < nv; ++k) idx[k] = (int32_t)k;
    int32_t *segn = malloc((size_t)nn * sizeof(int32_t)), *segs = malloc((size_t)nn * sizeof(int32_t)),
            *segl = malloc((size_t)nn * sizeof(int32_t)), *level_of = malloc((size_t)nn * sizeof(int32_t));
    double *blo = malloc((size_t)nn * 3 * sizeof(double)), *bhi = malloc((size_t)nn * 3 * sizeof(double));
    double *I = calloc((size_t)nn * 3, sizeof(double));
    for (int64_t f = 0; f < nn; ++f) { left[f] = -1; right[f] = -1; rep[f] = -1; }
    const float *pos[3] = {px, py, pz};
    /* level by level: segments (node, start, len) in breadth-first order */
    int64_t q0 = 0, q1 = 1, next_id = 1;
    segn[0] = 0; segs[0] = 0; segl[0] = (int32_t)nv; level_of[0] = 0;
    int32_t depth = 0;
    while (q0 < q1) {
        int64_t qe = q1;
        for (int64_t k = q0; k < qe; ++k) {
            int32_t f = segn[k], s = segs[k], n = segl[k];
            for (int a = 0; a < 3; ++a) { blo[3 * f + a] = INFINITY; bhi[3 * f + a] = -INFINITY; }
            for (int32_t t = s; t < s + n; ++t)
                for (int a = 0; a < 3; ++a) {
                    double v = pos[a][idx[t]];
                    if (v < blo[3 * f + a]) blo[3 * f + a] = v;
                    if (v > bhi[3 * f + a]) bhi[3 * f + a] = v;
                }
            if (n == 1) { rep[f] = idx[s]; continue; }
            int ax = 0;
            double best = bhi[3 * f] - blo[3 * f];
            for (int a = 1; a < 3; ++a)
                if (bhi[3 * f + a] - blo[3 * f + a] > best) { best = bhi[3 * f + a] - blo[3 * f + a]; ax = a; }
            lt_pos[0] = px; lt_pos[1] = py; lt_pos[2] = pz; lt_axis = ax;
            qsort(idx + s, (size_t)n, sizeof(int32_t), cmp_vpl_axis);
        }
        for (int64_t k = q0; k < qe; ++k) {   /* children ids in level order */
            int32_t f = segn[k], s = segs[k], n = segl[k];
            if (n == 1) continue;
            int32_t nl = (n + 1) / 2;
            left[f] = (int32_t)next_id;
            right[f] = (int32_t)(next_id + 1);
            segn[q1] = left[f]; segs[q1] = s; segl[q1] = nl; level_of[q1] = depth + 1; q1++;
            segn[q1] = right[f]; segs[q1] = s + nl; segl[q1] = n - nl; level_of[q1] = depth + 1; q1++;
            next_id += 2;
        }
        q0 = qe;
        depth++;
    }
    /* intensities and representatives bottom-up (reverse breadth-first order) */
    for (int64_t k = q1 - 1; k >= 0; --k) {
        int32_t f = segn[k];
        if (left[f] < 0) {
            int32_t v = rep[f];
            I[3 * f] = ir[v]; I[3 * f + 1] = ig[v]; I[3 * f + 2] = ib[v];
        } else {
            int32_t l = left[f], r = right[f];
            for (int c = 0; c < 3; ++c) I[3 * f + c] = I[3 * l + c] + I[3 * r + c];
            double ll = (0.2126 * I[3 * l] + 0.7152 * I[3 * l + 1]) + 0.0722 * I[3 * l + 2];
            double lr = (0.2126 * I[3 * r] + 0.7152 * I[3 * r + 1]) + 0.0722 * I[3 * r + 2];
            rep[f] = ll >= lr ? rep[l] : rep[r];
        }
    }
    for (int64_t f = 0; f < nn; ++f) { tir[f] = (float)I[3 * f]; tig[f] = (float)I[3 * f + 1]; tib[f] = (float)I[3 * f + 2]; }
    /* global cut: split the internal nodes by (bound desc, id asc) while the cut is short of cut_max */
    int64_t nint = 0;
    int32_t *ord = malloc((size_t)nn * sizeof(int32_t));
    double *bnd = malloc((size_t)nn * sizeof(double));
    for (int64_t f = 0; f < nn; ++f) {
        double dx = bhi[3 * f] - blo[3 * f], dy = bhi[3 * f + 1] - blo[3 * f + 1], dz = bhi[3 * f + 2] - blo[3 * f + 2];
        double lf = (0.2126 * I[3 * f] + 0.7152 * I[3 * f + 1]) + 0.0722 * I[3 * f + 2];
        bnd[f] = lf * sqrt((dx * dx + dy * dy) + dz * dz);
        if (left[f] >= 0) ord[nint++] = (int32_t)f;
    }
    /* insertion into order by (bound desc, id asc): plain selection of the next largest, nsplit times */
    int64_t nsplit = cut_max - 1 < nint ? cut_max - 1 : nint;
    uint8_t *split = calloc((size_t)nn, 1);
    for (int64_t k = 0; k < nsplit; ++k) {
        int64_t bk = k;
        for (int64_t t = k + 1; t < nint; ++t)
            if (bnd[ord[t]] > bnd[ord[bk]] || (bnd[ord[t]] == bnd[ord[bk]] && ord[t] < ord[bk])) bk = t;
        int32_t tmp = ord[k]; ord[k] = ord[bk]; ord[bk] = tmp;
        split[ord[k]] = 1;
    }
    int64_t nc = 0;
    for (int64_t f = 0; f < nn; ++f) {
        if (split[f]) continue;
        /* parent split (or the root itself) */
        int is_child_of_split = (f == 0);
        if (!is_child_of_split)
            for (int64_t k = 0; k < nsplit && !is_child_of_split; ++k)
                is_child_of_split = left[ord[k]] == f || right[ord[k]] == f;
        if (is_child_of_split) cut[nc++] = (int32_t)f;
    }
    *ncut = nc;
    free(idx); free(segn); free(segs); free(segl); free(level_of); free(blo); free(bhi); free(I);
    free(ord); free(bnd); free(split);
    return 0;
}
