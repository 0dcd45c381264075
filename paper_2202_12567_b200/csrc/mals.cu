// mals.cu — masked alternating least squares completion (BASELINE north_star), fp64 (sm_100a).
//
//   X half:  x_i = (sum_{j in Omega_i} y_j y_j^T + lam I)^{-1} sum_{j in Omega_i} M^_ij y_j
//   Y half:  y_j = (sum_{i in Omega^j} x_i x_i^T + lam I)^{-1} sum_{i in Omega^j} M^_ij x_i
//
// MALS factors are signed, so row sums of U V can cancel; fp32 normal equations miss the 1e-3
// per-pixel bar (DESIGN.md §MALS precision), hence the normal equations are accumulated and
// solved in fp64 (B200 runs fp64 FMA at half the fp32 rate).  One CTA per slice, X and Y in
// shared memory as fp64; each q x q system is owned by a group of q lanes, lane l holding row
// l of [A | b]; the solve is Gauss-Jordan without pivoting (A is SPD), pivot rows broadcast by
// shuffles.  Only the operand of the current half-step (Y for the row half, X for the column half)
// is gathered, so only it lives in shared memory (fp64, (max(m, n) + 1) x q: 131 KB at C4); both
// factors are kept in fp64 in global memory and the operand is reloaded at each half-step.
#include <algorithm>

#include "lmc_internal.h"
#include "philox.cuh"

namespace lmc {

struct MArgs {
    const int32_t *slice_off;
    int32_t s0, lbase, G, mmax;
    int32_t rs0, rss;   // global slice id of local slice ls: rs0 + ls * rss (the draws' key)
    int64_t ncap;
    int K;
    double lambda;
    uint64_t seed;
    const int32_t *cut_n, *rowptr, *colptr, *csc_src, *nnz;
    const uint16_t *col, *csc_row;
    const double *val;             // fp64 entry values (the fp32 copy would perturb MALS, R34)
    double *valc;                  // the same values in CSC order (filled per slice at start)
    float *U, *V, *resid;
    double *Xd, *Yd;               // fp64 factors [rows][q], [slice][G][q]
    int32_t fmax;                  // rows of the operand buffer in shared memory (max(mmax, G))
    int32_t *flags, *iters;
    const int32_t *order;          // CTA -> slice, or null for CTA = slice
};

constexpr int MT = 256;
// threads per CTA: q = 16 runs the tensor-core accumulation (few registers) with 16 warps.
// q = 32: one 32-lane system per warp; the operand rows (256 bytes each) would not fit in shared
// memory next to each other at |g| = 1024, so they are read from the fp64 factor in global memory
// (L2-resident per slice: 1025 x 256 bytes)
template <int Q>
struct MCfg {
    static constexpr int NT = Q == 16 ? 512 : MT;
    static constexpr bool FG = Q == 32;   // operand gathered from global memory
};
// operand layout in shared memory: at q = 16 the two 64-byte halves of odd rows are swapped, so the
// four rows a tensor-core fragment load touches fall into both bank halves
template <int Q>
__device__ __forceinline__ int fidx(int r, int c)
{
    if constexpr (Q == 16) return r * 16 + (c ^ ((r & 1) << 3));
    return r * Q + c;
}

__device__ __forceinline__ double dwarp_sum(double v)
{
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double dwarp_max(double v)
{
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

template <bool MAX>
__device__ double dblock_reduce(double v, double *red)
{
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    v = MAX ? dwarp_max(v) : dwarp_sum(v);
    __syncthreads();
    if (lane == 0) red[w] = v;
    __syncthreads();
    if (w == 0) {
        double t = lane < nw ? red[lane] : (MAX ? -1.0e300 : 0.0);
        t = MAX ? dwarp_max(t) : dwarp_sum(t);
        if (lane == 0) red[32] = t;
    }
    __syncthreads();
    return red[32];
}

// one ridge system per group of Q lanes: accumulate sum v v^T and sum m v over the system's
// samples (operand rows of F, row-major Q doubles), then solve in place; returns x_l on lane l.
// 1 / x for the (positive, normal) pivots: the hardware approximation refined by one Newton step
// (relative error ~2^-40, far below the 1e-4 completion bar; two steps measured 1% slower, none
// fails the MALS parity tests) instead of the IEEE division's longer sequence
#ifndef MALS_RCP_NEWTON
#define MALS_RCP_NEWTON 1
#endif
__device__ __forceinline__ double rcp_pivot(double x)
{
#ifdef MALS_IEEE_RCP
    return 1.0 / x;
#else
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
#pragma unroll
    for (int it = 0; it < MALS_RCP_NEWTON; ++it) {   // each step squares the relative error
        const double e = fma(-x, r, 1.0);
        r = fma(r, e, r);
    }
    return r;
#endif
}

template <int Q>
__device__ __forceinline__ double solve_group(double (&a)[Q], double b, int l, int lane0)
{
#pragma unroll
    for (int k = 0; k < Q; ++k) {
        double p[Q];
#pragma unroll
        for (int c = k; c < Q; ++c) p[c] = __shfl_sync(0xffffffffu, a[c], lane0 + k);
        const double pb = __shfl_sync(0xffffffffu, b, lane0 + k);
        const double ip = rcp_pivot(p[k]);
        if (l == k) {
#pragma unroll
            for (int c = k; c < Q; ++c) a[c] = p[c] * ip;
            b = pb * ip;
        } else {
            const double f = a[k] * ip;
#pragma unroll
            for (int c = k; c < Q; ++c) a[c] = fma(-f, p[c], a[c]);
            b = fma(-f, pb, b);
        }
    }
    return b;
}

// The in-register Cholesky alternative (MALS_CHOL=1 builds; measured against Gauss-Jordan, DESIGN
// §6): right-looking A = L L^T with the forward substitution fused (b becomes y = L^-1 b); at step
// k lane i receives l_jk of every j > k, and lane k keeps them (column k of L) for the back
// substitution x = L^-T y, which then needs one broadcast per step.
template <int Q>
__device__ __forceinline__ double solve_chol(double (&a)[Q], double b, int l, int lane0)
{
    double c[Q];   // lane l: c[j] = l_jl (j > l), column l of L
    double rown = 0.0;   // 1 / l_ll
#pragma unroll
    for (int j = 0; j < Q; ++j) c[j] = 0.0;
#pragma unroll Q
    for (int k = 0; k < Q; ++k) {
        const double akk = __shfl_sync(0xffffffffu, a[k], lane0 + k);
        const double r = rcp_pivot(sqrt(akk));    // 1 / l_kk
        const double lik = a[k] * r;               // l_ik (lane k: l_kk)
        const double yk = __shfl_sync(0xffffffffu, b * r, lane0 + k);
        if (l == k) { rown = r; b = yk; }
        else if (l > k) b = fma(-lik, yk, b);
#pragma unroll
        for (int j = 0; j < Q; ++j) {
            if (j > k) {   // compile-time after unrolling
                const double ljk = __shfl_sync(0xffffffffu, lik, lane0 + j);
                c[j] = l == k ? ljk : c[j];
                a[j] = fma(-lik, ljk, a[j]);
            }
        }
    }
    double x = 0.0;
#pragma unroll
    for (int jj = 0; jj < Q; ++jj) {
        const int j = Q - 1 - jj;
        const double xj = __shfl_sync(0xffffffffu, b * rown, lane0 + j);
        x = l == j ? xj : x;
        b = l < j ? fma(-c[j], xj, b) : b;
    }
    return x;
}
#ifndef MALS_CHOL
#define MALS_CHOL 0
#endif
template <int Q>
__device__ __forceinline__ double solve_sys(double (&a)[Q], double b, int l, int lane0)
{
    if constexpr (MALS_CHOL) return solve_chol<Q>(a, b, l, lane0);
    return solve_group<Q>(a, b, l, lane0);
}

// ---- q = 16: normal equations on the fp64 tensor cores ------------------------------------
// mma.sync m8n8k4 f64 (g = lane/4, t = lane%4): A (8x4) a0 = A[g][t]; B (4x8) b0 = B[t][g];
// C (8x8) c0, c1 = C[g][2t], C[g][2t+1].  For a system with samples k (gathered operand rows
// f_k): sum_k f_k f_k^T = F^T F and sum_k m_k f_k = F^T m are products with K = 4 samples per
// instruction; lane (g, t) loads f_t[g] and f_t[8 + g], which serve as both the A fragment (rows
// 8mt + g of F^T) and the B fragment (columns 8nt + g of F).  Exact fp64 products and sums
// (only the summation order differs from a sample-by-sample loop).
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b)
{
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

// accumulate [F^T F | F^T m] of one system (samples [p0, p1)) into the warp's scratch (16 x 17,
// row-major); `half` selects CSR (row system) or CSC (column system) indexing.  The system's
// (index, value) lists are read 32 entries at a time with coalesced loads, one batch ahead, and
// handed to the 4-sample steps by shuffles.  F^T F is symmetric: the tensor cores form the blocks
// (0,0), (0,1), (1,1) and (1,0) is written as the transpose of (0,1); F^T m is a per-lane fp64
// FMA sum over the lane's samples, reduced over the 4 lanes of a component at the end.
// the first 32-entry batch of a system's (index, value) list: lane k holds entry p0 + k (the zero
// row nf and value 0 past the end)
__device__ __forceinline__ void first_batch(const MArgs &A, int64_t ob, int half, int p0, int p1, int nf, int &bcol,
                                            double &bval)
{
    const int lane = threadIdx.x & 31;
    const uint16_t *idx = half == 0 ? A.col + ob : A.csc_row + ob;
    const double *val = half == 0 ? A.val + ob : A.valc + ob;
    bcol = nf;
    bval = 0.0;
    if (p0 + lane < p1) { bcol = idx[p0 + lane]; bval = val[p0 + lane]; }
}

__device__ __forceinline__ void accumulate_tc(const double *F, int nf, const MArgs &A, int64_t ob, int half, int p0,
                                              int p1, double inv_sigma, double *scr, int bcol, double bval)
{
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    double c00[2] = {0.0, 0.0}, c01[2] = {0.0, 0.0}, c11[2] = {0.0, 0.0};
    double b0 = 0.0, b1 = 0.0;
    const uint16_t *idx = half == 0 ? A.col + ob : A.csc_row + ob;
    const double *val = half == 0 ? A.val + ob : A.valc + ob;
    // (bcol, bval): the first batch, loaded by the caller ahead of time (first_batch)
    for (int pb = p0; pb < p1; pb += 32) {
        int ncol = nf;
        double nval = 0.0;
        if (pb + 32 + lane < p1) { ncol = idx[pb + 32 + lane]; nval = val[pb + 32 + lane]; }
        const int nst = min(8, (p1 - pb + 3) >> 2);   // warp-uniform
        for (int st = 0; st < nst; ++st) {
            const int oc = __shfl_sync(0xffffffffu, bcol, 4 * st + t);
            const double vc = __shfl_sync(0xffffffffu, bval, 4 * st + t);
            const double f0 = F[fidx<16>(oc, g)], f1 = F[fidx<16>(oc, 8 + g)];
            dmma(c00, f0, f0);
            dmma(c01, f0, f1);
            dmma(c11, f1, f1);
            b0 = fma(f0, vc, b0);
            b1 = fma(f1, vc, b1);
        }
        bcol = ncol;
        bval = nval;
    }
    b0 += __shfl_xor_sync(0xffffffffu, b0, 1);
    b0 += __shfl_xor_sync(0xffffffffu, b0, 2);
    b1 += __shfl_xor_sync(0xffffffffu, b1, 1);
    b1 += __shfl_xor_sync(0xffffffffu, b1, 2);
    double *r0 = scr + (size_t)g * 17, *r1 = scr + (size_t)(8 + g) * 17;
    r0[2 * t] = c00[0]; r0[2 * t + 1] = c00[1];
    r0[8 + 2 * t] = c01[0]; r0[8 + 2 * t + 1] = c01[1];
    scr[(size_t)(8 + 2 * t) * 17 + g] = c01[0];        // block (1,0) = (0,1)^T
    scr[(size_t)(8 + 2 * t + 1) * 17 + g] = c01[1];
    r1[8 + 2 * t] = c11[0]; r1[8 + 2 * t + 1] = c11[1];
    if (t == 0) {
        r0[16] = b0 * inv_sigma;
        r1[16] = b1 * inv_sigma;
    }
}

template <int Q>
__global__ void __launch_bounds__(MCfg<Q>::NT, 1) k_mals(MArgs A)
{
    extern __shared__ __align__(16) double dsm[];
    __shared__ double red[33];
    const int ls = A.order ? A.order[blockIdx.x] : (int)blockIdx.x, s = A.s0 + ls, tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5, nwarps = MCfg<Q>::NT >> 5;
    constexpr int GPW = 32 / Q;                  // systems per warp
    const int gi = lane / Q, l = lane % Q, lane0 = gi * Q;
    const int m = A.slice_off[s + 1] - A.slice_off[s];
    const int n = A.cut_n[ls];
    const int64_t lrow0 = A.slice_off[s] - A.lbase;
    const int64_t ob = (int64_t)ls * A.ncap, vb = (int64_t)ls * A.G * Q;
    const int32_t *rp = A.rowptr + (int64_t)ls * (A.mmax + 1);
    const int32_t *cp = A.colptr + (int64_t)ls * (A.G + 1);
    const int nnz = A.nnz[ls];
    double *F = dsm;                              // operand of the current half-step
    double *Xg = A.Xd + lrow0 * Q, *Yg = A.Yd + vb;
    float *Ug = A.U + lrow0 * Q, *Vg = A.V + vb;
    if (m <= Q || n <= Q) {
        if (tid == 0) { A.flags[ls] = LMC_SLICE_DIRECT; A.iters[ls] = 0; A.resid[ls] = 0.f; }
        return;
    }
    double mx = 0.0;
    for (int k = tid; k < nnz; k += MCfg<Q>::NT) mx = fmax(mx, A.val[ob + k]);
    const double sigma = dblock_reduce<true>(mx, red);
    if (sigma == 0.0) {
        for (int k = tid; k < m * Q; k += MCfg<Q>::NT) Ug[k] = 0.f;
        for (int k = tid; k < n * Q; k += MCfg<Q>::NT) Vg[k] = 0.f;
        if (tid == 0) { A.flags[ls] = LMC_SLICE_ZERO; A.iters[ls] = 0; A.resid[ls] = 0.f; }
        return;
    }
    for (int k = tid; k < nnz; k += MCfg<Q>::NT) A.valc[ob + k] = A.val[ob + A.csc_src[ob + k]];
    double sum = 0.0, sq = 0.0;
    for (int k = tid; k < nnz; k += MCfg<Q>::NT) {
        const double v = A.val[ob + k] / sigma;
        sum += v;
        sq = fma(v, v, sq);
    }
    sum = dblock_reduce<false>(sum, red);
    const double nrmM2 = dblock_reduce<false>(sq, red);
    const double c0 = 2.0 * sqrt((sum / (double)nnz) / (double)Q);
    for (int e = tid; e < m * Q; e += MCfg<Q>::NT)
        Xg[e] = c0 * (double)unif_f(philox4((uint32_t)(e / Q), (uint32_t)(e % Q), (uint32_t)(A.rs0 + ls * A.rss), TAG_X0, A.seed).x);
    for (int e = tid; e < n * Q; e += MCfg<Q>::NT)
        Yg[e] = c0 * (double)unif_f(philox4((uint32_t)(e % Q), (uint32_t)(e / Q), (uint32_t)(A.rs0 + ls * A.rss), TAG_Y0, A.seed).x);
    __syncthreads();
    const double lam = A.lambda;
    for (int it = 0; it < A.K; ++it) {
        for (int half = 0; half < 2; ++half) {
            const int nsys = half == 0 ? m : n, nf = half == 0 ? n : m;
            const int32_t *ptr = half == 0 ? rp : cp;
            const double *src = half == 0 ? Yg : Xg;     // operand gathered per sample
            double *O = half == 0 ? Xg : Yg;             // unknowns solved for
            if constexpr (!MCfg<Q>::FG) {
                for (int e = tid; e < nf * Q; e += MCfg<Q>::NT) F[fidx<Q>(e / Q, e % Q)] = src[e];
                for (int e = tid; e < Q; e += MCfg<Q>::NT) F[nf * Q + e] = 0.0;   // zero row for padding samples
            }
            const double *Fh = MCfg<Q>::FG ? src : F;
            __syncthreads();
            if constexpr (Q == 16) {
                // two systems per warp: tensor-core accumulation one after the other into the
                // warp's scratch, then one 16-lane Gauss-Jordan solve per system side by side
                double *scr = F + (size_t)(A.fmax + 1) * Q + (size_t)warp * 2 * 16 * 17;
                // the list bounds and first batches of both systems of the next pair are loaded
                // before this pair's accumulation / solve, so their global latency is hidden
                int q0n[2], q1n[2], bc[2];
                double bv[2];
#pragma unroll
                for (int h2 = 0; h2 < 2; ++h2) {
                    const int sy = warp * 2 + h2;
                    q0n[h2] = sy < nsys ? ptr[sy] : 0;
                    q1n[h2] = sy < nsys ? ptr[sy + 1] : 0;
                    first_batch(A, ob, half, q0n[h2], q1n[h2], nf, bc[h2], bv[h2]);
                }
                for (int sys0 = warp * 2; sys0 < nsys; sys0 += nwarps * 2) {
                    int q0[2], q1[2], bcc[2];
                    double bvc[2];
#pragma unroll
                    for (int h2 = 0; h2 < 2; ++h2) { q0[h2] = q0n[h2]; q1[h2] = q1n[h2]; bcc[h2] = bc[h2]; bvc[h2] = bv[h2]; }
#pragma unroll
                    for (int h2 = 0; h2 < 2; ++h2) {   // prefetch the next pair
                        const int sy = sys0 + nwarps * 2 + h2;
                        q0n[h2] = sy < nsys ? ptr[sy] : 0;
                        q1n[h2] = sy < nsys ? ptr[sy + 1] : 0;
                        first_batch(A, ob, half, q0n[h2], q1n[h2], nf, bc[h2], bv[h2]);
                    }
#pragma unroll
                    for (int h2 = 0; h2 < 2; ++h2)
                        accumulate_tc(F, nf, A, ob, half, q0[h2], q1[h2], 1.0 / sigma, scr + h2 * 16 * 17, bcc[h2], bvc[h2]);
                    __syncwarp();
                    const int sys = sys0 + gi;
                    double a[Q];
                    const double *row = scr + gi * 16 * 17 + l * 17;
#pragma unroll
                    for (int c = 0; c < Q; ++c) a[c] = row[c];
                    double b = row[16];
                    __syncwarp();
#pragma unroll
                    for (int c = 0; c < Q; ++c)
                        if (c == l) a[c] += lam;
                    const double x = solve_sys<Q>(a, b, l, lane0);
                    if (sys < nsys) O[(size_t)sys * Q + l] = x;
                }
                __syncthreads();
            } else {
            for (int sys0 = warp * GPW; sys0 < nsys; sys0 += nwarps * GPW) {
                const int sys = sys0 + gi;
                const bool valid = sys < nsys;
                double a[Q];
#pragma unroll
                for (int c = 0; c < Q; ++c) a[c] = 0.0;
                double b = 0.0;
                const int p0 = valid ? ptr[sys] : 0, p1 = valid ? ptr[sys + 1] : 0;
                for (int p = p0; p < p1; ++p) {
                    int other;
                    double v;
                    if (half == 0) {
                        other = A.col[ob + p];
                        v = A.val[ob + p];
                    } else {
                        other = A.csc_row[ob + p];
                        v = A.valc[ob + p];
                    }
                    const double mh = v / sigma;
                    const double *f = Fh + (size_t)other * Q;
                    const double fl = f[l];
#pragma unroll
                    for (int c = 0; c < Q; c += 2) {
                        const double2 t = *reinterpret_cast<const double2 *>(f + c);
                        a[c] = fma(fl, t.x, a[c]);
                        a[c + 1] = fma(fl, t.y, a[c + 1]);
                    }
                    b = fma(mh, fl, b);
                }
#pragma unroll
                for (int c = 0; c < Q; ++c)
                    if (c == l) a[c] += lam;   // static register index (no local-memory spill)
                const double x = solve_sys<Q>(a, b, l, lane0);
                if (valid) O[(size_t)sys * Q + l] = x;
            }
            __syncthreads();
            }
        }
    }
    // after the last column half F holds X (q = 32: X in global memory): residual on Omega (y from
    // global), outputs (X, sigma Y)
    double ss = 0.0;
    for (int i = tid; i < m; i += MCfg<Q>::NT) {
        for (int p = rp[i]; p < rp[i + 1]; ++p) {
            const double *y = Yg + (size_t)A.col[ob + p] * Q;
            double d = 0.0;
#pragma unroll
            for (int c = 0; c < Q; ++c) d = fma(MCfg<Q>::FG ? Xg[(size_t)i * Q + c] : F[fidx<Q>(i, c)], y[c], d);
            const double e = A.val[ob + p] / sigma - d;
            ss = fma(e, e, ss);
        }
    }
    ss = dblock_reduce<false>(ss, red);
    const double res = sqrt(ss / nrmM2);
    for (int e = tid; e < m * Q; e += MCfg<Q>::NT) Ug[e] = (float)(MCfg<Q>::FG ? Xg[e] : F[fidx<Q>(e / Q, e % Q)]);
    for (int e = tid; e < n * Q; e += MCfg<Q>::NT) Vg[e] = (float)(sigma * Yg[e]);
    if (tid == 0) {
        const bool bad = !(res == res) || isinf(res);
        A.flags[ls] = bad ? (LMC_SLICE_DIVERGED | LMC_SLICE_DIRECT) : 0;
        A.iters[ls] = A.K;
        A.resid[ls] = (float)res;
    }
}

size_t mals_smem_bytes(int q, int mmax, int G)
{
    // operand (max(m, n) + 1 zero row) x q fp64, plus at q = 16 a 2 x 16 x 17 scratch per warp
    const size_t scr = q == 16 ? (size_t)(MCfg<16>::NT / 32) * 2 * 16 * 17 * sizeof(double) : 0;
    if (q == 32) return 16;   // operand in global memory (MCfg<32>::FG)
    return ((size_t)std::max(mmax, G) + 1) * q * sizeof(double) + scr;
}

template <int Q>
static cudaError_t launch_mals(lmc_ctx *c, const MArgs &A)
{
    size_t sm = mals_smem_bytes(Q, c->mmax, c->G);
    cudaError_t e = cudaFuncSetAttribute(k_mals<Q>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    k_mals<Q><<<c->SL, MCfg<Q>::NT, sm, c->stream>>>(A);
    return cudaGetLastError();
}

cudaError_t run_mals(lmc_ctx *c)
{
    if (c->SL == 0) return cudaSuccess;
    MArgs A;
    A.slice_off = c->soff_k;
    A.s0 = c->s0k;
    A.lbase = c->lbase_k;
    A.rs0 = c->rs0;
    A.rss = c->rss;
    A.G = c->G;
    A.mmax = c->mmax;
    A.ncap = c->ncap;
    A.K = c->cfg.max_iter;
    A.lambda = c->cfg.lambda;
    A.seed = c->cfg.seed;
    A.cut_n = c->d.cut_n;
    A.rowptr = c->d.rowptr;
    A.colptr = c->d.colptr;
    A.csc_src = c->d.csc_src;
    A.nnz = c->d.nnz;
    A.col = c->d.col;
    A.csc_row = c->d.csc_row;
    A.val = c->d.val64;
    A.U = c->d.U;
    A.V = c->d.V;
    A.resid = c->d.resid;
    A.Xd = c->d.Xd;
    A.Yd = c->d.Yd;
    A.valc = c->d.val64c;
    A.fmax = std::max(c->mmax, c->G);
    A.flags = c->d.flags;
    A.iters = c->d.iters;
    A.order = c->adm_ordered ? c->d.adm_order : nullptr;
    switch (c->q) {
    case 4: return launch_mals<4>(c, A);
    case 8: return launch_mals<8>(c, A);
    case 16: return launch_mals<16>(c, A);
    case 32: return launch_mals<32>(c, A);
    default: return cudaErrorInvalidValue;
    }
}

}  // namespace lmc
