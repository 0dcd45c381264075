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
// shuffles.
#include "lmc_internal.h"
#include "philox.cuh"

namespace lmc {

struct MArgs {
    const int32_t *slice_off;
    int32_t s0, lbase, G, mmax;
    int64_t ncap;
    int K;
    double lambda;
    uint64_t seed;
    const int32_t *cut_n, *rowptr, *colptr, *csc_src, *nnz;
    const uint16_t *col, *csc_row;
    const double *val;             // fp64 entry values (the fp32 copy would perturb MALS, R34)
    float *U, *V, *resid;
    int32_t *flags, *iters;
};

constexpr int MT = 256;

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
template <int Q>
__device__ __forceinline__ double solve_group(double (&a)[Q], double b, int l, int lane0)
{
#pragma unroll
    for (int k = 0; k < Q; ++k) {
        double p[Q];
#pragma unroll
        for (int c = k; c < Q; ++c) p[c] = __shfl_sync(0xffffffffu, a[c], lane0 + k);
        const double pb = __shfl_sync(0xffffffffu, b, lane0 + k);
        const double ip = 1.0 / p[k];
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

template <int Q>
__global__ void __launch_bounds__(MT, 1) k_mals(MArgs A)
{
    extern __shared__ __align__(16) double dsm[];
    __shared__ double red[33];
    const int ls = blockIdx.x, s = A.s0 + ls, tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5, nwarps = MT >> 5;
    constexpr int GPW = 32 / Q;                  // systems per warp
    const int gi = lane / Q, l = lane % Q, lane0 = gi * Q;
    const int m = A.slice_off[s + 1] - A.slice_off[s];
    const int n = A.cut_n[ls];
    const int64_t lrow0 = A.slice_off[s] - A.lbase;
    const int64_t ob = (int64_t)ls * A.ncap, vb = (int64_t)ls * A.G * Q;
    const int32_t *rp = A.rowptr + (int64_t)ls * (A.mmax + 1);
    const int32_t *cp = A.colptr + (int64_t)ls * (A.G + 1);
    const int nnz = A.nnz[ls];
    double *X = dsm;
    double *Y = X + (size_t)A.mmax * Q;
    float *Ug = A.U + lrow0 * Q, *Vg = A.V + vb;
    if (m <= Q || n <= Q) {
        if (tid == 0) { A.flags[ls] = LMC_SLICE_DIRECT; A.iters[ls] = 0; A.resid[ls] = 0.f; }
        return;
    }
    double mx = 0.0;
    for (int k = tid; k < nnz; k += MT) mx = fmax(mx, A.val[ob + k]);
    const double sigma = dblock_reduce<true>(mx, red);
    if (sigma == 0.0) {
        for (int k = tid; k < m * Q; k += MT) Ug[k] = 0.f;
        for (int k = tid; k < n * Q; k += MT) Vg[k] = 0.f;
        if (tid == 0) { A.flags[ls] = LMC_SLICE_ZERO; A.iters[ls] = 0; A.resid[ls] = 0.f; }
        return;
    }
    double sum = 0.0, sq = 0.0;
    for (int k = tid; k < nnz; k += MT) {
        const double v = A.val[ob + k] / sigma;
        sum += v;
        sq = fma(v, v, sq);
    }
    sum = dblock_reduce<false>(sum, red);
    const double nrmM2 = dblock_reduce<false>(sq, red);
    const double c0 = 2.0 * sqrt((sum / (double)nnz) / (double)Q);
    for (int e = tid; e < m * Q; e += MT)
        X[e] = c0 * (double)unif_f(philox4((uint32_t)(e / Q), (uint32_t)(e % Q), (uint32_t)s, TAG_X0, A.seed).x);
    for (int e = tid; e < n * Q; e += MT)
        Y[e] = c0 * (double)unif_f(philox4((uint32_t)(e % Q), (uint32_t)(e / Q), (uint32_t)s, TAG_Y0, A.seed).x);
    __syncthreads();
    const double lam = A.lambda;
    for (int it = 0; it < A.K; ++it) {
        for (int half = 0; half < 2; ++half) {
            const int nsys = half == 0 ? m : n;
            const int32_t *ptr = half == 0 ? rp : cp;
            const double *F = half == 0 ? Y : X;     // operand gathered per sample
            double *O = half == 0 ? X : Y;           // unknowns solved for
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
                        v = A.val[ob + A.csc_src[ob + p]];
                    }
                    const double mh = v / sigma;
                    const double *f = F + (size_t)other * Q;
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
                const double x = solve_group<Q>(a, b, l, lane0);
                if (valid) O[(size_t)sys * Q + l] = x;
            }
            __syncthreads();
        }
    }
    // residual on Omega, outputs (X, sigma Y)
    double ss = 0.0;
    for (int i = tid; i < m; i += MT) {
        for (int p = rp[i]; p < rp[i + 1]; ++p) {
            const double *x = X + (size_t)i * Q, *y = Y + (size_t)A.col[ob + p] * Q;
            double d = 0.0;
#pragma unroll
            for (int c = 0; c < Q; ++c) d = fma(x[c], y[c], d);
            const double e = A.val[ob + p] / sigma - d;
            ss = fma(e, e, ss);
        }
    }
    ss = dblock_reduce<false>(ss, red);
    const double res = sqrt(ss / nrmM2);
    for (int e = tid; e < m * Q; e += MT) Ug[e] = (float)X[e];
    for (int e = tid; e < n * Q; e += MT) Vg[e] = (float)(sigma * Y[e]);
    if (tid == 0) {
        const bool bad = !(res == res) || isinf(res);
        A.flags[ls] = bad ? (LMC_SLICE_DIVERGED | LMC_SLICE_DIRECT) : 0;
        A.iters[ls] = A.K;
        A.resid[ls] = (float)res;
    }
}

size_t mals_smem_bytes(int q, int mmax, int G) { return ((size_t)mmax + (size_t)G) * q * sizeof(double); }

template <int Q>
static cudaError_t launch_mals(lmc_ctx *c, const MArgs &A)
{
    size_t sm = mals_smem_bytes(Q, c->mmax, c->G);
    cudaError_t e = cudaFuncSetAttribute(k_mals<Q>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    k_mals<Q><<<c->SL, MT, sm, c->stream>>>(A);
    return cudaGetLastError();
}

cudaError_t run_mals(lmc_ctx *c)
{
    if (c->SL == 0) return cudaSuccess;
    MArgs A;
    A.slice_off = c->d.slice_off;
    A.s0 = c->s0;
    A.lbase = c->h_slice_off[c->s0];
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
    A.flags = c->d.flags;
    A.iters = c->d.iters;
    switch (c->q) {
    case 4: return launch_mals<4>(c, A);
    case 8: return launch_mals<8>(c, A);
    case 16: return launch_mals<16>(c, A);
    default: return cudaErrorInvalidValue;
    }
}

}  // namespace lmc
