// complete.cu — per-slice low-rank completion and factored image rendering (sm_100a, fp32).
//
//   ADM      PAPER.md:149 and Appendix A, typo readings R18; Z kept implicit:
//            Z_k = X_k Y_k + S_k with S_k = P_Omega(M^ - X_k Y_k), so
//              Z_k Y_k^T   = X_k (Y_k Y_k^T) + S_k Y_k^T
//              X^T Z_k     = (X^T X_k) Y_k + X^T S_k
//            and X_{k+1} = X_k + (S_k Y_k^T + a U_k - L_k - a X_k)(Y_k Y_k^T + a I)^{-1}.
//   MALS     BASELINE north_star: per-row / per-column ridge normal equations over Omega,
//            accumulated in registers, solved by in-register Cholesky.
//   resolve  I(s) = X (Y e) with RGB weights w^k_c = I^k_c / lum(I_c) (R4).
//
// One CTA per slice; X (m x q) and Y (n x q, column j contiguous) stay in shared memory for
// all K iterations; Omega (CSR + CSC) streams from L2; U, Lambda, V, Pi and S live in global
// memory (L2-resident at the working-set sizes of a frame).
#include <cub/cub.cuh>

#include "lmc_internal.h"
#include "philox.cuh"

namespace lmc {

#define FULLM 0xffffffffu

struct CArgs {
    const int32_t *slice_off;
    int32_t s0, lbase, G, mmax;
    int64_t ncap;
    int K;
    float alpha, beta, gamma, tol, lambda;
    uint64_t seed;
    const int32_t *cut_n, *rowptr, *colptr, *csc_src, *nnz;
    const uint16_t *col, *csc_row;
    const float *val;
    float *U, *V, *Lam, *Pi, *Xold, *S, *resid;
    int32_t *flags, *iters;
};

template <int Q>
struct Cfg {
    static constexpr int QP = (Q >= 32) ? Q : Q + 4;          // padded row stride (floats)
    static constexpr int NT = (Q >= 32) ? 256 : 512;          // threads per CTA
    static constexpr int PART = 4096;                          // floats of Gram partials / GJ workspace
};

__device__ __forceinline__ float warp_sum(float v)
{
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULLM, v, o);
    return v;
}
__device__ __forceinline__ float warp_maxf(float v)
{
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(FULLM, v, o));
    return v;
}

// block-wide reduction (sum or max) of one float per thread; result broadcast to all threads
template <bool MAX>
__device__ float block_reduce(float v, float *red)
{
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    v = MAX ? warp_maxf(v) : warp_sum(v);
    __syncthreads();
    if (lane == 0) red[w] = v;
    __syncthreads();
    if (w == 0) {
        float t = lane < nw ? red[lane] : (MAX ? -INFINITY : 0.f);
        t = MAX ? warp_maxf(t) : warp_sum(t);
        if (lane == 0) red[32] = t;
    }
    __syncthreads();
    return red[32];
}

// out[a][b] = sum_i A[i][a] * B[i][b] over `rows` rows (A, B row-major with strides lda, ldb).
// Deterministic: fixed partition of rows and a fixed-order sum of the partials.
template <int Q>
__device__ void gram(const float *A, int lda, const float *B, int ldb, int rows, float *out, float *part)
{
    constexpr int TQ = Q / 4;
    constexpr int T = TQ * TQ;                 // 4x4 tiles
    int P = (int)blockDim.x / T;
    if (P * Q * Q > Cfg<Q>::PART) P = Cfg<Q>::PART / (Q * Q);
    const int tid = threadIdx.x;
    if (tid < P * T) {
        const int p = tid / T, tile = tid % T, ta = tile / TQ, tb = tile % TQ;
        float acc[4][4];
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
            for (int y = 0; y < 4; ++y) acc[x][y] = 0.f;
        for (int i = p; i < rows; i += P) {
            const float4 a = *reinterpret_cast<const float4 *>(A + (size_t)i * lda + 4 * ta);
            const float4 b = *reinterpret_cast<const float4 *>(B + (size_t)i * ldb + 4 * tb);
            const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
            for (int x = 0; x < 4; ++x)
#pragma unroll
                for (int y = 0; y < 4; ++y) acc[x][y] = fmaf(av[x], bv[y], acc[x][y]);
        }
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
            for (int y = 0; y < 4; ++y) part[(size_t)p * Q * Q + (4 * ta + x) * Q + 4 * tb + y] = acc[x][y];
    }
    __syncthreads();
    for (int e = tid; e < Q * Q; e += blockDim.x) {
        float s = 0.f;
        for (int p = 0; p < P; ++p) s += part[(size_t)p * Q * Q + e];
        out[e] = s;
    }
    __syncthreads();
}

// M <- (M + d I)^{-1} for SPD M (q x q), Gauss-Jordan without pivoting by warp 0; aug: 2 Q^2 floats
template <int Q>
__device__ void inv_spd(float *M, float d, float *aug)
{
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        constexpr int C2 = 2 * Q;
        for (int idx = lane; idx < Q * C2; idx += 32) {
            int r = idx / C2, c = idx % C2;
            aug[idx] = c < Q ? M[r * Q + c] + (r == c ? d : 0.f) : (c - Q == r ? 1.f : 0.f);
        }
        __syncwarp();
        for (int k = 0; k < Q; ++k) {
            const float ip = 1.0f / aug[k * C2 + k];
            __syncwarp();
            for (int c = lane; c < C2; c += 32) aug[k * C2 + c] *= ip;
            __syncwarp();
            for (int r = lane; r < Q; r += 32) {
                if (r == k) continue;
                const float f = aug[r * C2 + k];
#pragma unroll 8
                for (int c = 0; c < C2; ++c) aug[r * C2 + c] = fmaf(-f, aug[k * C2 + c], aug[r * C2 + c]);
            }
            __syncwarp();
        }
        for (int idx = lane; idx < Q * Q; idx += 32) M[idx] = aug[(idx / Q) * C2 + Q + idx % Q];
    }
    __syncthreads();
}

template <int Q>
__device__ __forceinline__ void load_vec(const float *p, float (&v)[Q])
{
#pragma unroll
    for (int l = 0; l < Q; l += 4) {
        float4 t = *reinterpret_cast<const float4 *>(p + l);
        v[l] = t.x; v[l + 1] = t.y; v[l + 2] = t.z; v[l + 3] = t.w;
    }
}
template <int Q>
__device__ __forceinline__ void store_vec(float *p, const float (&v)[Q])
{
#pragma unroll
    for (int l = 0; l < Q; l += 4) *reinterpret_cast<float4 *>(p + l) = make_float4(v[l], v[l + 1], v[l + 2], v[l + 3]);
}

// ------------------------------------------------------------------------------------------
// ADM (App. A): one CTA per slice
// ------------------------------------------------------------------------------------------
template <int Q>
__global__ void __launch_bounds__(Cfg<Q>::NT, 1) k_adm(CArgs A)
{
    constexpr int QP = Cfg<Q>::QP;
    extern __shared__ __align__(16) float sm[];
    __shared__ float red[33];
    const int ls = blockIdx.x, s = A.s0 + ls, tid = threadIdx.x, NT = blockDim.x;
    const int m = A.slice_off[s + 1] - A.slice_off[s];
    const int n = A.cut_n[ls];
    const int64_t lrow0 = A.slice_off[s] - A.lbase;
    const int64_t ob = (int64_t)ls * A.ncap, vb = (int64_t)ls * A.G * Q;
    const int32_t *rp = A.rowptr + (int64_t)ls * (A.mmax + 1);
    const int32_t *cp = A.colptr + (int64_t)ls * (A.G + 1);
    const int nnz = A.nnz[ls];
    float *X = sm;                                  // mmax x QP
    float *Y = X + (size_t)A.mmax * QP;             // G x QP
    float *Bm = Y + (size_t)A.G * QP;               // Q x Q : (Y Y^T + aI)^{-1}
    float *Dm = Bm + Q * Q;                         // (X^T X + bI)^{-1}
    float *Cm = Dm + Q * Q;                         // X_{k+1}^T X_k
    float *part = Cm + Q * Q;                       // PART
    float *Ug = A.U + (lrow0 * Q), *Lg = A.Lam + lrow0 * Q, *Xo = A.Xold + lrow0 * Q;
    float *Vg = A.V + vb, *Pg = A.Pi + vb;
    if (m <= Q || n <= Q) {   // R25: rank not below the slice dimensions -> direct rendering
        if (tid == 0) { A.flags[ls] = LMC_SLICE_DIRECT; A.iters[ls] = 0; A.resid[ls] = 0.f; }
        return;
    }
    // sigma = max_Omega M~ (R23); mean for the initial scale (R20)
    float mx = 0.f;
    for (int k = tid; k < nnz; k += NT) mx = fmaxf(mx, A.val[ob + k]);
    const float sigma = block_reduce<true>(mx, red);
    if (sigma == 0.f) {   // zero slice
        for (int k = tid; k < m * Q; k += NT) Ug[k] = 0.f;
        for (int k = tid; k < n * Q; k += NT) Vg[k] = 0.f;
        if (tid == 0) { A.flags[ls] = LMC_SLICE_ZERO; A.iters[ls] = 0; A.resid[ls] = 0.f; }
        return;
    }
    const float inv_sigma = 1.0f / sigma;
    float sum = 0.f, sq = 0.f;
    for (int k = tid; k < nnz; k += NT) {
        float v = A.val[ob + k] * inv_sigma;
        sum += v;
        sq = fmaf(v, v, sq);
    }
    sum = block_reduce<false>(sum, red);
    const float nrmM2 = block_reduce<false>(sq, red);
    const float mu = sum / (float)nnz;
    const float c0 = 2.0f * sqrtf(mu / (float)Q);
    // X_0, Y_0 (Philox uniform), U_0 = X_0, V_0 = Y_0, Lambda_0 = Pi_0 = 0
    for (int e = tid; e < m * Q; e += NT) {
        int i = e / Q, l = e % Q;
        float x = c0 * unif_f(philox4((uint32_t)i, (uint32_t)l, (uint32_t)s, TAG_X0, A.seed).x);
        X[i * QP + l] = x;
        Ug[e] = x;
        Lg[e] = 0.f;
    }
    for (int e = tid; e < n * Q; e += NT) {
        int j = e / Q, l = e % Q;
        float y = c0 * unif_f(philox4((uint32_t)l, (uint32_t)j, (uint32_t)s, TAG_Y0, A.seed).x);
        Y[j * QP + l] = y;
        Vg[e] = y;
        Pg[e] = 0.f;
    }
    __syncthreads();
    gram<Q>(Y, QP, Y, QP, n, Bm, part);
    inv_spd<Q>(Bm, A.alpha, part);
    const float al = A.alpha, be = A.beta, ga = A.gamma;
    int it = 0;
    for (; it < A.K; ++it) {
        const bool first = (it == 0);
        // ---- X_{k+1} = (Z_k Y_k^T + a U_k - L_k)(Y_k Y_k^T + a I)^{-1}; U, Lambda updates
        for (int i = tid; i < m; i += NT) {
            float x[Q], r[Q];
            load_vec<Q>(X + i * QP, x);
#pragma unroll
            for (int l = 0; l < Q; ++l) r[l] = 0.f;
            const int k1 = rp[i + 1];
            for (int k = rp[i]; k < k1; ++k) {
                const int j = A.col[ob + k];
                const float mh = A.val[ob + k] * inv_sigma;
                float y[Q];
                load_vec<Q>(Y + j * QP, y);
                float d = 0.f;
                if (!first) {
#pragma unroll
                    for (int l = 0; l < Q; ++l) d = fmaf(x[l], y[l], d);
                }
                const float sv = mh - d;
                A.S[ob + k] = sv;
#pragma unroll
                for (int l = 0; l < Q; ++l) r[l] = fmaf(sv, y[l], r[l]);
            }
            float u[Q], lam[Q];
            load_vec<Q>(Ug + i * Q, u);
            load_vec<Q>(Lg + i * Q, lam);
            float t[Q], xn[Q];
#pragma unroll
            for (int l = 0; l < Q; ++l) t[l] = r[l] + al * u[l] - lam[l] - (first ? 0.f : al * x[l]);
#pragma unroll
            for (int l = 0; l < Q; ++l) {
                float acc = first ? 0.f : x[l];
#pragma unroll
                for (int mm = 0; mm < Q; ++mm) acc = fmaf(t[mm], Bm[mm * Q + l], acc);
                xn[l] = acc;
            }
#pragma unroll
            for (int l = 0; l < Q; ++l) {
                const float un = fmaxf(0.f, xn[l] + lam[l] / al);
                lam[l] = lam[l] + ga * al * (xn[l] - un);
                u[l] = un;
            }
            store_vec<Q>(Xo + i * Q, x);
            store_vec<Q>(X + i * QP, xn);
            store_vec<Q>(Ug + i * Q, u);
            store_vec<Q>(Lg + i * Q, lam);
        }
        __syncthreads();
        // ---- (X^T X + bI)^{-1} and X_{k+1}^T X_k
        gram<Q>(X, QP, X, QP, m, Dm, part);
        inv_spd<Q>(Dm, be, part);
        if (!first) gram<Q>(X, QP, Xo, Q, m, Cm, part);
        // ---- Y_{k+1} = (X^T X + bI)^{-1} (X^T Z_k + b V_k - Pi_k); V, Pi updates
        for (int j = tid; j < n; j += NT) {
            float y[Q], t[Q];
            load_vec<Q>(Y + j * QP, y);
#pragma unroll
            for (int a = 0; a < Q; ++a) {
                float acc = 0.f;
                if (!first) {
#pragma unroll
                    for (int b = 0; b < Q; ++b) acc = fmaf(Cm[a * Q + b], y[b], acc);
                }
                t[a] = acc;
            }
            const int k1 = cp[j + 1];
            for (int k = cp[j]; k < k1; ++k) {
                const int i = A.csc_row[ob + k];
                const float sv = A.S[ob + A.csc_src[ob + k]];
                float xv[Q];
                load_vec<Q>(X + i * QP, xv);
#pragma unroll
                for (int l = 0; l < Q; ++l) t[l] = fmaf(sv, xv[l], t[l]);
            }
            float v[Q], pi[Q], yn[Q];
            load_vec<Q>(Vg + j * Q, v);
            load_vec<Q>(Pg + j * Q, pi);
#pragma unroll
            for (int l = 0; l < Q; ++l) t[l] = t[l] + be * v[l] - pi[l];
#pragma unroll
            for (int a = 0; a < Q; ++a) {
                float acc = 0.f;
#pragma unroll
                for (int b = 0; b < Q; ++b) acc = fmaf(Dm[a * Q + b], t[b], acc);
                yn[a] = acc;
            }
#pragma unroll
            for (int l = 0; l < Q; ++l) {
                const float vn = fmaxf(0.f, yn[l] + pi[l] / be);
                pi[l] = pi[l] + ga * be * (yn[l] - vn);
                v[l] = vn;
            }
            store_vec<Q>(Y + j * QP, yn);
            store_vec<Q>(Vg + j * Q, v);
            store_vec<Q>(Pg + j * Q, pi);
        }
        __syncthreads();
        // ---- (Y Y^T + aI)^{-1} for the next X step
        gram<Q>(Y, QP, Y, QP, n, Bm, part);
        inv_spd<Q>(Bm, al, part);
        // ---- optional tolerance stop on r_{k+1} = ||P_Omega(M^ - X_{k+1} Y_{k+1})|| / ||P_Omega M^||
        if (A.tol > 0.f) {
            float ss = 0.f;
            for (int i = tid; i < m; i += NT) {
                float x[Q];
                load_vec<Q>(X + i * QP, x);
                for (int k = rp[i]; k < rp[i + 1]; ++k) {
                    float y[Q];
                    load_vec<Q>(Y + A.col[ob + k] * QP, y);
                    float d = 0.f;
#pragma unroll
                    for (int l = 0; l < Q; ++l) d = fmaf(x[l], y[l], d);
                    const float e = A.val[ob + k] * inv_sigma - d;
                    ss = fmaf(e, e, ss);
                }
            }
            ss = block_reduce<false>(ss, red);
            if (!(ss == ss) || isinf(ss)) { ++it; break; }
            if (sqrtf(ss / nrmM2) < A.tol) { ++it; break; }
        }
    }
    // final residual on Omega and non-finite check
    float ss = 0.f;
    for (int i = tid; i < m; i += NT) {
        float x[Q];
        load_vec<Q>(X + i * QP, x);
        for (int k = rp[i]; k < rp[i + 1]; ++k) {
            float y[Q];
            load_vec<Q>(Y + A.col[ob + k] * QP, y);
            float d = 0.f;
#pragma unroll
            for (int l = 0; l < Q; ++l) d = fmaf(x[l], y[l], d);
            const float e = A.val[ob + k] * inv_sigma - d;
            ss = fmaf(e, e, ss);
        }
    }
    ss = block_reduce<false>(ss, red);
    const float res = sqrtf(ss / nrmM2);
    // output (U_K, sigma V_K) (R22)
    for (int e = tid; e < n * Q; e += NT) Vg[e] *= sigma;
    if (tid == 0) {
        const bool bad = !(res == res) || isinf(res);
        A.flags[ls] = bad ? (LMC_SLICE_DIVERGED | LMC_SLICE_DIRECT) : 0;
        A.iters[ls] = it;
        A.resid[ls] = res;
    }
}

// ------------------------------------------------------------------------------------------
// Masked ALS: x_i = (sum_{j in Omega_i} y_j y_j^T + lam I)^{-1} sum_j M^_ij y_j, then y_j alike.
// One thread per row (column); the packed upper triangle of the q x q Gram stays in registers.
// ------------------------------------------------------------------------------------------
template <int Q>
__device__ __forceinline__ void ridge_solve(float (&Ap)[Q * (Q + 1) / 2], float (&b)[Q], float lam, float (&x)[Q])
{
    // packed lower-triangular Cholesky in place: index (r, c<=r) -> r(r+1)/2 + c
#pragma unroll
    for (int r = 0; r < Q; ++r) Ap[r * (r + 1) / 2 + r] += lam;
#pragma unroll
    for (int j = 0; j < Q; ++j) {
        float d = Ap[j * (j + 1) / 2 + j];
#pragma unroll
        for (int k = 0; k < j; ++k) d = fmaf(-Ap[j * (j + 1) / 2 + k], Ap[j * (j + 1) / 2 + k], d);
        d = sqrtf(fmaxf(d, 1e-30f));
        const float id = 1.0f / d;
        Ap[j * (j + 1) / 2 + j] = d;
#pragma unroll
        for (int i = j + 1; i < Q; ++i) {
            float s = Ap[i * (i + 1) / 2 + j];
#pragma unroll
            for (int k = 0; k < j; ++k) s = fmaf(-Ap[i * (i + 1) / 2 + k], Ap[j * (j + 1) / 2 + k], s);
            Ap[i * (i + 1) / 2 + j] = s * id;
        }
    }
#pragma unroll
    for (int i = 0; i < Q; ++i) {
        float s = b[i];
#pragma unroll
        for (int k = 0; k < i; ++k) s = fmaf(-Ap[i * (i + 1) / 2 + k], x[k], s);
        x[i] = s / Ap[i * (i + 1) / 2 + i];
    }
#pragma unroll
    for (int i = Q - 1; i >= 0; --i) {
        float s = x[i];
#pragma unroll
        for (int k = i + 1; k < Q; ++k) s = fmaf(-Ap[k * (k + 1) / 2 + i], x[k], s);
        x[i] = s / Ap[i * (i + 1) / 2 + i];
    }
}

template <int Q>
__global__ void __launch_bounds__(256, 1) k_mals(CArgs A)
{
    constexpr int QP = Cfg<Q>::QP;
    constexpr int NP = Q * (Q + 1) / 2;
    extern __shared__ __align__(16) float sm[];
    __shared__ float red[33];
    const int ls = blockIdx.x, s = A.s0 + ls, tid = threadIdx.x, NT = blockDim.x;
    const int m = A.slice_off[s + 1] - A.slice_off[s];
    const int n = A.cut_n[ls];
    const int64_t lrow0 = A.slice_off[s] - A.lbase;
    const int64_t ob = (int64_t)ls * A.ncap, vb = (int64_t)ls * A.G * Q;
    const int32_t *rp = A.rowptr + (int64_t)ls * (A.mmax + 1);
    const int32_t *cp = A.colptr + (int64_t)ls * (A.G + 1);
    const int nnz = A.nnz[ls];
    float *X = sm;
    float *Y = X + (size_t)A.mmax * QP;
    float *Ug = A.U + lrow0 * Q, *Vg = A.V + vb;
    if (m <= Q || n <= Q) {
        if (tid == 0) { A.flags[ls] = LMC_SLICE_DIRECT; A.iters[ls] = 0; A.resid[ls] = 0.f; }
        return;
    }
    float mx = 0.f;
    for (int k = tid; k < nnz; k += NT) mx = fmaxf(mx, A.val[ob + k]);
    const float sigma = block_reduce<true>(mx, red);
    if (sigma == 0.f) {
        for (int k = tid; k < m * Q; k += NT) Ug[k] = 0.f;
        for (int k = tid; k < n * Q; k += NT) Vg[k] = 0.f;
        if (tid == 0) { A.flags[ls] = LMC_SLICE_ZERO; A.iters[ls] = 0; A.resid[ls] = 0.f; }
        return;
    }
    const float inv_sigma = 1.0f / sigma;
    float sum = 0.f, sq = 0.f;
    for (int k = tid; k < nnz; k += NT) {
        float v = A.val[ob + k] * inv_sigma;
        sum += v;
        sq = fmaf(v, v, sq);
    }
    sum = block_reduce<false>(sum, red);
    const float nrmM2 = block_reduce<false>(sq, red);
    const float c0 = 2.0f * sqrtf((sum / (float)nnz) / (float)Q);
    for (int e = tid; e < m * Q; e += NT)
        X[(e / Q) * QP + e % Q] = c0 * unif_f(philox4((uint32_t)(e / Q), (uint32_t)(e % Q), (uint32_t)s, TAG_X0, A.seed).x);
    for (int e = tid; e < n * Q; e += NT)
        Y[(e / Q) * QP + e % Q] = c0 * unif_f(philox4((uint32_t)(e % Q), (uint32_t)(e / Q), (uint32_t)s, TAG_Y0, A.seed).x);
    __syncthreads();
    for (int it = 0; it < A.K; ++it) {
        for (int i = tid; i < m; i += NT) {
            float Ap[NP], b[Q], x[Q];
#pragma unroll
            for (int e = 0; e < NP; ++e) Ap[e] = 0.f;
#pragma unroll
            for (int l = 0; l < Q; ++l) b[l] = 0.f;
            for (int k = rp[i]; k < rp[i + 1]; ++k) {
                float y[Q];
                load_vec<Q>(Y + A.col[ob + k] * QP, y);
                const float mh = A.val[ob + k] * inv_sigma;
#pragma unroll
                for (int r = 0; r < Q; ++r) {
#pragma unroll
                    for (int c = 0; c <= r; ++c) Ap[r * (r + 1) / 2 + c] = fmaf(y[r], y[c], Ap[r * (r + 1) / 2 + c]);
                    b[r] = fmaf(mh, y[r], b[r]);
                }
            }
            ridge_solve<Q>(Ap, b, A.lambda, x);
            store_vec<Q>(X + i * QP, x);
        }
        __syncthreads();
        for (int j = tid; j < n; j += NT) {
            float Ap[NP], b[Q], y[Q];
#pragma unroll
            for (int e = 0; e < NP; ++e) Ap[e] = 0.f;
#pragma unroll
            for (int l = 0; l < Q; ++l) b[l] = 0.f;
            for (int k = cp[j]; k < cp[j + 1]; ++k) {
                float xv[Q];
                load_vec<Q>(X + A.csc_row[ob + k] * QP, xv);
                const float mh = A.val[ob + A.csc_src[ob + k]] * inv_sigma;
#pragma unroll
                for (int r = 0; r < Q; ++r) {
#pragma unroll
                    for (int c = 0; c <= r; ++c) Ap[r * (r + 1) / 2 + c] = fmaf(xv[r], xv[c], Ap[r * (r + 1) / 2 + c]);
                    b[r] = fmaf(mh, xv[r], b[r]);
                }
            }
            ridge_solve<Q>(Ap, b, A.lambda, y);
            store_vec<Q>(Y + j * QP, y);
        }
        __syncthreads();
    }
    float ss = 0.f;
    for (int i = tid; i < m; i += NT) {
        float x[Q];
        load_vec<Q>(X + i * QP, x);
        for (int k = rp[i]; k < rp[i + 1]; ++k) {
            float y[Q];
            load_vec<Q>(Y + A.col[ob + k] * QP, y);
            float d = 0.f;
#pragma unroll
            for (int l = 0; l < Q; ++l) d = fmaf(x[l], y[l], d);
            const float e = A.val[ob + k] * inv_sigma - d;
            ss = fmaf(e, e, ss);
        }
    }
    ss = block_reduce<false>(ss, red);
    const float res = sqrtf(ss / nrmM2);
    for (int e = tid; e < m * Q; e += NT) Ug[e] = X[(e / Q) * QP + e % Q];
    for (int e = tid; e < n * Q; e += NT) Vg[e] = sigma * Y[(e / Q) * QP + e % Q];
    if (tid == 0) {
        const bool bad = !(res == res) || isinf(res);
        A.flags[ls] = bad ? (LMC_SLICE_DIVERGED | LMC_SLICE_DIRECT) : 0;
        A.iters[ls] = A.K;
        A.resid[ls] = res;
    }
}

size_t complete_smem_bytes(int q, int mmax, int G, int solver)
{
    int qp = q >= 32 ? q : q + 4;
    size_t base = ((size_t)mmax + (size_t)G) * qp * sizeof(float);
    if (solver == LMC_SOLVER_MALS) return base;
    return base + (3 * (size_t)q * q + 4096) * sizeof(float);
}

static CArgs cargs(lmc_ctx *c)
{
    CArgs A;
    A.slice_off = c->d.slice_off;
    A.s0 = c->s0;
    A.lbase = c->h_slice_off[c->s0];
    A.G = c->G;
    A.mmax = c->mmax;
    A.ncap = c->ncap;
    A.K = c->cfg.max_iter;
    A.alpha = (float)c->cfg.alpha;
    A.beta = (float)c->cfg.beta;
    A.gamma = (float)c->cfg.gamma;
    A.tol = (float)c->cfg.tol;
    A.lambda = (float)c->cfg.lambda;
    A.seed = c->cfg.seed;
    A.cut_n = c->d.cut_n;
    A.rowptr = c->d.rowptr;
    A.colptr = c->d.colptr;
    A.csc_src = c->d.csc_src;
    A.nnz = c->d.nnz;
    A.col = c->d.col;
    A.csc_row = c->d.csc_row;
    A.val = c->d.val;
    A.U = c->d.U;
    A.V = c->d.V;
    A.Lam = c->d.Lam;
    A.Pi = c->d.Pi;
    A.Xold = c->d.Xold;
    A.S = c->d.S;
    A.resid = c->d.resid;
    A.flags = c->d.flags;
    A.iters = c->d.iters;
    return A;
}

template <int Q>
static cudaError_t launch_q(lmc_ctx *c, const CArgs &A)
{
    size_t sm = complete_smem_bytes(Q, c->mmax, c->G, c->cfg.solver);
    cudaError_t e;
    if (c->cfg.solver == LMC_SOLVER_MALS) {
        e = cudaFuncSetAttribute(k_mals<Q>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        if (e != cudaSuccess) return e;
        k_mals<Q><<<c->SL, 256, sm, c->stream>>>(A);
    } else {
        e = cudaFuncSetAttribute(k_adm<Q>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        if (e != cudaSuccess) return e;
        k_adm<Q><<<c->SL, Cfg<Q>::NT, sm, c->stream>>>(A);
    }
    return cudaGetLastError();
}

cudaError_t run_complete(lmc_ctx *c)
{
    if (c->SL == 0) return cudaSuccess;
    CArgs A = cargs(c);
    switch (c->q) {
    case 4: return launch_q<4>(c, A);
    case 8: return launch_q<8>(c, A);
    case 16: return launch_q<16>(c, A);
    case 32: return launch_q<32>(c, A);
    default: return cudaErrorInvalidValue;
    }
}

// ------------------------------------------------------------------------------------------
// Resolve: t^k = V w^k (q-vectors), out^k_i = tint^k_i <U_i, t^k>
// ------------------------------------------------------------------------------------------
struct RArgs {
    const int32_t *slice_off, *rows, *pixel, *cut_n, *cut_cols, *flags;
    int32_t s0, lbase, G, q;
    int64_t row0;
    const float *U, *V, *I, *direct_rgb;
    const float4 *prow;
    float *image, *rows_rgb;
};

__global__ void __launch_bounds__(256) k_resolve(RArgs A)
{
    __shared__ float t[3 * MAX_Q];
    __shared__ float wsum[8][3 * MAX_Q];
    const int ls = blockIdx.x, s = A.s0 + ls, tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int m = A.slice_off[s + 1] - A.slice_off[s], n = A.cut_n[ls], q = A.q;
    const int64_t lrow0 = A.slice_off[s] - A.lbase;
    const int fl = A.flags[ls];
    const float *V = A.V + (int64_t)ls * A.G * q;
    const int64_t cb = (int64_t)ls * A.G;
    if (!(fl & (LMC_SLICE_DIRECT | LMC_SLICE_ZERO))) {
        // each warp: partial t over a strided subset of columns
        for (int e = lane; e < 3 * q; e += 32) {
            const int k = e / q, a = e % q;
            float acc = 0.f;
            for (int cidx = w; cidx < n; cidx += 8) {
                const int u = A.cut_cols[cb + cidx];
                const float i0 = A.I[3 * u], i1 = A.I[3 * u + 1], i2 = A.I[3 * u + 2];
                const float li = (0.2126f * i0 + 0.7152f * i1) + 0.0722f * i2;
                const float wk = li != 0.f ? A.I[3 * u + k] / li : 0.f;
                acc = fmaf(V[(int64_t)cidx * q + a], wk, acc);
            }
            wsum[w][e] = acc;
        }
        __syncthreads();
        for (int e = tid; e < 3 * q; e += blockDim.x) {
            float acc = 0.f;
            for (int k = 0; k < 8; ++k) acc += wsum[k][e];
            t[e] = acc;
        }
        __syncthreads();
    }
    for (int i = tid; i < m; i += blockDim.x) {
        const int64_t li = lrow0 + i;
        float o0 = 0.f, o1 = 0.f, o2 = 0.f;
        if (fl & LMC_SLICE_DIRECT) {
            o0 = A.direct_rgb[3 * li];
            o1 = A.direct_rgb[3 * li + 1];
            o2 = A.direct_rgb[3 * li + 2];
        } else if (!(fl & LMC_SLICE_ZERO)) {
            const float *u = A.U + li * q;
            float d0 = 0.f, d1 = 0.f, d2 = 0.f;
            for (int a = 0; a < q; ++a) {
                const float ua = u[a];
                d0 = fmaf(ua, t[a], d0);
                d1 = fmaf(ua, t[q + a], d1);
                d2 = fmaf(ua, t[2 * q + a], d2);
            }
            const float4 C = A.prow[4 * li + 2], D = A.prow[4 * li + 3];
            const float lr = (0.2126f * C.z + 0.7152f * C.w) + 0.0722f * D.x;
            const float ir = lr != 0.f ? 1.0f / lr : 0.f;
            o0 = C.z * ir * d0;
            o1 = C.w * ir * d1;
            o2 = D.x * ir * d2;
        }
        if (A.rows_rgb) {
            A.rows_rgb[3 * li] = o0;
            A.rows_rgb[3 * li + 1] = o1;
            A.rows_rgb[3 * li + 2] = o2;
        }
        if (A.image) {
            const int64_t p = A.pixel[A.rows[A.row0 + li]];
            A.image[3 * p] = o0;
            A.image[3 * p + 1] = o1;
            A.image[3 * p + 2] = o2;
        }
    }
}

cudaError_t run_resolve(lmc_ctx *c, float *image, float *rows_rgb)
{
    if (c->SL == 0) return cudaSuccess;
    RArgs A;
    A.slice_off = c->d.slice_off;
    A.rows = c->d.rows;
    A.pixel = c->d.pixel;
    A.cut_n = c->d.cut_n;
    A.cut_cols = c->d.cut_cols;
    A.flags = c->d.flags;
    A.s0 = c->s0;
    A.lbase = c->h_slice_off[c->s0];
    A.G = c->G;
    A.q = c->q;
    A.row0 = c->row0;
    A.U = c->d.U;
    A.V = c->d.V;
    A.I = c->d.ut_I;
    A.direct_rgb = c->d.direct_rgb;
    A.prow = c->d.prow;
    A.image = image;
    A.rows_rgb = rows_rgb;
    k_resolve<<<c->SL, 256, 0, c->stream>>>(A);
    return cudaGetLastError();
}

__global__ void k_scatter(int64_t M, const int32_t *__restrict__ rows, const int32_t *__restrict__ pixel,
                          const float *__restrict__ all_rows, float *image)
{
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= M) return;
    const int64_t p = pixel[rows[k]];
    image[3 * p] = all_rows[3 * k];
    image[3 * p + 1] = all_rows[3 * k + 1];
    image[3 * p + 2] = all_rows[3 * k + 2];
}

cudaError_t run_scatter(lmc_ctx *c, const float *all_rows, float *image)
{
    if (c->M == 0) return cudaSuccess;
    k_scatter<<<(unsigned)((c->M + 255) / 256), 256, 0, c->stream>>>(c->M, c->d.rows, c->d.pixel, all_rows, image);
    return cudaGetLastError();
}

}  // namespace lmc
