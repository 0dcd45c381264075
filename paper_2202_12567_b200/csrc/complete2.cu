// complete2.cu — ADM completion, lane-per-segment design (q = 4, 8, 16), sm_100a.
//
//   ADM  PAPER.md:149 and Appendix A, typo readings R18, fp32, Z never formed
//        (same algebra as complete.cu's header):
//          X_{k+1} = X_k + (S_k Y_k^T + a U_k - L_k - a X_k)(Y_k Y_k^T + a I)^{-1},
//          X_{k+1}^T Z_k = (X_{k+1}^T X_k) Y_k + X_{k+1}^T S_k,  S_k = P_Omega(M^ - X_k Y_k).
//
// Work decomposition.  One CTA per slice; X (rows) and Y (columns) stay in shared memory for all
// K iterations, stored row-major with the 16-byte blocks of row r XOR-swizzled by swz(r).  A lane
// owns one *segment* of a member (a row in the row phase, a column in the column phase): it holds
// the member's q-vector and its accumulator in registers and walks the segment's samples, so a
// sample costs one q-vector gather (q/4 16-byte shared loads), 2q FMAs and no shuffles.  Long
// members are split into a power-of-two number of segments on aligned neighbouring lanes, summed
// by an xor butterfly before the update.  The residual s_ij of the row phase is written at the
// sample's column-layout position: into shared memory for the leading column groups that fit
// next to X and Y, into global memory for the rest; the column phase reads S coalesced.
// Omega streams straight into registers (coalesced 16-byte loads one 8-k-step batch ahead).
//
// Bank conflicts.  Every X / Y row takes 64 bytes (q = 8 and q = 4 rows are stored 2x / 4x), so
// row r's 16-byte blocks sit in bank group 4 (r & 1) + block.  Lane l reads the blocks of a row
// in the order c ^ rot(l), rot(l) = (l >> 1) & 3 (its q-vectors live in registers in that rotated
// order), and at k-step k takes, when it can, a sample whose gathered index has parity (l + k) & 1.
// The eight lanes of a quarter warp (one 128-byte shared-memory phase of a 16-byte load) then form
// four rotation pairs of opposite parity: eight distinct bank groups, no conflict.  Padding
// entries gather one of two zero rows, the one with the wanted parity.
#include <cub/cub.cuh>
#include <cstdio>
#include <cstdlib>
#include <algorithm>

#include "lmc_internal.h"
#include "philox.cuh"

namespace lmc {

#define FULLM2 0xffffffffu

// zero row of the wanted parity among the two sentinel rows cnt, cnt + 1
__host__ __device__ __forceinline__ int zrow(int cnt, int want) { return cnt + ((cnt + want) & 1); }

// ------------------------------------------------------------------------------------------
// Layout (one CTA of 1024 threads per slice)
// ------------------------------------------------------------------------------------------
constexpr int LT2 = 1024;
#ifndef ADM2_KB
#define ADM2_KB 8
#endif
constexpr int KB = ADM2_KB;   // k-steps per register batch (group lengths are multiples of it)

struct L2Args {
    const int32_t *slice_off, *cut_n, *rowptr, *colptr, *csc_src, *nnz;
    const uint16_t *col, *csc_row;
    const float *val;
    int32_t s0, G, mmax, q, Tr, Tc;
    int64_t ncap, scap, gcap;
    int4 *r_grp, *c_grp;         // [SL][gcap] (goff, Kg, maxlg, 0)
    uint32_t *r_slot, *c_slot;   // [SL][gcap * 32] member | seg << 11 | lg << 16
    int32_t *ngrp;               // [SL][2] row groups, column groups
    int32_t *ctot;               // [SL] column-layout size (the dummy S slot)
    unsigned long long *r_ent;   // [SL][scap] (M^ bits << 32) | (S position << 11) | column
    uint16_t *c_code;            // [SL][scap] row
    float *S;                    // [SL][scap]
    int32_t *map;                // [SL][ncap] CSR index -> S position
    float4 *norm;                // [SL] sigma, 1/sigma, sum M^, sum M^^2
    unsigned long long *counters;
};

__device__ __forceinline__ float warp_sum2(float v)
{
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULLM2, v, o);
    return v;
}
__device__ __forceinline__ float warp_max2(float v)
{
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(FULLM2, v, o));
    return v;
}
template <bool MAX>
__device__ float block_reduce2(float v, float *red)
{
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    v = MAX ? warp_max2(v) : warp_sum2(v);
    __syncthreads();
    if (lane == 0) red[w] = v;
    __syncthreads();
    if (w == 0) {
        float t = lane < nw ? red[lane] : (MAX ? -INFINITY : 0.f);
        t = MAX ? warp_max2(t) : warp_sum2(t);
        if (lane == 0) red[32] = t;
    }
    __syncthreads();
    return red[32];
}

// positions inside a group (base = goff): row entries in pairs of k-steps, column codes in
// eights, column S in fours, each lane-interleaved so a warp reads one contiguous span
__device__ __forceinline__ int pos_rent(int k, int l) { return (k >> 1) * 64 + l * 2 + (k & 1); }
__device__ __forceinline__ int pos_ccode(int k, int l) { return (k >> 3) * 256 + l * 8 + (k & 7); }
__device__ __forceinline__ int pos_cs(int k, int l) { return (k >> 2) * 128 + l * 4 + (k & 3); }

template <int Q>
__global__ void __launch_bounds__(LT2, 1) k_layout2(L2Args A)
{
    typedef cub::BlockRadixSort<uint32_t, LT2, 1> Sort;
    typedef cub::BlockScan<int32_t, LT2> Scan;
    union TmpU {
        typename Sort::TempStorage sort;
        typename Scan::TempStorage scan;
    };
    extern __shared__ __align__(16) unsigned char lsm2[];
    TmpU &tmp = *reinterpret_cast<TmpU *>(lsm2);
    __shared__ int32_t sh_kg[LT2];      // per group: max segment length, then rounded
    __shared__ int32_t sh_lg[LT2];      // per group: max log2 segments
    __shared__ int32_t sh_goff[LT2 + 1];
    __shared__ int32_t sh_who[LT2], sh_len[LT2], sh_slot0[LT2], sh_mlg[LT2];
    __shared__ float red[33];
    const int ls = blockIdx.x, s = A.s0 + ls, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int m = A.slice_off[s + 1] - A.slice_off[s], n = A.cut_n[ls];
    const int64_t ob = (int64_t)ls * A.ncap, sb = (int64_t)ls * A.scap, gb = (int64_t)ls * A.gcap;
    const int32_t *rp = A.rowptr + (int64_t)ls * (A.mmax + 1);
    const int32_t *cp = A.colptr + (int64_t)ls * (A.G + 1);
    const int nnz = A.nnz[ls];
    float mx = 0.f;
    for (int k = tid; k < nnz; k += LT2) mx = fmaxf(mx, A.val[ob + k]);
    const float sigma = block_reduce2<true>(mx, red);   // R23: sigma = max_Omega M~
    const float inv_sigma = sigma > 0.f ? 1.0f / sigma : 0.f;
    float sum = 0.f, sq = 0.f;
    for (int k = tid; k < nnz; k += LT2) {
        const float v = A.val[ob + k] * inv_sigma;
        sum += v;
        sq = fmaf(v, v, sq);
    }
    sum = block_reduce2<false>(sum, red);
    sq = block_reduce2<false>(sq, red);
    if (tid == 0) A.norm[ls] = make_float4(sigma, inv_sigma, sum, sq);
    int dummy = 0;
    const unsigned lt_mask = (1u << lane) - 1u;
    for (int pass = 0; pass < 2; ++pass) {
        const bool rows = pass == 1;   // columns first: the row entries carry S positions
        const int cnt = rows ? m : n, T = rows ? A.Tr : A.Tc;
        const int32_t *ptr = rows ? rp : cp;
        int4 *grp = (rows ? A.r_grp : A.c_grp) + gb;
        uint32_t *slot = (rows ? A.r_slot : A.c_slot) + gb * 32;
        // segments: nseg = next power of two >= ceil(len / T) (<= 32), lengths differ by <= 1
        int len = 0, lg = 0, smax = 0;
        if (tid < cnt) {
            len = ptr[tid + 1] - ptr[tid];
            const int need = max(1, (len + T - 1) / T);
            while ((1 << lg) < need && lg < 5) ++lg;
            smax = (len + (1 << lg) - 1) >> lg;
        }
        // members by (segments desc, segment length desc, id): power-of-two segment counts in
        // descending order keep every member's lanes inside one group, aligned
        uint32_t key[1] = {tid < cnt ? ((uint32_t)(5 - lg) << 21) | ((uint32_t)(2047 - min(smax, 2047)) << 10) | (uint32_t)tid
                                     : 0xFFFFFFFFu};
        Sort(tmp.sort).Sort(key, 0, 24);
        __syncthreads();
        const int who = (int)(key[0] & 1023u);
        const bool mem = tid < cnt;
        const int mlg = mem ? 5 - (int)(key[0] >> 21) : 0;
        const int nsg = mem ? (1 << mlg) : 0;
        int s0, tot;
        Scan(tmp.scan).ExclusiveSum(nsg, s0, tot);
        const int ng = (tot + 31) >> 5;
        if (tid < LT2) { sh_kg[tid] = 0; sh_lg[tid] = 0; }
        __syncthreads();
        if (mem) {
            const int l2 = ptr[who + 1] - ptr[who];
            sh_who[tid] = who;
            sh_len[tid] = l2;
            sh_slot0[tid] = s0;
            sh_mlg[tid] = mlg;
            for (int sg = 0; sg < nsg; ++sg) {
                const int e0 = (l2 * sg) >> mlg, e1 = (l2 * (sg + 1)) >> mlg;
                atomicMax(&sh_kg[(s0 + sg) >> 5], e1 - e0);
            }
            atomicMax(&sh_lg[s0 >> 5], mlg);
        }
        __syncthreads();
        int gsz = 0;
        if (tid < ng) {
            const int kg = (sh_kg[tid] + KB - 1) / KB * KB;
            sh_kg[tid] = kg;
            gsz = 32 * kg;
        }
        int pre, gtot;
        Scan(tmp.scan).ExclusiveSum(gsz, pre, gtot);
        if (gtot + 1 > A.scap || ng > A.gcap || (!rows && gtot >= (1 << 21))) {   // block-uniform
            if (tid == 0) {
                atomicOr(&A.counters[3], 4ull);   // reported by the next getter / stats call
                A.ngrp[2 * ls] = 0;
                A.ngrp[2 * ls + 1] = 0;
            }
            return;
        }
        if (tid < ng) {
            sh_goff[tid] = pre;
            grp[tid] = make_int4(pre, sh_kg[tid], sh_lg[tid], 0);
        }
        if (tid == 0) {
            sh_goff[ng] = gtot;
            A.ngrp[2 * ls + (rows ? 0 : 1)] = ng;
            if (!rows) A.ctot[ls] = gtot;
            atomicAdd(&A.counters[rows ? 6 : 7], (unsigned long long)gtot);   // padded layout sizes (stats)
        }
        if (!rows) dummy = gtot;
        __syncthreads();
        // empty lanes of the last group: sentinel member (zero row m / zero column n)
        for (int sl = tot + tid; sl < ng * 32; sl += LT2) {
            slot[sl] = (uint32_t)cnt;
            const int g = sl >> 5, l = sl & 31, base = sh_goff[g], kg = sh_kg[g];
            for (int k = 0; k < kg; ++k) {
                if (rows) {
                    A.r_ent[sb + base + pos_rent(k, l)] = ((unsigned long long)(uint32_t)dummy << 11) | (unsigned long long)zrow(n, (l + k) & 1);
                } else {
                    A.c_code[sb + base + pos_ccode(k, l)] = (uint16_t)zrow(m, (l + k) & 1);
                    A.S[sb + base + pos_cs(k, l)] = 0.f;
                }
            }
        }
        // a warp per segment: entries of the member in [e0, e1), placed so that k-step k takes an
        // entry whose gathered index has parity (l + k) & 1 when it can; the leftover entries of
        // the more frequent parity fill the positions the other one could not (closed form)
        const uint16_t *gidx = rows ? (A.col + ob) : (A.csc_row + ob);
        for (int r = warp; r < cnt; r += LT2 / 32) {
            const int mw = sh_who[r], ml = sh_len[r], mlg2 = sh_mlg[r], ms0 = sh_slot0[r];
            const int mp0 = ptr[mw];
            for (int sg = 0; sg < (1 << mlg2); ++sg) {
                const int sl = ms0 + sg, g = sl >> 5, l = sl & 31;
                const int e0 = (ml * sg) >> mlg2, e1 = (ml * (sg + 1)) >> mlg2, Ls = e1 - e0;
                const int base = sh_goff[g], kg = sh_kg[g];
                if (lane == 0) slot[sl] = (uint32_t)mw | ((uint32_t)sg << 11) | ((uint32_t)mlg2 << 16);
                int nodd = 0;
                for (int k0 = 0; k0 < Ls; k0 += 32) {
                    const int k = k0 + lane;
                    nodd += __popc(__ballot_sync(FULLM2, k < Ls && (gidx[mp0 + e0 + k] & 1)));
                }
                // positions k = 2 j + rb[b] want parity b, rb[b] = (b - l) & 1
                const int cnt2[2] = {Ls - nodd, nodd};
                int rb[2], npos[2], fill[2];
#pragma unroll
                for (int b = 0; b < 2; ++b) {
                    rb[b] = (b - l) & 1;
                    npos[b] = Ls > rb[b] ? (Ls - rb[b] + 1) >> 1 : 0;
                    fill[b] = min(cnt2[b], npos[b]);
                }
                int seen[2] = {0, 0};
                for (int k0 = 0; k0 < Ls; k0 += 32) {
                    const int kk = k0 + lane;
                    const bool in = kk < Ls;
                    const int e = mp0 + e0 + kk;
                    const int res = in ? (int)(gidx[e] & 1) : -1;
                    int j = 0;
#pragma unroll
                    for (int b = 0; b < 2; ++b) {
                        const unsigned bm = __ballot_sync(FULLM2, res == b);
                        if (res == b) j = seen[b] + __popc(bm & lt_mask);
                        seen[b] += __popc(bm);
                    }
                    if (!in) continue;
                    // own parity while its positions last, then the other parity's spare positions
                    const int k = j < fill[res] ? 2 * j + rb[res] : 2 * (fill[res ^ 1] + (j - fill[res])) + rb[res ^ 1];
                    if (rows) {
                        const float mh = A.val[ob + e] * inv_sigma;
                        A.r_ent[sb + base + pos_rent(k, l)] = ((unsigned long long)__float_as_uint(mh) << 32) |
                                                              ((unsigned long long)(uint32_t)A.map[ob + e] << 11) |
                                                              (unsigned long long)A.col[ob + e];
                    } else {
                        const int sp = base + pos_cs(k, l);
                        A.c_code[sb + base + pos_ccode(k, l)] = A.csc_row[ob + e];
                        A.map[ob + A.csc_src[ob + e]] = sp;
                        A.S[sb + sp] = 0.f;
                    }
                }
                for (int k = Ls + lane; k < kg; k += 32) {   // padding k-steps of this lane
                    if (rows) {
                        A.r_ent[sb + base + pos_rent(k, l)] = ((unsigned long long)(uint32_t)dummy << 11) | (unsigned long long)zrow(n, (l + k) & 1);
                    } else {
                        A.c_code[sb + base + pos_ccode(k, l)] = (uint16_t)zrow(m, (l + k) & 1);
                        A.S[sb + base + pos_cs(k, l)] = 0.f;
                    }
                }
            }
        }
        __syncthreads();
    }
    if (tid == 0) A.S[sb + dummy] = 0.f;
}

// ------------------------------------------------------------------------------------------
// ADM kernel
// ------------------------------------------------------------------------------------------
struct C2Args {
    const int32_t *slice_off;
    int32_t s0, lbase, G, mmax;
    int32_t rs0, rss;   // global slice id of local slice ls: rs0 + ls * rss (the draws' key)
    int64_t scap, gcap;
    int K;
    float alpha, beta, gamma, tol;
    uint64_t seed;
    int32_t smem_bytes;
    const int32_t *cut_n, *nnz, *ngrp, *ctot;
    const float4 *norm;
    const int4 *r_grp, *c_grp;
    const uint32_t *r_slot, *c_slot;
    const unsigned long long *r_ent;
    const uint16_t *c_code;
    float *U, *V, *Lam, *Pi, *Xold, *S, *resid;
    float *Us, *Ls, *Xs, *Vs, *Ps;   // per-slot state [SL][gcap * 32 * Q] (see st_slot)
    int32_t *flags, *iters;
    const int32_t *order;
    unsigned long long *prof;   // optional phase clocks (LMC_ADM_PROF=1)
    int32_t force_nf;           // test hook (LMC_TEST_NONFINITE_SLICE): this slice's residual is made NaN
    const int32_t *warm_ok;     // warm start: per slice, start from the previous U, V / sigma
    int32_t warm_iters;
    int32_t dbg;                // diagnostic timing switches (LMC_ADM2_DBG, wrong results): 1 no Grams after it 1, 2 no epilogue matvecs, 4 no S stores
};

template <int Q>
struct K2 {
    static constexpr int NB = Q / 4;
#ifndef ADM2_NT
#define ADM2_NT 512
#endif
    static constexpr int NT = ADM2_NT;
    static constexpr int NW = NT / 32;
    static constexpr int GWN = NW < 16 ? NW : 16;   // warps that form Gram partials
    static constexpr int RB = 64;   // bytes per X / Y row slot (q < 16 rows stored 16 / q times)
};

// Rotated row access.  off = base + 64 r + 16 rot(lane): register block c of the lane holds
// logical block lb(c) = (c ^ rot) mod NB, read from physical block c ^ rot (one of the copies).
template <int Q>
__device__ __forceinline__ int lblk(int c, int rot) { return (c ^ rot) & (Q / 4 - 1); }
template <int Q>
__device__ __forceinline__ void ld_rot(const char *smc, int off, float (&v)[Q])
{
#pragma unroll
    for (int c = 0; c < Q / 4; ++c) {
        const float4 t = *reinterpret_cast<const float4 *>(smc + (off ^ (c << 4)));
        v[4 * c] = t.x; v[4 * c + 1] = t.y; v[4 * c + 2] = t.z; v[4 * c + 3] = t.w;
    }
}
// store a rotated register row into every copy of the row slot
template <int Q>
__device__ __forceinline__ void st_rot(char *smc, int off, const float (&v)[Q])
{
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const int rc = c & (Q / 4 - 1);
        *reinterpret_cast<float4 *>(smc + (off ^ (c << 4))) = make_float4(v[4 * rc], v[4 * rc + 1], v[4 * rc + 2], v[4 * rc + 3]);
    }
}
// global rows (plain logical order) into / from rotated registers
template <int Q>
__device__ __forceinline__ void ld_grot(const float *p, int rot, float (&v)[Q])
{
#pragma unroll
    for (int c = 0; c < Q / 4; ++c) {
        const float4 t = reinterpret_cast<const float4 *>(p)[lblk<Q>(c, rot)];
        v[4 * c] = t.x; v[4 * c + 1] = t.y; v[4 * c + 2] = t.z; v[4 * c + 3] = t.w;
    }
}
template <int Q>
__device__ __forceinline__ void st_grot(float *p, int rot, const float (&v)[Q])
{
#pragma unroll
    for (int c = 0; c < Q / 4; ++c)
        reinterpret_cast<float4 *>(p)[lblk<Q>(c, rot)] = make_float4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
}
// Per-slot state (U, Lambda, X_k rows; V, Pi columns): the q-vector of lane slot (g, l) is stored
// logical block lb at float4 index (g NB + lb) 32 + l, so a warp's access to its group is four
// contiguous 128-byte lines per block instead of 32 scattered rows.
template <int Q>
__device__ __forceinline__ void ld_slot(const float *base, int g, int lane, int rot, float (&v)[Q])
{
#pragma unroll
    for (int c = 0; c < Q / 4; ++c) {
        const float4 t = reinterpret_cast<const float4 *>(base)[(g * (Q / 4) + lblk<Q>(c, rot)) * 32 + lane];
        v[4 * c] = t.x; v[4 * c + 1] = t.y; v[4 * c + 2] = t.z; v[4 * c + 3] = t.w;
    }
}
template <int Q>
__device__ __forceinline__ void st_slot(float *base, int g, int lane, int rot, const float (&v)[Q])
{
#pragma unroll
    for (int c = 0; c < Q / 4; ++c)
        reinterpret_cast<float4 *>(base)[(g * (Q / 4) + lblk<Q>(c, rot)) * 32 + lane] =
            make_float4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
}
template <int Q>
__device__ __forceinline__ float dotq(const float (&a)[Q], const float (&b)[Q])
{
    float p[4];
#pragma unroll
    for (int h = 0; h < 4; ++h) p[h] = a[h] * b[h];
#pragma unroll
    for (int c = 4; c < Q; ++c) p[c & 3] = fmaf(a[c], b[c], p[c & 3]);
    return (p[0] + p[1]) + (p[2] + p[3]);
}
// out[a] += sum_b t[b] M[b][a] in rotated register order (M row-major Q x Q in shared memory)
template <int Q>
__device__ __forceinline__ void matvec_rot(const float (&t)[Q], const float *M, int rot, float (&out)[Q])
{
#pragma unroll
    for (int cb = 0; cb < Q / 4; ++cb) {
        const float *Mr = M + 4 * lblk<Q>(cb, rot) * Q;
#pragma unroll
        for (int eb = 0; eb < 4; ++eb) {
            const float tb = t[4 * cb + eb];
#pragma unroll
            for (int c = 0; c < Q / 4; ++c) {
                const float4 r = reinterpret_cast<const float4 *>(Mr + eb * Q)[lblk<Q>(c, rot)];
                out[4 * c] = fmaf(tb, r.x, out[4 * c]);
                out[4 * c + 1] = fmaf(tb, r.y, out[4 * c + 1]);
                out[4 * c + 2] = fmaf(tb, r.z, out[4 * c + 2]);
                out[4 * c + 3] = fmaf(tb, r.w, out[4 * c + 3]);
            }
        }
    }
}
// xor butterfly over the aligned lanes of multi-segment members (levels < this lane's lg).  The
// partner's rotation differs from this lane's by d = ((1 << lv) >> 1) & 3 for every lane, so its
// register block c ^ d holds this lane's logical block of register block c.
template <int Q>
__device__ __forceinline__ void seg_allreduce(float (&acc)[Q], int maxlg, int lg)
{
#pragma unroll
    for (int lv = 0; lv < 5; ++lv) {
        if (lv >= maxlg) break;
        const bool on = lv < lg;
        const int d = ((1 << lv) >> 1) & 3;
        float o[Q];
#pragma unroll
        for (int c = 0; c < Q / 4; ++c) {
            const int sc = (c ^ d) & (Q / 4 - 1);
#pragma unroll
            for (int e = 0; e < 4; ++e) o[4 * c + e] = __shfl_xor_sync(FULLM2, acc[4 * sc + e], 1 << lv);
        }
#pragma unroll
        for (int c = 0; c < Q; ++c) acc[c] += on ? o[c] : 0.f;
    }
}

// Gram partial sums sum_i A_i^T B_i over rows [0, rows): A rows in shared memory (logical block b
// at byte 64 i + 16 b), B likewise or plain global rows; 4 x 4 tiles per thread, reduced over the
// warp into part[warp][Q * Q]
template <int Q, bool BGLOB>
__device__ __forceinline__ void gram2(const char *Ab, const void *Bb, int rows, float *part)
{
    constexpr int TQ = Q / 4, T = TQ * TQ, NT = K2<Q>::NT, P = NT / T;
    const int tid = threadIdx.x, p = tid / T, tile = tid % T, ta = tile / TQ, tb = tile % TQ;
    float acc[4][4];
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) acc[x][y] = 0.f;
#pragma unroll 4
    for (int i = p; i < rows; i += P) {
        const float4 a = *reinterpret_cast<const float4 *>(Ab + i * 64 + 16 * ta);
        float4 b;
        if constexpr (BGLOB) b = reinterpret_cast<const float4 *>(reinterpret_cast<const float *>(Bb) + (size_t)i * Q)[tb];
        else b = *reinterpret_cast<const float4 *>(reinterpret_cast<const char *>(Bb) + i * 64 + 16 * tb);
        const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
            for (int y = 0; y < 4; ++y) acc[x][y] = fmaf(av[x], bv[y], acc[x][y]);
    }
#pragma unroll
    for (int o = T; o < 32; o <<= 1)
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
            for (int y = 0; y < 4; ++y) acc[x][y] += __shfl_xor_sync(FULLM2, acc[x][y], o);
    const int lane = tid & 31, warp = tid >> 5;
    if (lane < T) {
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
            for (int y = 0; y < 4; ++y) part[warp * Q * Q + (4 * ta + x) * Q + 4 * tb + y] = acc[x][y];
    }
}
// Gram partials over rows [0, rows) by all warps.  Per partition, slot s < T accumulates a 4 x 4
// tile of A^T A (A rows in shared memory), slot T + s (with_c) a tile of A^T B with B = plain
// global rows (X_k); 8 rows' loads in flight per step.  Partitions of a warp are summed by
// shuffles; part[w][0 or 1][Q * Q] holds warp w's partials.
template <int Q>
__device__ __forceinline__ void gram_all(const char *Ab, const float *Bg, int rows, float *part, bool with_c)
{
    constexpr int TQ = Q / 4, T = TQ * TQ, NW = K2<Q>::GWN;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (w >= NW) return;
    const int SLT = with_c ? 2 * T : T, PW = 32 / SLT, PP = NW * PW;
    const int p = w * PW + lane / SLT, slot = lane % SLT, which = slot / T, tile = slot % T;
    const int ta = tile / TQ, tb = tile % TQ;
    float acc[4][4];
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) acc[x][y] = 0.f;
    for (int i0 = p; i0 < rows; i0 += 8 * PP) {
        float4 a[8], b[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {   // all loads of 8 rows in flight before the FMAs
            const int i = i0 + u * PP;
            const bool in = i < rows;
            const int r = in ? i : 0;
            if (which) b[u] = __ldcg(reinterpret_cast<const float4 *>(Bg + (size_t)r * Q) + tb);
            else b[u] = *reinterpret_cast<const float4 *>(Ab + r * 64 + 16 * tb);
            a[u] = *reinterpret_cast<const float4 *>(Ab + r * 64 + 16 * ta);
            if (!in) a[u] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const float av[4] = {a[u].x, a[u].y, a[u].z, a[u].w}, bv[4] = {b[u].x, b[u].y, b[u].z, b[u].w};
#pragma unroll
            for (int x = 0; x < 4; ++x)
#pragma unroll
                for (int y = 0; y < 4; ++y) acc[x][y] = fmaf(av[x], bv[y], acc[x][y]);
        }
    }
    for (int o = SLT; o < 32; o <<= 1)
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
            for (int y = 0; y < 4; ++y) acc[x][y] += __shfl_xor_sync(FULLM2, acc[x][y], o);
    if (lane < SLT) {
        float *pw = part + (w * 2 + which) * Q * Q;
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
            for (int y = 0; y < 4; ++y) pw[(4 * ta + x) * Q + 4 * tb + y] = acc[x][y];
    }
}
// one warp: out = sum over the GWN warps' partials `which` (transposed if asked), fixed order
template <int Q>
__device__ __forceinline__ void gram_reduce_warp(float *out, const float *part, int which, bool transpose)
{
    constexpr int NW = K2<Q>::GWN;
    const int lane = threadIdx.x & 31;
    for (int e = lane; e < Q * Q; e += 32) {
        float s = 0.f;
#pragma unroll
        for (int w = 0; w < NW; ++w) s += part[(w * 2 + which) * Q * Q + e];
        const int r = e / Q, c = e % Q;
        out[transpose ? c * Q + r : e] = s;
    }
}
__device__ __forceinline__ void nbar_sync(int id, int cnt) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(cnt) : "memory"); }
__device__ __forceinline__ void nbar_arrive(int id, int cnt) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(cnt) : "memory"); }

template <int Q>
__device__ __forceinline__ void gram2_reduce(float *out, const float *part, bool transpose, int t0, int nthr)
{
    constexpr int NW = K2<Q>::NW;
    for (int e = (int)threadIdx.x - t0; e < Q * Q; e += nthr) {
        if (e < 0) break;
        float s = 0.f;
        for (int w = 0; w < NW; ++w) s += part[w * Q * Q + e];
        const int r = e / Q, c = e % Q;
        out[transpose ? c * Q + r : e] = s;
    }
}
// M <- (M + d I)^{-1} for SPD M by Gauss-Jordan without pivoting in one warp's registers
template <int Q>
__device__ void inv2_warp(float *M, float d)
{
    const int lane = threadIdx.x & 31;
    const int r = lane < Q ? lane : 0;
    float a[Q], b[Q];
#pragma unroll
    for (int c = 0; c < Q; ++c) {
        a[c] = M[r * Q + c] + (r == c ? d : 0.f);
        b[c] = (r == c) ? 1.f : 0.f;
    }
#pragma unroll
    for (int k = 0; k < Q; ++k) {
        const float ip = 1.0f / __shfl_sync(FULLM2, a[k], k);
        const bool piv = lane == k;
        const float f = piv ? 0.f : a[k] * ip;
#pragma unroll
        for (int c = k; c < Q; ++c) {
            const float p = __shfl_sync(FULLM2, a[c], k);
            a[c] = piv ? p * ip : fmaf(-f, p, a[c]);
        }
#pragma unroll
        for (int c = 0; c <= k; ++c) {
            const float p = __shfl_sync(FULLM2, b[c], k);
            b[c] = piv ? p * ip : fmaf(-f, p, b[c]);
        }
    }
    __syncwarp();
    if (lane < Q) {
#pragma unroll
        for (int c = 0; c < Q; ++c) M[lane * Q + c] = b[c];
    }
}

__device__ __forceinline__ int next_grp(int *ctr, int lane)
{
    int g = 0;
    if (lane == 0) g = atomicAdd(ctr, 1);
    return __shfl_sync(FULLM2, g, 0);
}

// squared residual of the row layout: sum over Omega of (M^ - x_i . y_j)^2 (this thread's share)
template <int Q>
__device__ float resid2(const char *smc, int xo_l, int yo_l, const int4 *rg, const uint32_t *rs,
                        const unsigned long long *re, int ngr, int m, int warp, int lane)
{
    float ss = 0.f;
    for (int g = warp; g < ngr; g += K2<Q>::NW) {
        const int4 gi = rg[g];
        const uint32_t sl = rs[g * 32 + lane];
        const int mem = (int)(sl & 2047u);
        const bool own = mem < m && ((sl >> 11) & 31u) == 0u;   // no double count of segments
        float x[Q];
        ld_rot<Q>(smc, xo_l + (mem < m ? mem : m) * 64, x);
        const ulonglong2 *e = reinterpret_cast<const ulonglong2 *>(re + gi.x) + lane;
        for (int kp = 0; kp < gi.y / 2; ++kp) {
            const ulonglong2 w = __ldg(e + kp * 32);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const unsigned long long ww = h ? w.y : w.x;
                float y[Q];
                ld_rot<Q>(smc, yo_l + (int)((uint32_t)ww & 2047u) * 64, y);
                const float err = __uint_as_float((uint32_t)(ww >> 32)) - dotq<Q>(x, y);
                ss = fmaf(err, err, ss);
            }
        }
        (void)own;
    }
    return ss;
}

#define PCLK(var) asm volatile("mov.u64 %0, %%clock64;" : "=l"(var)::"memory")

template <int Q, bool PROF>
__global__ void __launch_bounds__(K2<Q>::NT, 1) k_adm2(C2Args A)
{
    constexpr int NT = K2<Q>::NT, NW = K2<Q>::NW, RB = K2<Q>::RB;
    extern __shared__ __align__(128) char smc[];
    __shared__ float red[33];
    __shared__ int sh_ctr[2];
    __shared__ int sh_cap;
    const int ls = A.order ? A.order[blockIdx.x] : (int)blockIdx.x, s = A.s0 + ls, tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5, rot = (lane >> 1) & 3;
    const int m = A.slice_off[s + 1] - A.slice_off[s];
    const int n = A.cut_n[ls];
    const int64_t lrow0 = A.slice_off[s] - A.lbase;
    const int64_t sb = (int64_t)ls * A.scap, vb = (int64_t)ls * A.G * Q, gb = (int64_t)ls * A.gcap;
    float *Ug = A.U + lrow0 * Q, *Lg = A.Lam + lrow0 * Q, *Xo = A.Xold + lrow0 * Q;
    float *Vg = A.V + vb, *Pg = A.Pi + vb;
    const int64_t stb = (int64_t)ls * A.gcap * 32 * Q;
    float *Usl = A.Us + stb, *Lsl = A.Ls + stb, *Xsl = A.Xs + stb, *Vsl = A.Vs + stb, *Psl = A.Ps + stb;
    unsigned long long pacc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long pt0 = 0, pt1 = 0;
    if (PROF) PCLK(pt0);
    if (m <= Q || n <= Q) {   // R25: rank not below the slice dimensions -> direct rendering
        if (tid == 0) { A.flags[ls] = LMC_SLICE_DIRECT; A.iters[ls] = 0; A.resid[ls] = 0.f; }
        return;
    }
    const float4 nm = A.norm[ls];   // sigma, 1/sigma, sum M^, sum M^^2
    const float sigma = nm.x;
    if (sigma == 0.f) {
        for (int k = tid; k < m * Q; k += NT) Ug[k] = 0.f;
        for (int k = tid; k < n * Q; k += NT) Vg[k] = 0.f;
        if (tid == 0) { A.flags[ls] = LMC_SLICE_ZERO; A.iters[ls] = 0; A.resid[ls] = 0.f; }
        return;
    }
    // shared memory: X (m + 2 row slots: two zero rows), Y (n + 2), B, D, C (Q x Q), Gram
    // partials, then S (the leading column groups that fit)
    const int xo = 0, xbytes = ((m + 2) * RB + 127) & ~127;
    const int yo = xbytes, ybytes = ((n + 2) * RB + 127) & ~127;
    char *Xb = smc + xo;
    char *Yb = smc + yo;
    float *Bm = reinterpret_cast<float *>(smc + yo + ybytes);
    float *Dm = Bm + Q * Q;
    float *Cm = Dm + Q * Q;
    float *part = Cm + Q * Q;
    float *Ss = part + 2 * (K2<Q>::GWN > NW / 2 ? K2<Q>::GWN : NW / 2 + 1) * Q * Q;
    const int soff = (int)(reinterpret_cast<char *>(Ss) - smc);
    const int capS_raw = soff < A.smem_bytes ? (A.smem_bytes - soff) / 4 : 0;
    const int xo_l = xo + 16 * rot, yo_l = yo + 16 * rot;   // this lane's rotated row bases
    const int ngr = A.ngrp[2 * ls], ngc = A.ngrp[2 * ls + 1];
    const int4 *rgrp = A.r_grp + gb, *cgrp = A.c_grp + gb;
    const uint32_t *rslot = A.r_slot + gb * 32, *cslot = A.c_slot + gb * 32;
    const unsigned long long *rent = A.r_ent + sb;
    const uint16_t *ccode = A.c_code + sb;
    float *gS = A.S + sb;
    if (tid == 0) { sh_cap = A.ctot[ls]; sh_ctr[0] = 0; sh_ctr[1] = 0; }
    __syncthreads();
    for (int g = tid; g < ngc; g += NT) {
        const int4 gi = cgrp[g];
        if (gi.x + 32 * gi.y > capS_raw) atomicMin(&sh_cap, gi.x);
    }
    __syncthreads();
    const int capS = sh_cap;
    for (int k = tid; k < capS; k += NT) Ss[k] = 0.f;   // padding slots read 0
    // R20: X_0, Y_0 Philox-uniform with E[X_0 Y_0] = mean_Omega M^ (every copy of a row slot)
    const float c0 = 2.0f * sqrtf((nm.z / (float)A.nnz[ls]) / (float)Q);
    constexpr int CP = 16 / Q;   // copies per row slot
    const bool warm = A.warm_ok && A.warm_ok[ls];   // the previous frame's U and V / sigma
    const int Keff = warm && A.warm_iters > 0 ? A.warm_iters : A.K;
    for (int e = tid; e < (m + 2) * 16; e += NT) {
        const int i = e >> 4, ph = e & 15, l = ph % Q;   // physical float ph of slot i holds element l
        const float x = i >= m ? 0.f : warm ? Ug[i * Q + l]
                                            : c0 * unif_f(philox4((uint32_t)i, (uint32_t)l, (uint32_t)(A.rs0 + ls * A.rss), TAG_X0, A.seed).x);
        reinterpret_cast<float *>(Xb + i * RB)[ph] = x;
    }
    for (int e = tid; e < (n + 2) * 16; e += NT) {
        const int j = e >> 4, ph = e & 15, l = ph % Q;
        const float y = j >= n ? 0.f : warm ? Vg[j * Q + l] * nm.y
                                            : c0 * unif_f(philox4((uint32_t)l, (uint32_t)j, (uint32_t)(A.rs0 + ls * A.rss), TAG_Y0, A.seed).x);
        reinterpret_cast<float *>(Yb + j * RB)[ph] = y;
    }
    (void)CP;
    for (int e = tid; e < Q * Q; e += NT) Cm[e] = 0.f;
    __syncthreads();
    // U_0 = X_0, Lambda_0 = 0, V_0 = Y_0, Pi_0 = 0 in slot order (sentinel slots: zero rows)
    constexpr int NB = Q / 4;
    for (int e = tid; e < ngr * 32 * NB; e += NT) {
        const int s2 = e / NB, lb = e % NB, g = s2 >> 5, l = s2 & 31;
        const int mem = (int)(rslot[s2] & 2047u);
        const float4 v = *reinterpret_cast<const float4 *>(Xb + (mem < m ? mem : m) * RB + 16 * lb);
        reinterpret_cast<float4 *>(Usl)[(g * NB + lb) * 32 + l] = v;
        reinterpret_cast<float4 *>(Lsl)[(g * NB + lb) * 32 + l] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    for (int e = tid; e < ngc * 32 * NB; e += NT) {
        const int s2 = e / NB, lb = e % NB, g = s2 >> 5, l = s2 & 31;
        const int mem = (int)(cslot[s2] & 2047u);
        const float4 v = *reinterpret_cast<const float4 *>(Yb + (mem < n ? mem : n) * RB + 16 * lb);
        reinterpret_cast<float4 *>(Vsl)[(g * NB + lb) * 32 + l] = v;
        reinterpret_cast<float4 *>(Psl)[(g * NB + lb) * 32 + l] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    gram2<Q, false>(Yb, Yb, n, part);
    __syncthreads();
    gram2_reduce<Q>(Bm, part, false, 0, NT);
    __syncthreads();
    if (warp == 0) inv2_warp<Q>(Bm, A.alpha);
    __syncthreads();
    const float al = A.alpha, be = A.beta, ga = A.gamma;
    const float inv_al = 1.0f / al, inv_be = 1.0f / be;
    const float nrmM2 = nm.w;
    if (PROF) { PCLK(pt1); pacc[0] += pt1 - pt0; pt0 = pt1; }
    int it = 0;
    for (; it < Keff; ++it) {
        const float fd = (it == 0) ? 0.f : 1.f;   // Z_0 = P_Omega(M^): no X_0 Y_0 part in step 0
        // ---- row phase: s_ij = M^_ij - x_i.y_j, r_i = sum_j s_ij y_j, X / U / Lambda update
        // B = (Y Y^T + aI)^{-1} of the previous iteration is produced by warp 0 while the other warps
        // run their first sample loop: they wait for it (named barrier 4) before their first update
        bool wait_b = it > 0 && warp != 0;
        for (int g = next_grp(&sh_ctr[0], lane); g < ngr; g = next_grp(&sh_ctr[0], lane)) {
            const int4 gi = rgrp[g];
            const uint32_t sl = rslot[g * 32 + lane];
            const int mem = (int)(sl & 2047u), lg = (int)(sl >> 16);
            const bool valid = mem < m, head = ((sl >> 11) & 31u) == 0u;
            const int xoff = xo_l + (valid ? mem : m) * RB;
            float x[Q], acc[Q];
            ld_rot<Q>(smc, xoff, x);
#pragma unroll
            for (int c = 0; c < Q; ++c) acc[c] = 0.f;
            const ulonglong2 *e = reinterpret_cast<const ulonglong2 *>(rent + gi.x) + lane;
            const int nbat = gi.y / KB;
            ulonglong2 cur[KB / 2], nxt[KB / 2];
#pragma unroll
            for (int p = 0; p < KB / 2; ++p) cur[p] = __ldg(e + p * 32);
            // software pipeline: the gather of k-step k + 1 is issued before k-step k is computed
            float y[Q];
            ld_rot<Q>(smc, yo_l + (int)((uint32_t)cur[0].x & 2047u) * RB, y);
            for (int b = 0; b < nbat; ++b) {
                const bool more = b + 1 < nbat;
                if (more) {
#pragma unroll
                    for (int p = 0; p < KB / 2; ++p) nxt[p] = __ldg(e + ((b + 1) * (KB / 2) + p) * 32);
                }
#pragma unroll
                for (int k = 0; k < KB; ++k) {
                    const unsigned long long w = (k & 1) ? cur[k >> 1].y : cur[k >> 1].x;
                    const uint32_t lo = (uint32_t)w;
                    int jn;
                    if (k + 1 < KB) jn = (int)((uint32_t)(((k + 1) & 1) ? cur[(k + 1) >> 1].y : cur[(k + 1) >> 1].x) & 2047u);
                    else jn = more ? (int)((uint32_t)nxt[0].x & 2047u) : n;   // n: a zero row
                    float yn[Q];
                    ld_rot<Q>(smc, yo_l + jn * RB, yn);
                    const float sv = fmaf(-fd, dotq<Q>(x, y), __uint_as_float((uint32_t)(w >> 32)));
#pragma unroll
                    for (int c = 0; c < Q; ++c) acc[c] = fmaf(sv, y[c], acc[c]);
                    const int sp = (int)(lo >> 11);
                    if (!(A.dbg & 4)) {
                        if (sp < capS) Ss[sp] = sv;
                        else gS[sp] = sv;
                    }
#pragma unroll
                    for (int c = 0; c < Q; ++c) y[c] = yn[c];
                }
#pragma unroll
                for (int p = 0; p < KB / 2; ++p) cur[p] = nxt[p];
            }
            if (gi.z) seg_allreduce<Q>(acc, gi.z, lg);
            if (wait_b) { nbar_sync(4, NT); wait_b = false; }
            float u[Q], lam[Q], xn[Q];
            ld_slot<Q>(Usl, g, lane, rot, u);
            ld_slot<Q>(Lsl, g, lane, rot, lam);
            const float fx = fd * al;
#pragma unroll
            for (int c = 0; c < Q; ++c) {
                acc[c] = acc[c] + al * u[c] - lam[c] - fx * x[c];   // t
                xn[c] = fd * x[c];
            }
            if (!(A.dbg & 2)) matvec_rot<Q>(acc, Bm, rot, xn);
#pragma unroll
            for (int c = 0; c < Q; ++c) {
                u[c] = fmaxf(0.f, xn[c] + lam[c] * inv_al);
                lam[c] = lam[c] + ga * al * (xn[c] - u[c]);
            }
            if (valid && head) {
                st_grot<Q>(Xo + (size_t)mem * Q, rot, x);
                st_rot<Q>(smc, xoff, xn);
                st_slot<Q>(Usl, g, lane, rot, u);
                st_slot<Q>(Lsl, g, lane, rot, lam);
            }
        }
        if (wait_b) nbar_sync(4, NT);
        if (PROF) { PCLK(pt1); pacc[1] += pt1 - pt0; pt0 = pt1; }
        __syncthreads();
        if (PROF) { PCLK(pt1); pacc[2] += pt1 - pt0; pt0 = pt1; }
        // ---- (X^T X + bI)^{-1} and C = X_{k+1}^T X_k: the Gram warps form partials, warp 0 sums
        // and inverts while every other warp starts the column phase (named barriers 1, 2)
        if (tid == 0) sh_ctr[0] = 0;
        const bool skipg = (A.dbg & 1) && it > 1;
        if (!skipg) gram_all<Q>(Xb, Xo, m, part, it > 0);
        __syncthreads();
        if (warp == 0) {   // everyone else starts the column phase (named barrier 2 before updates)
            if (!skipg) {
                gram_reduce_warp<Q>(Dm, part, 0, false);
                if (it > 0) gram_reduce_warp<Q>(Cm, part, 1, true);   // Cm[b][a] = (X_{k+1}^T X_k)[a][b]
                __syncwarp();
                inv2_warp<Q>(Dm, be);
            }
            __syncwarp();
            nbar_arrive(2, NT);
        }
        if (PROF) { PCLK(pt1); pacc[3] += pt1 - pt0; pt0 = pt1; }
        // ---- column phase: Y_{k+1} = (X^T X + bI)^{-1}(X^T Z_k + b V_k - Pi_k), V / Pi update
        bool wait_d = warp != 0;
        for (int g = next_grp(&sh_ctr[1], lane); g < ngc; g = next_grp(&sh_ctr[1], lane)) {
            const int4 gi = cgrp[g];
            const uint32_t sl = cslot[g * 32 + lane];
            const int mem = (int)(sl & 2047u), lg = (int)(sl >> 16);
            const bool valid = mem < n, head = ((sl >> 11) & 31u) == 0u;
            const bool sin = gi.x + 32 * gi.y <= capS;   // warp-uniform: S of this group in shared memory
            float acc[Q];
#pragma unroll
            for (int c = 0; c < Q; ++c) acc[c] = 0.f;
            const uint4 *cc = reinterpret_cast<const uint4 *>(ccode + gi.x) + lane;
            const float4 *sg4 = reinterpret_cast<const float4 *>((sin ? Ss : gS) + gi.x) + lane;
            const int nbat = gi.y / KB;
            uint4 ccur = __ldg(cc), cnx = ccur;
            float4 scur0, scur1, snx0, snx1;
            if (sin) { scur0 = sg4[0]; scur1 = sg4[32]; }
            else { scur0 = __ldcg(sg4); scur1 = __ldcg(sg4 + 32); }
            snx0 = scur0; snx1 = scur1;
            float xv[Q];
            ld_rot<Q>(smc, xo_l + (int)(ccur.x & 0xffffu) * RB, xv);
            for (int b = 0; b < nbat; ++b) {
                const bool more = b + 1 < nbat;
                if (more) {
                    cnx = __ldg(cc + (b + 1) * 32);
                    if (sin) { snx0 = sg4[(2 * b + 2) * 32]; snx1 = sg4[(2 * b + 3) * 32]; }
                    else { snx0 = __ldcg(sg4 + (2 * b + 2) * 32); snx1 = __ldcg(sg4 + (2 * b + 3) * 32); }
                }
                const uint32_t cw[4] = {ccur.x, ccur.y, ccur.z, ccur.w};
                const float sv[8] = {scur0.x, scur0.y, scur0.z, scur0.w, scur1.x, scur1.y, scur1.z, scur1.w};
#pragma unroll
                for (int k = 0; k < KB; ++k) {
                    int rn;
                    if (k + 1 < KB) rn = (int)((cw[(k + 1) >> 1] >> (16 * ((k + 1) & 1))) & 0xffffu);
                    else rn = more ? (int)(cnx.x & 0xffffu) : m;   // m: a zero row
                    float xn2[Q];
                    ld_rot<Q>(smc, xo_l + rn * RB, xn2);
#pragma unroll
                    for (int c = 0; c < Q; ++c) acc[c] = fmaf(sv[k], xv[c], acc[c]);
#pragma unroll
                    for (int c = 0; c < Q; ++c) xv[c] = xn2[c];
                }
                ccur = cnx; scur0 = snx0; scur1 = snx1;
            }
            if (gi.z) seg_allreduce<Q>(acc, gi.z, lg);
            if (wait_d) { nbar_sync(2, NT); wait_d = false; }
            const int mj = valid ? mem : n;
            const int yoff = yo_l + mj * RB;
            float y[Q], v[Q], pi[Q], yn[Q];
            ld_rot<Q>(smc, yoff, y);
#pragma unroll
            for (int c = 0; c < Q; ++c) y[c] *= fd;
            if (!(A.dbg & 2)) matvec_rot<Q>(y, Cm, rot, acc);   // + (X_{k+1}^T X_k) y_j
            ld_slot<Q>(Vsl, g, lane, rot, v);
            ld_slot<Q>(Psl, g, lane, rot, pi);
#pragma unroll
            for (int c = 0; c < Q; ++c) {
                acc[c] = acc[c] + be * v[c] - pi[c];
                yn[c] = 0.f;
            }
            if (!(A.dbg & 2)) matvec_rot<Q>(acc, Dm, rot, yn);
#pragma unroll
            for (int c = 0; c < Q; ++c) {
                v[c] = fmaxf(0.f, yn[c] + pi[c] * inv_be);
                pi[c] = pi[c] + ga * be * (yn[c] - v[c]);
            }
            if (valid && head) {
                st_rot<Q>(smc, yoff, yn);
                st_slot<Q>(Vsl, g, lane, rot, v);
                st_slot<Q>(Psl, g, lane, rot, pi);
            }
        }
        if (wait_d) nbar_sync(2, NT);
        if (PROF) { PCLK(pt1); pacc[4] += pt1 - pt0; pt0 = pt1; }
        __syncthreads();
        if (PROF) { PCLK(pt1); pacc[5] += pt1 - pt0; pt0 = pt1; }
        if (tid == 0) sh_ctr[1] = 0;
        if (A.tol > 0.f) {   // r_{k+1} = ||P_Omega(M^ - X_{k+1} Y_{k+1})|| / ||P_Omega M^|| (R21)
            const float ss = block_reduce2<false>(resid2<Q>(smc, xo_l, yo_l, rgrp, rslot, rent, ngr, m, warp, lane), red);
            if (!(ss == ss) || isinf(ss) || sqrtf(ss / nrmM2) < A.tol) { ++it; break; }
        }
        // ---- (Y Y^T + aI)^{-1} for the next row phase: Gram warps + warp 0, barriers 3, 4 ------
        if (it + 1 < Keff) {
            const bool skipy = (A.dbg & 1) && it > 1;
            if (!skipy) gram_all<Q>(Yb, nullptr, n, part, false);
            __syncthreads();
            if (warp == 0) {   // the other warps start the next row phase (named barrier 4)
                if (!skipy) gram_reduce_warp<Q>(Bm, part, 0, false);
                __syncwarp();
                if (!skipy) inv2_warp<Q>(Bm, al);
                __syncwarp();
                nbar_arrive(4, NT);
            }
        }
        if (PROF) { PCLK(pt1); pacc[6] += pt1 - pt0; pt0 = pt1; }
    }
    const float ss = block_reduce2<false>(resid2<Q>(smc, xo_l, yo_l, rgrp, rslot, rent, ngr, m, warp, lane), red);
    const float res = s == A.force_nf ? __int_as_float(0x7fc00000) : sqrtf(ss / nrmM2);
    // R22: output (U_K, sigma V_K) in row / column order from the head lane slots
    for (int e = tid; e < ngr * 32 * NB; e += NT) {
        const int s2 = e / NB, lb = e % NB, g = s2 >> 5, l = s2 & 31;
        const uint32_t sl = rslot[s2];
        const int mem = (int)(sl & 2047u);
        if (mem < m && ((sl >> 11) & 31u) == 0u)
            reinterpret_cast<float4 *>(Ug + (size_t)mem * Q)[lb] = reinterpret_cast<const float4 *>(Usl)[(g * NB + lb) * 32 + l];
    }
    for (int e = tid; e < ngc * 32 * NB; e += NT) {
        const int s2 = e / NB, lb = e % NB, g = s2 >> 5, l = s2 & 31;
        const uint32_t sl = cslot[s2];
        const int mem = (int)(sl & 2047u);
        if (mem < n && ((sl >> 11) & 31u) == 0u) {
            const float4 v = reinterpret_cast<const float4 *>(Vsl)[(g * NB + lb) * 32 + l];
            reinterpret_cast<float4 *>(Vg + (size_t)mem * Q)[lb] = make_float4(sigma * v.x, sigma * v.y, sigma * v.z, sigma * v.w);
        }
    }
    if (PROF) {
        PCLK(pt1);
        pacc[7] += pt1 - pt0;
        if (lane == 0)
            for (int k = 0; k < 8; ++k) atomicAdd(&A.prof[k], pacc[k]);
    }
    if (tid == 0) {
        const bool bad = !(res == res) || isinf(res);
        A.flags[ls] = bad ? (LMC_SLICE_DIVERGED | LMC_SLICE_DIRECT) : 0;
        A.iters[ls] = it;
        A.resid[ls] = res;
    }
}

// ------------------------------------------------------------------------------------------
// host
// ------------------------------------------------------------------------------------------
cudaError_t run_layout2(lmc_ctx *c)
{
    if (c->SL == 0) return cudaSuccess;
    L2Args A;
    A.slice_off = c->soff_k;
    A.cut_n = c->d.cut_n;
    A.rowptr = c->d.rowptr;
    A.colptr = c->d.colptr;
    A.csc_src = c->d.csc_src;
    A.nnz = c->d.nnz;
    A.col = c->d.col;
    A.csc_row = c->d.csc_row;
    A.val = c->d.val;
    A.s0 = c->s0k;
    A.G = c->G;
    A.mmax = c->mmax;
    A.q = c->q;
    A.Tr = c->adm2_Tr;
    A.Tc = c->adm2_Tc;
    A.ncap = c->ncap;
    A.scap = c->scap;
    A.gcap = c->gcap;
    A.r_grp = c->d.r_grp;
    A.c_grp = c->d.c_grp;
    A.r_slot = c->d.r_slot;
    A.c_slot = c->d.c_slot;
    A.ngrp = c->d.ngrp;
    A.ctot = c->d.ctot;
    A.r_ent = c->d.r_ent;
    A.c_code = c->d.c_ent;
    A.S = c->d.S;
    A.map = c->d.newpos;
    A.norm = c->d.norm;
    A.counters = c->d.counters;
    auto kern = c->q == 4 ? k_layout2<4> : c->q == 8 ? k_layout2<8> : k_layout2<16>;
    if (!(c->q == 4 || c->q == 8 || c->q == 16)) return cudaErrorInvalidValue;
    const size_t sm = std::max(sizeof(typename cub::BlockRadixSort<uint32_t, LT2, 1>::TempStorage),
                               sizeof(typename cub::BlockScan<int32_t, LT2>::TempStorage));
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    kern<<<c->SL, LT2, sm, c->stream>>>(A);
    return cudaGetLastError();
}

template <int Q, bool PROF>
static cudaError_t launch_adm2(lmc_ctx *c, C2Args A)
{
    int dev = 0, maxsm = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    e = cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (e != cudaSuccess) return e;
    cudaFuncAttributes fa;
    e = cudaFuncGetAttributes(&fa, k_adm2<Q, PROF>);
    if (e != cudaSuccess) return e;
    A.smem_bytes = (maxsm - (int)fa.sharedSizeBytes) & ~127;   // all of it: the slice decides how much S fits
    e = cudaFuncSetAttribute(k_adm2<Q, PROF>, cudaFuncAttributeMaxDynamicSharedMemorySize, A.smem_bytes);
    if (e != cudaSuccess) return e;
    k_adm2<Q, PROF><<<c->SL, K2<Q>::NT, A.smem_bytes, c->stream>>>(A);
    return cudaGetLastError();
}

cudaError_t run_adm2(lmc_ctx *c)
{
    if (c->SL == 0) return cudaSuccess;
    C2Args A;
    A.slice_off = c->soff_k;
    A.s0 = c->s0k;
    A.lbase = c->lbase_k;
    A.rs0 = c->rs0;
    A.rss = c->rss;
    A.G = c->G;
    A.mmax = c->mmax;
    A.scap = c->scap;
    A.gcap = c->gcap;
    A.K = c->cfg.max_iter;
    A.alpha = (float)c->cfg.alpha;
    A.beta = (float)c->cfg.beta;
    A.gamma = (float)c->cfg.gamma;
    A.tol = (float)c->cfg.tol;
    A.seed = c->cfg.seed;
    A.cut_n = c->d.cut_n;
    A.nnz = c->d.nnz;
    A.ngrp = c->d.ngrp;
    A.ctot = c->d.ctot;
    A.norm = c->d.norm;
    A.r_grp = c->d.r_grp;
    A.c_grp = c->d.c_grp;
    A.r_slot = c->d.r_slot;
    A.c_slot = c->d.c_slot;
    A.r_ent = c->d.r_ent;
    A.c_code = c->d.c_ent;
    A.U = c->d.U;
    A.V = c->d.V;
    A.Lam = c->d.Lam;
    A.Pi = c->d.Pi;
    A.Xold = c->d.Xold;
    A.S = c->d.S;
    A.resid = c->d.resid;
    A.flags = c->d.flags;
    A.iters = c->d.iters;
    A.Us = c->d.slot_st;
    A.Ls = A.Us + (size_t)c->SL * c->gcap * 32 * c->q;
    A.Xs = A.Ls + (size_t)c->SL * c->gcap * 32 * c->q;
    A.Vs = A.Xs + (size_t)c->SL * c->gcap * 32 * c->q;
    A.Ps = A.Vs + (size_t)c->SL * c->gcap * 32 * c->q;
    A.order = c->adm_ordered ? c->d.adm_order : nullptr;
    // LMC_ADM_PROF=1: per-phase clock64 totals (diagnostic only; synchronises, prints to stderr)
    const char *pe = getenv("LMC_ADM_PROF");
    const bool prof = pe && pe[0] == '1';
    A.prof = nullptr;
    const char *dbe = getenv("LMC_ADM2_DBG");
    A.dbg = dbe ? atoi(dbe) : 0;
    const char *fe = getenv("LMC_TEST_NONFINITE_SLICE");
    A.force_nf = fe ? atoi(fe) : -1;
    A.warm_ok = c->cfg.warm_start ? c->d.warm_ok : nullptr;
    A.warm_iters = c->cfg.warm_iters;
    if (prof) {
        if (cudaMalloc(&A.prof, 8 * sizeof(unsigned long long)) != cudaSuccess) return cudaErrorMemoryAllocation;
        cudaMemsetAsync(A.prof, 0, 8 * sizeof(unsigned long long), c->stream);
    }
    cudaError_t e;
    switch (c->q) {
    case 4: e = prof ? launch_adm2<4, true>(c, A) : launch_adm2<4, false>(c, A); break;
    case 8: e = prof ? launch_adm2<8, true>(c, A) : launch_adm2<8, false>(c, A); break;
    case 16: e = prof ? launch_adm2<16, true>(c, A) : launch_adm2<16, false>(c, A); break;
    default: e = cudaErrorInvalidValue;
    }
    if (prof) {
        unsigned long long h[8] = {0};
        cudaStreamSynchronize(c->stream);
        cudaMemcpy(h, A.prof, sizeof h, cudaMemcpyDeviceToHost);
        cudaFree(A.prof);
        double t = 0;
        for (int k = 0; k < 8; ++k) t += (double)h[k];
        const char *nm[8] = {"prologue", "row-loop", "row-barrier", "gramX+inv+C", "col-loop", "col-barrier", "gramY+inv", "epilogue"};
        fprintf(stderr, "[adm2 prof] warp-cycles:");
        for (int k = 0; k < 8; ++k) fprintf(stderr, " %s=%.1f%%", nm[k], 100.0 * (double)h[k] / (t > 0 ? t : 1));
        fprintf(stderr, "\n");
    }
    return e;
}

}  // namespace lmc
