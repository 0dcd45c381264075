// complete.cu — per-slice ADM completion, Omega layout and factored image rendering (sm_100a).
//
//   ADM      PAPER.md:149 and Appendix A, typo readings R18, fp32.  Z is never
//            formed: Z_k = X_k Y_k + S_k with S_k = P_Omega(M^ - X_k Y_k), so
//              Z_k Y_k^T = X_k (Y_k Y_k^T) + S_k Y_k^T,   X^T Z_k = (X^T X_k) Y_k + X^T S_k
//            and X_{k+1} = X_k + (S_k Y_k^T + a U_k - L_k - a X_k)(Y_k Y_k^T + a I)^{-1}
//            (Z_0 = P_Omega(M^) has no X_0 Y_0 part: the k = 0 step drops the X_k terms).
//   resolve  I(s) = X (Y e) with RGB weights w^k_c = I^k_c / lum(I_c) (R4).
//
// Work decomposition (one CTA per slice, X and Y resident in shared memory for all K
// iterations): a row (column) is owned by a group of L = q/4 lanes, each holding four of its q
// components as a float4, so a warp advances R = 32/L rows at once.  Omega streams from L2 in a
// sliced-ELL layout (k_layout: rows sorted by length, groups of R rows interleaved) so every
// warp-wide load of column ids / values is coalesced and the y_j / x_i gathers are 64-byte
// contiguous per lane group.
#include <cub/cub.cuh>
#include <cstdio>
#include <cstdlib>

#include "lmc_internal.h"
#include "philox.cuh"

namespace lmc {

#define FULLM 0xffffffffu

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

__device__ __forceinline__ float4 f4fma(float s, float4 y, float4 a)
{
    return make_float4(fmaf(s, y.x, a.x), fmaf(s, y.y, a.y), fmaf(s, y.z, a.z), fmaf(s, y.w, a.w));
}
__device__ __forceinline__ float f4dot(float4 a, float4 b) { return fmaf(a.w, b.w, fmaf(a.z, b.z, fmaf(a.y, b.y, a.x * b.x))); }
__device__ __forceinline__ float f4get(float4 v, int c) { return c == 0 ? v.x : c == 1 ? v.y : c == 2 ? v.z : v.w; }

// ------------------------------------------------------------------------------------------
// Omega layout: sliced ELL over rows and over columns (groups of R, sorted by length).
// Row entries: (float bits of M^ = M~/sigma) << 32 | (index of the entry in the column layout)
// << 10 | column;  column entries: row.  The residual S of the row phase is stored at the
// column-layout index, so the column phase streams it coalesced.  Also the per-slice
// normalisation sigma = max_Omega M~ (R23).
// ------------------------------------------------------------------------------------------
struct LArgs {
    const int32_t *slice_off, *cut_n, *rowptr, *colptr, *csc_src, *nnz;
    const uint16_t *col, *csc_row;
    const float *val;
    int32_t s0, G, mmax, R, P, D, KAR, KAC, solo_min;
    int64_t ncap, scap;
    uint16_t *r_perm, *r_len, *c_perm, *c_len;
    int32_t *r_goff, *c_goff, *map, *c_nsolo;
    unsigned long long *r_ent;
    uint16_t *c_ent;
    float *S;
    float4 *norm;
};

constexpr int LT = 1024;
#ifndef ADM_COL_CHUNK
#define ADM_COL_CHUNK 128
#endif
// (S, row) entries per column-phase chunk of the ADM kernel (Cfg<Q>::COL_CHUNK)
__host__ __device__ constexpr int adm_col_chunk(int q) { return q >= 32 ? 64 : ADM_COL_CHUNK; }

// Within a cp.async chunk (KA k-steps of R members, canonical position k * R + r) the entries are
// stored V k-steps per member together: position (k - k % V) * R + r * V + k % V.  A lane group
// then reads V consecutive k-steps of its member with one vector load, and the R groups of a warp
// read one contiguous span (row entries: V = 2 x 8 bytes; column S: V = 4 x 4 bytes; column rows:
// V = 8 x 2 bytes) -- a quarter to a half of the shared-memory wavefronts of per-k-step loads.
constexpr int VROW = 2, VS = 4, VCR = 8;
__host__ __device__ __forceinline__ int vperm(int rel, int R, int KA, int V)
{
    // rel: canonical position relative to a chunk-aligned group base
    const int ch = R * KA, c = rel / ch, w = rel - c * ch, k = w / R, r = w - k * R;
    const int v = V < KA ? V : KA;
    return c * ch + (k - k % v) * R + r * v + k % v;
}


// The entries of the P rows (columns) that share a shared-memory phase of the ADM kernel are
// scheduled so that at step k member t takes, when it can, an entry whose gathered index has
// residue (t + k) mod P: the P gathers of a phase then fall into different bank sets.  Member
// r of a group has t = (r / D) mod P (D = 1: a lane group owns a row).
#ifndef LAYOUT_MINB
#define LAYOUT_MINB 1
#endif
template <int PP>
__global__ void __launch_bounds__(LT, LAYOUT_MINB) k_layout(LArgs A)
{
    typedef cub::BlockRadixSort<uint32_t, LT, 1> Sort;
    typedef cub::BlockScan<int32_t, LT> Scan;
    extern __shared__ __align__(16) unsigned char lsm[];
    typename Sort::TempStorage &sort_tmp = *reinterpret_cast<typename Sort::TempStorage *>(lsm);
    __shared__ typename Scan::TempStorage scan_tmp;
    __shared__ int32_t sh_goff[LT + 1];
    __shared__ int32_t sh_len[LT];
    __shared__ int32_t sh_who[LT];
    __shared__ float red[33];
    const int ls = blockIdx.x, s = A.s0 + ls, tid = threadIdx.x;
    constexpr int P = PP;   // residues (bank sets) of a shared-memory phase: 32 / q
    // compile-time shape (q = 32 / P): members per group R = 128 / q, k-steps per row chunk
    // (512 bytes of 8-byte entries) and per column chunk -- the host's A.R / A.KAR / A.KAC
    constexpr int R = 4 * PP, KAR = 64 / R, KAC = adm_col_chunk(32 / PP) / R;
    const int m = A.slice_off[s + 1] - A.slice_off[s], n = A.cut_n[ls];
    const int64_t ob = (int64_t)ls * A.ncap, sb = (int64_t)ls * A.scap;
    const int32_t *rp = A.rowptr + (int64_t)ls * (A.mmax + 1);
    const int32_t *cp = A.colptr + (int64_t)ls * (A.G + 1);
    const int nnz = A.nnz[ls];
    float mx = 0.f;
    for (int k = tid; k < nnz; k += LT) mx = fmaxf(mx, A.val[ob + k]);
    const float sigma = block_reduce<true>(mx, red);   // R23: sigma = max_Omega M~
    const float inv_sigma = sigma > 0.f ? 1.0f / sigma : 0.f;
    float sum = 0.f, sq = 0.f;
    for (int k = tid; k < nnz; k += LT) {
        const float v = A.val[ob + k] * inv_sigma;
        sum += v;
        sq = fmaf(v, v, sq);
    }
    sum = block_reduce<false>(sum, red);
    sq = block_reduce<false>(sq, red);
    if (tid == 0) A.norm[ls] = make_float4(sigma, inv_sigma, sum, sq);
    int dummy = 0;   // row-layout padding stores its (zero) residual here, after the column layout
    for (int pass = 0; pass < 2; ++pass) {
        const bool rows_pass = pass == 1;
        const int cnt = rows_pass ? m : n;
        const int KA = rows_pass ? KAR : KAC;   // k-steps per cp.async chunk
        const int32_t *ptr = rows_pass ? rp : cp;
        uint16_t *perm = (rows_pass ? A.r_perm : A.c_perm) + (int64_t)ls * (rows_pass ? A.mmax : A.G);
        uint16_t *lens = (rows_pass ? A.r_len : A.c_len) + (int64_t)ls * (rows_pass ? A.mmax : A.G);
        int32_t *goff = (rows_pass ? A.r_goff : A.c_goff) + (int64_t)ls * ((rows_pass ? A.mmax : A.G) + 1);
        // sort by (length desc, index asc): unique keys -> deterministic permutation
        const int len = tid < cnt ? ptr[tid + 1] - ptr[tid] : 0;
        uint32_t key[1] = {tid < cnt ? ((uint32_t)(2047 - len) << 10) | (uint32_t)tid : 0xFFFFFFFFu};
        Sort(sort_tmp).Sort(key, 0, 32);
        const int rank = tid;                       // blocked arrangement: thread = rank
        const int who = (int)(key[0] & 1023u);
        const int wlen = rank < cnt ? 2047 - (int)(key[0] >> 10) : 0;
        if (rank < cnt) {
            perm[rank] = (uint16_t)who;
            lens[rank] = (uint16_t)wlen;
        }
        sh_len[rank] = wlen;
        sh_who[rank] = who;
        // solo members (columns only): at least one chunk of entries; each gets a group of its own
        // whose R lane groups split its entries (the longest columns no longer bound the phase)
        const int solo_min = rows_pass ? (1 << 30) : A.solo_min;
        const int nsolo = __syncthreads_count(rank < cnt && wlen >= solo_min);
        if (!rows_pass && tid == 0) A.c_nsolo[ls] = nsolo;
        // groups: nsolo solo groups, then groups of R members, all padded to whole cp.async chunks
        const int ng = nsolo + (cnt - nsolo + R - 1) / R;
        int gsz = 0;
        if (tid < nsolo) {
            gsz = ((sh_len[tid] + R * KA - 1) / (R * KA)) * (R * KA);
        } else if (tid < ng) {
            gsz = R * (((sh_len[nsolo + (tid - nsolo) * R] + KA - 1) / KA) * KA);
        }
        int pre, tot;
        Scan(scan_tmp).ExclusiveSum(gsz, pre, tot);
        if (tid < ng) { sh_goff[tid] = pre; goff[tid] = pre; }
        if (tid == 0) { sh_goff[ng] = tot; goff[ng] = tot; }
        if (!rows_pass) dummy = tot;
        __syncthreads();
        const uint16_t *gidx = rows_pass ? (A.col + ob) : (A.csc_row + ob);   // gathered index per position
        // a warp per member (ranks lane-strided over the warps, so the long solo members spread):
        // residue counts and within-residue ranks come from ballots over 32-entry chunks, and
        // every entry's position has a closed form, so the member's entries are placed in parallel
        const int lane = tid & 31, warp = tid >> 5;
        const unsigned lt_mask = (1u << lane) - 1u;
        const int nmem = nsolo + (ng - nsolo) * R;
        // the next member's list start is loaded one member ahead; the residues of a member's first
        // LCH x 32 entries are loaded together (independent loads) and kept for the placement sweep
        constexpr int LCH = 4;
        int mp0_next = warp < cnt ? ptr[sh_who[warp]] : 0;
        for (int mr = warp; mr < nmem; mr += LT / 32) {
            const int mown = mr < cnt ? sh_len[mr] : 0;
            const int mp0 = mp0_next;
            {
                const int mn = mr + LT / 32;
                mp0_next = mn < cnt ? ptr[sh_who[mn]] : 0;
            }
            int cntr[P];
#pragma unroll
            for (int b2 = 0; b2 < P; ++b2) cntr[b2] = 0;
            int rc[LCH];
#pragma unroll
            for (int c4 = 0; c4 < LCH; ++c4) {
                const int k = 32 * c4 + lane;
                rc[c4] = k < mown ? (int)gidx[mp0 + k] % P : -1;
            }
#pragma unroll
            for (int c4 = 0; c4 < LCH; ++c4)
                if (32 * c4 < mown) {
#pragma unroll
                    for (int b2 = 0; b2 < P; ++b2) cntr[b2] += __popc(__ballot_sync(FULLM, rc[c4] == b2));
                }
            for (int k0 = 32 * LCH; k0 < mown; k0 += 32) {
                const int k = k0 + lane;
                const int res = k < mown ? (int)gidx[mp0 + k] % P : -1;
#pragma unroll
                for (int b2 = 0; b2 < P; ++b2)
                    cntr[b2] += __popc(__ballot_sync(FULLM, res == b2));
            }
            const bool solo = mr < nsolo;
            int base, glen, r = 0, start[P], npos[P], fill[P];
            if (solo) {
                // position p wants residue p mod P (lane group p mod R, D = 1); residue b fills
                // its own positions b, b + P, ... first, the overflow takes the positions left
                // by residues short of entries (in residue order)
                base = sh_goff[mr];
                glen = sh_goff[mr + 1] - base;
#pragma unroll
                for (int b2 = 0; b2 < P; ++b2) {
                    npos[b2] = mown > b2 ? (mown - b2 + P - 1) / P : 0;
                    fill[b2] = min(cntr[b2], npos[b2]);
                }
            } else {
                const int g = nsolo + (mr - nsolo) / R;
                r = (mr - nsolo) % R;
                const int t = r % P;   // D = 1: a lane group owns a member
                base = sh_goff[g];
                glen = (sh_goff[g + 1] - base) / R;
                int acc = 0;
#pragma unroll
                for (int b2 = 0; b2 < P; ++b2) {
                    {
                        const int res = (t + b2) % P;
                        int c2 = 0;
#pragma unroll
                        for (int b3 = 0; b3 < P; ++b3)
                            if (b3 == res) c2 = cntr[b3];
#pragma unroll
                        for (int b3 = 0; b3 < P; ++b3)
                            if (b3 == res) start[b3] = acc;
                        acc += c2;
                    }
                }
            }
            int seen[P];   // entries of each residue in earlier chunks
#pragma unroll
            for (int b2 = 0; b2 < P; ++b2) seen[b2] = 0;
            for (int k0 = 0; k0 < mown; k0 += 32) {
                const int k = k0 + lane;
                const bool in = k < mown;
                const int pos = mp0 + k;
                int res = -1;
                if (k0 < 32 * LCH) {
#pragma unroll
                    for (int c4 = 0; c4 < LCH; ++c4)
                        if (k0 == 32 * c4) res = rc[c4];
                } else {
                    res = in ? (int)gidx[pos] % P : -1;
                }
                int j = 0, sres = 0, fres = 0;
#pragma unroll
                for (int b2 = 0; b2 < P; ++b2) {
                    {
                        const unsigned bm = __ballot_sync(FULLM, res == b2);
                        if (res == b2) {
                            j = seen[b2] + __popc(bm & lt_mask);
                            sres = solo ? 0 : start[b2];
                            fres = solo ? fill[b2] : 0;
                        }
                        seen[b2] += __popc(bm);
                    }
                }
                if (!in) continue;
                int rel;
                if (solo) {
                    int p;
                    if (j < fres) {
                        p = P * j + res;
                    } else {
                        int o = j - fres;
#pragma unroll
                        for (int b2 = 0; b2 < P; ++b2)
                            if (b2 < res) o += max(0, cntr[b2] - npos[b2]);
                        p = -1;
#pragma unroll
                        for (int b2 = 0; b2 < P; ++b2) {
                            if (p < 0) {
                                const int def = npos[b2] - fill[b2];
                                if (o < def) p = P * (fill[b2] + o) + b2;
                                else o -= def;
                            }
                        }
                    }
                    rel = p;
                } else {
                    rel = (sres + j) * R + r;
                }
                if (rows_pass) {
                    const float mh = A.val[ob + pos] * inv_sigma;
                    A.r_ent[sb + base + vperm(rel, R, KAR, VROW)] =
                        ((unsigned long long)__float_as_uint(mh) << 32) |
                        ((unsigned long long)(uint32_t)A.map[ob + pos] << 11) | (unsigned long long)A.col[ob + pos];
                } else {
                    const int is = base + vperm(rel, R, KAC, VS);
                    A.c_ent[sb + base + vperm(rel, R, KAC, VCR)] = A.csc_row[ob + pos];
                    A.map[ob + A.csc_src[ob + pos]] = is;
                    A.S[sb + is] = 0.f;
                }
            }
            // padding: sentinel entries up to the group length
            for (int k = mown + lane; k < glen; k += 32) {
                const int rel = solo ? k : k * R + r;
                if (rows_pass) {
                    // sentinel: zero row n of Y, residual parked in the dummy slot
                    A.r_ent[sb + base + vperm(rel, R, KAR, VROW)] = ((unsigned long long)(uint32_t)dummy << 11) | (unsigned long long)n;
                } else {
                    A.c_ent[sb + base + vperm(rel, R, KAC, VCR)] = (uint16_t)m;   // sentinel: zero row m of X
                    A.S[sb + base + vperm(rel, R, KAC, VS)] = 0.f;                // padding slots stay finite
                }
            }
        }
        __syncthreads();
    }
    if (tid == 0) A.S[sb + dummy] = 0.f;
}

// ------------------------------------------------------------------------------------------
// ADM
// ------------------------------------------------------------------------------------------
struct CArgs {
    const int32_t *slice_off;
    int32_t s0, lbase, G, mmax, nmax;
    int32_t rs0, rss;   // global slice id of local slice ls: rs0 + ls * rss (the draws' key)
    int64_t scap;
    int K;
    float alpha, beta, gamma, tol;
    uint64_t seed;
    const int32_t *cut_n, *nnz;
    const float4 *norm;
    const uint16_t *r_perm, *r_len, *c_perm, *c_len;
    const int32_t *r_goff, *c_goff, *c_nsolo;
    const unsigned long long *r_ent;
    const uint16_t *c_ent;
    float *U, *V, *Lam, *Pi, *Xold, *S, *resid;
    int32_t *flags, *iters;
    const int32_t *order;       // CTA -> slice, or null for CTA = slice
    unsigned long long *prof;   // optional phase clocks (LMC_ADM_PROF=1), else null
    int32_t force_nf;           // test hook (LMC_TEST_NONFINITE_SLICE): this slice's residual is made NaN
    const int32_t *warm_ok;     // warm start: per slice, start from the previous U, V / sigma
    int32_t warm_iters;
};

// Per-rank kernel shape.  q <= 16: 32 warps, a 2 KB ring per warp, 128-entry column chunks.
// q = 32: X and Y take twice the shared memory (a 1024-node cut at 512-row slices needs 197 KB),
// so 16 warps with a 1 KB ring each and 64-entry column chunks (the same ring stages in half the
// bytes); 512 threads leave 128 registers per thread.
template <int Q>
struct Cfg {
    static constexpr int L = Q / 4;           // lanes per row / column
    static constexpr int R = 32 / L;          // rows per warp step
    static constexpr int NT = Q >= 32 ? 512 : 1024;                  // threads per CTA
    static constexpr int SLOT = Q >= 32 ? 512 : 1024;                // bytes per ring slot (2 per warp)
    static constexpr int COL_CHUNK = Q >= 32 ? 64 : ADM_COL_CHUNK;   // (S, row) entries per column chunk
    static constexpr int PART = NT / 32 * 2 * SLOT / 4;             // floats of Gram partials (the ring area)
};
__host__ __device__ constexpr int adm_threads(int q) { return q >= 32 ? 512 : 1024; }
__host__ __device__ constexpr int adm_slot(int q) { return q >= 32 ? 512 : 1024; }

// ---- q = 16: the q x q products of the updates on the fp64 tensor cores ---------------------
// mma.sync m8n8k4 f64 (g = lane / 4, t = lane % 4): a0 = A[g][t], b0 = B[t][g], c = C[g][2t..2t+1].
// A warp step holds 8 rows (g = lane group) x 16 components, lane t holding components 4t..4t+3
// as a float4.  Taking k-step kk over the components {4t + kk : t = 0..3}, the A fragment is the
// lane's own component kk (no shuffles); with output column n of half h standing for component
// 4(n / 2) + 2h + n % 2, lane (g, t) receives components 4t + 2h, 4t + 2h + 1 of row g -- its own
// float4 again.  The matrix is kept in shared memory in this fragment order (MatFrag16), 8 floats
// per lane as two float4.  Products and sums are exact fp64 (one rounding to fp32 at the end):
// 8 DMMA instead of 16 shuffles and 16 16-byte shared loads per warp step.
#ifndef ADM_TC_MATVEC
#define ADM_TC_MATVEC 1
#endif
__device__ __forceinline__ int frag16(int r, int c)
{
    // element (r, c) of the 16 x 16 matrix -> its slot in the fragment-ordered copy
    const int t = r >> 2, kk = r & 3, g = 2 * (c >> 2) + (c & 1), h = (c >> 1) & 1;
    return (kk >> 1) * 128 + (4 * g + t) * 4 + (kk & 1) * 2 + h;
}
__device__ __forceinline__ void dmma16(double (&d)[2], double a, double b)
{
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}
__device__ __forceinline__ float4 matvec_tc16(float4 t4, const float *Mf, float4 acc)
{
    const int lane = threadIdx.x & 31;
    const float4 f0 = reinterpret_cast<const float4 *>(Mf)[lane];        // kk 0, 1 (h 0, 1)
    const float4 f1 = reinterpret_cast<const float4 *>(Mf + 128)[lane];  // kk 2, 3
    double c0[2] = {0.0, 0.0}, c1[2] = {0.0, 0.0};
    dmma16(c0, (double)t4.x, (double)f0.x);
    dmma16(c1, (double)t4.x, (double)f0.y);
    dmma16(c0, (double)t4.y, (double)f0.z);
    dmma16(c1, (double)t4.y, (double)f0.w);
    dmma16(c0, (double)t4.z, (double)f1.x);
    dmma16(c1, (double)t4.z, (double)f1.y);
    dmma16(c0, (double)t4.w, (double)f1.z);
    dmma16(c1, (double)t4.w, (double)f1.w);
    acc.x += (float)c0[0];
    acc.y += (float)c0[1];
    acc.z += (float)c1[0];
    acc.w += (float)c1[1];
    return acc;
}
template <int Q>
struct TcMatvec {
    static constexpr bool on = Q == 16 && ADM_TC_MATVEC;
};
// index of element (r, c) of a q x q matrix consumed by matvec(): fragment order at q = 16
template <int Q>
__device__ __forceinline__ int mat_idx(int r, int c)
{
    if constexpr (TcMatvec<Q>::on) return frag16(r, c);
    return r * Q + c;
}
#ifndef GRAM_UNROLL
#define GRAM_UNROLL 8   // 8 rows in flight per thread: k_adm 136.7 -> 136.1 ms at C4 (4: HEAD of round 1)
#endif
constexpr int kGramUnroll = GRAM_UNROLL;   // rows per unrolled step of the Gram partials
// partial Gram sums of out[a][b] = sum_i A[i][a] B[i][b] over threads [t0, t0 + nthr):
// P = nthr / (Q/4)^2 row partitions, each producing a Q x Q partial in part[p]
template <int Q>
__device__ __forceinline__ int gram_partial(const float *A, const float *B, int rows, float *part, int t0, int nthr)
{
    constexpr int TQ = Q / 4, T = TQ * TQ;
    int P = nthr / T;
    if (P * Q * Q > Cfg<Q>::PART) P = Cfg<Q>::PART / (Q * Q);
    const int tid = (int)threadIdx.x - t0;
    if (tid >= 0 && tid < P * T) {
        const int p = tid / T, tile = tid % T, ta = tile / TQ, tb = tile % TQ;
        float acc[4][4];
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
            for (int y = 0; y < 4; ++y) acc[x][y] = 0.f;
#pragma unroll kGramUnroll
        for (int i = p; i < rows; i += P) {
            const float4 a = *reinterpret_cast<const float4 *>(A + (size_t)i * Q + 4 * ta);
            const float4 b = *reinterpret_cast<const float4 *>(B + (size_t)i * Q + 4 * tb);
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
    return P;
}

template <int Q, bool MATVEC_ORDER = false>
__device__ __forceinline__ void gram_reduce(float *out, const float *part, int P)
{
#if GRAM_RED4
    // every thread sums a quarter of the partials of one element (a warp reads 32 consecutive
    // elements: no bank conflicts), the four quarters meet in part[0..3] after a barrier
    if ((int)blockDim.x >= 4 * Q * Q) {   // block-uniform; called by every thread of the block
        const int e = threadIdx.x % (Q * Q), j = threadIdx.x / (Q * Q);
        const int pq = (P + 3) / 4, pa = j * pq, pb = min(P, pa + pq);
        float s = 0.f;
        if (j < 4)
            for (int p = pa; p < pb; ++p) s += part[(size_t)p * Q * Q + e];
        __syncthreads();
        float *q4 = const_cast<float *>(part);
        if (j < 4) q4[j * Q * Q + e] = s;
        __syncthreads();
        if (j == 0) {
            s = (q4[e] + q4[Q * Q + e]) + (q4[2 * Q * Q + e] + q4[3 * Q * Q + e]);
            if constexpr (MATVEC_ORDER) out[mat_idx<Q>(e / Q, e % Q)] = s;
            else out[e] = s;
        }
        return;
    }
#endif
    for (int e = threadIdx.x; e < Q * Q; e += blockDim.x) {
        float s = 0.f;
        for (int p = 0; p < P; ++p) s += part[(size_t)p * Q * Q + e];
        if constexpr (MATVEC_ORDER) out[mat_idx<Q>(e / Q, e % Q)] = s;
        else out[e] = s;
    }
}

// M <- (M + d I)^{-1} for SPD M (Q x Q) by Gauss-Jordan without pivoting in the registers of the
// calling warp (lane r holds row r of [M + dI | I]); pivot rows are broadcast by shuffles.
template <int Q>
__device__ void inv_spd_warp(float *M, float d)
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
        const float ip = 1.0f / __shfl_sync(FULLM, a[k], k);
        const bool piv = lane == k;
        const float f = piv ? 0.f : a[k] * ip;
        // every pivot-row element is broadcast before the element is updated in this step
#pragma unroll
        for (int c = k; c < Q; ++c) {
            const float p = __shfl_sync(FULLM, a[c], k);
            a[c] = piv ? p * ip : fmaf(-f, p, a[c]);
        }
#pragma unroll
        for (int c = 0; c <= k; ++c) {
            const float p = __shfl_sync(FULLM, b[c], k);
            b[c] = piv ? p * ip : fmaf(-f, p, b[c]);
        }
    }
    __syncwarp();
    if (lane < Q) {
#pragma unroll
        for (int c = 0; c < Q; ++c) M[mat_idx<Q>(lane, c)] = b[c];
    }
}

// out[4sub..] = sum_m t[m] * Mt[m][4sub..] with t spread over the L lanes of the lane group
template <int Q>
__device__ __forceinline__ float4 group_matvec(float4 t4, const float *Mt, int grp_lane0, int sub, float4 acc)
{
    constexpr int L = Q / 4;
#pragma unroll
    for (int sp = 0; sp < L; ++sp) {
        float4 tt;
        tt.x = __shfl_sync(FULLM, t4.x, grp_lane0 + sp);
        tt.y = __shfl_sync(FULLM, t4.y, grp_lane0 + sp);
        tt.z = __shfl_sync(FULLM, t4.z, grp_lane0 + sp);
        tt.w = __shfl_sync(FULLM, t4.w, grp_lane0 + sp);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            acc = f4fma(f4get(tt, c), *reinterpret_cast<const float4 *>(Mt + (4 * sp + c) * Q + 4 * sub), acc);
        }
    }
    return acc;
}

template <int Q>
__device__ __forceinline__ float4 matvec(float4 t4, const float *Mt, int grp_lane0, int sub, float4 acc)
{
    if constexpr (TcMatvec<Q>::on) return matvec_tc16(t4, Mt, acc);
    return group_matvec<Q>(t4, Mt, grp_lane0, sub, acc);
}

template <int Q>
__device__ __forceinline__ float group_sum(float v)
{
#pragma unroll
    for (int o = 1; o < Q / 4; o <<= 1) v += __shfl_xor_sync(FULLM, v, o);
    return v;
}

__device__ __forceinline__ int next_group(int *ctr, int lane)
{
    int g = 0;
    if (lane == 0) g = atomicAdd(ctr, 1);
    return __shfl_sync(FULLM, g, 0);
}

__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem)
{
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }
// 1-D bulk copies (TMA engine, no tensor map) completing on a per-stage mbarrier: one elected lane
// issues a whole ring stage, the warp waits on the barrier's phase
__device__ __forceinline__ void mbar_init(unsigned long long *bar, int count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, unsigned long long *bar)
{
    asm volatile("fence.proxy.async.shared::cta;\n"
                 "mbarrier.arrive.expect_tx.shared::cta.b64 _, [%2], %3;\n"
                 "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %3, [%2];\n"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long *bar, uint32_t parity)
{
    asm volatile("{\n .reg .pred p;\n WAIT_%=:\n"
                 " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
                 " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)), "r"(parity)
                 : "memory");
}
#ifndef ADM_TMA_ROW
#define ADM_TMA_ROW 0
#endif
// predicated global store without a branch
__device__ __forceinline__ void st_pred(float *addr, float v, bool p)
{
    asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q st.global.f32 [%0], %1;\n}\n" ::"l"(addr), "f"(v),
                 "r"((int)p)
                 : "memory");
}

// Omega streaming: each warp double-buffers its group's entries through a 2 x 1 KB ring in shared
// memory with cp.async (chunk = 512 B of row entries, or 512 B of S + 256 B of rows).
// stages of the per-warp ring (2 x Cfg<Q>::SLOT bytes): row phase 512-byte chunks, column phase
// chunks of Cfg<Q>::COL_CHUNK (S, row) entries
#ifndef ADM_ROW_NS
#define ADM_ROW_NS 2
#endif
#ifndef ADM_COL_NS
#define ADM_COL_NS 2
#endif
constexpr int ROW_NS = ADM_ROW_NS, COL_NS = ADM_COL_NS;

// entries per column-phase chunk (4-byte S + 2-byte row each).  64 pads the column groups less
// (14% -> 7% padding at C4) but measured no faster (more chunk waits)

template <int Q>
__device__ __forceinline__ float row_residual_ss(const float *X, const float *Y, const CArgs &A, int ls, int m,
                                                 int warp, int nwarps, int lane)
{
    constexpr int L = Cfg<Q>::L, R = Cfg<Q>::R;
    const int grp = lane / L, sub = lane % L;
    const uint16_t *rperm = A.r_perm + (int64_t)ls * A.mmax, *rlen = A.r_len + (int64_t)ls * A.mmax;
    const int32_t *rgoff = A.r_goff + (int64_t)ls * (A.mmax + 1);
    const unsigned long long *rent = A.r_ent + (int64_t)ls * A.scap;
    const int ngr = (m + R - 1) / R;
    float ss = 0.f;
    for (int g = warp; g < ngr; g += nwarps) {
        const int rank = g * R + grp;
        const bool valid = rank < m;
        const int row = valid ? rperm[rank] : m;
        const int len = rlen[g * R];   // group length (warp-uniform); padding entries add 0
        const unsigned long long *e = rent + rgoff[g];
        const float4 x4 = *reinterpret_cast<const float4 *>(X + row * Q + 4 * sub);
        for (int k = 0; k < len; ++k) {
            const unsigned long long w = e[vperm(k * R + grp, R, 64 / R, VROW)];
            const float4 y4 = *reinterpret_cast<const float4 *>(Y + (int)((uint32_t)w & 2047u) * Q + 4 * sub);
            const float err = __uint_as_float((uint32_t)(w >> 32)) - group_sum<Q>(f4dot(x4, y4));
            if (sub == 0) ss = fmaf(err, err, ss);
        }
    }
    return ss;
}

// phase clocks of the instrumented builds (PROF): PMARK(k) charges the time since the last mark
// to phase k; PEXIT(k) closes a dynamically scheduled loop (own time -> k - 1, wait for the
// slowest warp -> k) and is the phase barrier.
#define PEXIT(k)                                                  \
    if (PROF) {                                                   \
        long long pt1;                                            \
        asm volatile("mov.u64 %0, %%clock64;" : "=l"(pt1)::"memory"); \
        pacc[k - 1] += (unsigned long long)(pt1 - pt0);           \
        pt0 = pt1;                                                \
        if (lane == 0) sh_exit[warp] = pt1;                       \
        __syncthreads();                                          \
        long long mx = sh_exit[0];                                \
        for (int w = 1; w < nwarps; ++w) mx = max(mx, sh_exit[w]); \
        pacc[k] += (unsigned long long)(mx - pt0);                \
        __syncthreads();                                          \
        asm volatile("mov.u64 %0, %%clock64;" : "=l"(pt0)::"memory"); \
    } else {                                                      \
        __syncthreads();                                          \
    }
#define PMARK(k)                                                  \
    if (PROF) {                                                   \
        long long pt1;                                            \
        asm volatile("mov.u64 %0, %%clock64;" : "=l"(pt1)::"memory"); \
        pacc[k] += (unsigned long long)(pt1 - pt0);               \
        pt0 = pt1;                                                \
    }

template <int Q, bool PROF>
__global__ void __launch_bounds__(Cfg<Q>::NT, 1) k_adm(CArgs A)
{
    constexpr int L = Cfg<Q>::L, R = Cfg<Q>::R;
    constexpr int CKR = 64 / R;                 // row-phase k-steps per 512-byte chunk (8-byte entries)
    constexpr int COL_CHUNK = Cfg<Q>::COL_CHUNK, RING_SLOT = Cfg<Q>::SLOT;
    static_assert(ROW_NS >= 2 && ROW_NS * 512 <= 2 * RING_SLOT, "row ring stages");
    constexpr int CKC = COL_CHUNK / R;          // column-phase k-steps per chunk (4-byte S + 2-byte rows)
    constexpr int SB = COL_CHUNK * 4, RB = COL_CHUNK * 2;   // bytes of S and of rows per chunk
    constexpr int CST = (SB + RB + 127) / 128 * 128;       // bytes per column-phase ring stage
    static_assert(COL_NS >= 2 && COL_NS * CST <= 2 * RING_SLOT, "column ring stages");
    constexpr int VC = CKC < VCR ? CKC : VCR;   // column rows per vector load (layout: vperm)
    static_assert(CKR % VROW == 0 && CKC % VS == 0 && VC % VS == 0 && (VC == 8 || VC == 4), "vector widths");
    extern __shared__ __align__(16) float sm[];
    __shared__ float red[33];
    __shared__ int sh_ctr[2];
    __shared__ unsigned long long sh_prof[8];
    __shared__ long long sh_exit[32];
#if ADM_TMA_ROW
    __shared__ unsigned long long sh_bar[32 * ROW_NS];   // per warp: one mbarrier per row-ring stage
#endif
    const int ls = A.order ? A.order[blockIdx.x] : (int)blockIdx.x, s = A.s0 + ls, tid = threadIdx.x, NT = blockDim.x;
    long long pt0 = PROF ? clock64() : 0;
    unsigned long long pacc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const int lane = tid & 31, warp = tid >> 5, nwarps = NT >> 5;
    const int grp = lane / L, sub = lane % L, lane0 = grp * L;
    const int m = A.slice_off[s + 1] - A.slice_off[s];
    const int n = A.cut_n[ls];
    const int64_t lrow0 = A.slice_off[s] - A.lbase;
    const int64_t sb = (int64_t)ls * A.scap, vb = (int64_t)ls * A.G * Q;
    const uint16_t *rperm = A.r_perm + (int64_t)ls * A.mmax;
    const uint16_t *cperm = A.c_perm + (int64_t)ls * A.G;
    const int32_t *rgoff = A.r_goff + (int64_t)ls * (A.mmax + 1), *cgoff = A.c_goff + (int64_t)ls * (A.G + 1);
    // rank-level element index of this slice's layout base (SL * scap < 2^32, checked at create):
    // the hot loops form their global addresses from 32-bit indices and the kernel-parameter bases
    const uint32_t sb32 = (uint32_t)sb;
    float *X = sm;                                  // (mmax + 1) x Q, row m_s is the zero sentinel
    float *Y = X + (size_t)(A.mmax + 1) * Q;        // (nmax + 1) x Q (column j contiguous), row n_s zero
    float *Bm = Y + (size_t)(A.nmax + 1) * Q;       // (Y Y^T + aI)^{-1}
    float *Dm = Bm + Q * Q;                         // (X^T X + bI)^{-1}
    float *Cm = Dm + Q * Q;                         // (X_{k+1}^T X_k)^T
    char *ring = reinterpret_cast<char *>(Cm + Q * Q);   // nwarps x 2 x RING_SLOT, also Gram partials
    float *part = reinterpret_cast<float *>(ring);
    char *slot0 = ring + (size_t)warp * 2 * RING_SLOT;
#if ADM_TMA_ROW
    unsigned long long *wbar = sh_bar + warp * ROW_NS;
    uint32_t wph = 0;   // phase parity of each of the warp's stage barriers
    if (lane < ROW_NS) mbar_init(wbar + lane, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    __syncwarp();
#endif
    float *Ug = A.U + lrow0 * Q, *Lg = A.Lam + lrow0 * Q, *Xo = A.Xold + lrow0 * Q;
    float *Vg = A.V + vb, *Pg = A.Pi + vb;
    if (m <= Q || n <= Q) {   // R25: rank not below the slice dimensions -> direct rendering
        if (tid == 0) { A.flags[ls] = LMC_SLICE_DIRECT; A.iters[ls] = 0; A.resid[ls] = 0.f; }
        return;
    }
    const float4 nm = A.norm[ls];            // sigma, 1/sigma, sum M^, sum M^^2
    const float sigma = nm.x;
    if (sigma == 0.f) {
        for (int k = tid; k < m * Q; k += NT) Ug[k] = 0.f;
        for (int k = tid; k < n * Q; k += NT) Vg[k] = 0.f;
        if (tid == 0) { A.flags[ls] = LMC_SLICE_ZERO; A.iters[ls] = 0; A.resid[ls] = 0.f; }
        return;
    }
    const float nrmM2 = nm.w;
    // R20: X_0, Y_0 Philox-uniform with E[X_0 Y_0] = mean_Omega M^
    const float c0 = 2.0f * sqrtf((nm.z / (float)A.nnz[ls]) / (float)Q);
    const bool warm = A.warm_ok && A.warm_ok[ls];   // the previous frame's U and V / sigma
    const int Keff = warm && A.warm_iters > 0 ? A.warm_iters : A.K;
    for (int e = tid; e < m * Q; e += NT) {
        const int i = e / Q, l = e % Q;
        const float x = warm ? Ug[e] : c0 * unif_f(philox4((uint32_t)i, (uint32_t)l, (uint32_t)(A.rs0 + ls * A.rss), TAG_X0, A.seed).x);
        X[e] = x;
        Ug[e] = x;
        Lg[e] = 0.f;
    }
    for (int e = tid; e < n * Q; e += NT) {
        const int j = e / Q, l = e % Q;
        const float y = warm ? Vg[e] * nm.y : c0 * unif_f(philox4((uint32_t)l, (uint32_t)j, (uint32_t)(A.rs0 + ls * A.rss), TAG_Y0, A.seed).x);
        Y[e] = y;
        Vg[e] = y;
        Pg[e] = 0.f;
    }
    if (tid == 0) { sh_ctr[0] = 0; sh_ctr[1] = 0; }
    for (int e = tid; e < Q * Q; e += NT) Cm[e] = 0.f;   // step 0 multiplies it by 0: keep it finite
    for (int e = tid; e < Q; e += NT) { X[m * Q + e] = 0.f; Y[n * Q + e] = 0.f; }   // sentinel rows
    __syncthreads();
    {
        const int P = gram_partial<Q>(Y, Y, n, part, 0, NT);
        __syncthreads();
        gram_reduce<Q>(Bm, part, P);
        __syncthreads();
        if (warp == 0) inv_spd_warp<Q>(Bm, A.alpha);
        __syncthreads();
    }
    const float al = A.alpha, be = A.beta, ga = A.gamma;
    const float inv_al = 1.0f / al, inv_be = 1.0f / be;
    const int nsolo = A.c_nsolo[ls];
    const int ngr = (m + R - 1) / R, ngc = nsolo + (n - nsolo + R - 1) / R;
    int it = 0;
    for (; it < Keff; ++it) {
        const float fd = (it == 0) ? 0.f : 1.f;   // Z_0 = P_Omega(M^): no X_0 Y_0 part in step 0
        // ---- row phase: s_ij = M^_ij - x_i.y_j on Omega_i, r_i = sum_j s_ij y_j, X/U/Lambda update
        for (int g = next_group(&sh_ctr[0], lane); g < ngr; g = next_group(&sh_ctr[0], lane)) {
            const int rank = g * R + grp;
            const bool valid = rank < m;
            const int row = valid ? rperm[rank] : m;          // m: the zero sentinel row
            const int nch = (rgoff[g + 1] - rgoff[g]) / (CKR * R);
            const uint32_t eg32 = sb32 + (uint32_t)rgoff[g] + 2u * (uint32_t)lane;   // this lane's 16 bytes of a chunk
            const float4 x4 = *reinterpret_cast<const float4 *>(X + row * Q + 4 * sub);
            float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
            // gathers address byte offsets from the lane's own float4 slot: column * 4Q + this base
            const char *ysub = reinterpret_cast<const char *>(Y + 4 * sub);
#if ADM_TMA_ROW
            const unsigned long long *egb = A.r_ent + (sb32 + (uint32_t)rgoff[g]);   // the group's entries
            if (lane == 0) {
#pragma unroll
                for (int p = 0; p < ROW_NS - 1; ++p)
                    if (p < nch) bulk_g2s(slot0 + p * 512, egb + 64 * p, 512u, wbar + p);
            }
#else
#pragma unroll
            for (int p = 0; p < ROW_NS - 1; ++p) {
                if (p < nch) cp_async16(slot0 + p * 512 + lane * 16, A.r_ent + (eg32 + 64u * p));
                cp_commit();
            }
#endif
            int cs = 0;   // ring stage of chunk c
            for (int c = 0; c < nch; ++c) {
                const int pf = c + ROW_NS - 1;
#if ADM_TMA_ROW
                if (lane == 0 && pf < nch) {
                    const int ps = cs == 0 ? ROW_NS - 1 : cs - 1;
                    bulk_g2s(slot0 + ps * 512, egb + 64 * pf, 512u, wbar + ps);
                }
                mbar_wait(wbar + cs, (wph >> cs) & 1u);
                wph ^= 1u << cs;
#else
                if (pf < nch) cp_async16(slot0 + (cs == 0 ? ROW_NS - 1 : cs - 1) * 512 + lane * 16, A.r_ent + (eg32 + 64u * pf));
                cp_commit();
                cp_wait<ROW_NS - 1>();
#endif
                __syncwarp();
                const unsigned long long *wb = reinterpret_cast<const unsigned long long *>(slot0 + cs * 512) + VROW * grp;
                cs = cs + 1 == ROW_NS ? 0 : cs + 1;
#pragma unroll
                for (int kk = 0; kk < CKR; kk += VROW) {
                    // two k-steps of this row in one 16-byte load (vperm layout)
                    const ulonglong2 wp = *reinterpret_cast<const ulonglong2 *>(wb + kk * R);
#pragma unroll
                    for (int h = 0; h < VROW; ++h) {
                        // padding entries gather the zero row n of Y: they add exactly 0 and park a
                        // zero residual in the dummy slot, so no masking is needed
                        const unsigned long long w = h == 0 ? wp.x : wp.y;
                        const float4 y4 = *reinterpret_cast<const float4 *>(ysub + ((uint32_t)w & 2047u) * (4u * Q));
                        const float d = group_sum<Q>(f4dot(x4, y4));
                        const float sv = fmaf(-fd, d, __uint_as_float((uint32_t)(w >> 32)));
                        acc = f4fma(sv, y4, acc);
                        st_pred(A.S + (sb32 + (((uint32_t)w) >> 11)), sv, sub == 0);
                    }
                }
                __syncwarp();
            }
            const float4 u4 = *reinterpret_cast<const float4 *>(Ug + row * Q + 4 * sub);
            const float4 l4 = *reinterpret_cast<const float4 *>(Lg + row * Q + 4 * sub);
            const float fx = fd * al;
            float4 t4;
            t4.x = acc.x + al * u4.x - l4.x - fx * x4.x;
            t4.y = acc.y + al * u4.y - l4.y - fx * x4.y;
            t4.z = acc.z + al * u4.z - l4.z - fx * x4.z;
            t4.w = acc.w + al * u4.w - l4.w - fx * x4.w;
            const float4 x0 = make_float4(fd * x4.x, fd * x4.y, fd * x4.z, fd * x4.w);
            const float4 xn = matvec<Q>(t4, Bm, lane0, sub, x0);
            float4 un, ln;
            un.x = fmaxf(0.f, xn.x + l4.x * inv_al); ln.x = l4.x + ga * al * (xn.x - un.x);
            un.y = fmaxf(0.f, xn.y + l4.y * inv_al); ln.y = l4.y + ga * al * (xn.y - un.y);
            un.z = fmaxf(0.f, xn.z + l4.z * inv_al); ln.z = l4.z + ga * al * (xn.z - un.z);
            un.w = fmaxf(0.f, xn.w + l4.w * inv_al); ln.w = l4.w + ga * al * (xn.w - un.w);
            if (valid) {
                *reinterpret_cast<float4 *>(Xo + row * Q + 4 * sub) = x4;
                *reinterpret_cast<float4 *>(X + row * Q + 4 * sub) = xn;
                *reinterpret_cast<float4 *>(Ug + row * Q + 4 * sub) = un;
                *reinterpret_cast<float4 *>(Lg + row * Q + 4 * sub) = ln;
            }
        }
        PEXIT(1);
        // ---- (X^T X + bI)^{-1}; warp 0 inverts while the other warps form X_{k+1}^T X_k
        {
            int P = gram_partial<Q>(X, X, m, part, 0, NT);
            __syncthreads();
            gram_reduce<Q>(Dm, part, P);
            if (tid == 0) sh_ctr[0] = 0;
            __syncthreads();
            PMARK(2);
            if (warp == 0) {
                inv_spd_warp<Q>(Dm, be);
            } else if (it > 0) {
                P = gram_partial<Q>(Xo, X, m, part, 32, NT - 32);
            }
            __syncthreads();
            if (it > 0) {
                P = (NT - 32) / ((Q / 4) * (Q / 4));
                if (P * Q * Q > Cfg<Q>::PART) P = Cfg<Q>::PART / (Q * Q);
                gram_reduce<Q, true>(Cm, part, P);   // Cm[b][a] = (X_{k+1}^T X_k)[a][b]
                __syncthreads();
            }
        }
        PMARK(3);
        // ---- column phase: Y_{k+1} = (X^T X + bI)^{-1}(X^T Z_k + b V_k - Pi_k), V/Pi update
        for (int g = next_group(&sh_ctr[1], lane); g < ngc; g = next_group(&sh_ctr[1], lane)) {
            const bool solo = g < nsolo;                       // warp-uniform
            const int rank = solo ? g : nsolo + (g - nsolo) * R + grp;
            const bool valid = rank < n;
            const int colj = valid ? cperm[rank] : n;         // n: the zero sentinel column
            const int cb = cgoff[g];
            const int nch = (cgoff[g + 1] - cb) / (CKC * R);
            const uint32_t sg32 = sb32 + (uint32_t)cb + 4u * (uint32_t)lane;   // this lane's 16 bytes of S
            const uint32_t rg32 = sb32 + (uint32_t)cb + 8u * (uint32_t)lane;   // and of rows
            const float4 y4 = *reinterpret_cast<const float4 *>(Y + colj * Q + 4 * sub);
            float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
            const char *xsub = reinterpret_cast<const char *>(X + 4 * sub);
#pragma unroll
            for (int p = 0; p < COL_NS - 1; ++p) {
                if (p < nch) {
                    if (lane < SB / 16) cp_async16(slot0 + p * CST + lane * 16, A.S + (sg32 + (uint32_t)(COL_CHUNK * p)));
                    if (lane < RB / 16) cp_async16(slot0 + p * CST + SB + lane * 16, A.c_ent + (rg32 + (uint32_t)(COL_CHUNK * p)));
                }
                cp_commit();
            }
            int cs = 0;   // ring stage of chunk c
            for (int c = 0; c < nch; ++c) {
                const int pf = c + COL_NS - 1;
                if (pf < nch) {
                    char *nx = slot0 + (cs == 0 ? COL_NS - 1 : cs - 1) * CST;
                    if (lane < SB / 16) cp_async16(nx + lane * 16, A.S + (sg32 + (uint32_t)(COL_CHUNK * pf)));
                    if (lane < RB / 16) cp_async16(nx + SB + lane * 16, A.c_ent + (rg32 + (uint32_t)(COL_CHUNK * pf)));
                }
                cp_commit();
                cp_wait<COL_NS - 1>();
                __syncwarp();
                const char *cur = slot0 + cs * CST;
                cs = cs + 1 == COL_NS ? 0 : cs + 1;
                // vperm layout: VS k-steps of S and VC k-steps of rows per vector load
                const float *sbuf = reinterpret_cast<const float *>(cur) + VS * grp;
                const uint16_t *rbuf = reinterpret_cast<const uint16_t *>(cur + SB) + VC * grp;
#pragma unroll
                for (int kq = 0; kq < CKC; kq += VC) {
                    uint32_t rw[VC / 2];
                    if constexpr (VC == 8) {
                        const uint4 t = *reinterpret_cast<const uint4 *>(rbuf + kq * R);
                        rw[0] = t.x; rw[1] = t.y; rw[2] = t.z; rw[3] = t.w;
                    } else {
                        const uint2 t = *reinterpret_cast<const uint2 *>(rbuf + kq * R);
                        rw[0] = t.x; rw[1] = t.y;
                    }
#pragma unroll
                    for (int k4 = 0; k4 < VC; k4 += VS) {
                        const float4 s4 = *reinterpret_cast<const float4 *>(sbuf + (kq + k4) * R);
#pragma unroll
                        for (int h = 0; h < VS; ++h) {
                            // padding: zero row m of X and a zero S slot
                            const int k = k4 + h;
                            const uint32_t row = (k & 1) ? (rw[k >> 1] >> 16) : (rw[k >> 1] & 0xffffu);
                            const float4 xv = *reinterpret_cast<const float4 *>(xsub + row * (4u * Q));
                            acc = f4fma(f4get(s4, h), xv, acc);
                        }
                    }
                }
                __syncwarp();
            }
            if (solo) {   // the R lane groups hold partial sums of one column
#pragma unroll
                for (int o = L; o < 32; o <<= 1) {
                    acc.x += __shfl_xor_sync(FULLM, acc.x, o);
                    acc.y += __shfl_xor_sync(FULLM, acc.y, o);
                    acc.z += __shfl_xor_sync(FULLM, acc.z, o);
                    acc.w += __shfl_xor_sync(FULLM, acc.w, o);
                }
            }
            acc = matvec<Q>(make_float4(fd * y4.x, fd * y4.y, fd * y4.z, fd * y4.w), Cm, lane0, sub, acc);
            const float4 v4 = *reinterpret_cast<const float4 *>(Vg + colj * Q + 4 * sub);
            const float4 p4 = *reinterpret_cast<const float4 *>(Pg + colj * Q + 4 * sub);
            float4 t4;
            t4.x = acc.x + be * v4.x - p4.x;
            t4.y = acc.y + be * v4.y - p4.y;
            t4.z = acc.z + be * v4.z - p4.z;
            t4.w = acc.w + be * v4.w - p4.w;
            const float4 yn = matvec<Q>(t4, Dm, lane0, sub, make_float4(0.f, 0.f, 0.f, 0.f));
            float4 vn, pn;
            vn.x = fmaxf(0.f, yn.x + p4.x * inv_be); pn.x = p4.x + ga * be * (yn.x - vn.x);
            vn.y = fmaxf(0.f, yn.y + p4.y * inv_be); pn.y = p4.y + ga * be * (yn.y - vn.y);
            vn.z = fmaxf(0.f, yn.z + p4.z * inv_be); pn.z = p4.z + ga * be * (yn.z - vn.z);
            vn.w = fmaxf(0.f, yn.w + p4.w * inv_be); pn.w = p4.w + ga * be * (yn.w - vn.w);
            if (valid && (!solo || grp == 0)) {
                *reinterpret_cast<float4 *>(Y + colj * Q + 4 * sub) = yn;
                *reinterpret_cast<float4 *>(Vg + colj * Q + 4 * sub) = vn;
                *reinterpret_cast<float4 *>(Pg + colj * Q + 4 * sub) = pn;
            }
        }
        PEXIT(5);
        {
            const int P = gram_partial<Q>(Y, Y, n, part, 0, NT);
            __syncthreads();
            gram_reduce<Q>(Bm, part, P);
            if (tid == 0) sh_ctr[1] = 0;
            __syncthreads();
            PMARK(6);
            if (warp == 0) inv_spd_warp<Q>(Bm, al);
            __syncthreads();
        }
        PMARK(7);
        if (A.tol > 0.f) {   // r_{k+1} = ||P_Omega(M^ - X_{k+1} Y_{k+1})|| / ||P_Omega M^|| (R21)
            const float ss = block_reduce<false>(row_residual_ss<Q>(X, Y, A, ls, m, warp, nwarps, lane), red);
            if (!(ss == ss) || isinf(ss) || sqrtf(ss / nrmM2) < A.tol) { ++it; break; }
        }
    }
    const float ss = block_reduce<false>(row_residual_ss<Q>(X, Y, A, ls, m, warp, nwarps, lane), red);
    const float res = s == A.force_nf ? __int_as_float(0x7fc00000) : sqrtf(ss / nrmM2);
    for (int e = tid; e < n * Q; e += NT) Vg[e] *= sigma;   // R22: output (U_K, sigma V_K)
    if (PROF) {
        if (tid < 8) sh_prof[tid] = 0;
        __syncthreads();
        if (lane == 0)
            for (int k = 0; k < 8; ++k) atomicAdd(&sh_prof[k], pacc[k]);
        __syncthreads();
        if (tid < 8) atomicAdd(&A.prof[tid], sh_prof[tid]);
    }
    if (tid == 0) {
        const bool bad = !(res == res) || isinf(res);
        A.flags[ls] = bad ? (LMC_SLICE_DIVERGED | LMC_SLICE_DIRECT) : 0;
        A.iters[ls] = it;
        A.resid[ls] = res;
    }
}

size_t adm_smem_bytes(int q, int mmax, int nmax)
{
    // X, Y, three q x q matrices, 2 ring slots per warp (reused for the Gram partials)
    return ((size_t)mmax + (size_t)nmax + 2) * q * sizeof(float) + 3 * (size_t)q * q * sizeof(float) +
           (size_t)(adm_threads(q) / 32) * 2 * adm_slot(q);
}

static int layout_R(int q) { return 128 / q; }

cudaError_t run_layout(lmc_ctx *c)
{
    if (c->SL == 0) return cudaSuccess;
    LArgs A;
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
    A.R = layout_R(c->q);
    A.ncap = c->ncap;
    A.scap = c->scap;
    A.r_perm = c->d.r_perm;
    A.r_len = c->d.r_len;
    A.c_perm = c->d.c_perm;
    A.c_len = c->d.c_len;
    A.r_goff = c->d.r_goff;
    A.c_goff = c->d.c_goff;
    A.map = c->d.newpos;
    A.c_nsolo = c->d.c_nsolo;
    A.r_ent = c->d.r_ent;
    A.c_ent = c->d.c_ent;
    A.norm = c->d.norm;
    A.S = c->d.S;
    A.P = c->q >= 32 ? 1 : 32 / c->q;
    A.D = 1;
    A.KAR = 64 / A.R;      // k-steps per 512-byte chunk of 8-byte row entries
    A.KAC = adm_col_chunk(c->q) / A.R;   // k-steps per chunk of 4-byte S (+ 2-byte rows)
    A.solo_min = 128;      // columns of >= 128 entries get a warp of their own (a solo column pays the
                           // whole warp's update, so the threshold stays well above a group's share)
    const size_t sm = sizeof(typename cub::BlockRadixSort<uint32_t, LT, 1>::TempStorage);
    auto kern = A.P == 8 ? k_layout<8> : A.P == 4 ? k_layout<4> : A.P == 2 ? k_layout<2> : k_layout<1>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    kern<<<c->SL, LT, sm, c->stream>>>(A);
    return cudaGetLastError();
}

template <int Q, bool PROF = false>
static cudaError_t launch_adm(lmc_ctx *c, const CArgs &A)
{
    const size_t sm = adm_smem_bytes(Q, c->mmax, A.nmax);
    cudaError_t e = cudaFuncSetAttribute(k_adm<Q, PROF>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    const int nt = Cfg<Q>::NT;   // 32 warps (64 registers per thread) or 16 (q = 32), one CTA per SM
    k_adm<Q, PROF><<<c->SL, nt, sm, c->stream>>>(A);
    return cudaGetLastError();
}

cudaError_t run_adm(lmc_ctx *c, int nmax)
{
    if (c->SL == 0) return cudaSuccess;
    CArgs A;
    A.slice_off = c->soff_k;
    A.s0 = c->s0k;
    A.lbase = c->lbase_k;
    A.rs0 = c->rs0;
    A.rss = c->rss;
    A.G = c->G;
    A.mmax = c->mmax;
    A.nmax = nmax;
    A.scap = c->scap;
    A.K = c->cfg.max_iter;
    A.alpha = (float)c->cfg.alpha;
    A.beta = (float)c->cfg.beta;
    A.gamma = (float)c->cfg.gamma;
    A.tol = (float)c->cfg.tol;
    A.seed = c->cfg.seed;
    A.cut_n = c->d.cut_n;
    A.nnz = c->d.nnz;
    A.norm = c->d.norm;
    A.r_perm = c->d.r_perm;
    A.r_len = c->d.r_len;
    A.c_perm = c->d.c_perm;
    A.c_len = c->d.c_len;
    A.r_goff = c->d.r_goff;
    A.c_goff = c->d.c_goff;
    A.c_nsolo = c->d.c_nsolo;
    A.r_ent = c->d.r_ent;
    A.c_ent = c->d.c_ent;
    A.U = c->d.U;
    A.V = c->d.V;
    A.Lam = c->d.Lam;
    A.Pi = c->d.Pi;
    A.Xold = c->d.Xold;
    A.S = c->d.S;
    A.resid = c->d.resid;
    A.flags = c->d.flags;
    A.iters = c->d.iters;
    A.prof = nullptr;
    A.order = c->adm_ordered ? c->d.adm_order : nullptr;
    const char *fe = getenv("LMC_TEST_NONFINITE_SLICE");
    A.force_nf = fe ? atoi(fe) : -1;
    A.warm_ok = c->cfg.warm_start ? c->d.warm_ok : nullptr;
    A.warm_iters = c->cfg.warm_iters;
    // LMC_ADM_PROF=1: per-phase clock64 totals (diagnostic only; synchronises and prints to stderr)
    const char *pe = getenv("LMC_ADM_PROF");
    const bool prof = pe && pe[0] == '1' && c->q == 16;   // instrumented build for q = 16 only
    if (prof) {
        if (cudaMalloc(&A.prof, 8 * sizeof(unsigned long long)) != cudaSuccess) return cudaErrorMemoryAllocation;
        cudaMemsetAsync(A.prof, 0, 8 * sizeof(unsigned long long), c->stream);
    }
    cudaError_t e;
    switch (c->q) {
    case 4: e = launch_adm<4>(c, A); break;
    case 8: e = launch_adm<8>(c, A); break;
    case 16: e = prof ? launch_adm<16, true>(c, A) : launch_adm<16>(c, A); break;
    case 32: e = launch_adm<32>(c, A); break;
    default: e = cudaErrorInvalidValue;
    }
    if (prof) {
        unsigned long long h[8] = {0};
        cudaStreamSynchronize(c->stream);
        cudaMemcpy(h, A.prof, sizeof h, cudaMemcpyDeviceToHost);
        cudaFree(A.prof);
        double t = 0;
        for (int k = 0; k < 8; ++k) t += (double)h[k];
        const char *nm[8] = {"row-loop", "row-barrier", "gramX", "inv+Cm", "col-loop", "col-barrier", "gramY", "invB"};
        fprintf(stderr, "[adm prof] warp-cycles:");
        for (int k = 0; k < 8; ++k) fprintf(stderr, " %s=%.1f%%", nm[k], 100.0 * (double)h[k] / (t > 0 ? t : 1));
        fprintf(stderr, "\n");
    }
    return e;
}

// ------------------------------------------------------------------------------------------
// Resolve: t^k = V w^k (q-vectors), out^k_i = tint^k_i <U_i, t^k>
// ------------------------------------------------------------------------------------------
struct RArgs {
    const int32_t *slice_off, *rows, *pixel, *cut_n, *cut_cols, *flags;
    int32_t s0, lbase, G, q;
    int64_t row0, npix;                 // npix = width * height (image writes are bounds-checked)
    const float *U, *V, *I, *direct_rgb;
    const float4 *prow;
    float *image, *rows_rgb;
    float4 *tile4;   // optional packed (r, g, b, pixel index bits) per row of this rank (image gather)
    // Z-mode (resolve_mode 1): the slice's Omega in CSR order
    int32_t resolve_mode, mmax;
    int64_t ncap;
    const int32_t *rowptr;
    const uint16_t *col;
    const float *val;
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
            if (A.resolve_mode) {
                // Z-mode: + sum over row i's samples of (M~_ij - <U_i, V_j>) w^k_j (A24)
                const int32_t *rp = A.rowptr + (int64_t)ls * (A.mmax + 1);
                const int64_t ob = (int64_t)ls * A.ncap;
                for (int e = rp[i]; e < rp[i + 1]; ++e) {
                    const int j = A.col[ob + e];
                    const float *vj = V + (int64_t)j * q;
                    float uv = 0.f;
                    for (int a = 0; a < q; ++a) uv = fmaf(u[a], vj[a], uv);
                    const float r = A.val[ob + e] - uv;
                    const int un = A.cut_cols[cb + j];
                    const float i0 = A.I[3 * un], i1 = A.I[3 * un + 1], i2 = A.I[3 * un + 2];
                    const float lj = (0.2126f * i0 + 0.7152f * i1) + 0.0722f * i2;
                    if (lj != 0.f) {
                        d0 = fmaf(r, i0 / lj, d0);
                        d1 = fmaf(r, i1 / lj, d1);
                        d2 = fmaf(r, i2 / lj, d2);
                    }
                }
            }
            const float4 C = A.prow[4 * li + 2], D = A.prow[4 * li + 3];
            const float lr = (0.2126f * C.z + 0.7152f * C.w) + 0.0722f * D.x;
            const float ir = lr != 0.f ? 1.0f / lr : 0.f;
            o0 = C.z * ir * d0;
            o1 = C.w * ir * d1;
            o2 = D.x * ir * d2;
        }
        if (A.tile4) A.tile4[li] = make_float4(o0, o1, o2, __int_as_float(A.pixel[A.rows[A.row0 + li]]));
        if (A.rows_rgb) {
            A.rows_rgb[3 * li] = o0;
            A.rows_rgb[3 * li + 1] = o1;
            A.rows_rgb[3 * li + 2] = o2;
        }
        if (A.image) {
            const int64_t p = A.pixel[A.rows[A.row0 + li]];
            if (p < 0 || p >= A.npix) continue;   // rejected at lmc_create / lmc_upload_inputs
            A.image[3 * p] = o0;
            A.image[3 * p + 1] = o1;
            A.image[3 * p + 2] = o2;
        }
    }
}

cudaError_t run_resolve(lmc_ctx *c, float *image, float *rows_rgb, float4 *tile4)
{
    if (c->SL == 0) return cudaSuccess;
    RArgs A;
    A.slice_off = c->soff_k;
    A.rows = c->rows_k;
    A.pixel = c->d.pixel;
    A.cut_n = c->d.cut_n;
    A.cut_cols = c->d.cut_cols;
    A.flags = c->d.flags;
    A.s0 = c->s0k;
    A.lbase = c->lbase_k;
    A.G = c->G;
    A.q = c->q;
    A.row0 = c->row0_k;
    A.npix = (int64_t)c->W * c->H;
    A.U = c->d.U;
    A.V = c->d.V;
    A.I = c->d.ut_I;
    A.direct_rgb = c->d.direct_rgb;
    A.prow = c->d.prow;
    A.image = image;
    A.rows_rgb = rows_rgb;
    A.tile4 = tile4;
    A.resolve_mode = c->cfg.resolve_mode;
    A.mmax = c->mmax;
    A.ncap = c->ncap;
    A.rowptr = c->d.rowptr;
    A.col = c->d.col;
    A.val = c->d.val;
    k_resolve<<<c->SL, 256, 0, c->stream>>>(A);
    return cudaGetLastError();
}

__global__ void k_scatter(int64_t M, const int32_t *__restrict__ rows, const int32_t *__restrict__ pixel,
                          const float *__restrict__ all_rows, float *image, int64_t npix)
{
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= M) return;
    const int64_t p = pixel[rows[k]];
    if (p < 0 || p >= npix) return;
    image[3 * p] = all_rows[3 * k];
    image[3 * p + 1] = all_rows[3 * k + 1];
    image[3 * p + 2] = all_rows[3 * k + 2];
}

cudaError_t run_scatter(lmc_ctx *c, const float *all_rows, float *image)
{
    if (c->M == 0) return cudaSuccess;
    k_scatter<<<(unsigned)((c->M + 255) / 256), 256, 0, c->stream>>>(c->M, c->d.rows, c->d.pixel, all_rows, image,
                                                                       (int64_t)c->W * c->H);
    return cudaGetLastError();
}

// packed (r, g, b, pixel) rows of every rank (rank 0 of an NCCL image gather) into the image
__global__ void k_scatter4(int64_t n, const float4 *__restrict__ all4, float *image, int64_t npix)
{
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const float4 v = all4[k];
    const int64_t p = __float_as_int(v.w);
    if (p < 0 || p >= npix) return;
    image[3 * p] = v.x;
    image[3 * p + 1] = v.y;
    image[3 * p + 2] = v.z;
}
cudaError_t run_scatter4(lmc_ctx *c, const float4 *all4, int64_t n, float *image)
{
    if (n == 0) return cudaSuccess;
    k_scatter4<<<(unsigned)((n + 255) / 256), 256, 0, c->stream>>>(n, all4, image, (int64_t)c->W * c->H);
    return cudaGetLastError();
}

// image index of every row of this rank (slice-row order) -- the host-buffer resolve scatters with it
__global__ void k_rank_pixels(int64_t ML, int64_t row0, const int32_t *__restrict__ rows, const int32_t *__restrict__ pixel,
                              int32_t *out)
{
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < ML) out[k] = pixel[rows[row0 + k]];
}
cudaError_t run_rank_pixels(lmc_ctx *c, int32_t *out)
{
    if (c->ML == 0) return cudaSuccess;
    k_rank_pixels<<<(unsigned)((c->ML + 255) / 256), 256, 0, c->stream>>>(c->ML, c->row0_k, c->rows_k, c->d.pixel, out);
    return cudaGetLastError();
}

// G-buffer pixel indices must lie in [0, width * height) (lmc.h: LMC_EINVAL otherwise)
// bit 0: a pixel index outside [0, npix); bit 1: a non-finite position / normal (the slicing keys
// are exact 32-bit encodings of finite floats, slice.cu)
__global__ void k_check_pixels(int64_t M, const int32_t *__restrict__ pixel, int64_t npix, const float *__restrict__ px,
                               const float *__restrict__ py, const float *__restrict__ pz, const float *__restrict__ nx,
                               const float *__restrict__ ny, const float *__restrict__ nz, unsigned long long *flag)
{
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= M) return;
    if (pixel[k] < 0 || pixel[k] >= npix) atomicOr(flag, 1ull);
    if (!(isfinite(px[k]) && isfinite(py[k]) && isfinite(pz[k]) && isfinite(nx[k]) && isfinite(ny[k]) && isfinite(nz[k])))
        atomicOr(flag, 2ull);
}
cudaError_t run_check_pixels(lmc_ctx *c, unsigned long long *flag)
{
    cudaError_t e = cudaMemsetAsync(flag, 0, sizeof(unsigned long long), c->stream);
    if (e != cudaSuccess || c->M == 0) return e;
    k_check_pixels<<<(unsigned)((c->M + 255) / 256), 256, 0, c->stream>>>(c->M, c->d.pixel, (int64_t)c->W * c->H, c->d.g[0], c->d.g[1],
                                                                 c->d.g[2], c->d.g[3], c->d.g[4], c->d.g[5], flag);
    return cudaGetLastError();
}

// Completion launch order on the device (no host round trip): slice order, except that the nsm
// slices with the fewest samples run last, largest first, so the final wave holds the shortest
// CTAs.  sorted = slices by ascending |Omega| (stable radix sort); one CTA compacts the rest.
__global__ void __launch_bounds__(1024) k_launch_order(int32_t SL, int32_t ntail, const int32_t *__restrict__ sorted,
                                                       int32_t *mark, int32_t *order)
{
    typedef cub::BlockScan<int32_t, 1024> Scan;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ int32_t base;
    for (int k = threadIdx.x; k < SL; k += 1024) mark[k] = 0;
    __syncthreads();
    for (int k = threadIdx.x; k < ntail; k += 1024) mark[sorted[k]] = 1;
    if (threadIdx.x == 0) base = 0;
    __syncthreads();
    for (int k0 = 0; k0 < SL; k0 += 1024) {
        const int k = k0 + (int)threadIdx.x;
        const int keep = k < SL && !mark[k];
        int pos, tot;
        Scan(tmp).ExclusiveSum(keep, pos, tot);
        if (keep) order[base + pos] = k;
        __syncthreads();
        if (threadIdx.x == 0) base += tot;
        __syncthreads();
    }
    for (int k = threadIdx.x; k < ntail; k += 1024) order[SL - ntail + k] = sorted[ntail - 1 - k];
}
__global__ void k_iota(int32_t n, int32_t *a)
{
    int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n) a[k] = k;
}
cudaError_t launch_order_bytes(int32_t SL, size_t *bytes)
{
    *bytes = 0;
    return cub::DeviceRadixSort::SortPairs(nullptr, *bytes, (const int32_t *)nullptr, (int32_t *)nullptr,
                                           (const int32_t *)nullptr, (int32_t *)nullptr, SL);
}
cudaError_t run_launch_order(lmc_ctx *c, int ntail)
{
    const int SL = c->SL;
    int32_t *keys_out = c->d.ord_tmp, *iota = c->d.ord_tmp + SL, *sorted = c->d.ord_tmp + 2 * SL, *mark = c->d.ord_tmp + 3 * SL;
    k_iota<<<(SL + 255) / 256, 256, 0, c->stream>>>(SL, iota);
    size_t bytes = c->d.ord_cub_bytes;
    cudaError_t e = cub::DeviceRadixSort::SortPairs(c->d.ord_cub, bytes, c->d.nnz, keys_out, iota, sorted, SL, 0, 32, c->stream);
    if (e != cudaSuccess) return e;
    k_launch_order<<<1, 1024, 0, c->stream>>>(SL, ntail, sorted, mark, c->d.adm_order);
    return cudaGetLastError();
}

}  // namespace lmc

namespace lmc {
// ------------------------------------------------------------------------------------------
// Warm start: a slice starts from the previous frame's factors iff its rows and its
// cut equal the previous frame's and the previous result was a regular completion (flags 0)
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_warm_check(const int32_t *__restrict__ slice_off, int32_t s0, int64_t lbase,
                                                    int64_t row0, const int32_t *__restrict__ rows,
                                                    const int32_t *__restrict__ cut_n, const int32_t *__restrict__ cut_cols,
                                                    const int32_t *__restrict__ prev_rows, const int32_t *__restrict__ prev_n,
                                                    const int32_t *__restrict__ prev_cut, const int32_t *__restrict__ prev_flags,
                                                    int G, int have_prev, int32_t *warm_ok)
{
    const int ls = blockIdx.x, s = s0 + ls;
    const int64_t lr0 = slice_off[s] - lbase;
    const int m = slice_off[s + 1] - slice_off[s], n = cut_n[ls];
    int same = have_prev && prev_flags[ls] == 0 && prev_n[ls] == n;
    if (same) {
        for (int k = threadIdx.x; k < m; k += blockDim.x)
            if (rows[row0 + lr0 + k] != prev_rows[lr0 + k]) same = 0;
        for (int k = threadIdx.x; k < n; k += blockDim.x)
            if (cut_cols[(int64_t)ls * G + k] != prev_cut[(int64_t)ls * G + k]) same = 0;
    }
    same = __syncthreads_and(same);
    if (threadIdx.x == 0) warm_ok[ls] = same;
}

__global__ void k_warm_save(int SL, int G, int64_t ML, int64_t row0, const int32_t *__restrict__ rows,
                            const int32_t *__restrict__ cut_n, const int32_t *__restrict__ cut_cols,
                            const int32_t *__restrict__ flags, int32_t *prev_rows, int32_t *prev_n, int32_t *prev_cut,
                            int32_t *prev_flags)
{
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < ML) prev_rows[k] = rows[row0 + k];
    if (k < (int64_t)SL * G) prev_cut[k] = cut_cols[k];
    if (k < SL) { prev_n[k] = cut_n[k]; prev_flags[k] = flags[k]; }
}

cudaError_t run_warm_check(lmc_ctx *c)
{
    if (c->SL == 0) return cudaSuccess;
    k_warm_check<<<c->SL, 256, 0, c->stream>>>(c->soff_k, c->s0k, c->lbase_k, c->row0_k, c->rows_k, c->d.cut_n,
                                               c->d.cut_cols, c->d.prev_rows, c->d.prev_n, c->d.prev_cut, c->d.prev_flags,
                                               c->G, c->have_prev ? 1 : 0, c->d.warm_ok);
    return cudaGetLastError();
}

cudaError_t run_warm_save(lmc_ctx *c)
{
    if (c->SL == 0) return cudaSuccess;
    const int64_t n = std::max<int64_t>(std::max<int64_t>(c->ML, (int64_t)c->SL * c->G), c->SL);
    k_warm_save<<<(unsigned)((n + 255) / 256), 256, 0, c->stream>>>(c->SL, c->G, c->ML, c->row0_k, c->rows_k, c->d.cut_n,
                                                                   c->d.cut_cols, c->d.flags, c->d.prev_rows, c->d.prev_n,
                                                                   c->d.prev_cut, c->d.prev_flags);
    c->have_prev = true;
    return cudaGetLastError();
}
}  // namespace lmc
