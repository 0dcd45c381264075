// slice.cu — matrix slicing (DESIGN R26) by per-tile radix select (sm_100a).
//
// A tile of n rows (ascending row order) splits on the dimension d of largest key extent; the
// lower ceil(n/2) rows by (key_d, row) go left, both children keep ascending row order.  Only the
// threshold is needed, not the order: with k* the ceil(n/2)-th smallest key and `need` = how many
// rows with key k* still go left, a row goes left iff key < k*, or key == k* and it is among the
// first `need` rows with key k* (rows ascend within the tile, so that is the (key, row) order).
//
// Keys are 32-bit: key_d = x_d / D (d < 3) or w_n n_d (d >= 3) is a strictly increasing function
// of the fp32 coordinate for every finite input when D, w_n lie in [1e-30, 1e30] (checked at
// lmc_create; finite G-buffer checked at upload): two floats differ by >= 2^-24 relative and the
// fp64 quotient / product rounds by <= 2^-53, so the order and the ties of the fp64 keys are those
// of the floats (with -0 == +0); w_n = 0 makes the three normal keys all tie at 0.  k* is found by
// four 8-bit MSB-first histogram passes.  Extents are computed in fp64 from the float extremes
// exactly as the fp64 keys would give them.
//
// Levels with many tiles (or only tiles of <= 8192 rows) run one CTA per tile, one launch per
// level; the top levels (few, large tiles) run as chunks of <= 4096 rows over extent /
// 4 histogram passes / count / scatter launches with per-tile histograms in HBM.
#include <cstdint>
#include <cstdio>

#include "lmc_internal.h"

namespace lmc {

#define SFULL 0xffffffffu

__device__ __forceinline__ uint32_t enc32(float f)
{
    uint32_t u = __float_as_uint(f);
    if (u == 0x80000000u) u = 0u;   // -0 == +0
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float dec32(uint32_t u)
{
    u = (u & 0x80000000u) ? (u & 0x7fffffffu) : ~u;
    return __uint_as_float(u);
}

struct SliceKeys {   // 6 SoA key arrays of one ping-pong buffer, each M long
    uint32_t *k[6];
};

__device__ __forceinline__ const uint32_t *key_dim(const SliceKeys &K, int d)
{
    // select without indexing the parameter array (no local-memory copy)
    return d == 0 ? K.k[0] : d == 1 ? K.k[1] : d == 2 ? K.k[2] : d == 3 ? K.k[3] : d == 4 ? K.k[4] : K.k[5];
}

// fp64 key of dimension d of the float decoded from an extreme, +0 canonical (as the fp64 keys)
__device__ __forceinline__ double key64(uint32_t e, int d, double diag, double wn)
{
    const double f = (double)dec32(e);
    const double k = d < 3 ? f / diag : wn * f;
    return __dadd_rn(k, 0.0);
}

// dimension of largest extent (first maximum; R26), from the 6 encoded maxima and minima
__device__ int best_dim(const uint32_t *mx, const uint32_t *mn, double diag, double wn)
{
    int best = 0;
    double bext = -1.0;
    for (int d = 0; d < 6; ++d) {
        double e;
        if (d >= 3 && wn == 0.0) e = 0.0;
        else e = key64(mx[d], d, diag, wn) - key64(mn[d], d, diag, wn);
        if (e > bext) { bext = e; best = d; }
    }
    return best;
}

__global__ void k_sl_keys0(const float *__restrict__ px, const float *__restrict__ py, const float *__restrict__ pz,
                           const float *__restrict__ nx, const float *__restrict__ ny, const float *__restrict__ nz,
                           int64_t M, int wn_zero, SliceKeys K, int32_t *rows)
{
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= M) return;
    rows[r] = (int32_t)r;
    K.k[0][r] = enc32(px[r]);
    K.k[1][r] = enc32(py[r]);
    K.k[2][r] = enc32(pz[r]);
    K.k[3][r] = wn_zero ? 0u : enc32(nx[r]);
    K.k[4][r] = wn_zero ? 0u : enc32(ny[r]);
    K.k[5][r] = wn_zero ? 0u : enc32(nz[r]);
}

// block-wide (256 threads) resolution of one radix pass: the bucket of the k-th smallest key
// among the histogram h (thread t holds bin t); returns (bucket, keys below it) via shared memory
__device__ __forceinline__ void pick_bucket(uint32_t h, uint32_t k, uint32_t *sh_w, uint32_t *sh_out)
{
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    uint32_t v = h;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t n = __shfl_up_sync(SFULL, v, o);
        if (lane >= o) v += n;
    }
    if (lane == 31) sh_w[w] = v;
    __syncthreads();
    uint32_t base = 0;
    for (int j = 0; j < w; ++j) base += sh_w[j];
    const uint32_t incl = base + v, excl = incl - h;
    if (h > 0 && excl < k && incl >= k) { sh_out[0] = (uint32_t)t; sh_out[1] = excl; }
    __syncthreads();
}

// ---- chunked path (the top levels) --------------------------------------------------------
// work item w: (tile, start, len, first work item of the tile), positions relative to the level
struct LvArgs {
    const int32_t *tbeg, *tend, *tslot, *work;
    int64_t lo;
    const int32_t *rows_in;
    int32_t *rows_out;
    SliceKeys kin, kout;
    uint32_t *ext;     // [slot][12]: 6 maxima, 6 minima (encoded)
    uint32_t *hist;    // [slot][4][256]
    uint32_t *cnt;     // [2 x work item]: rows of the chunk below k* and equal to k*
    uint32_t *state;   // [slot][4]: k*, need, dim, nl
    double diag, wn;
};

__global__ void k_sl_init(uint32_t *ext, uint32_t *hist, int nslots)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < (int64_t)nslots * 12) ext[i] = (i % 12) < 6 ? 0u : 0xffffffffu;
    if (i < (int64_t)nslots * 1024) hist[i] = 0u;
}

__global__ void __launch_bounds__(256) k_sl_ext(LvArgs A)
{
    const int *wk = A.work + 4 * blockIdx.x;
    const int slot = A.tslot[wk[0]], start = wk[1], len = wk[2];
    if (slot < 0) return;
    const int64_t b = A.lo + start;
    uint32_t mx[6], mn[6];
#pragma unroll
    for (int d = 0; d < 6; ++d) { mx[d] = 0u; mn[d] = 0xffffffffu; }
    for (int i = threadIdx.x; i < len; i += blockDim.x) {
#pragma unroll
        for (int d = 0; d < 6; ++d) {
            const uint32_t e = A.kin.k[d][b + i];
            mx[d] = max(mx[d], e);
            mn[d] = min(mn[d], e);
        }
    }
    __shared__ uint32_t red[8][12];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int d = 0; d < 6; ++d) {
        mx[d] = __reduce_max_sync(SFULL, mx[d]);
        mn[d] = __reduce_min_sync(SFULL, mn[d]);
        if (lane == 0) { red[w][d] = mx[d]; red[w][6 + d] = mn[d]; }
    }
    __syncthreads();
    if (threadIdx.x < 12) {
        const int d = threadIdx.x;
        uint32_t v = red[0][d];
        for (int j = 1; j < 8; ++j) v = d < 6 ? max(v, red[j][d]) : min(v, red[j][d]);
        if (d < 6) atomicMax(&A.ext[slot * 12 + d], v);
        else atomicMin(&A.ext[slot * 12 + d], v);
    }
}

// radix state after `npass` resolved passes of slot's histograms (whole CTA of 256 threads)
__device__ void sl_state(const LvArgs &A, int slot, int n, int npass, uint32_t &prefix, uint32_t &mask, uint32_t &k,
                         int &dim)
{
    __shared__ uint32_t sh_w[8], sh_out[2];
    __shared__ int sh_dim;
    if (threadIdx.x == 0) sh_dim = best_dim(A.ext + slot * 12, A.ext + slot * 12 + 6, A.diag, A.wn);
    prefix = 0u;
    mask = 0u;
    k = (uint32_t)((n + 1) / 2);
    for (int p = 0; p < npass; ++p) {
        const uint32_t h = A.hist[((size_t)slot * 4 + p) * 256 + threadIdx.x];
        pick_bucket(h, k, sh_w, sh_out);
        const int sh = 24 - 8 * p;
        prefix |= sh_out[0] << sh;
        mask |= 0xffu << sh;
        k -= sh_out[1];
        __syncthreads();
    }
    __syncthreads();
    dim = sh_dim;
}

__global__ void __launch_bounds__(256) k_sl_hist(LvArgs A, int pass)
{
    const int *wk = A.work + 4 * blockIdx.x;
    const int tile = wk[0], slot = A.tslot[tile], start = wk[1], len = wk[2];
    if (slot < 0) return;
    uint32_t prefix, mask, k;
    int dim;
    sl_state(A, slot, A.tend[tile] - A.tbeg[tile], pass, prefix, mask, k, dim);
    __shared__ uint32_t h[256];
    h[threadIdx.x] = 0u;
    __syncthreads();
    const uint32_t *kd = key_dim(A.kin, dim) + A.lo + start;
    const int sh = 24 - 8 * pass;
    for (int i = threadIdx.x; i < len; i += blockDim.x) {
        const uint32_t e = kd[i];
        if (((e ^ prefix) & mask) == 0u) atomicAdd(&h[(e >> sh) & 0xffu], 1u);
    }
    __syncthreads();
    const uint32_t v = h[threadIdx.x];
    if (v) atomicAdd(&A.hist[((size_t)slot * 4 + pass) * 256 + threadIdx.x], v);
}

__global__ void __launch_bounds__(256) k_sl_count(LvArgs A)
{
    const int *wk = A.work + 4 * blockIdx.x;
    const int tile = wk[0], slot = A.tslot[tile], start = wk[1], len = wk[2];
    if (slot < 0) return;
    const int n = A.tend[tile] - A.tbeg[tile];
    uint32_t kstar, mask, need;
    int dim;
    sl_state(A, slot, n, 4, kstar, mask, need, dim);
    if (threadIdx.x == 0 && start == A.tbeg[tile]) {
        uint32_t *st = A.state + 4 * slot;
        st[0] = kstar; st[1] = need; st[2] = (uint32_t)dim; st[3] = (uint32_t)((n + 1) / 2);
    }
    const uint32_t *kd = key_dim(A.kin, dim) + A.lo + start;
    uint32_t c = 0;
    for (int i = threadIdx.x; i < len; i += blockDim.x) {
        const uint32_t e = kd[i];
        c += e < kstar ? 0x10000u : (e == kstar ? 1u : 0u);
    }
    __shared__ uint32_t red[8];
    c = __reduce_add_sync(SFULL, c);   // a chunk has < 2^16 rows: the halves do not carry
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t s = 0;
        for (int j = 0; j < 8; ++j) s += red[j];
        A.cnt[2 * blockIdx.x] = s >> 16;
        A.cnt[2 * blockIdx.x + 1] = s & 0xffffu;
    }
}

// exclusive block scan (256 threads) of one u32 per thread; returns the exclusive prefix
__device__ __forceinline__ uint32_t block_excl_256(uint32_t v, uint32_t *sh_w)
{
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t n = __shfl_up_sync(SFULL, x, o);
        if (lane >= o) x += n;
    }
    if (lane == 31) sh_w[w] = x;
    __syncthreads();
    uint32_t base = 0;
    for (int j = 0; j < w; ++j) base += sh_w[j];
    __syncthreads();
    return base + x - v;
}

// Staged output of a run of nr rows (source positions src .. src + nr): row i goes to local slot
// sl[i]; slots [0, nleft) are the left child's positions L0 .., the rest the right child's R0 ..
// (both contiguous).  Each array is scattered into shared memory and written out coalesced.
__device__ __forceinline__ void staged_copy(const int32_t *rows_in, int32_t *rows_out, const SliceKeys &kin,
                                            const SliceKeys &kout, int64_t src, int nr, const uint16_t *sl,
                                            uint32_t *stage, int nleft, int64_t L0, int64_t R0)
{
    const int t = threadIdx.x, NT = blockDim.x;
#pragma unroll
    for (int a = 0; a < 7; ++a) {   // unrolled: the key arrays are picked at compile time
        const uint32_t *in = a == 0 ? reinterpret_cast<const uint32_t *>(rows_in) : kin.k[a - 1];
        uint32_t *out = a == 0 ? reinterpret_cast<uint32_t *>(rows_out) : kout.k[a - 1];
        for (int i = t; i < nr; i += NT) stage[sl[i]] = in[src + i];
        __syncthreads();
        for (int q = t; q < nr; q += NT) out[q < nleft ? L0 + q : R0 + (q - nleft)] = stage[q];
        __syncthreads();
    }
}

constexpr int SC_EPT = 16;   // rows per thread of a 4096-row chunk
__global__ void __launch_bounds__(256) k_sl_scatter(LvArgs A)
{
    const int *wk = A.work + 4 * blockIdx.x;
    const int tile = wk[0], slot = A.tslot[tile], start = wk[1], len = wk[2], w0 = wk[3];
    const int64_t b = A.lo + start;
    if (slot < 0) {   // a leaf carried through this level: copy
        for (int i = threadIdx.x; i < len; i += blockDim.x) {
            A.rows_out[b + i] = A.rows_in[b + i];
#pragma unroll
            for (int d = 0; d < 6; ++d) A.kout.k[d][b + i] = A.kin.k[d][b + i];
        }
        return;
    }
    const uint32_t *st = A.state + 4 * slot;
    const uint32_t kstar = st[0], need = st[1], nl = st[3];
    const int dim = (int)st[2];
    // counts of the tile's earlier chunks (below k*, equal to k*)
    __shared__ uint32_t sh_w[8], sh_w2[8];
    uint32_t offl = 0, offe = 0;
    for (int j = w0 + threadIdx.x; j < (int)blockIdx.x; j += blockDim.x) { offl += A.cnt[2 * j]; offe += A.cnt[2 * j + 1]; }
    offl = __reduce_add_sync(SFULL, offl);
    offe = __reduce_add_sync(SFULL, offe);
    if ((threadIdx.x & 31) == 0) { sh_w[threadIdx.x >> 5] = offl; sh_w2[threadIdx.x >> 5] = offe; }
    __syncthreads();
    offl = 0;
    offe = 0;
    for (int j = 0; j < 8; ++j) { offl += sh_w[j]; offe += sh_w2[j]; }
    __syncthreads();
    // blocked: thread t owns rows [t * EPT, t * EPT + EPT) of the chunk
    const int i0 = threadIdx.x * SC_EPT;
    const uint32_t *kd = key_dim(A.kin, dim) + b;
    uint32_t fl[SC_EPT], tsum = 0;
#pragma unroll
    for (int j = 0; j < SC_EPT; ++j) {
        const int i = i0 + j;
        uint32_t f = 0;
        if (i < len) {
            const uint32_t e = kd[i];
            f = e < kstar ? 0x10000u : (e == kstar ? 1u : 0u);
        }
        fl[j] = f;
        tsum += f;
    }
    uint32_t pre = block_excl_256(tsum, sh_w);   // packed in-chunk prefix (< 2^16 per half)
    __shared__ uint32_t sh_tot;
    if (threadIdx.x == blockDim.x - 1) sh_tot = pre + tsum;
    __syncthreads();
    const uint32_t tot = sh_tot;
    const int tb = A.tbeg[tile];
    const int64_t tbase = A.lo + tb;
    const int ic0 = start - tb;                    // chunk offset in the tile
    const uint32_t lbf = offl + min(offe, need);   // left rows of the tile before this chunk
    const int nleft = (int)(offl + (tot >> 16) + min(offe + (tot & 0xffffu), need) - lbf);
    __shared__ uint16_t sl[4096];
    __shared__ uint32_t stage[4096];
#pragma unroll
    for (int j = 0; j < SC_EPT; ++j) {
        const int i = i0 + j;
        if (i < len) {
            const uint32_t less = offl + (pre >> 16), eq = offe + (pre & 0xffffu);
            const uint32_t lb = less + min(eq, need) - lbf;   // left rows of this chunk before i
            const bool left = fl[j] == 0x10000u || (fl[j] == 1u && eq < need);
            sl[i] = (uint16_t)(left ? lb : (uint32_t)nleft + ((uint32_t)i - lb));
        }
        pre += fl[j];
    }
    __syncthreads();
    staged_copy(A.rows_in, A.rows_out, A.kin, A.kout, b, len, sl, stage, nleft, tbase + lbf,
                tbase + nl + ((uint32_t)ic0 - lbf));
}

// ---- fused path: one CTA (1024 threads) per tile -------------------------------------------
// Tiles of <= 8192 rows keep their keys in registers over the four passes; larger tiles stream
// rounds of 8192 rows from L2 per pass.  Positions: rounds of 8192 with running totals.
constexpr int FT = 1024, FEPT = 8, FROUND = FT * FEPT;
constexpr int FT_SMEM = FROUND * 6;   // bytes: staging words + slots


__global__ void __launch_bounds__(FT, 1) k_sl_tile(const int32_t *__restrict__ tbeg, const int32_t *__restrict__ tend,
                                                  const int32_t *__restrict__ tslot, int64_t lo, const int32_t *rows_in,
                                                  int32_t *rows_out, SliceKeys kin, SliceKeys kout, double diag, double wn)
{
    const int tile = blockIdx.x, slot = tslot[tile];
    const int n = tend[tile] - tbeg[tile];
    const int64_t b = lo + tbeg[tile];
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    if (slot < 0) {
        for (int i = t; i < n; i += FT) {
            rows_out[b + i] = rows_in[b + i];
#pragma unroll
            for (int d = 0; d < 6; ++d) kout.k[d][b + i] = kin.k[d][b + i];
        }
        return;
    }
    __shared__ uint32_t red[32][12];
    __shared__ uint32_t h[256], sh_w[32], sh_out[2];
    __shared__ int sh_dim;
    extern __shared__ __align__(16) uint32_t sl_dyn[];   // FROUND staging words + FROUND u16 slots
    uint32_t *stage = sl_dyn;
    uint16_t *sl = reinterpret_cast<uint16_t *>(sl_dyn + FROUND);
    // extents over the tile (strided loads, coalesced)
    uint32_t mx[6], mn[6];
#pragma unroll
    for (int d = 0; d < 6; ++d) { mx[d] = 0u; mn[d] = 0xffffffffu; }
    for (int i = t; i < n; i += FT) {
#pragma unroll
        for (int d = 0; d < 6; ++d) {
            const uint32_t e = kin.k[d][b + i];
            mx[d] = max(mx[d], e);
            mn[d] = min(mn[d], e);
        }
    }
#pragma unroll
    for (int d = 0; d < 6; ++d) {
        mx[d] = __reduce_max_sync(SFULL, mx[d]);
        mn[d] = __reduce_min_sync(SFULL, mn[d]);
        if (lane == 0) { red[w][d] = mx[d]; red[w][6 + d] = mn[d]; }
    }
    if (t < 256) h[t] = 0u;
    __syncthreads();
    if (t < 12) {
        uint32_t v = red[0][t];
        for (int j = 1; j < FT / 32; ++j) v = t < 6 ? max(v, red[j][t]) : min(v, red[j][t]);
        red[0][t] = v;
    }
    __syncthreads();
    if (t == 0) sh_dim = best_dim(&red[0][0], &red[0][6], diag, wn);
    __syncthreads();
    const uint32_t *kdim = key_dim(kin, sh_dim) + b;
    const bool resident = n <= FROUND;
    // rows of round r owned by this thread, blocked: [r * FROUND + t * FEPT, ... + FEPT)
    const int i0 = t * FEPT;
    uint32_t kd[FEPT];
    if (resident) {
#pragma unroll
        for (int j = 0; j < FEPT; ++j) kd[j] = i0 + j < n ? kdim[i0 + j] : 0u;
    }
    uint32_t prefix = 0u, mask = 0u, k = (uint32_t)((n + 1) / 2);
    for (int p = 0; p < 4; ++p) {
        const int sh = 24 - 8 * p;
        if (resident) {
#pragma unroll
            for (int j = 0; j < FEPT; ++j)
                if (i0 + j < n && ((kd[j] ^ prefix) & mask) == 0u) atomicAdd(&h[(kd[j] >> sh) & 0xffu], 1u);
        } else {
            for (int i = t; i < n; i += FT) {   // strided: coalesced L2 reads
                const uint32_t e = kdim[i];
                if (((e ^ prefix) & mask) == 0u) atomicAdd(&h[(e >> sh) & 0xffu], 1u);
            }
        }
        __syncthreads();
        if (t < 256) {
            const uint32_t hv = h[t];
            uint32_t v = hv;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t nn = __shfl_up_sync(SFULL, v, o);
                if (lane >= o) v += nn;
            }
            if (lane == 31) sh_w[w] = v;
            asm volatile("bar.sync 1, 256;" ::: "memory");
            uint32_t base = 0;
            for (int j = 0; j < w; ++j) base += sh_w[j];
            const uint32_t incl = base + v, excl = incl - hv;
            if (hv > 0 && excl < k && incl >= k) { sh_out[0] = (uint32_t)t; sh_out[1] = excl; }
            h[t] = 0u;
        }
        __syncthreads();
        prefix |= sh_out[0] << sh;
        mask |= 0xffu << sh;
        k -= sh_out[1];
        __syncthreads();
    }
    const uint32_t kstar = prefix, need = k, nl = (uint32_t)((n + 1) / 2);
    uint32_t offl = 0, offe = 0;   // rows below / equal to k* in the earlier rounds
    for (int r0 = 0; r0 < n; r0 += FROUND) {
        if (!resident) {
#pragma unroll
            for (int j = 0; j < FEPT; ++j) kd[j] = r0 + i0 + j < n ? kdim[r0 + i0 + j] : 0u;
        }
        uint32_t fl[FEPT], tsum = 0;
#pragma unroll
        for (int j = 0; j < FEPT; ++j) {
            fl[j] = r0 + i0 + j < n ? (kd[j] < kstar ? 0x10000u : (kd[j] == kstar ? 1u : 0u)) : 0u;
            tsum += fl[j];
        }
        // exclusive block scan of tsum (1024 threads; a round has < 2^16 rows per half)
        uint32_t x = tsum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t nn = __shfl_up_sync(SFULL, x, o);
            if (lane >= o) x += nn;
        }
        if (lane == 31) sh_w[w] = x;
        __syncthreads();
        if (w == 0) {
            const uint32_t s = sh_w[lane];
            uint32_t y = s;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t nn = __shfl_up_sync(SFULL, y, o);
                if (lane >= o) y += nn;
            }
            sh_w[lane] = y - s;
            if (lane == 31) { sh_out[0] = y >> 16; sh_out[1] = y & 0xffffu; }   // round totals
        }
        __syncthreads();
        uint32_t pre = sh_w[w] + x - tsum;
        const int nr = min(FROUND, n - r0);
        const uint32_t rl = sh_out[0], re = sh_out[1];   // round totals
        const uint32_t lbf = offl + min(offe, need);      // left rows before the round
        const int nleft = (int)(offl + rl + min(offe + re, need) - lbf);
#pragma unroll
        for (int j = 0; j < FEPT; ++j) {
            const int i = i0 + j;   // round-relative
            if (r0 + i < n) {
                const uint32_t less = offl + (pre >> 16), eq = offe + (pre & 0xffffu);
                const uint32_t lb = less + min(eq, need) - lbf;
                const bool left = fl[j] == 0x10000u || (fl[j] == 1u && eq < need);
                sl[i] = (uint16_t)(left ? lb : (uint32_t)nleft + ((uint32_t)i - lb));
            }
            pre += fl[j];
        }
        __syncthreads();
        staged_copy(rows_in, rows_out, kin, kout, b + r0, nr, sl, stage, nleft, b + lbf, b + nl + ((uint32_t)r0 - lbf));
        offl += rl;
        offe += re;
    }
}

static SliceKeys keys_of(uint32_t *base, int64_t M)
{
    SliceKeys K;
    for (int d = 0; d < 6; ++d) K.k[d] = base + (size_t)d * M;
    return K;
}

cudaError_t run_slicing(lmc_ctx *c)
{
    cudaStream_t st = c->stream;
    const int64_t M = c->M;
    if (M == 0) return cudaSuccess;
    Dev &d = c->d;
    int32_t *rbuf[2] = {d.rows, d.rows_alt};
    SliceKeys kbuf[2] = {keys_of(d.sk, M), keys_of(d.sk + 6 * M, M)};
    const double diag = c->diag, wn = c->cfg.normal_weight;
    k_sl_keys0<<<(unsigned)((M + 255) / 256), 256, 0, st>>>(d.g[0], d.g[1], d.g[2], d.g[3], d.g[4], d.g[5], M,
                                                             wn == 0.0 ? 1 : 0, kbuf[0], rbuf[0]);
    int cur = 0;
    for (const auto &L : c->levels) {
        const int32_t *tbeg = d.lvl_begin + L.tile_off, *tend = d.lvl_end + L.tile_off, *tslot = d.lvl_slot + L.tile_off;
        if (L.fused) {
            // per device (a process may drive several GPUs): set on every call, a cheap host call
            cudaError_t e = cudaFuncSetAttribute(k_sl_tile, cudaFuncAttributeMaxDynamicSharedMemorySize, FT_SMEM);
            if (e != cudaSuccess) return e;
            k_sl_tile<<<L.tile_n, FT, FT_SMEM, st>>>(tbeg, tend, tslot, L.lo, rbuf[cur], rbuf[cur ^ 1], kbuf[cur], kbuf[cur ^ 1],
                                               diag, wn);
        } else {
            LvArgs A;
            A.tbeg = tbeg; A.tend = tend; A.tslot = tslot;
            A.work = d.lvl_work + 4 * L.work_off;
            A.lo = L.lo;
            A.rows_in = rbuf[cur]; A.rows_out = rbuf[cur ^ 1];
            A.kin = kbuf[cur]; A.kout = kbuf[cur ^ 1];
            A.ext = d.sl_ext; A.hist = d.sl_hist; A.cnt = d.sl_cnt; A.state = d.sl_state;
            A.diag = diag; A.wn = wn;
            const int64_t ni = (int64_t)L.nslots * 1024;
            k_sl_init<<<(unsigned)((ni + 255) / 256), 256, 0, st>>>(d.sl_ext, d.sl_hist, L.nslots);
            k_sl_ext<<<L.work_n, 256, 0, st>>>(A);
            for (int p = 0; p < 4; ++p) k_sl_hist<<<L.work_n, 256, 0, st>>>(A, p);
            k_sl_count<<<L.work_n, 256, 0, st>>>(A);
            k_sl_scatter<<<L.work_n, 256, 0, st>>>(A);
        }
        cur ^= 1;
    }
    if (cur == 1) {   // the result of the last level is in rows_alt: this rank's range to rows
        const int64_t lo = c->levels.empty() ? 0 : c->levels.back().lo;
        const int64_t n = c->levels.empty() ? M : c->levels.back().n;
        cudaError_t e = cudaMemcpyAsync(d.rows + lo, d.rows_alt + lo, n * sizeof(int32_t), cudaMemcpyDeviceToDevice, st);
        if (e != cudaSuccess) return e;
    }
    return cudaGetLastError();
}

// interleaved partition: rank r's slices r, r + P, ... copied row by row into its local
// array (local slice offsets soff_loc, planned on the host); one thread per local row
__global__ void k_rank_rows(int64_t ML, int SL, int rank, int P, const int32_t *__restrict__ soff_loc,
                            const int32_t *__restrict__ slice_off, const int32_t *__restrict__ rows, int32_t *rows_loc)
{
    const int64_t li = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (li >= ML) return;
    int lo = 0, hi = SL - 1;   // last local slice with offset <= li
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (soff_loc[mid] <= li) lo = mid; else hi = mid - 1;
    }
    const int s = rank + lo * P;
    rows_loc[li] = rows[slice_off[s] + (li - soff_loc[lo])];
}

cudaError_t run_rank_rows(lmc_ctx *c)
{
    if (c->ML == 0 || c->SL == 0) return cudaSuccess;
    k_rank_rows<<<(unsigned)((c->ML + 255) / 256), 256, 0, c->stream>>>(c->ML, c->SL, c->cfg.rank, c->cfg.world,
                                                                        c->d.soff_loc, c->d.slice_off, c->d.rows,
                                                                        c->d.rows_loc);
    return cudaGetLastError();
}

// launches of run_slicing (the launch counter of lmc_stats)
int64_t slicing_launches(const lmc_ctx *c)
{
    if (c->M == 0) return 0;
    int64_t n = 1;
    for (const auto &L : c->levels) n += L.fused ? 1 : 8;
    return n;
}

}  // namespace lmc
