// lighttree.cu — step 1 of the method on the GPU (DESIGN
// reading R38): the binary light tree of the VPLs and the conservative global lightcut g.
//
//   tree  median split: a node's VPLs split on the axis of its largest bounding-box extent (first
//         maximum), ordered by (coordinate, VPL index), the left child taking ceil(n/2); node ids
//         breadth-first.  The shape (node ids, ranges, leaves) depends on the VPL count only and is
//         planned on the host; every level is one segmented sort of 64-bit keys (coordinate bits,
//         VPL index) on the device.  I_f = I_l + I_r in fp64, rep(f) = rep of the brighter child.
//   cut   the internal nodes with the largest bounds lum(I_f) |bbox diagonal| (ties: smaller id)
//         are split until the cut has cut_max nodes: bounds never grow down the tree, so this is
//         the per-node split test "bound above the cut_max-th largest bound", evaluated for all
//         nodes at once (one radix sort of the bounds).
#include <cub/cub.cuh>

#include <algorithm>
#include <cstring>
#include <functional>
#include <vector>

#include "lmc.h"

namespace {

struct LtLevel { int64_t seg0, nseg; };   // this level's segments [seg0, seg0 + nseg) of the plan

__device__ __forceinline__ uint32_t ord_f(float v)
{
    uint32_t u = __float_as_uint(v == 0.f ? 0.f : v);   // -0 -> +0: the comparison order of the oracle
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float unord_f(uint32_t u) { return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u); }

// internal segment of the level holding position `pos` (segments sorted by start), or -1 (a leaf)
__device__ __forceinline__ int seg_of(const int32_t *__restrict__ seg, int nseg, int64_t pos)
{
    int lo = 0, hi = nseg - 1;
    while (lo < hi) {   // last segment with start <= pos
        const int mid = (lo + hi + 1) >> 1;
        if (seg[3 * mid + 1] <= pos) lo = mid; else hi = mid - 1;
    }
    return pos < (int64_t)seg[3 * lo + 1] + seg[3 * lo + 2] && pos >= seg[3 * lo + 1] ? lo : -1;
}

// bounding boxes of the level's segments: a CTA per (segment, chunk) work item, block min/max, one
// atomic per chunk on the ordered encodings
__global__ void __launch_bounds__(256) k_lt_bbox(const int32_t *__restrict__ work, const int32_t *__restrict__ idx,
                                                 const float *__restrict__ px, const float *__restrict__ py,
                                                 const float *__restrict__ pz, uint32_t *bb /* [node][6] */)
{
    const int node = work[3 * blockIdx.x], start = work[3 * blockIdx.x + 1], len = work[3 * blockIdx.x + 2];
    uint32_t lo[3] = {~0u, ~0u, ~0u}, hi[3] = {0u, 0u, 0u};
    for (int k = threadIdx.x; k < len; k += blockDim.x) {
        const int v = idx[start + k];
        const uint32_t e[3] = {ord_f(px[v]), ord_f(py[v]), ord_f(pz[v])};
#pragma unroll
        for (int a = 0; a < 3; ++a) { lo[a] = min(lo[a], e[a]); hi[a] = max(hi[a], e[a]); }
    }
#pragma unroll
    for (int a = 0; a < 3; ++a)
        for (int o = 16; o > 0; o >>= 1) {
            lo[a] = min(lo[a], __shfl_xor_sync(0xffffffffu, lo[a], o));
            hi[a] = max(hi[a], __shfl_xor_sync(0xffffffffu, hi[a], o));
        }
    __shared__ uint32_t red[8][6];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0)
        for (int a = 0; a < 3; ++a) { red[w][a] = lo[a]; red[w][3 + a] = hi[a]; }
    __syncthreads();
    if (threadIdx.x < 6) {
        const int a = threadIdx.x;
        uint32_t v = red[0][a];
        for (int k = 1; k < (int)(blockDim.x >> 5); ++k) v = a < 3 ? min(v, red[k][a]) : max(v, red[k][a]);
        if (a < 3) atomicMin(&bb[6 * node + a], v);
        else atomicMax(&bb[6 * node + a], v);
    }
}

__global__ void k_lt_bbox_init(int64_t n, uint32_t *bb)
{
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n) bb[k] = (k % 6) < 3 ? ~0u : 0u;
}

// sort keys of the level's internal segments: (coordinate on the longest axis, VPL index)
__global__ void k_lt_keys(const int32_t *__restrict__ seg /* [s][3] node, start, len */, int nseg,
                          const int32_t *__restrict__ idx, const float *__restrict__ px, const float *__restrict__ py,
                          const float *__restrict__ pz, const uint32_t *__restrict__ bb, int64_t base, int64_t n,
                          unsigned long long *keys)
{
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const int s = seg_of(seg, nseg, base + k);
    if (s < 0) return;   // a leaf of this level between two sorted segments
    const int node = seg[3 * s];
    double best = -1.0;
    int ax = 0;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const double e = (double)unord_f(bb[6 * node + 3 + a]) - (double)unord_f(bb[6 * node + a]);
        if (e > best) { best = e; ax = a; }
    }
    const int v = idx[base + k];
    const float c = ax == 0 ? px[v] : ax == 1 ? py[v] : pz[v];
    keys[k] = ((unsigned long long)ord_f(c) << 32) | (uint32_t)v;
}

__global__ void k_lt_unkey(const unsigned long long *__restrict__ keys, const int32_t *__restrict__ seg, int nseg,
                           int64_t base, int64_t n, int32_t *idx_out)
{
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n && seg_of(seg, nseg, base + k) >= 0) idx_out[k] = (int32_t)(uint32_t)keys[k];
}

// bottom-up intensities / representatives of one level's nodes
__global__ void k_lt_sum(const int32_t *__restrict__ nodes, int n, const int32_t *__restrict__ left,
                         const int32_t *__restrict__ right, const int32_t *__restrict__ leaf_start,
                         const int32_t *__restrict__ idx, const float *__restrict__ ir, const float *__restrict__ ig,
                         const float *__restrict__ ib, double *I, int32_t *rep)
{
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const int f = nodes[k];
    if (left[f] < 0) {
        const int v = idx[leaf_start[f]];
        rep[f] = v;
        I[3 * f] = ir[v];
        I[3 * f + 1] = ig[v];
        I[3 * f + 2] = ib[v];
        return;
    }
    const int l = left[f], r = right[f];
    I[3 * f] = I[3 * l] + I[3 * r];
    I[3 * f + 1] = I[3 * l + 1] + I[3 * r + 1];
    I[3 * f + 2] = I[3 * l + 2] + I[3 * r + 2];
    const double ll = (0.2126 * I[3 * l] + 0.7152 * I[3 * l + 1]) + 0.0722 * I[3 * l + 2];
    const double lr = (0.2126 * I[3 * r] + 0.7152 * I[3 * r + 1]) + 0.0722 * I[3 * r + 2];
    rep[f] = ll >= lr ? rep[l] : rep[r];
}

// bound of every internal node as a descending sort key; leaves sort last
__global__ void k_lt_bound(int64_t nn, const int32_t *__restrict__ left, const double *__restrict__ I,
                           const uint32_t *__restrict__ bb, unsigned long long *key, int32_t *id, float *ir, float *ig,
                           float *ib)
{
    const int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= nn) return;
    ir[f] = (float)I[3 * f];
    ig[f] = (float)I[3 * f + 1];
    ib[f] = (float)I[3 * f + 2];
    id[f] = (int32_t)f;
    if (left[f] < 0) { key[f] = ~0ull; return; }
    double d[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) d[a] = (double)unord_f(bb[6 * f + 3 + a]) - (double)unord_f(bb[6 * f + a]);
    const double lf = (0.2126 * I[3 * f] + 0.7152 * I[3 * f + 1]) + 0.0722 * I[3 * f + 2];
    const double bnd = lf * sqrt((d[0] * d[0] + d[1] * d[1]) + d[2] * d[2]);   // >= 0
    // descending bound: ~bits of a finite bound >= 0 always has the top bit set, so clearing it
    // loses nothing and keeps every internal node ahead of the leaves (key ~0)
    key[f] = ~(unsigned long long)__double_as_longlong(bnd) & 0x7fffffffffffffffull;
}

__global__ void k_lt_split(const int32_t *__restrict__ sorted_id, int64_t nsplit, uint8_t *split)
{
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < nsplit) split[sorted_id[k]] = 1;
}

__global__ void k_lt_incut(int64_t nn, const int32_t *__restrict__ parent, const uint8_t *__restrict__ split, int32_t *flag)
{
    const int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= nn) return;
    flag[f] = !split[f] && (f == 0 || split[parent[f]]);
}

__global__ void k_lt_compact(int64_t nn, const int32_t *__restrict__ flag, const int32_t *__restrict__ pre, int32_t *cut)
{
    const int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (f < nn && flag[f]) cut[pre[f]] = (int32_t)f;
}

template <typename T>
cudaError_t dmal(T **p, size_t n) { return cudaMalloc((void **)p, std::max<size_t>(n, 1) * sizeof(T)); }

}  // namespace

extern "C" lmc_status lmc_build_light_tree(const lmc_vpls *v, int32_t cut_max, int32_t memory, void *stream_,
                                           int32_t *left_out, int32_t *right_out, int32_t *rep_out, float *ir_out,
                                           float *ig_out, float *ib_out, int32_t *cut_out, int64_t *cut_size)
{
    if (!v || v->count < 1 || v->count > (1ll << 30) || cut_max < 1 || !cut_size ||
        (memory != LMC_MEM_DEVICE && memory != LMC_MEM_HOST))
        return LMC_EINVAL;
    if (!v->px || !v->py || !v->pz || !v->ir || !v->ig || !v->ib) return LMC_EINVAL;
    cudaStream_t st = (cudaStream_t)stream_;
    const int64_t nv = v->count, nn = 2 * nv - 1;
    // ---- the shape, planned on the host: breadth-first segments (node, start, len) per level
    std::vector<int32_t> seg, left(nn, -1), right(nn, -1), parent(nn, -1), leaf_start(nn, 0);
    std::vector<LtLevel> levels;
    std::vector<int32_t> level_nodes;            // breadth-first node list
    std::vector<int64_t> level_off(1, 0);
    seg.insert(seg.end(), {0, 0, (int32_t)nv});
    int64_t next_id = 1;
    for (int64_t s0 = 0, s1 = 1; s0 < s1;) {
        levels.push_back({s0, s1 - s0});
        for (int64_t s = s0; s < s1; ++s) level_nodes.push_back(seg[3 * s]);
        level_off.push_back((int64_t)level_nodes.size());
        int64_t e = s1;
        for (int64_t s = s0; s < s1; ++s) {
            const int32_t f = seg[3 * s], st0 = seg[3 * s + 1], n = seg[3 * s + 2];
            if (n == 1) { leaf_start[f] = st0; continue; }
            const int32_t nl = (n + 1) / 2;
            left[f] = (int32_t)next_id;
            right[f] = (int32_t)next_id + 1;
            parent[next_id] = f;
            parent[next_id + 1] = f;
            seg.insert(seg.end(), {(int32_t)next_id, st0, nl, (int32_t)next_id + 1, st0 + nl, n - nl});
            next_id += 2;
            e += 2;
        }
        s0 = s1;
        s1 = e;
    }
    // per level: internal segments (sort ranges) and bbox work chunks
    struct LvlDev { int64_t base, n; int nint; size_t seg_off, work_off; int nwork; };
    std::vector<LvlDev> lv;
    std::vector<int32_t> iseg, work;
    std::vector<int64_t> pos_off;
    for (auto &L : levels) {
        LvlDev d;
        d.seg_off = iseg.size() / 3;
        d.work_off = work.size() / 3;
        int64_t lo = -1, hi = -1;
        int nint = 0;
        for (int64_t s = L.seg0; s < L.seg0 + L.nseg; ++s) {
            const int32_t f = seg[3 * s], st0 = seg[3 * s + 1], n = seg[3 * s + 2];
            for (int32_t o = 0; o < n; o += 4096) work.insert(work.end(), {f, st0 + o, std::min<int32_t>(4096, n - o)});
            if (n == 1) continue;
            if (lo < 0) lo = st0;
            hi = st0 + n;
            iseg.insert(iseg.end(), {f, st0, n});
            ++nint;
        }
        d.nwork = (int)(work.size() / 3 - d.work_off);
        d.nint = nint;
        d.base = lo < 0 ? 0 : lo;
        d.n = lo < 0 ? 0 : hi - lo;
        lv.push_back(d);
    }
    // ---- device buffers
    lmc_status ret = LMC_OK;
    cudaError_t e = cudaSuccess;
    int32_t *d_idx = nullptr, *d_idx2 = nullptr, *d_iseg = nullptr, *d_work = nullptr, *d_beg = nullptr,
            *d_end = nullptr, *d_left = nullptr, *d_right = nullptr, *d_parent = nullptr, *d_leaf = nullptr,
            *d_nodes = nullptr, *d_rep = nullptr, *d_id = nullptr, *d_id2 = nullptr, *d_flag = nullptr, *d_pre = nullptr,
            *d_cut = nullptr;
    float *d_pos3[3] = {nullptr, nullptr, nullptr}, *d_I3[3] = {nullptr, nullptr, nullptr}, *d_io[3] = {nullptr, nullptr, nullptr};
    uint32_t *d_bb = nullptr;
    double *d_I = nullptr;
    unsigned long long *d_key = nullptr, *d_key2 = nullptr;
    uint8_t *d_split = nullptr;
    void *d_tmp = nullptr;
    size_t tmp_bytes = 0;
    const float *in3[3] = {v->px, v->py, v->pz}, *inI[3] = {v->ir, v->ig, v->ib};
    auto ck = [&](cudaError_t x) { if (x != cudaSuccess && e == cudaSuccess) e = x; return e == cudaSuccess; };
    ck(dmal(&d_idx, nv));
    ck(dmal(&d_idx2, nv));
    ck(dmal(&d_iseg, iseg.size()));
    ck(dmal(&d_work, work.size()));
    ck(dmal(&d_left, nn));
    ck(dmal(&d_right, nn));
    ck(dmal(&d_parent, nn));
    ck(dmal(&d_leaf, nn));
    ck(dmal(&d_nodes, nn));
    ck(dmal(&d_rep, nn));
    ck(dmal(&d_id, nn));
    ck(dmal(&d_id2, nn));
    ck(dmal(&d_flag, nn));
    ck(dmal(&d_pre, nn));
    ck(dmal(&d_cut, nn));
    ck(dmal(&d_bb, 6 * nn));
    ck(dmal(&d_I, 3 * nn));
    ck(dmal(&d_key, nn));
    ck(dmal(&d_key2, nn));
    ck(dmal(&d_split, nn));
    ck(dmal(&d_beg, std::max<size_t>(iseg.size() / 3, 1)));
    ck(dmal(&d_end, std::max<size_t>(iseg.size() / 3, 1)));
    for (int a = 0; a < 3; ++a) {
        ck(dmal(&d_pos3[a], nv));
        ck(dmal(&d_I3[a], nv));
        ck(dmal(&d_io[a], nn));
    }
    if (e == cudaSuccess) {
        const cudaMemcpyKind kin = memory == LMC_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
        for (int a = 0; a < 3; ++a) {
            ck(cudaMemcpyAsync(d_pos3[a], in3[a], nv * 4, kin, st));
            ck(cudaMemcpyAsync(d_I3[a], inI[a], nv * 4, kin, st));
        }
        std::vector<int32_t> iota(nv), bg, en;
        for (int64_t k = 0; k < nv; ++k) iota[k] = (int32_t)k;
        ck(cudaMemcpyAsync(d_idx, iota.data(), nv * 4, cudaMemcpyHostToDevice, st));
        ck(cudaMemcpyAsync(d_iseg, iseg.data(), iseg.size() * 4, cudaMemcpyHostToDevice, st));
        ck(cudaMemcpyAsync(d_work, work.data(), work.size() * 4, cudaMemcpyHostToDevice, st));
        ck(cudaMemcpyAsync(d_left, left.data(), nn * 4, cudaMemcpyHostToDevice, st));
        ck(cudaMemcpyAsync(d_right, right.data(), nn * 4, cudaMemcpyHostToDevice, st));
        ck(cudaMemcpyAsync(d_parent, parent.data(), nn * 4, cudaMemcpyHostToDevice, st));
        ck(cudaMemcpyAsync(d_leaf, leaf_start.data(), nn * 4, cudaMemcpyHostToDevice, st));
        ck(cudaMemcpyAsync(d_nodes, level_nodes.data(), nn * 4, cudaMemcpyHostToDevice, st));
        // segment bounds relative to each level's base, for the segmented sorts
        for (size_t li = 0; li < lv.size(); ++li)
            for (int k = 0; k < lv[li].nint; ++k) {
                bg.push_back((int32_t)(iseg[3 * (lv[li].seg_off + k) + 1] - lv[li].base));
                en.push_back((int32_t)(iseg[3 * (lv[li].seg_off + k) + 1] + iseg[3 * (lv[li].seg_off + k) + 2] - lv[li].base));
            }
        if (!bg.empty()) {
            ck(cudaMemcpyAsync(d_beg, bg.data(), bg.size() * 4, cudaMemcpyHostToDevice, st));
            ck(cudaMemcpyAsync(d_end, en.data(), en.size() * 4, cudaMemcpyHostToDevice, st));
        }
        int max_nint = 1;
        for (auto &d : lv) max_nint = std::max(max_nint, d.nint);
        size_t b1 = 0, b2 = 0, b3 = 0;
        ck(cub::DeviceSegmentedSort::SortKeys(nullptr, b1, d_key, d_key2, (int)nv, max_nint, d_beg, d_end, st));
        ck(cub::DeviceRadixSort::SortPairs(nullptr, b2, d_key, d_key2, d_id, d_id2, (int)nn, 0, 64, st));
        ck(cub::DeviceScan::ExclusiveSum(nullptr, b3, d_flag, d_pre, (int)nn, st));
        tmp_bytes = std::max(b1, std::max(b2, b3));
        ck(cudaMalloc(&d_tmp, std::max<size_t>(tmp_bytes, 16)));
        ck(cudaMemsetAsync(d_split, 0, nn, st));
        k_lt_bbox_init<<<(unsigned)((6 * nn + 255) / 256), 256, 0, st>>>(6 * nn, d_bb);
        // ---- levels: bboxes of every segment, then a segmented sort of the internal ones
        size_t boff = 0;
        for (size_t li = 0; li < lv.size() && e == cudaSuccess; ++li) {
            const LvlDev &d = lv[li];
            if (d.nwork > 0) k_lt_bbox<<<d.nwork, 256, 0, st>>>(d_work + 3 * d.work_off, d_idx, d_pos3[0], d_pos3[1], d_pos3[2], d_bb);
            if (d.nint == 0) continue;
            const unsigned nb = (unsigned)((d.n + 255) / 256);
            k_lt_keys<<<nb, 256, 0, st>>>(d_iseg + 3 * d.seg_off, d.nint, d_idx, d_pos3[0], d_pos3[1], d_pos3[2], d_bb,
                                          d.base, d.n, d_key);
            size_t bytes = tmp_bytes;
            ck(cub::DeviceSegmentedSort::SortKeys(d_tmp, bytes, d_key, d_key2, (int)d.n, d.nint, d_beg + boff,
                                                  d_end + boff, st));
            k_lt_unkey<<<nb, 256, 0, st>>>(d_key2, d_iseg + 3 * d.seg_off, d.nint, d.base, d.n, d_idx + d.base);
            boff += d.nint;
            ck(cudaGetLastError());
        }
        // ---- intensities and representatives bottom-up
        for (size_t li = levels.size(); li-- > 0 && e == cudaSuccess;) {
            const int n = (int)(level_off[li + 1] - level_off[li]);
            k_lt_sum<<<(n + 255) / 256, 256, 0, st>>>(d_nodes + level_off[li], n, d_left, d_right, d_leaf, d_idx, d_I3[0],
                                                      d_I3[1], d_I3[2], d_I, d_rep);
        }
        // ---- global cut: split the cut_max - 1 internal nodes of largest bound (ties: smaller id)
        const unsigned nbn = (unsigned)((nn + 255) / 256);
        k_lt_bound<<<nbn, 256, 0, st>>>(nn, d_left, d_I, d_bb, d_key, d_id, d_io[0], d_io[1], d_io[2]);
        size_t bytes = tmp_bytes;
        ck(cub::DeviceRadixSort::SortPairs(d_tmp, bytes, d_key, d_key2, d_id, d_id2, (int)nn, 0, 64, st));   // stable
        const int64_t nsplit = std::min<int64_t>(cut_max - 1, nv - 1);
        if (nsplit > 0) k_lt_split<<<(unsigned)((nsplit + 255) / 256), 256, 0, st>>>(d_id2, nsplit, d_split);
        k_lt_incut<<<nbn, 256, 0, st>>>(nn, d_parent, d_split, d_flag);
        bytes = tmp_bytes;
        ck(cub::DeviceScan::ExclusiveSum(d_tmp, bytes, d_flag, d_pre, (int)nn, st));
        k_lt_compact<<<nbn, 256, 0, st>>>(nn, d_flag, d_pre, d_cut);
        ck(cudaGetLastError());
        int32_t last_pre = 0, last_flag = 0;
        ck(cudaMemcpyAsync(&last_pre, d_pre + nn - 1, 4, cudaMemcpyDeviceToHost, st));
        ck(cudaMemcpyAsync(&last_flag, d_flag + nn - 1, 4, cudaMemcpyDeviceToHost, st));
        ck(cudaStreamSynchronize(st));
        const int64_t ncut = (int64_t)last_pre + last_flag;
        *cut_size = ncut;
        const cudaMemcpyKind kout = memory == LMC_MEM_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
        if (left_out) ck(cudaMemcpyAsync(left_out, d_left, nn * 4, kout, st));
        if (right_out) ck(cudaMemcpyAsync(right_out, d_right, nn * 4, kout, st));
        if (rep_out) ck(cudaMemcpyAsync(rep_out, d_rep, nn * 4, kout, st));
        if (ir_out) ck(cudaMemcpyAsync(ir_out, d_io[0], nn * 4, kout, st));
        if (ig_out) ck(cudaMemcpyAsync(ig_out, d_io[1], nn * 4, kout, st));
        if (ib_out) ck(cudaMemcpyAsync(ib_out, d_io[2], nn * 4, kout, st));
        if (cut_out) ck(cudaMemcpyAsync(cut_out, d_cut, ncut * 4, kout, st));
        ck(cudaStreamSynchronize(st));
    }
    if (e == cudaErrorMemoryAllocation) ret = LMC_ENOMEM;
    else if (e != cudaSuccess) ret = LMC_ECUDA;
    void *all[] = {d_idx, d_idx2, d_iseg, d_work, d_beg, d_end, d_left, d_right, d_parent, d_leaf, d_nodes, d_rep,
                   d_id, d_id2, d_flag, d_pre, d_cut, d_bb, d_I, d_key, d_key2, d_split, d_tmp,
                   d_pos3[0], d_pos3[1], d_pos3[2], d_I3[0], d_I3[1], d_I3[2], d_io[0], d_io[1], d_io[2]};
    for (void *p : all)
        if (p) cudaFree(p);
    return ret;
}
