// lmc_api.cu — host side of liblmc: context, validation, upper light tree, capacities, stage
// state machine and getters.  No per-slice arithmetic runs here; every stage of the path is a
// kernel in exact.cu / complete.cu.
#include <cuda_runtime.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <functional>
#include <new>
#include <vector>

#include "lmc_internal.h"

using namespace lmc;

namespace {

// NVTX range over one C-ABI call (a no-op unless a profiler injects itself): nsys / ncu timelines
// show the stages by name (SURVEY §5 tooling)
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

lmc_status fail(lmc_ctx *c, lmc_status s, const char *fmt, ...)
{
    if (c) {
        char buf[512];
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(buf, sizeof buf, fmt, ap);
        va_end(ap);
        c->err = buf;
        if (s == LMC_ECUDA) c->sticky = LMC_ECUDA;
    }
    return s;
}

lmc_status cuda_fail(lmc_ctx *c, cudaError_t e, const char *where)
{
    if (e == cudaErrorMemoryAllocation) return fail(c, LMC_ENOMEM, "%s: %s", where, cudaGetErrorString(e));
    return fail(c, LMC_ECUDA, "%s: %s", where, cudaGetErrorString(e));
}

#define CK(expr, where)                                   \
    do {                                                  \
        cudaError_t e_ = (expr);                          \
        if (e_ != cudaSuccess) return cuda_fail(c, e_, where); \
    } while (0)

double lum3(double r, double g, double b) { return (0.2126 * r + 0.7152 * g) + 0.0722 * b; }

template <typename T>
cudaError_t dalloc(T **p, size_t n)
{
    *p = nullptr;
    if (n == 0) n = 1;
    return cudaMalloc((void **)p, n * sizeof(T));
}

// copy n elements of an input array (device or host) into device memory
template <typename T>
cudaError_t dcopy_in(T *dst, const T *src, size_t n, int memory, cudaStream_t st)
{
    if (n == 0) return cudaSuccess;
    return cudaMemcpyAsync(dst, src, n * sizeof(T), memory == LMC_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice,
                           st);
}

template <typename T>
cudaError_t hcopy_in(std::vector<T> &dst, const T *src, size_t n, int memory, cudaStream_t st)
{
    dst.resize(n);
    if (n == 0) return cudaSuccess;
    if (memory == LMC_MEM_HOST) {
        memcpy(dst.data(), src, n * sizeof(T));
        return cudaSuccess;
    }
    cudaError_t e = cudaMemcpyAsync(dst.data(), src, n * sizeof(T), cudaMemcpyDeviceToHost, st);
    if (e != cudaSuccess) return e;
    return cudaStreamSynchronize(st);
}

void free_all(lmc_ctx *c)
{
    if (c->comm) {
        ncclCommDestroy((ncclComm_t)c->comm);
        c->comm = nullptr;
    }
    Dev &d = c->d;
    void *ptrs[] = {d.pixel, d.g[0], d.g[1], d.g[2], d.g[3], d.g[4], d.g[5], d.g[6], d.g[7], d.g[8], d.g[9], d.g[10],
                    d.g[11], d.g[12], d.expo, d.vpl, d.ut_i32, d.ut_lum, d.ut_I, d.rows, d.rows_alt, d.sk,
                    d.sl_ext, d.sl_hist, d.sl_cnt, d.sl_state, d.lvl_begin, d.lvl_end, d.lvl_slot, d.lvl_work, d.slice_off, d.prow, d.sbox,
                    d.p1_rows, d.p1_Ta, d.p1_Tb, d.p1_cnt, d.pool_rows, d.pool_Ta, d.pool_Tb, d.pool_used, d.cs_flags,
                    d.cs_eps, d.cs_cost, d.cs_zoff, d.cs_zlen, d.cut_n, d.cut_cols, d.src_off, d.src_len, d.src_side,
                    d.rowptr, d.col, d.val, d.val64, d.Xd, d.Yd, d.val64c, d.carried, d.colptr, d.csc_row, d.csc_src, d.nnz, d.target_n, d.n_new,
                    d.newpos, d.U, d.V, d.Lam, d.Pi, d.Xold, d.S, d.flags, d.iters, d.resid,
                    d.direct_rgb, d.counters, d.img, d.rows_rgb, d.vpl_soa, d.r_perm, d.r_len, d.c_perm, d.c_len,
                    d.r_goff, d.c_goff, d.c_nsolo, d.adm_order, d.r_ent, d.c_ent, d.norm, d.r_grp, d.c_grp,
                    d.r_slot, d.c_slot, d.ngrp, d.ctot, d.slot_st, d.ord_tmp, d.ord_cub, d.rank_pix, d.all4, d.prev_cut, d.prev_n, d.prev_flags, d.prev_rows, d.warm_ok, d.bvh, d.tri4, d.soff_loc, d.rows_loc};
    for (void *p : ptrs)
        if (p) cudaFree(p);
    if (c->h_stage) cudaFreeHost(c->h_stage);
    if (c->h_pix) cudaFreeHost(c->h_pix);
    c->h_pix = nullptr;
    memset(&c->d, 0, sizeof(c->d));
    c->h_stage = nullptr;
    if (c->ev_ok)
        for (auto &e : c->ev) cudaEventDestroy(e);
    c->ev_ok = false;
    release_scene_slot(c->scene_slot);
    c->scene_slot = -1;
}

// ------------------------------------------------------------------------------------------
// upper light tree (global cut + ancestors) on the host
// ------------------------------------------------------------------------------------------
struct HostTree {
    std::vector<int32_t> left, right, rep, cut;
    std::vector<float> ir, ig, ib;
};

lmc_status build_upper(lmc_ctx *c, const HostTree &t)
{
    const int64_t NN = c->NN;
    std::vector<int32_t> parent(NN, -1);
    for (int64_t f = 0; f < NN; ++f) {
        int32_t l = t.left[f], r = t.right[f];
        if ((l < 0) != (r < 0)) return fail(c, LMC_EINVAL, "node %lld has exactly one child", (long long)f);
        if (l >= 0) {
            if (l >= NN || r >= NN) return fail(c, LMC_EINVAL, "child index out of range at node %lld", (long long)f);
            if (parent[l] >= 0 || parent[r] >= 0) return fail(c, LMC_EINVAL, "node with two parents under %lld", (long long)f);
            parent[l] = (int32_t)f;
            parent[r] = (int32_t)f;
            if (!(t.rep[f] == t.rep[l] || t.rep[f] == t.rep[r]))
                return fail(c, LMC_EINVAL, "rep(%lld) is not the rep of a child (R5)", (long long)f);
        } else if (t.rep[f] < 0 || t.rep[f] >= c->NV) {
            return fail(c, LMC_EINVAL, "leaf %lld has an invalid VPL id", (long long)f);
        }
    }
    // antichain cover: every leaf has exactly one ancestor-or-self in the cut
    std::vector<uint8_t> in_cut(NN, 0);
    for (int32_t g : t.cut) {
        if (g < 0 || g >= NN) return fail(c, LMC_EINVAL, "global cut node out of range");
        if (in_cut[g]) return fail(c, LMC_EINVAL, "duplicate node in the global cut");
        in_cut[g] = 1;
    }
    std::vector<uint8_t> upper(NN, 0);
    for (int32_t g : t.cut) {
        for (int32_t a = parent[g]; a >= 0; a = parent[a]) {
            if (in_cut[a]) return fail(c, LMC_EINVAL, "global cut is not an antichain");
            if (upper[a]) break;
            upper[a] = 1;
        }
    }
    // leaf coverage by counting leaves under cut nodes
    {
        int64_t leaves = 0, covered = 0;
        for (int64_t f = 0; f < NN; ++f) leaves += t.left[f] < 0;
        std::vector<int32_t> st;
        for (int32_t g : t.cut) {
            st.push_back(g);
            while (!st.empty()) {
                int32_t f = st.back();
                st.pop_back();
                if (t.left[f] < 0) ++covered;
                else { st.push_back(t.left[f]); st.push_back(t.right[f]); }
            }
        }
        if (covered != leaves) return fail(c, LMC_EINVAL, "global cut does not cover every leaf exactly once");
    }
    std::vector<int32_t> nodes;
    for (int64_t f = 0; f < NN; ++f)
        if (upper[f] || in_cut[f]) nodes.push_back((int32_t)f);
    const int U = (int)nodes.size();
    std::vector<int32_t> loc(NN, -1);
    for (int u = 0; u < U; ++u) loc[nodes[u]] = u;
    std::vector<int32_t> L(U), R(U), P(U), rep(U), height(U, 0), nunc(U), base_of(U, -1);
    std::vector<double> lum(U);
    std::vector<float> I(3 * (size_t)U);
    for (int u = 0; u < U; ++u) {
        int32_t f = nodes[u];
        L[u] = in_cut[f] ? -1 : loc[t.left[f]];
        R[u] = in_cut[f] ? -1 : loc[t.right[f]];
        P[u] = parent[f] >= 0 ? loc[parent[f]] : -1;
        rep[u] = t.rep[f];
        lum[u] = lum3(t.ir[f], t.ig[f], t.ib[f]);
        I[3 * u] = t.ir[f];
        I[3 * u + 1] = t.ig[f];
        I[3 * u + 2] = t.ib[f];
    }
    // heights (children before parents: iterate until stable over reverse local order)
    std::function<int(int)> hgt = [&](int u) -> int {
        if (L[u] < 0) return 0;
        if (height[u] > 0) return height[u];
        int h = 1 + std::max(hgt(L[u]), hgt(R[u]));
        height[u] = h;
        return h;
    };
    int H = 0;
    for (int u = 0; u < U; ++u) H = std::max(H, hgt(u));
    std::vector<int32_t> hlist, hoff(H + 2, 0), base_list;
    for (int h = 1; h <= H; ++h) {
        hoff[h] = (int32_t)hlist.size();
        for (int u = 0; u < U; ++u)
            if (L[u] >= 0 && height[u] == h) hlist.push_back(u);
    }
    hoff[H + 1] = (int32_t)hlist.size();
    if (H == 0) hoff[1] = 0;
    double lmax = 0.0;
    for (int u = 0; u < U; ++u)
        if (L[u] >= 0 && L[L[u]] < 0 && L[R[u]] < 0) {
            base_of[u] = (int32_t)base_list.size();
            base_list.push_back(u);
            lmax = std::max(lmax, lum[u]);
        }
    for (int u = 0; u < U; ++u) {
        // P:104 n_f proportional to I_f (R6): max(nmin, ceil(nmax lum / l_max)), clamped by m in-kernel
        if (lmax > 0.0) {
            double x = ceil(((double)c->cfg.p1_nmax * lum[u]) / lmax);
            if (x > 1073741824.0) x = 1073741824.0;
            nunc[u] = x > (double)c->cfg.p1_nmin ? (int32_t)x : c->cfg.p1_nmin;
        } else {
            nunc[u] = c->cfg.p1_nmin;
        }
    }
    // capacity of the per-slice sample pool: sum over internal nodes of a bound on |zeta_f|
    {
        const int64_t m = c->mmax;
        std::vector<int64_t> zb(U, 0);
        std::function<int64_t(int)> zbound = [&](int u) -> int64_t {
            if (L[u] < 0) return std::min<int64_t>(m, nunc[u]);
            if (zb[u] > 0) return zb[u];
            int64_t v;
            if (base_of[u] >= 0) v = std::min<int64_t>(m, nunc[u]);
            else v = std::min<int64_t>(m, zbound(L[u]) + zbound(R[u]));
            zb[u] = v;
            return v;
        };
        int64_t tot = 0;
        for (int u = 0; u < U; ++u)
            if (L[u] >= 0) tot += zbound(u);
        c->pool_cap = std::max<int64_t>(tot, 32);
    }
    // upload: int32 block [node L R P rep nunc hlist hoff base_list base_of]
    std::vector<int32_t> blk;
    auto put = [&](const std::vector<int32_t> &v) { size_t o = blk.size(); blk.insert(blk.end(), v.begin(), v.end()); return o; };
    size_t o_node = put(nodes), o_L = put(L), o_R = put(R), o_P = put(P), o_rep = put(rep), o_n = put(nunc),
           o_hl = put(hlist), o_ho = put(hoff), o_bl = put(base_list), o_bo = put(base_of);
    Dev &d = c->d;
    CK(dalloc(&d.ut_i32, blk.size()), "alloc upper tree");
    CK(dalloc(&d.ut_lum, (size_t)U), "alloc upper tree");
    CK(dalloc(&d.ut_I, 3 * (size_t)U), "alloc upper tree");
    CK(cudaMemcpy(d.ut_i32, blk.data(), blk.size() * 4, cudaMemcpyHostToDevice), "upload upper tree");
    CK(cudaMemcpy(d.ut_lum, lum.data(), (size_t)U * 8, cudaMemcpyHostToDevice), "upload upper tree");
    CK(cudaMemcpy(d.ut_I, I.data(), (size_t)U * 12, cudaMemcpyHostToDevice), "upload upper tree");
    Upper &up = c->up;
    up.U = U;
    up.H = H;
    up.nB = (int32_t)base_list.size();
    up.node = d.ut_i32 + o_node;
    up.left = d.ut_i32 + o_L;
    up.right = d.ut_i32 + o_R;
    up.parent = d.ut_i32 + o_P;
    up.rep = d.ut_i32 + o_rep;
    up.nunc = d.ut_i32 + o_n;
    up.hlist = d.ut_i32 + o_hl;
    up.hoff = d.ut_i32 + o_ho;
    up.base_list = d.ut_i32 + o_bl;
    up.base_of = d.ut_i32 + o_bo;
    up.lum = d.ut_lum;
    up.I = d.ut_I;
    c->h_up_node = nodes;
    return LMC_OK;
}

// ------------------------------------------------------------------------------------------
// slicing structure: sizes depend only on (M, target): left child takes ceil(n/2)
// ------------------------------------------------------------------------------------------
// ------------------------------------------------------------------------------------------
// slicing tree shape (sizes depend only on (M, target): the left child takes ceil(n/2)) and the
// ranks' shares of it.  P = 2^k ranks and every node above depth k internal: rank r
// owns the r-th depth-k subtree (slicing levels >= k then run on that rank only); otherwise the
// slice index range [S r / P, S (r + 1) / P) of a replicated slicing.  Returns k, or -1.
// ------------------------------------------------------------------------------------------
struct TNode { int32_t start, len, depth; bool leaf; };

static std::vector<TNode> slicing_tree(int64_t M, int32_t target)
{
    std::vector<TNode> all;
    std::function<void(int32_t, int32_t, int32_t)> rec = [&](int32_t start, int32_t len, int32_t depth) {
        bool leaf = len <= target;
        all.push_back({start, len, depth, leaf});
        if (leaf) return;
        int32_t nl = (len + 1) / 2;
        rec(start, nl, depth + 1);
        rec(start + nl, len - nl, depth + 1);
    };
    if (M > 0) rec(0, (int32_t)M, 0);
    return all;
}

static std::vector<int32_t> leaf_offsets(const std::vector<TNode> &all)
{
    std::vector<TNode> leaves;
    for (auto &n : all)
        if (n.leaf) leaves.push_back(n);
    std::sort(leaves.begin(), leaves.end(), [](const TNode &a, const TNode &b) { return a.start < b.start; });
    std::vector<int32_t> off(1, 0);
    for (auto &n : leaves) off.push_back(n.start + n.len);
    return off;
}

static int plan_partition(const std::vector<TNode> &all, const std::vector<int32_t> &slice_off, int64_t M, int world,
                          std::vector<int32_t> &part_slice, std::vector<int64_t> &part_row)
{
    const int32_t S = (int32_t)slice_off.size() - 1;
    int k = -1;
    std::vector<int32_t> sub_lo;
    if (world > 1 && (world & (world - 1)) == 0) {
        int kk = 0;
        while ((1 << kk) < world) ++kk;
        std::vector<TNode> at;
        bool ok = true;
        for (auto &n : all) {
            if (n.depth == kk) at.push_back(n);
            if (n.depth < kk && n.leaf) ok = false;
        }
        if (ok && (int)at.size() == world) {
            std::sort(at.begin(), at.end(), [](const TNode &a, const TNode &b) { return a.start < b.start; });
            k = kk;
            for (auto &n : at) sub_lo.push_back(n.start);
        }
    }
    part_slice.assign(world + 1, 0);
    part_row.assign(world + 1, 0);
    for (int r = 0; r <= world; ++r) {
        if (k >= 0) {
            const int64_t row = r < world ? sub_lo[r] : M;
            part_row[r] = row;
            part_slice[r] = r < world ? (int32_t)(std::lower_bound(slice_off.begin(), slice_off.end() - 1, (int32_t)row) -
                                                  slice_off.begin())
                                      : S;
        } else {
            const int32_t s = (int32_t)((int64_t)S * r / world);
            part_slice[r] = s;
            part_row[r] = slice_off[s];
        }
    }
    return k;
}

lmc_status build_levels(lmc_ctx *c)
{
    typedef TNode Node;
    std::vector<Node> all = slicing_tree(c->M, c->cfg.slice_target);
    c->levels.clear();
    int32_t maxd = 0;
    for (auto &n : all) maxd = std::max(maxd, n.depth);
    c->h_slice_off = leaf_offsets(all);
    c->S = (int32_t)c->h_slice_off.size() - 1;
    // ---- the ranks' shares, see plan_partition
    int k;
    if (c->cfg.world > 1 && c->cfg.partition == 1) {
        // interleaved shares: rank r takes slices r, r + P, ...; every rank slices the whole frame.
        // part_slice / part_row: cumulative slice / row counts per rank (the gather's tile offsets)
        const int P = c->cfg.world;
        k = -1;
        c->h_part_slice.assign(P + 1, 0);
        c->h_part_row.assign(P + 1, 0);
        for (int r = 0; r < P; ++r) {
            int32_t ns = 0;
            int64_t nr = 0;
            for (int s = r; s < c->S; s += P) { ++ns; nr += c->h_slice_off[s + 1] - c->h_slice_off[s]; }
            c->h_part_slice[r + 1] = c->h_part_slice[r] + ns;
            c->h_part_row[r + 1] = c->h_part_row[r] + nr;
        }
    } else {
        k = plan_partition(all, c->h_slice_off, c->M, c->cfg.world, c->h_part_slice, c->h_part_row);
    }
    c->sub_k = k;
    const int64_t sub_a = c->h_part_row[c->cfg.rank], sub_b = c->h_part_row[c->cfg.rank + 1];
    // tilings per depth: nodes at depth d + leaves at depth < d; from depth k on only this rank's
    // subtree, positions relative to the level's first row
    std::vector<int32_t> beg, end, slot, work;
    auto tiling = [&](int d, int64_t lo, int64_t hi, std::vector<Node> &out) {
        out.clear();
        for (auto &n : all)
            if ((n.depth == d || (n.leaf && n.depth < d)) && n.start >= lo && n.start < hi) out.push_back(n);
        std::sort(out.begin(), out.end(), [](const Node &a, const Node &b) { return a.start < b.start; });
    };
    int max_tiles = 1, max_slots = 1, max_work = 1;
    std::vector<Node> cur;
    for (int d = 0; d < maxd; ++d) {
        const bool sub = k >= 0 && d >= k;
        const int64_t lo = sub ? sub_a : 0, hi = sub ? sub_b : c->M;
        tiling(d, lo, hi, cur);
        lmc_ctx::Level L;
        L.lo = lo;
        L.n = hi - lo;
        L.tile_off = (int32_t)beg.size();
        L.tile_n = (int32_t)cur.size();
        int ns = 0;
        int32_t maxlen = 0;
        for (auto &n : cur) maxlen = std::max(maxlen, n.len);
        L.fused = maxlen <= 8192 || (int)cur.size() >= 64;   // slice.cu: one CTA per tile
        const size_t w0 = work.size();
        L.work_off = (int32_t)(work.size() / 4);
        for (int ti = 0; ti < (int)cur.size(); ++ti) {
            const Node &n = cur[ti];
            beg.push_back(n.start - (int32_t)lo);
            end.push_back(n.start + n.len - (int32_t)lo);
            const bool split = n.depth == d && !n.leaf;
            slot.push_back(split ? ns++ : -1);
            if (!L.fused) {   // chunks of <= 4096 rows of every tile (leaves: copied through)
                const int32_t first = (int32_t)((work.size() - w0) / 4);
                for (int32_t o = 0; o < n.len; o += 4096) {
                    work.push_back(ti);
                    work.push_back(n.start - (int32_t)lo + o);
                    work.push_back(std::min<int32_t>(4096, n.len - o));
                    work.push_back(first);
                }
            }
        }
        L.work_n = (int32_t)(work.size() / 4) - L.work_off;
        L.nslots = ns;
        max_tiles = std::max(max_tiles, (int)cur.size());
        if (L.n > 0 && ns > 0) {
            c->levels.push_back(L);
            if (!L.fused) { max_slots = std::max(max_slots, ns); max_work = std::max(max_work, (int)L.work_n); }
        } else {
            work.resize(w0);
        }
    }
    c->max_tiles = max_tiles;
    Dev &d = c->d;
    CK(dalloc(&d.lvl_begin, beg.size()), "alloc slicing");
    CK(dalloc(&d.lvl_end, end.size()), "alloc slicing");
    CK(dalloc(&d.lvl_slot, slot.size()), "alloc slicing");
    CK(dalloc(&d.lvl_work, work.size()), "alloc slicing");
    CK(dalloc(&d.sl_ext, (size_t)max_slots * 12), "alloc slicing");
    CK(dalloc(&d.sl_hist, (size_t)max_slots * 1024), "alloc slicing");
    CK(dalloc(&d.sl_state, (size_t)max_slots * 4), "alloc slicing");
    CK(dalloc(&d.sl_cnt, (size_t)max_work * 2), "alloc slicing");
    if (!beg.empty()) {
        CK(cudaMemcpy(d.lvl_begin, beg.data(), beg.size() * 4, cudaMemcpyHostToDevice), "upload slicing");
        CK(cudaMemcpy(d.lvl_end, end.data(), end.size() * 4, cudaMemcpyHostToDevice), "upload slicing");
        CK(cudaMemcpy(d.lvl_slot, slot.data(), slot.size() * 4, cudaMemcpyHostToDevice), "upload slicing");
    }
    if (!work.empty()) CK(cudaMemcpy(d.lvl_work, work.data(), work.size() * 4, cudaMemcpyHostToDevice), "upload slicing");
    CK(dalloc(&d.slice_off, c->h_slice_off.size()), "alloc slicing");
    CK(cudaMemcpy(d.slice_off, c->h_slice_off.data(), c->h_slice_off.size() * 4, cudaMemcpyHostToDevice), "upload slicing");
    return LMC_OK;
}

lmc_status check_stage(lmc_ctx *c, int need)
{
    if (!c) return LMC_EINVAL;
    if (c->sticky != LMC_OK) return c->sticky;
    if (c->state < need) return fail(c, LMC_ESTATE, "stage called out of order (state %d, needs %d)", c->state, need);
    return LMC_OK;
}

lmc_status check_overflow(lmc_ctx *c)
{
    unsigned long long cnt[5];
    CK(cudaMemcpyAsync(cnt, c->d.counters, sizeof cnt, cudaMemcpyDeviceToHost, c->stream), "read counters");
    CK(cudaStreamSynchronize(c->stream), "sync");
    if (cnt[3] & 1ull) return fail(c, LMC_EOVERFLOW, "coarsening sample pool overflow (cap %lld)", (long long)c->pool_cap);
    if (cnt[3] & 2ull) return fail(c, LMC_EOVERFLOW, "pass-2 sample capacity overflow (cap %lld)", (long long)c->ncap);
    if (cnt[3] & 4ull) return fail(c, LMC_EOVERFLOW, "completion layout capacity overflow (cap %lld)", (long long)c->scap);
    return LMC_OK;
}

template <typename T>
cudaError_t d2h(T *dst, const T *src, size_t n)
{
    if (!dst || n == 0) return cudaSuccess;
    return cudaMemcpy(dst, src, n * sizeof(T), cudaMemcpyDeviceToHost);
}

void ev_rec(lmc_ctx *c, int k)
{
    if (c->timing && c->ev_ok) cudaEventRecord(c->ev[k], c->stream);
}

}  // namespace

// Triangle BVH: median split of the triangle centroids on the longest axis of their
// bounds, ties by triangle index (deterministic), at most 4 triangles per leaf; children of a
// node are adjacent (first, first + 1).  Node bounds are the exact float32 min / max of the
// vertices.  Only acceleration: the decision per triangle is the exact fp64 test in exact.cu.
static void build_tri_bvh(const float *tri, int32_t n, std::vector<float4> &nodes, std::vector<float4> &tris,
                          std::vector<int32_t> *order_out = nullptr)
{
    std::vector<int32_t> idx(n);
    for (int32_t k = 0; k < n; ++k) idx[k] = k;
    std::vector<float> cen(3 * (size_t)n);
    for (int32_t k = 0; k < n; ++k)
        for (int a = 0; a < 3; ++a) cen[3 * (size_t)k + a] = (tri[9 * (size_t)k + a] + tri[9 * (size_t)k + 3 + a] + tri[9 * (size_t)k + 6 + a]) / 3.0f;
    struct Job {
        int32_t node, lo, hi;
    };
    nodes.assign(2, make_float4(0, 0, 0, 0));
    std::vector<Job> stack{{0, 0, n}};
    while (!stack.empty()) {
        Job j = stack.back();
        stack.pop_back();
        float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
        float clo[3] = {INFINITY, INFINITY, INFINITY}, chi[3] = {-INFINITY, -INFINITY, -INFINITY};
        for (int32_t i = j.lo; i < j.hi; ++i) {
            const float *t = tri + 9 * (size_t)idx[i];
            for (int a = 0; a < 3; ++a) {
                lo[a] = std::min(lo[a], std::min(t[a], std::min(t[3 + a], t[6 + a])));
                hi[a] = std::max(hi[a], std::max(t[a], std::max(t[3 + a], t[6 + a])));
                clo[a] = std::min(clo[a], cen[3 * (size_t)idx[i] + a]);
                chi[a] = std::max(chi[a], cen[3 * (size_t)idx[i] + a]);
            }
        }
        float4 &A = nodes[2 * (size_t)j.node];
        float4 &B = nodes[2 * (size_t)j.node + 1];
        A = make_float4(lo[0], lo[1], lo[2], 0.f);
        B = make_float4(hi[0], hi[1], hi[2], 0.f);
        const int32_t cnt = j.hi - j.lo;
        if (cnt <= 4) {
            int32_t first = j.lo, c4 = cnt;
            memcpy(&A.w, &first, 4);
            memcpy(&B.w, &c4, 4);
            continue;
        }
        int ax = 0;
        for (int a = 1; a < 3; ++a)
            if (chi[a] - clo[a] > chi[ax] - clo[ax]) ax = a;
        const int32_t mid = j.lo + cnt / 2;
        std::nth_element(idx.begin() + j.lo, idx.begin() + mid, idx.begin() + j.hi, [&](int32_t p, int32_t q) {
            const float cp = cen[3 * (size_t)p + ax], cq = cen[3 * (size_t)q + ax];
            return cp < cq || (cp == cq && p < q);
        });
        const int32_t child = (int32_t)(nodes.size() / 2);
        nodes.resize(nodes.size() + 4);
        float4 &A2 = nodes[2 * (size_t)j.node];   // (re-fetch: resize may move the storage)
        int32_t zero = 0;
        memcpy(&A2.w, &child, 4);
        memcpy(&nodes[2 * (size_t)j.node + 1].w, &zero, 4);
        stack.push_back({child + 1, mid, j.hi});
        stack.push_back({child, j.lo, mid});
    }
    if (order_out) *order_out = idx;
    tris.resize(3 * (size_t)n);
    for (int32_t i = 0; i < n; ++i) {
        const float *t = tri + 9 * (size_t)idx[i];
        tris[3 * (size_t)i + 0] = make_float4(t[0], t[1], t[2], t[3]);
        tris[3 * (size_t)i + 1] = make_float4(t[4], t[5], t[6], t[7]);
        tris[3 * (size_t)i + 2] = make_float4(t[8], 0.f, 0.f, 0.f);
    }
}

// ==========================================================================================
extern "C" {

const char *lmc_status_str(lmc_status s)
{
    switch (s) {
    case LMC_OK: return "LMC_OK";
    case LMC_EINVAL: return "LMC_EINVAL";
    case LMC_ESTATE: return "LMC_ESTATE";
    case LMC_ENOMEM: return "LMC_ENOMEM";
    case LMC_ECUDA: return "LMC_ECUDA";
    case LMC_EOVERFLOW: return "LMC_EOVERFLOW";
    case LMC_ENCCL: return "LMC_ENCCL";
    }
    return "LMC_UNKNOWN";
}

const char *lmc_last_error(const lmc_ctx *c) { return c ? c->err.c_str() : "null context"; }

void lmc_destroy(lmc_ctx *c)
{
    if (!c) return;
    free_all(c);
    delete c;
}

static lmc_status create_impl(lmc_ctx *c, const lmc_gbuffer *g, const lmc_vpls *v, const lmc_light_tree *t,
                              const lmc_scene *sc)
{
    const lmc_config &cfg = c->cfg;
    c->stream = (cudaStream_t)cfg.stream;
    if (cfg.slice_target < 1 || cfg.slice_target > MAX_SLICE) return fail(c, LMC_EINVAL, "slice_target must be in [1, %d]", MAX_SLICE);
    if (!(cfg.rate > 0.0 && cfg.rate <= 1.0)) return fail(c, LMC_EINVAL, "rate must be in (0, 1]");
    if (!(cfg.gamma > 0.0 && cfg.gamma < 1.618)) return fail(c, LMC_EINVAL, "gamma must be in (0, 1.618)");
    if (!(cfg.alpha > 0.0 && cfg.beta > 0.0)) return fail(c, LMC_EINVAL, "alpha, beta must be > 0");
    if (!(cfg.rank_q == 4 || cfg.rank_q == 8 || cfg.rank_q == 16 || cfg.rank_q == 32))
        return fail(c, LMC_EINVAL, "rank_q must be one of 4, 8, 16, 32");
    if (cfg.solver == LMC_SOLVER_MALS && !(cfg.lambda > 0.0)) return fail(c, LMC_EINVAL, "MALS needs lambda > 0");
    if (cfg.solver != LMC_SOLVER_ADM && cfg.solver != LMC_SOLVER_MALS) return fail(c, LMC_EINVAL, "unknown solver");
    if (cfg.p1_nmax < 1 || cfg.p1_nmax > MAX_NMAX || cfg.p1_nmin < 1) return fail(c, LMC_EINVAL, "p1_nmax must be in [1, 32], p1_nmin >= 1");
    if (cfg.max_iter < 0) return fail(c, LMC_EINVAL, "max_iter must be >= 0");
    if (cfg.solver == LMC_SOLVER_MALS && cfg.max_iter < 1) return fail(c, LMC_EINVAL, "MALS needs max_iter >= 1");
    if (cfg.world < 1 || cfg.rank < 0 || cfg.rank >= cfg.world) return fail(c, LMC_EINVAL, "bad rank/world");
    if (cfg.input_memory != LMC_MEM_DEVICE && cfg.input_memory != LMC_MEM_HOST) return fail(c, LMC_EINVAL, "bad input_memory");
    if (!g || !v || !t || !sc) return fail(c, LMC_EINVAL, "null input struct");
    if (g->count < 0 || g->count > (1ll << 31) - 1) return fail(c, LMC_EINVAL, "bad gbuffer count");
    if (g->width < 0 || g->height < 0 || (int64_t)g->width * g->height > (1ll << 31) - 1 ||
        (g->count > 0 && (g->width < 1 || g->height < 1)))
        return fail(c, LMC_EINVAL, "bad image size %d x %d", g->width, g->height);
    if (g->count > 0 && (!g->pixel || !g->px || !g->py || !g->pz || !g->nx || !g->ny || !g->nz || !g->vx || !g->vy ||
                         !g->vz || !g->rho_r || !g->rho_g || !g->rho_b || !g->spec || !g->exponent))
        return fail(c, LMC_EINVAL, "null gbuffer array");
    if (v->count < 1 || !v->px || !v->py || !v->pz || !v->nx || !v->ny || !v->nz) return fail(c, LMC_EINVAL, "bad VPL set");
    if (t->num_nodes < 1 || !t->left || !t->right || !t->rep || !t->ir || !t->ig || !t->ib || !t->global_cut)
        return fail(c, LMC_EINVAL, "bad light tree");
    if (t->cut_size < 1 || t->cut_size > MAX_CUT) return fail(c, LMC_EINVAL, "global cut size must be in [1, %d]", MAX_CUT);
    if (sc->n_sph < 0 || sc->n_sph > MAX_PRIMS || sc->n_box < 0 || sc->n_box > MAX_PRIMS || sc->n_rect < 0 ||
        sc->n_rect > MAX_PRIMS)
        return fail(c, LMC_EINVAL, "at most %d occluders of each kind", MAX_PRIMS);
    if ((sc->n_sph && !sc->sph) || (sc->n_box && !sc->box) || (sc->n_rect && !sc->rect)) return fail(c, LMC_EINVAL, "null occluder array");
    if (!(sc->diag >= 1e-30 && sc->diag <= 1e30)) return fail(c, LMC_EINVAL, "scene diagonal must be in [1e-30, 1e30]");
    if (!(cfg.normal_weight == 0.0 || (cfg.normal_weight >= 1e-30 && cfg.normal_weight <= 1e30)))
        return fail(c, LMC_EINVAL, "normal_weight must be 0 or in [1e-30, 1e30]");
    if (sc->n_tri < 0 || sc->n_tri > (1 << 26) || (sc->n_tri && !sc->tri)) return fail(c, LMC_EINVAL, "bad triangle array");
    c->M = g->count;
    c->W = g->width;
    c->H = g->height;
    c->NV = v->count;
    c->NN = t->num_nodes;
    c->G = (int32_t)t->cut_size;
    c->diag = sc->diag;
    c->q = cfg.rank_q;
    c->nmax = cfg.p1_nmax;
    // scene constants
    memset(&c->scene, 0, sizeof c->scene);
    c->scene.nsph = sc->n_sph;
    c->scene.nbox = sc->n_box;
    c->scene.nrect = sc->n_rect;
    c->scene.dc2 = sc->clamp_dist * sc->clamp_dist;
    c->scene.eps = sc->shadow_eps;
    if (sc->n_sph) memcpy(c->scene.sph, sc->sph, sizeof(float) * 4 * sc->n_sph);
    if (sc->n_box) memcpy(c->scene.box, sc->box, sizeof(float) * 6 * sc->n_box);
    if (sc->n_rect) memcpy(c->scene.rect, sc->rect, sizeof(float) * 12 * sc->n_rect);
    c->scene.margin = (float)(1e-3 * sc->diag);
    for (int k = 0; k < sc->n_rect; ++k) {   // screening data of the rectangles (not used by exact tests)
        const float *r = sc->rect + 12 * k;
        for (int a = 0; a < 3; ++a) {
            float c0 = r[a], c1 = r[a] + r[3 + a], c2 = r[a] + r[6 + a], c3 = r[a] + r[3 + a] + r[6 + a];
            c->scene.rbox[6 * k + a] = std::min(std::min(c0, c1), std::min(c2, c3));
            c->scene.rbox[6 * k + 3 + a] = std::max(std::max(c0, c1), std::max(c2, c3));
        }
        c->scene.rnorm[k] = (float)std::sqrt((double)r[9] * r[9] + (double)r[10] * r[10] + (double)r[11] * r[11]);
    }
    if (sc->n_tri > 0) {   // triangle BVH, device-resident for the context's lifetime
        for (int64_t k = 0; k < 9ll * sc->n_tri; ++k)
            if (!std::isfinite(sc->tri[k])) return fail(c, LMC_EINVAL, "non-finite triangle vertex");
        std::vector<float4> nodes, tris;
        build_tri_bvh(sc->tri, sc->n_tri, nodes, tris);
        CK(cudaMalloc(&c->d.bvh, nodes.size() * sizeof(float4)), "alloc bvh");
        CK(cudaMalloc(&c->d.tri4, tris.size() * sizeof(float4)), "alloc triangles");
        CK(cudaMemcpy(c->d.bvh, nodes.data(), nodes.size() * sizeof(float4), cudaMemcpyHostToDevice), "upload bvh");
        CK(cudaMemcpy(c->d.tri4, tris.data(), tris.size() * sizeof(float4), cudaMemcpyHostToDevice), "upload triangles");
        c->scene.bvh = c->d.bvh;
        c->scene.tri4 = c->d.tri4;
        c->scene.ntri = sc->n_tri;
        c->scene.nbvh = (int32_t)(nodes.size() / 2);
    }
    c->scene_slot = acquire_scene_slot();
    if (c->scene_slot < 0) return fail(c, LMC_EINVAL, "more than %d live contexts in this process", SCENE_SLOTS);
    CK(upload_scene(c->scene_slot, c->scene), "upload scene");
    // slicing structure and this rank's share
    lmc_status st = build_levels(c);
    if (st != LMC_OK) return st;
    c->s0 = c->h_part_slice[cfg.rank];
    c->s1 = c->h_part_slice[cfg.rank + 1];
    c->SL = c->s1 - c->s0;
    c->interleaved = cfg.world > 1 && cfg.partition == 1;
    c->h_lrow.assign(c->SL + 1, 0);
    if (c->interleaved) {
        // this rank's slices r, r + P, ... gathered into local arrays each frame (slice.cu)
        c->row0 = c->h_part_row[cfg.rank];
        c->ML = c->h_part_row[cfg.rank + 1] - c->row0;
        for (int ls = 0; ls < c->SL; ++ls) {
            const int s = cfg.rank + ls * cfg.world;
            c->h_lrow[ls + 1] = c->h_lrow[ls] + (c->h_slice_off[s + 1] - c->h_slice_off[s]);
        }
        c->s0k = 0;
        c->lbase_k = 0;
        c->row0_k = 0;
        c->rs0 = cfg.rank;
        c->rss = cfg.world;
    } else {
        c->row0 = c->h_slice_off[c->s0];
        c->ML = c->h_slice_off[c->s1] - c->row0;
        for (int ls = 0; ls <= c->SL; ++ls) c->h_lrow[ls] = c->h_slice_off[c->s0 + ls] - (int32_t)c->row0;
        c->s0k = c->s0;
        c->lbase_k = c->h_slice_off[c->s0];
        c->row0_k = c->row0;
        c->rs0 = c->s0;
        c->rss = 1;
    }
    c->mmax = 1;
    for (int s = 0; s < c->S; ++s) c->mmax = std::max(c->mmax, c->h_slice_off[s + 1] - c->h_slice_off[s]);
    // light tree on the host for the upper-tree construction
    HostTree ht;
    CK(hcopy_in(ht.left, t->left, (size_t)c->NN, cfg.input_memory, c->stream), "read tree");
    CK(hcopy_in(ht.right, t->right, (size_t)c->NN, cfg.input_memory, c->stream), "read tree");
    CK(hcopy_in(ht.rep, t->rep, (size_t)c->NN, cfg.input_memory, c->stream), "read tree");
    CK(hcopy_in(ht.ir, t->ir, (size_t)c->NN, cfg.input_memory, c->stream), "read tree");
    CK(hcopy_in(ht.ig, t->ig, (size_t)c->NN, cfg.input_memory, c->stream), "read tree");
    CK(hcopy_in(ht.ib, t->ib, (size_t)c->NN, cfg.input_memory, c->stream), "read tree");
    CK(hcopy_in(ht.cut, t->global_cut, (size_t)c->G, cfg.input_memory, c->stream), "read tree");
    st = build_upper(c, ht);
    if (st != LMC_OK) return st;
    c->up.rs0 = c->rs0;   // random draws keyed by the global slice id
    c->up.rss = c->rss;
    const int64_t G = c->G, SL = c->SL, ML = c->ML, M = c->M;
    {
        int64_t nt = (int64_t)std::ceil((double)(c->mmax * G) * cfg.rate);
        c->ncap = std::min<int64_t>((int64_t)c->mmax * G, std::max<int64_t>(nt, 2 * c->pool_cap) + G);
        // sliced-ELL bound: padding to the longest row of a group (<= 32 max(m, G)) plus whole
        // cp.async chunks per group (<= 128 entries per group) plus the dummy slot; multiple of 8
        const int64_t mg = std::max<int64_t>(c->mmax, G);
        c->scap = (c->ncap + 32 * mg + 128 * mg + 256 + 7) & ~7ll;
        // lane-per-segment layout (complete2.cu): a member of len entries takes the next power of
        // two >= ceil(len / T) segments (< 2 len / T + 2), groups of 32 segments of <= T entries
        // padded to multiples of 8 k-steps
        // q <= 8: lane-per-segment kernel (complete2.cu; 1.6-2.6x faster than the lane-group kernel
        // on the C5 sweep).  q = 16: lane-per-segment while a slice's expected samples rate * m * |g|
        // stay <= 64k (its residuals S then mostly fit in shared memory: 1-4% faster at C2, C3 and
        // 5% rates), else the lane-group kernel of complete.cu (C4 and 20% rates: S spills to
        // global memory and the lane-per-segment kernel is 7-10% slower).
        // LMC_ADM2=1 / 0 forces the choice at q = 16, LMC_ADM_V1=1 forces complete.cu at every q.
        const char *ev = getenv("LMC_ADM_V1"), *e2 = getenv("LMC_ADM2");
        const double per_slice = cfg.rate * ((double)c->M / std::max(c->S, 1)) * (double)G;
        const bool q16_adm2 = e2 && e2[0] ? e2[0] == '1' : per_slice <= 65536.0;
        c->use_adm2 = cfg.solver == LMC_SOLVER_ADM && (cfg.rank_q <= 8 || (cfg.rank_q == 16 && q16_adm2)) &&
                      !(ev && ev[0] == '1');
        if (c->use_adm2) {
            const int64_t T = std::min(c->adm2_Tr, c->adm2_Tc), Tmax = std::max(c->adm2_Tr, c->adm2_Tc);
            c->gcap = (2 * c->ncap / T + 2 * mg + 31) / 32 + 2;
            const int64_t cap2 = 32 * ((Tmax + 7) / 8 * 8) * c->gcap + 256;
            if (cap2 >= (1ll << 19)) c->use_adm2 = false;   // S positions are 19-bit in the row entries
            else c->scap = std::max(c->scap, cap2);
        }
        c->scap = (c->scap + 255) & ~255ll;
    }
    // device arena
    Dev &d = c->d;
    CK(dalloc(&d.pixel, M), "alloc gbuffer");
    for (int k = 0; k < 13; ++k) CK(dalloc(&d.g[k], M), "alloc gbuffer");
    CK(dalloc(&d.expo, M), "alloc gbuffer");
    CK(dalloc(&d.vpl, 2 * (size_t)c->NV), "alloc vpls");
    CK(dalloc(&d.vpl_soa, 6 * (size_t)c->NV), "alloc vpls");
    CK(dalloc(&d.rows, M), "alloc slicing");
    CK(dalloc(&d.rows_alt, M), "alloc slicing");
    if (c->interleaved) {   // this rank's slice offsets and rows, gathered after the slicing of each frame
        CK(dalloc(&d.soff_loc, SL + 1), "alloc slicing");
        CK(dalloc(&d.rows_loc, std::max<int64_t>(ML, 1)), "alloc slicing");
        CK(cudaMemcpy(d.soff_loc, c->h_lrow.data(), (SL + 1) * sizeof(int32_t), cudaMemcpyHostToDevice), "upload slicing");
        c->soff_k = d.soff_loc;
        c->rows_k = d.rows_loc;
    } else {
        c->soff_k = d.slice_off;
        c->rows_k = d.rows;
    }
    CK(dalloc(&d.sk, 12 * M), "alloc slicing");
    CK(dalloc(&d.prow, 4 * (size_t)ML), "alloc rows");
    const int64_t nB = c->up.nB, U = c->up.U;
    CK(dalloc(&d.p1_rows, SL * nB * c->nmax), "alloc pass1");
    CK(dalloc(&d.p1_Ta, SL * nB * c->nmax), "alloc pass1");
    CK(dalloc(&d.p1_Tb, SL * nB * c->nmax), "alloc pass1");
    CK(dalloc(&d.p1_cnt, SL * nB), "alloc pass1");
    CK(dalloc(&d.pool_rows, SL * c->pool_cap), "alloc pool");
    CK(dalloc(&d.pool_Ta, SL * c->pool_cap), "alloc pool");
    CK(dalloc(&d.pool_Tb, SL * c->pool_cap), "alloc pool");
    CK(dalloc(&d.pool_used, SL), "alloc pool");
    CK(dalloc(&d.cs_flags, SL * U), "alloc coarsen");
    CK(dalloc(&d.cs_eps, SL * U), "alloc coarsen");
    CK(dalloc(&d.cs_cost, SL * U), "alloc coarsen");
    CK(dalloc(&d.cs_zoff, SL * U), "alloc coarsen");
    CK(dalloc(&d.cs_zlen, SL * U), "alloc coarsen");
    CK(dalloc(&d.cut_n, SL), "alloc cut");
    CK(dalloc(&d.cut_cols, SL * G), "alloc cut");
    CK(dalloc(&d.src_off, SL * G), "alloc cut");
    CK(dalloc(&d.src_len, SL * G), "alloc cut");
    CK(dalloc(&d.src_side, SL * G), "alloc cut");
    CK(dalloc(&d.rowptr, SL * (c->mmax + 1)), "alloc pass2");
    CK(dalloc(&d.col, SL * c->ncap), "alloc pass2");
    CK(dalloc(&d.val, SL * c->ncap), "alloc pass2");
    if (cfg.solver == LMC_SOLVER_MALS) {
        CK(dalloc(&d.val64, SL * c->ncap), "alloc pass2");
        CK(dalloc(&d.Xd, ML * c->q), "alloc MALS factors");
        CK(dalloc(&d.val64c, SL * c->ncap), "alloc MALS values");
        CK(dalloc(&d.Yd, SL * G * c->q), "alloc MALS factors");
    }
    CK(dalloc(&d.carried, SL * c->ncap), "alloc pass2");
    CK(dalloc(&d.colptr, SL * (G + 1)), "alloc pass2");
    CK(dalloc(&d.csc_row, SL * c->ncap), "alloc pass2");
    CK(dalloc(&d.csc_src, SL * c->ncap), "alloc pass2");
    CK(dalloc(&d.nnz, SL), "alloc pass2");
    CK(dalloc(&d.target_n, SL), "alloc pass2");
    CK(dalloc(&d.n_new, SL), "alloc pass2");
    CK(dalloc(&d.newpos, SL * c->ncap), "alloc pass2");
    // + q: the lane-group ADM kernel reads (and discards) the zero sentinel row m / column n
    CK(dalloc(&d.U, ML * c->q + c->q), "alloc factors");
    CK(dalloc(&d.Lam, ML * c->q + c->q), "alloc factors");
    CK(dalloc(&d.Xold, ML * c->q + c->q), "alloc factors");
    CK(dalloc(&d.V, SL * G * c->q + c->q), "alloc factors");
    CK(dalloc(&d.Pi, SL * G * c->q + c->q), "alloc factors");
    CK(dalloc(&d.S, SL * c->scap), "alloc factors");
    CK(dalloc(&d.r_perm, SL * c->mmax), "alloc layout");
    CK(dalloc(&d.r_len, SL * c->mmax), "alloc layout");
    CK(dalloc(&d.c_perm, SL * G), "alloc layout");
    CK(dalloc(&d.c_len, SL * G), "alloc layout");
    CK(dalloc(&d.r_goff, SL * (c->mmax + 1)), "alloc layout");
    CK(dalloc(&d.c_goff, SL * (G + 1)), "alloc layout");
    CK(dalloc(&d.c_nsolo, SL), "alloc layout");
    CK(dalloc(&d.adm_order, SL), "alloc layout");
    CK(dalloc(&d.ord_tmp, 4 * SL), "alloc layout");
    CK(launch_order_bytes((int32_t)std::max<int64_t>(SL, 1), &d.ord_cub_bytes), "cub sizing");
    CK(cudaMalloc(&d.ord_cub, std::max<size_t>(d.ord_cub_bytes, 16)), "alloc cub");
    CK(dalloc(&d.rank_pix, ML), "alloc resolve");
    if (cfg.warm_start) {
        if (cfg.warm_iters < 0) return fail(c, LMC_EINVAL, "warm_iters must be >= 0");
        CK(dalloc(&d.prev_cut, SL * G), "alloc warm start");
        CK(dalloc(&d.prev_n, SL), "alloc warm start");
        CK(dalloc(&d.prev_flags, SL), "alloc warm start");
        CK(dalloc(&d.prev_rows, ML), "alloc warm start");
        CK(dalloc(&d.warm_ok, SL), "alloc warm start");
        CK(cudaMemsetAsync(d.warm_ok, 0, sizeof(int32_t) * (size_t)std::max<int64_t>(SL, 1), c->stream), "memset");
    }
    CK(cudaMallocHost(&c->h_pix, sizeof(int32_t) * (size_t)std::max<int64_t>(ML, 1)), "alloc staging");
    CK(dalloc(&d.r_ent, SL * c->scap), "alloc layout");
    CK(dalloc(&d.c_ent, SL * c->scap), "alloc layout");
    CK(dalloc(&d.norm, SL), "alloc layout");
    if (c->use_adm2) {
        CK(dalloc(&d.r_grp, SL * c->gcap), "alloc layout");
        CK(dalloc(&d.c_grp, SL * c->gcap), "alloc layout");
        CK(dalloc(&d.r_slot, SL * c->gcap * 32), "alloc layout");
        CK(dalloc(&d.c_slot, SL * c->gcap * 32), "alloc layout");
        CK(dalloc(&d.ngrp, 2 * SL), "alloc layout");
        CK(dalloc(&d.ctot, SL), "alloc layout");
        CK(dalloc(&d.slot_st, 5 * SL * c->gcap * 32 * c->q), "alloc slot state");
    }
    CK(dalloc(&d.sbox, 6 * SL), "alloc slices");
    CK(dalloc(&d.flags, SL), "alloc factors");
    CK(dalloc(&d.iters, SL), "alloc factors");
    CK(dalloc(&d.resid, SL), "alloc factors");
    CK(dalloc(&d.direct_rgb, 3 * ML), "alloc resolve");
    CK(dalloc(&d.rows_rgb, 3 * ML), "alloc resolve");
    CK(dalloc(&d.img, 3 * (size_t)std::max<int64_t>((int64_t)c->W * c->H, 1)), "alloc resolve");
    CK(cudaMallocHost(&c->h_stage, 3 * sizeof(float) * (size_t)std::max<int64_t>((int64_t)c->W * c->H, 1)), "alloc staging");
    CK(dalloc(&d.counters, 16), "alloc counters");
    CK(cudaMemsetAsync(d.counters, 0, 16 * sizeof(unsigned long long), c->stream), "memset");
    CK(cudaMemsetAsync(d.flags, 0, SL * sizeof(int32_t), c->stream), "memset");
    CK(cudaMemsetAsync(d.img, 0, 3 * sizeof(float) * (size_t)std::max<int64_t>((int64_t)c->W * c->H, 1), c->stream), "memset");
    size_t need = cfg.solver == LMC_SOLVER_MALS ? mals_smem_bytes(c->q, c->mmax, (int)G) : adm_smem_bytes(c->q, c->mmax, (int)G);
    if (c->scap >= (1ll << 21)) return fail(c, LMC_EINVAL, "per-slice sample capacity %lld exceeds 2^21", (long long)c->scap);
    if ((double)SL * (double)c->scap >= 4294967296.0)   // the ADM kernels index the layout with 32-bit element offsets
        return fail(c, LMC_EINVAL, "%lld slices x %lld samples of layout capacity exceed 2^32", (long long)SL, (long long)c->scap);

    int maxsm = 0, dev = 0;
    CK(cudaGetDevice(&dev), "device");
    CK(cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev), "device attr");
    CK(cudaDeviceGetAttribute(&c->nsm, cudaDevAttrMultiProcessorCount, dev), "device attr");
    if (need > (size_t)maxsm)
        return fail(c, LMC_EINVAL, "rank %d with slices of %d rows and a %lld-node cut needs %zu B of shared memory (max %d)",
                    c->q, c->mmax, (long long)G, need, maxsm);
    for (auto &e : c->ev) CK(cudaEventCreate(&e), "events");
    c->ev_ok = true;
    // NCCL communicator of the image gather (world > 1 with an id from lmc_nccl_unique_id)
    bool has_id = false;
    for (int k = 0; k < 128; ++k) has_id = has_id || cfg.nccl_id[k] != 0;
    if (cfg.world > 1 && has_id) {
        ncclUniqueId id;
        static_assert(sizeof(id.internal) == 128, "ncclUniqueId is 128 bytes");
        memcpy(id.internal, cfg.nccl_id, 128);
        ncclComm_t comm = nullptr;
        ncclResult_t r = ncclCommInitRank(&comm, cfg.world, id, cfg.rank);
        if (r != ncclSuccess) {
            c->sticky = LMC_ENCCL;
            return fail(c, LMC_ENCCL, "ncclCommInitRank: %s", ncclGetErrorString(r));
        }
        c->comm = comm;
        CK(dalloc(&d.all4, (size_t)std::max<int64_t>(cfg.rank == 0 ? c->M : c->ML, 1)), "alloc gather");
    }
    return lmc_upload_inputs(c, g, v, t);
}

lmc_status lmc_create(const lmc_gbuffer *g, const lmc_vpls *v, const lmc_light_tree *t, const lmc_scene *sc,
                      const lmc_config *cfg, lmc_ctx **out)
{
    NvtxRange nvtx_("lmc_create");
    if (!cfg || !out) return LMC_EINVAL;
    lmc_ctx *c = new (std::nothrow) lmc_ctx();
    if (!c) return LMC_ENOMEM;
    memset(&c->d, 0, sizeof(c->d));
    c->cfg = *cfg;
    lmc_status st = create_impl(c, g, v, t, sc);
    if (st != LMC_OK) {
        static thread_local std::string last;
        last = c->err;
        fprintf(stderr, "lmc_create: %s: %s\n", lmc_status_str(st), c->err.c_str());
        lmc_destroy(c);
        return st;
    }
    *out = c;
    return LMC_OK;
}

lmc_status lmc_upload_inputs(lmc_ctx *c, const lmc_gbuffer *g, const lmc_vpls *v, const lmc_light_tree *t)
{
    NvtxRange nvtx_("lmc_upload_inputs");
    if (!c || !g || !v) return LMC_EINVAL;
    if (c->sticky != LMC_OK) return c->sticky;
    (void)t;
    if (g->count != c->M || v->count != c->NV) return fail(c, LMC_EINVAL, "upload: sizes differ from lmc_create");
    const int mem = c->cfg.input_memory;
    cudaStream_t st = c->stream;
    Dev &d = c->d;
    const float *src[13] = {g->px, g->py, g->pz, g->nx, g->ny, g->nz, g->vx, g->vy, g->vz, g->rho_r, g->rho_g, g->rho_b, g->spec};
    CK(dcopy_in(d.pixel, g->pixel, (size_t)c->M, mem, st), "copy gbuffer");
    for (int k = 0; k < 13; ++k) CK(dcopy_in(d.g[k], src[k], (size_t)c->M, mem, st), "copy gbuffer");
    CK(dcopy_in(d.expo, g->exponent, (size_t)c->M, mem, st), "copy gbuffer");
    // VPLs packed as (px,py,pz,nx)(ny,nz,0,0) by a kernel from a SoA staging copy
    {
        const size_t nv = (size_t)c->NV;
        const float *vs[6] = {v->px, v->py, v->pz, v->nx, v->ny, v->nz};
        for (int k = 0; k < 6; ++k) CK(dcopy_in(d.vpl_soa + k * nv, vs[k], nv, mem, st), "copy vpls");
        CK(run_pack_vpls(c), "pack vpls");
    }
    CK(run_check_pixels(c, d.counters + 8), "check pixels");
    unsigned long long bad = 0;
    CK(cudaMemcpyAsync(&bad, d.counters + 8, sizeof bad, cudaMemcpyDeviceToHost, st), "check pixels");
    CK(cudaStreamSynchronize(st), "sync");
    if (bad & 1ull) return fail(c, LMC_EINVAL, "a G-buffer pixel index is outside [0, width * height)");
    if (bad & 2ull) return fail(c, LMC_EINVAL, "a G-buffer position or normal is not finite");
    c->state = 0;
    return LMC_OK;
}

lmc_status lmc_set_timing(lmc_ctx *c, int32_t enabled)
{
    if (!c) return LMC_EINVAL;
    c->timing = enabled;
    return LMC_OK;
}

lmc_status lmc_build_slices(lmc_ctx *c)
{
    NvtxRange nvtx_("lmc_build_slices");
    lmc_status s = check_stage(c, 0);
    if (s != LMC_OK) return s;
    ev_rec(c, 0);
    CK(cudaMemsetAsync(c->d.counters, 0, 8 * sizeof(unsigned long long), c->stream), "memset counters");
    CK(run_slicing(c), "slicing");
    if (c->interleaved) CK(run_rank_rows(c), "slicing");
    CK(run_pack_rows(c), "pack rows");
    c->launches += slicing_launches(c) + (c->M > 0 ? 1 : 0) + (c->interleaved && c->ML > 0 ? 1 : 0);   // + row packing (+ rank rows)
    ev_rec(c, 1);
    c->state = 1;
    return LMC_OK;
}

lmc_status lmc_sample_pass1(lmc_ctx *c)
{
    NvtxRange nvtx_("lmc_sample_pass1");
    lmc_status s = check_stage(c, 1);
    if (s != LMC_OK) return s;
    CK(run_pass1(c), "pass 1");
    c->launches += (c->SL > 0 ? 1 : 0) + ((c->SL > 0 && c->up.nB > 0) ? 1 : 0);   // k_slice_bbox, k_pass1
    ev_rec(c, 2);
    c->state = 2;
    return LMC_OK;
}

lmc_status lmc_coarsen_cut(lmc_ctx *c)
{
    NvtxRange nvtx_("lmc_coarsen_cut");
    lmc_status s = check_stage(c, 2);
    if (s != LMC_OK) return s;
    CK(run_coarsen(c), "coarsening");
    c->launches += c->SL > 0 ? 1 : 0;
    ev_rec(c, 3);
    c->state = 3;
    return LMC_OK;
}

lmc_status lmc_sample_pass2(lmc_ctx *c)
{
    NvtxRange nvtx_("lmc_sample_pass2");
    lmc_status s = check_stage(c, 3);
    if (s != LMC_OK) return s;
    CK(run_pass2(c), "pass 2");
    c->launches += c->SL > 0 ? 2 : 0;
    ev_rec(c, 4);
    c->state = 4;
    return LMC_OK;
}

// Launch order of the completion CTAs: slice order, except that the nsm slices with the fewest
// samples run last, largest first, so the final wave holds the shortest CTAs (a slice's result
// does not depend on when its CTA runs).  Computed on the device (run_launch_order): no host sync.
// LMC_ADM_TAIL=k moves k x nsm slices (diagnostic; 0 keeps slice order).
static cudaError_t completion_order(lmc_ctx *c)
{
    const char *te = getenv("LMC_ADM_TAIL");
    const int ntail = std::min<int>((te ? atoi(te) : 1) * c->nsm, c->SL);   // SL: all slices, largest first
    c->adm_ordered = false;
    if (!(ntail > 0 && (c->SL > ntail || (te && ntail == c->SL)))) return cudaSuccess;
    cudaError_t e = run_launch_order(c, ntail);
    if (e != cudaSuccess) return e;
    c->adm_ordered = true;
    c->launches += 3;
    return cudaSuccess;
}

lmc_status lmc_complete(lmc_ctx *c)
{
    NvtxRange nvtx_("lmc_complete");
    lmc_status s = check_stage(c, 4);
    if (s != LMC_OK) return s;
    if (c->cfg.solver == LMC_SOLVER_MALS) {
        CK(completion_order(c), "completion order");
        ev_rec(c, 8);
        CK(run_mals(c), "completion (MALS)");
        ev_rec(c, 9);
    } else if (c->use_adm2) {
        if (c->cfg.warm_start) { CK(run_warm_check(c), "warm start"); c->launches += c->SL > 0 ? 1 : 0; }
        CK(run_layout2(c), "Omega layout");
        CK(completion_order(c), "completion order");
        ev_rec(c, 8);
        CK(run_adm2(c), "completion (ADM)");
        ev_rec(c, 9);
        c->launches += c->SL > 0 ? 2 : 0;
    } else {
        if (c->cfg.warm_start) { CK(run_warm_check(c), "warm start"); c->launches += c->SL > 0 ? 1 : 0; }
        CK(run_layout(c), "Omega layout");
        // shared memory of the ADM kernel is sized by the cut bound G (validated at lmc_create), so
        // nothing of this frame has to be read back: the call only enqueues
        CK(completion_order(c), "completion order");
        ev_rec(c, 8);
        CK(run_adm(c, c->G), "completion (ADM)");
        ev_rec(c, 9);
        c->launches += c->SL > 0 ? 1 : 0;
    }
    CK(run_direct(c), "direct slices");
    c->launches += c->SL > 0 ? 2 : 0;
    if (c->cfg.warm_start && c->cfg.solver == LMC_SOLVER_ADM) {
        CK(run_warm_save(c), "warm start");   // this frame's cut, rows and flags for the next frame
        c->launches += c->SL > 0 ? 1 : 0;
    }
    ev_rec(c, 5);
    c->state = 5;
    return LMC_OK;
}

// world > 1: every rank packs its rows as (r, g, b, pixel index) float4s; rank 0 receives every
// other rank's tile at that rank's row offset and scatters all of them into the image -- one
// NCCL group of P - 1 send / receive pairs, no all-gather
static lmc_status resolve_gather(lmc_ctx *c, float *image, int32_t image_memory)
{
    const int world = c->cfg.world, rank = c->cfg.rank;
    ncclComm_t comm = (ncclComm_t)c->comm;
    const size_t f4 = sizeof(float4) / sizeof(float);
    if (rank == 0) {
        if (!image) return fail(c, LMC_EINVAL, "null image on rank 0");
        if (image_memory != LMC_MEM_DEVICE && image_memory != LMC_MEM_HOST) return fail(c, LMC_EINVAL, "bad image_memory");
        CK(run_resolve(c, nullptr, nullptr, c->d.all4), "resolve");   // rank 0's rows come first
        ncclResult_t r = ncclGroupStart();
        for (int p = 1; p < world && r == ncclSuccess; ++p) {
            const int64_t r0 = c->h_part_row[p], r1 = c->h_part_row[p + 1];
            if (r1 > r0) r = ncclRecv(c->d.all4 + r0, (size_t)(f4 * (r1 - r0)), ncclFloat, p, comm, c->stream);
        }
        ncclResult_t r2 = ncclGroupEnd();
        if (r != ncclSuccess || r2 != ncclSuccess) {
            c->sticky = LMC_ENCCL;
            return fail(c, LMC_ENCCL, "image gather: %s", ncclGetErrorString(r != ncclSuccess ? r : r2));
        }
        c->launches += (c->SL > 0 ? 1 : 0) + (c->M > 0 ? 1 : 0);
        if (image_memory == LMC_MEM_DEVICE) {
            CK(run_scatter4(c, c->d.all4, c->M, image), "scatter");
            ev_rec(c, 6);
            return LMC_OK;
        }
        // host image: the packed rows come down and are scattered here (other pixels untouched)
        ev_rec(c, 6);
        std::vector<float4> h((size_t)c->M);
        CK(cudaMemcpyAsync(h.data(), c->d.all4, sizeof(float4) * (size_t)c->M, cudaMemcpyDeviceToHost, c->stream),
           "image download");
        CK(cudaStreamSynchronize(c->stream), "sync");
        const int64_t npix = (int64_t)c->W * c->H;
        for (const float4 &v : h) {
            int32_t p;
            memcpy(&p, &v.w, 4);
            if (p < 0 || p >= npix) continue;
            image[3 * (int64_t)p] = v.x;
            image[3 * (int64_t)p + 1] = v.y;
            image[3 * (int64_t)p + 2] = v.z;
        }
        return LMC_OK;
    }
    CK(run_resolve(c, nullptr, nullptr, c->d.all4), "resolve");
    c->launches += c->SL > 0 ? 1 : 0;
    ev_rec(c, 6);
    if (c->ML > 0) {
        ncclResult_t r = ncclSend(c->d.all4, (size_t)(f4 * c->ML), ncclFloat, 0, comm, c->stream);
        if (r != ncclSuccess) {
            c->sticky = LMC_ENCCL;
            return fail(c, LMC_ENCCL, "image gather: %s", ncclGetErrorString(r));
        }
    }
    if (image_memory == LMC_MEM_HOST) CK(cudaStreamSynchronize(c->stream), "sync");
    return LMC_OK;
}

lmc_status lmc_resolve_image(lmc_ctx *c, float *image, int32_t image_memory)
{
    NvtxRange nvtx_("lmc_resolve_image");
    lmc_status s = check_stage(c, 5);
    if (s != LMC_OK) return s;
    if (!image && !(c->comm && c->cfg.rank != 0)) return fail(c, LMC_EINVAL, "null image");
    if (c->comm) return resolve_gather(c, image, image_memory);
    c->launches += c->SL > 0 ? 1 : 0;
    if (image_memory == LMC_MEM_DEVICE) {
        CK(run_resolve(c, image, nullptr), "resolve");
        ev_rec(c, 6);
        return LMC_OK;
    }
    if (image_memory != LMC_MEM_HOST) return fail(c, LMC_EINVAL, "bad image_memory");
    if (c->cfg.world == 1 && c->M == (int64_t)c->W * c->H) {
        // every pixel is a row of this rank: the whole image is this rank's output
        CK(run_resolve(c, c->d.img, nullptr), "resolve");
        ev_rec(c, 6);
        const size_t bytes = 3 * sizeof(float) * (size_t)c->W * c->H;
        CK(cudaMemcpyAsync(image, c->d.img, bytes, cudaMemcpyDeviceToHost, c->stream), "image download");
        CK(cudaStreamSynchronize(c->stream), "sync");
        return LMC_OK;
    }
    // otherwise only this rank's pixels are written: packed rows + their image indices, scattered here
    CK(run_resolve(c, nullptr, c->d.rows_rgb), "resolve");
    CK(run_rank_pixels(c, c->d.rank_pix), "resolve");
    c->launches += c->ML > 0 ? 1 : 0;
    ev_rec(c, 6);
    CK(cudaMemcpyAsync(c->h_stage, c->d.rows_rgb, 3 * sizeof(float) * (size_t)c->ML, cudaMemcpyDeviceToHost, c->stream),
       "image download");
    CK(cudaMemcpyAsync(c->h_pix, c->d.rank_pix, sizeof(int32_t) * (size_t)c->ML, cudaMemcpyDeviceToHost, c->stream),
       "image download");
    CK(cudaStreamSynchronize(c->stream), "sync");
    for (int64_t k = 0; k < c->ML; ++k) {
        const int64_t p = c->h_pix[k];
        image[3 * p] = c->h_stage[3 * k];
        image[3 * p + 1] = c->h_stage[3 * k + 1];
        image[3 * p + 2] = c->h_stage[3 * k + 2];
    }
    return LMC_OK;
}

lmc_status lmc_resolve_rows(lmc_ctx *c, float *tile)
{
    NvtxRange nvtx_("lmc_resolve_rows");
    lmc_status s = check_stage(c, 5);
    if (s != LMC_OK) return s;
    if (!tile) return fail(c, LMC_EINVAL, "null tile");
    CK(run_resolve(c, nullptr, nullptr, reinterpret_cast<float4 *>(tile)), "resolve");
    c->launches += c->SL > 0 ? 1 : 0;
    ev_rec(c, 6);
    return LMC_OK;
}

lmc_status lmc_scatter_rows(lmc_ctx *c, const float *tiles, int64_t n_rows, float *image)
{
    NvtxRange nvtx_("lmc_scatter_rows");
    lmc_status s = check_stage(c, 0);
    if (s != LMC_OK) return s;
    if (n_rows < 0 || (n_rows > 0 && (!tiles || !image))) return fail(c, LMC_EINVAL, "null buffer");
    CK(run_scatter4(c, reinterpret_cast<const float4 *>(tiles), n_rows, image), "scatter");
    c->launches += n_rows > 0 ? 1 : 0;
    return LMC_OK;
}

// ---- introspection -------------------------------------------------------------------------
static lmc_status sync_check(lmc_ctx *c, int need)
{
    lmc_status s = check_stage(c, need);
    if (s != LMC_OK) return s;
    CK(cudaStreamSynchronize(c->stream), "sync");
    return check_overflow(c);
}

static lmc_status local_slice(lmc_ctx *c, int32_t slice, int *ls)
{
    if (c->interleaved) {
        if (slice < 0 || slice >= c->S || slice % c->cfg.world != c->cfg.rank)
            return fail(c, LMC_EINVAL, "slice %d is not on this rank (%d of %d, interleaved)", slice, c->cfg.rank, c->cfg.world);
        *ls = slice / c->cfg.world;
        return LMC_OK;
    }
    if (slice < c->s0 || slice >= c->s1) return fail(c, LMC_EINVAL, "slice %d is not on this rank [%d, %d)", slice, c->s0, c->s1);
    *ls = slice - c->s0;
    return LMC_OK;
}

lmc_status lmc_get_slices(lmc_ctx *c, int32_t *off, int32_t *rows, int64_t *n_slices)
{
    lmc_status s = sync_check(c, 1);
    if (s != LMC_OK) return s;
    if (n_slices) *n_slices = c->S;
    if (off) memcpy(off, c->h_slice_off.data(), c->h_slice_off.size() * 4);
    CK(d2h(rows, c->d.rows, (size_t)c->M), "get slices");
    return LMC_OK;
}

lmc_status lmc_get_pass1(lmc_ctx *c, int32_t slice, int32_t *node, int32_t *count, int32_t *rows, double *Ta, double *Tb,
                         int32_t *n_pairs, int32_t *nmax)
{
    lmc_status s = sync_check(c, 2);
    if (s != LMC_OK) return s;
    int ls;
    if ((s = local_slice(c, slice, &ls)) != LMC_OK) return s;
    const int nB = c->up.nB, nm = c->nmax;
    if (n_pairs) *n_pairs = nB;
    if (nmax) *nmax = nm;
    if (node) {
        std::vector<int32_t> bl(nB);
        CK(d2h(bl.data(), c->up.base_list, (size_t)nB), "get pass1");
        for (int k = 0; k < nB; ++k) node[k] = c->h_up_node[bl[k]];
    }
    const size_t o = (size_t)ls * nB * nm;
    CK(d2h(count, c->d.p1_cnt + (size_t)ls * nB, (size_t)nB), "get pass1");
    if (rows) {
        std::vector<uint16_t> r((size_t)nB * nm);
        CK(d2h(r.data(), c->d.p1_rows + o, r.size()), "get pass1");
        for (size_t k = 0; k < r.size(); ++k) rows[k] = r[k];
    }
    CK(d2h(Ta, c->d.p1_Ta + o, (size_t)nB * nm), "get pass1");
    CK(d2h(Tb, c->d.p1_Tb + o, (size_t)nB * nm), "get pass1");
    return LMC_OK;
}

lmc_status lmc_get_coarsen(lmc_ctx *c, int32_t slice, int32_t *node, int32_t *processed, int32_t *merged, double *eps,
                           double *cost, int32_t *n_nodes)
{
    lmc_status s = sync_check(c, 3);
    if (s != LMC_OK) return s;
    int ls;
    if ((s = local_slice(c, slice, &ls)) != LMC_OK) return s;
    const int U = c->up.U;
    if (n_nodes) *n_nodes = U;
    if (node) memcpy(node, c->h_up_node.data(), (size_t)U * 4);
    std::vector<uint8_t> fl(U);
    CK(d2h(fl.data(), c->d.cs_flags + (size_t)ls * U, (size_t)U), "get coarsen");
    for (int u = 0; u < U; ++u) {
        if (processed) processed[u] = (fl[u] & 4) ? 1 : 0;
        if (merged) merged[u] = (fl[u] & 2) ? 1 : 0;
    }
    CK(d2h(eps, c->d.cs_eps + (size_t)ls * U, (size_t)U), "get coarsen");
    CK(d2h(cost, c->d.cs_cost + (size_t)ls * U, (size_t)U), "get coarsen");
    return LMC_OK;
}

lmc_status lmc_get_cut(lmc_ctx *c, int32_t slice, int32_t *nodes, int32_t *n)
{
    lmc_status s = sync_check(c, 3);
    if (s != LMC_OK) return s;
    int ls;
    if ((s = local_slice(c, slice, &ls)) != LMC_OK) return s;
    int32_t cnt = 0;
    CK(d2h(&cnt, c->d.cut_n + ls, 1), "get cut");
    if (n) *n = cnt;
    if (nodes) {
        std::vector<int32_t> u(cnt);
        CK(d2h(u.data(), c->d.cut_cols + (size_t)ls * c->G, (size_t)cnt), "get cut");
        for (int k = 0; k < cnt; ++k) nodes[k] = c->h_up_node[u[k]];
    }
    return LMC_OK;
}

lmc_status lmc_get_samples(lmc_ctx *c, int32_t slice, int32_t *row, int32_t *col, float *val, int32_t *carried,
                           int64_t *n, int64_t *target_n)
{
    lmc_status s = sync_check(c, 4);
    if (s != LMC_OK) return s;
    int ls;
    if ((s = local_slice(c, slice, &ls)) != LMC_OK) return s;
    int32_t nnz = 0, tn = 0;
    CK(d2h(&nnz, c->d.nnz + ls, 1), "get samples");
    CK(d2h(&tn, c->d.target_n + ls, 1), "get samples");
    if (n) *n = nnz;
    if (target_n) *target_n = tn;
    const int m = c->h_slice_off[slice + 1] - c->h_slice_off[slice];
    const size_t ob = (size_t)ls * c->ncap;
    if (row) {
        std::vector<int32_t> rp(m + 1);
        CK(d2h(rp.data(), c->d.rowptr + (size_t)ls * (c->mmax + 1), (size_t)m + 1), "get samples");
        for (int i = 0; i < m; ++i)
            for (int k = rp[i]; k < rp[i + 1]; ++k) row[k] = i;
    }
    if (col) {
        std::vector<uint16_t> cc(nnz);
        CK(d2h(cc.data(), c->d.col + ob, (size_t)nnz), "get samples");
        for (int k = 0; k < nnz; ++k) col[k] = cc[k];
    }
    CK(d2h(val, c->d.val + ob, (size_t)nnz), "get samples");
    if (carried) {
        std::vector<uint8_t> cr(nnz);
        CK(d2h(cr.data(), c->d.carried + ob, (size_t)nnz), "get samples");
        for (int k = 0; k < nnz; ++k) carried[k] = cr[k];
    }
    return LMC_OK;
}

lmc_status lmc_get_factors(lmc_ctx *c, int32_t slice, float *U, float *V, int32_t *m, int32_t *n, int32_t *q,
                           int32_t *flags, int32_t *iters, float *resid)
{
    lmc_status s = sync_check(c, 5);
    if (s != LMC_OK) return s;
    int ls;
    if ((s = local_slice(c, slice, &ls)) != LMC_OK) return s;
    const int mm = c->h_slice_off[slice + 1] - c->h_slice_off[slice];
    int32_t nn = 0;
    CK(d2h(&nn, c->d.cut_n + ls, 1), "get factors");
    if (m) *m = mm;
    if (n) *n = nn;
    if (q) *q = c->q;
    CK(d2h(flags, c->d.flags + ls, 1), "get factors");
    CK(d2h(iters, c->d.iters + ls, 1), "get factors");
    CK(d2h(resid, c->d.resid + ls, 1), "get factors");
    const int64_t lrow0 = c->h_lrow[ls];
    CK(d2h(U, c->d.U + lrow0 * c->q, (size_t)mm * c->q), "get factors");
    if (V) {   // device layout: column j contiguous (n x q); returned q x n row-major
        std::vector<float> vt((size_t)nn * c->q);
        CK(d2h(vt.data(), c->d.V + (size_t)ls * c->G * c->q, vt.size()), "get factors");
        for (int j = 0; j < nn; ++j)
            for (int a = 0; a < c->q; ++a) V[(size_t)a * nn + j] = vt[(size_t)j * c->q + a];
    }
    return LMC_OK;
}

int64_t lmc_sizeof_struct(int32_t which)
{
    switch (which) {
    case 0: return (int64_t)sizeof(lmc_gbuffer);
    case 1: return (int64_t)sizeof(lmc_vpls);
    case 2: return (int64_t)sizeof(lmc_light_tree);
    case 3: return (int64_t)sizeof(lmc_scene);
    case 4: return (int64_t)sizeof(lmc_config);
    case 5: return (int64_t)sizeof(lmc_stats);
    }
    return -1;
}

lmc_status lmc_nccl_unique_id(uint8_t out[128])
{
    if (!out) return LMC_EINVAL;
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return LMC_ENCCL;
    memcpy(out, id.internal, 128);
    return LMC_OK;
}

lmc_status lmc_plan_bvh(const float *tri, int32_t n_tri, float *nodes, int32_t *n_nodes, float *tris, int32_t *order)
{
    if (n_tri < 1 || n_tri > (1 << 26) || !tri) return LMC_EINVAL;
    for (int64_t k = 0; k < 9ll * n_tri; ++k)
        if (!std::isfinite(tri[k])) return LMC_EINVAL;
    std::vector<float4> nd, tr;
    std::vector<int32_t> ord;
    build_tri_bvh(tri, n_tri, nd, tr, &ord);
    if (nodes) memcpy(nodes, nd.data(), nd.size() * sizeof(float4));
    if (n_nodes) *n_nodes = (int32_t)(nd.size() / 2);
    if (tris) memcpy(tris, tr.data(), tr.size() * sizeof(float4));
    if (order) memcpy(order, ord.data(), ord.size() * sizeof(int32_t));
    return LMC_OK;
}

lmc_status lmc_plan_partition(int64_t rows, int32_t slice_target, int32_t world, int32_t *slice_first,
                              int64_t *row_first, int64_t *n_slices)
{
    if (rows < 0 || slice_target < 1 || world < 1) return LMC_EINVAL;
    std::vector<TNode> all = slicing_tree(rows, slice_target);
    std::vector<int32_t> off = leaf_offsets(all), ps;
    std::vector<int64_t> pr;
    plan_partition(all, off, rows, world, ps, pr);
    if (slice_first) memcpy(slice_first, ps.data(), ps.size() * sizeof(int32_t));
    if (row_first) memcpy(row_first, pr.data(), pr.size() * sizeof(int64_t));
    if (n_slices) *n_slices = (int64_t)off.size() - 1;
    return LMC_OK;
}

lmc_status lmc_get_partition(lmc_ctx *c, int32_t *slice_first, int64_t *row_first)
{
    if (!c) return LMC_EINVAL;
    if (slice_first) memcpy(slice_first, c->h_part_slice.data(), c->h_part_slice.size() * sizeof(int32_t));
    if (row_first) memcpy(row_first, c->h_part_row.data(), c->h_part_row.size() * sizeof(int64_t));
    return LMC_OK;
}

lmc_status lmc_get_stats(lmc_ctx *c, lmc_stats *st)
{
    if (!c || !st) return LMC_EINVAL;
    lmc_status s = sync_check(c, 0);
    if (s != LMC_OK) return s;
    memset(st, 0, sizeof *st);
    st->n_slices = c->S;
    st->slice_begin = c->s0;
    st->slice_end = c->s1;
    st->rows = c->ML;
    st->pool_cap = c->pool_cap;
    st->launches = c->launches;
    unsigned long long cnt[5];
    CK(d2h(cnt, c->d.counters, 5), "stats");
    st->evals_pass1 = (int64_t)cnt[0];
    st->evals_coarsen = (int64_t)cnt[1];
    st->evals_pass2 = (int64_t)cnt[2];
    st->pool_used_max = (int64_t)cnt[4];
    {
        unsigned long long c67[2];
        CK(d2h(c67, c->d.counters + 6, 2), "stats");
        st->layout_row_slots = (int64_t)c67[0];
        st->layout_col_slots = (int64_t)c67[1];
    }
    if (c->state >= 3) {
        std::vector<int32_t> cn(c->SL);
        CK(d2h(cn.data(), c->d.cut_n, (size_t)c->SL), "stats");
        for (int ls = 0; ls < c->SL; ++ls) {
            int64_t m = c->h_lrow[ls + 1] - c->h_lrow[ls];
            st->sum_cols += cn[ls];
            st->sum_completed += m * cn[ls];
        }
    }
    if (c->state >= 4) {
        std::vector<int32_t> nz(c->SL);
        CK(d2h(nz.data(), c->d.nnz, (size_t)c->SL), "stats");
        for (int v : nz) st->sum_samples += v;
    }
    if (c->state >= 5 && c->cfg.warm_start && c->d.warm_ok) {
        std::vector<int32_t> wk(c->SL);
        CK(d2h(wk.data(), c->d.warm_ok, (size_t)c->SL), "stats");
        for (int v : wk) st->n_warm += v;
    }
    if (c->state >= 5) {
        std::vector<int32_t> fl(c->SL);
        CK(d2h(fl.data(), c->d.flags, (size_t)c->SL), "stats");
        for (int f : fl) {
            st->n_direct += (f & LMC_SLICE_DIRECT) ? 1 : 0;
            st->n_zero += (f & LMC_SLICE_ZERO) ? 1 : 0;
            st->n_diverged += (f & LMC_SLICE_DIVERGED) ? 1 : 0;
        }
    }
    if (c->timing && c->ev_ok && c->state >= 5) {
        float *ms[6] = {&st->ms_slices, &st->ms_pass1, &st->ms_coarsen, &st->ms_pass2, &st->ms_complete, &st->ms_resolve};
        for (int k = 0; k < 6; ++k) {
            float v = 0.f;
            if (cudaEventElapsedTime(&v, c->ev[k], c->ev[k + 1]) == cudaSuccess) *ms[k] = v;
        }
        float v = 0.f;
        if (cudaEventElapsedTime(&v, c->ev[8], c->ev[9]) == cudaSuccess) st->ms_solver = v;
        v = 0.f;
        if (cudaEventElapsedTime(&v, c->ev[10], c->ev[11]) == cudaSuccess) st->ms_eval2 = v;
        cudaGetLastError();
    }
    return LMC_OK;
}

lmc_status lmc_eval_entries(lmc_ctx *c, int64_t n, const int32_t *rows, const int32_t *vpls, double *out)
{
    NvtxRange nvtx_("lmc_eval_entries");
    if (!c || n < 0 || (n > 0 && (!rows || !vpls || !out))) return LMC_EINVAL;
    if (c->sticky != LMC_OK) return c->sticky;
    for (int64_t k = 0; k < n; ++k)
        if (rows[k] < 0 || rows[k] >= c->M || vpls[k] < 0 || vpls[k] >= c->NV) return fail(c, LMC_EINVAL, "pair %lld out of range", (long long)k);
    int32_t *dr = nullptr, *dv = nullptr;
    double *dout = nullptr;
    float4 *tmp = nullptr;
    lmc_status st = LMC_OK;
    cudaError_t e;
    if ((e = dalloc(&dr, (size_t)n)) != cudaSuccess || (e = dalloc(&dv, (size_t)n)) != cudaSuccess ||
        (e = dalloc(&dout, (size_t)n)) != cudaSuccess || (e = dalloc(&tmp, 4 * (size_t)n)) != cudaSuccess) {
        st = cuda_fail(c, e, "eval alloc");
    } else if ((e = cudaMemcpy(dr, rows, n * 4, cudaMemcpyHostToDevice)) != cudaSuccess ||
               (e = cudaMemcpy(dv, vpls, n * 4, cudaMemcpyHostToDevice)) != cudaSuccess ||
               (e = run_eval_entries(c, n, dr, dv, dout, tmp)) != cudaSuccess ||
               (e = cudaStreamSynchronize(c->stream)) != cudaSuccess ||
               (e = cudaMemcpy(out, dout, n * 8, cudaMemcpyDeviceToHost)) != cudaSuccess) {
        st = cuda_fail(c, e, "eval entries");
    }
    cudaFree(dr);
    cudaFree(dv);
    cudaFree(dout);
    cudaFree(tmp);
    return st;
}

}  // extern "C"
