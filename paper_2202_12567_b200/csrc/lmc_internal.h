// lmc_internal.h — device views and launcher declarations shared by the liblmc translation units.
// (Internal to the CUDA path; the oracle never sees this file.)
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "lmc.h"

namespace lmc {

constexpr int TAG_P1 = 1, TAG_P2 = 2, TAG_FORCE = 3, TAG_X0 = 4, TAG_Y0 = 5;
constexpr int MAX_PRIMS = 32;
constexpr int SCENE_SLOTS = 16;   // live contexts per process (one __constant__ scene each)
constexpr int MAX_Q = 32;
constexpr int MAX_SLICE = 1024;   // rows per slice (bitmap words per row set = 32)
constexpr int MAX_CUT = 1024;     // |global cut| (columns per slice)
constexpr int MAX_NMAX = 32;      // pass-1 rows per pair (one warp)

// Analytic occluders + entry constants (host-filled, uploaded to __constant__ of the exact TU)
struct SceneConst {
    int32_t nsph, nbox, nrect, pad;
    double dc2;        // clamp_dist * clamp_dist
    double eps;        // shadow_eps
    float margin;      // conservative screening margin (1e-3 D) of the fp32 visibility pre-tests
    float pad3[3];
    // triangle meshes: BVH nodes, 2 float4 each: (lo3, first child | first triangle),
    // (hi3, triangle count; 0 = internal node, children at first, first + 1); triangles 3 float4
    // each: (v0, v1.x) (v1.yz, v2.xy) (v2.z, 0, 0, 0), in leaf order
    const float4 *bvh;
    const float4 *tri4;
    int32_t ntri, nbvh, pad5[2];
    float sph[MAX_PRIMS * 4];
    float box[MAX_PRIMS * 6];
    float rect[MAX_PRIMS * 12];
    float rbox[MAX_PRIMS * 6];   // bounding boxes of the rectangles (lo3, hi3)
    float rnorm[MAX_PRIMS];      // |e1 x e2| (scale of the plane-side screen)
};
static_assert(sizeof(SceneConst) % 16 == 0, "SceneConst is copied as int4 words");

// Upper light tree: the global cut g and all its ancestors, local ids in ascending node id.
struct Upper {
    int32_t U;                // nodes
    int32_t H;                // max height (g nodes have height 0)
    int32_t nB;               // base pairs (both children in g)
    const int32_t *node;      // global node id
    const int32_t *left, *right, *parent;   // local ids, -1 if none
    const int32_t *rep;       // representative VPL
    const int32_t *nunc;      // max(nmin, ceil(nmax lum / l_max)) (unclamped by m)
    const int32_t *hlist;     // internal nodes ordered by (height, id)
    const int32_t *hoff;      // H+2 offsets into hlist by height (height 1..H)
    const int32_t *base_list; // local ids of base pairs (ascending)
    const int32_t *base_of;   // local id -> base index or -1
    const double *lum;        // lum(I_f), fp64 from the float32 intensities
    const float *I;           // 3 per node
    int32_t rs0, rss;         // global id of this rank's local slice ls: rs0 + ls * rss (random-draw key)
};

// Per-frame device state (all allocated in lmc_create)
struct Dev {
    // inputs
    int32_t *pixel;
    float *g[13];             // px py pz nx ny nz vx vy vz rho_r rho_g rho_b spec
    int32_t *expo;
    float4 *vpl;              // 2 per VPL: (px,py,pz,nx) (ny,nz,0,0)
    float4 *bvh, *tri4;       // triangle BVH + triangles (SceneConst.bvh / tri4)
    // upper tree arrays (backing store of Upper)
    int32_t *ut_i32;
    double *ut_lum;
    float *ut_I;
    // slicing
    int32_t *rows, *rows_alt;          // M each: slicing order, ping-pong
    uint32_t *sk;                      // 2 x 6 M: order-preserving 32-bit keys of the 6 dimensions (SoA, ping-pong)
    int32_t *lvl_begin, *lvl_end;      // concatenated level tilings
    int32_t *lvl_slot;                 // per tile: slot of a splitting tile, -1 otherwise
    int32_t *lvl_work;                 // chunked levels: work items (tile, start, len, first item of the tile)
    uint32_t *sl_ext;                  // [slots][12] encoded per-dimension maxima / minima
    uint32_t *sl_hist;                 // [slots][4][256] radix-select histograms
    uint32_t *sl_cnt;                  // [2 x work items] rows below / equal to the threshold per chunk
    uint32_t *sl_state;                // [slots][4] threshold key, rows of it going left, dimension, ceil(n/2)
    int32_t *slice_off;                // S+1
    int32_t *soff_loc, *rows_loc;      // interleaved partition: this rank's slice offsets (SL+1) and rows (ML)
    float4 *prow;                      // 4 per local row (slice order)
    float *sbox;                       // [SL][6] bounding box (lo3, hi3) of each slice's points (fp32, exact)
    // pass 1: [SL][nB][nmax]
    uint16_t *p1_rows;
    double *p1_Ta, *p1_Tb;
    int32_t *p1_cnt;                   // [SL][nB]
    // coarsening
    uint16_t *pool_rows;               // [SL][pool_cap]
    double *pool_Ta, *pool_Tb;
    int32_t *pool_used;                // [SL]
    uint8_t *cs_flags;                 // [SL][U]  bit0 in_cut, bit1 merged, bit2 processed
    double *cs_eps, *cs_cost;          // [SL][U]
    int32_t *cs_zoff, *cs_zlen;        // [SL][U]
    int32_t *cut_n;                    // [SL]
    int32_t *cut_cols;                 // [SL][G] local upper ids
    int32_t *src_off, *src_len, *src_side; // [SL][G] carried-observation source per column
    // pass 2: per slice capacity ncap
    int32_t *rowptr;                   // [SL][mmax+1]
    uint16_t *col;                     // [SL][ncap]
    float *val;                        // [SL][ncap]
    double *val64;                     // [SL][ncap] (MALS only)
    double *Xd, *Yd;                   // MALS fp64 factors [ML][q], [SL][G][q] (MALS only)
    double *val64c;                    // [SL][ncap] values in CSC order (MALS only)
    uint8_t *carried;                  // [SL][ncap]
    int32_t *colptr;                   // [SL][G+1]
    uint16_t *csc_row;                 // [SL][ncap]
    int32_t *csc_src;                  // [SL][ncap]
    int32_t *nnz, *target_n, *n_new;   // [SL]
    int32_t *newpos;                   // [SL][ncap] scratch: the completion layouts' CSR index -> S position map
    // completion
    // sliced-ELL layout of Omega for the completion (k_layout)
    uint16_t *r_perm, *r_len;          // [SL][mmax] rows by (length desc, id)
    uint16_t *c_perm, *c_len;          // [SL][G]
    int32_t *r_goff, *c_goff;          // [SL][mmax+1], [SL][G+1]
    int32_t *c_nsolo;                  // [SL] leading column groups that hold a single (long) column
    int32_t *adm_order;                // [SL] completion CTA -> slice (the smallest slices last)
    int32_t *ord_tmp;                  // [4 SL] launch-order scratch (sorted keys, iota, sorted ids, marks)
    void *ord_cub;                     // CUB radix-sort temp of the launch order
    size_t ord_cub_bytes;
    int32_t *rank_pix;                 // [ML] image index of this rank's rows (host-buffer resolve)
    // warm start: the previous frame's cut, rows and flags of this rank's slices
    int32_t *prev_cut, *prev_n, *prev_flags, *prev_rows, *warm_ok;   // [SL][G], [SL], [SL], [ML], [SL]
    float4 *all4;                      // world > 1 with NCCL: [ML] this rank's packed (r, g, b, pixel) rows;
                                       // rank 0: [M], every rank's tile at its row offset
    unsigned long long *r_ent;         // [SL][scap] (M^ bits << 32) | (column-layout index << 10) | column
    uint16_t *c_ent;                   // [SL][scap] row of the column-layout entry
    float4 *norm;                      // [SL] sigma, 1/sigma, sum M^, sum M^^2
    // lane-per-segment layout of the q <= 16 ADM kernel (complete2.cu)
    int4 *r_grp, *c_grp;               // [SL][gcap] (entry offset, k-steps, max log2 segments, 0)
    uint32_t *r_slot, *c_slot;         // [SL][gcap * 32] member | segment << 11 | log2 segments << 16
    int32_t *ngrp;                     // [SL][2] row groups, column groups
    int32_t *ctot;                     // [SL] column-layout size
    float *slot_st;                    // 5 x [SL][gcap * 32 * q]: U, Lambda, X_k, V, Pi by lane slot
    float *U, *V, *Lam, *Pi, *Xold, *S; // U/Lam/Xold [ML][q], V/Pi [SL][G][q], S [SL][scap]
    int32_t *flags, *iters;            // [SL]
    float *resid;                      // [SL]
    float *direct_rgb;                 // [ML][3]
    float *rows_rgb;                   // [ML][3]
    float *img;                        // [H*W][3] staging image for host output
    float *vpl_soa;                    // 6 * NV staging for the VPL packing kernel
    // counters: 0 evals_pass1, 1 evals_coarsen, 2 evals_pass2, 3 overflow flags, 4 pool_used_max, 5 max n_s,
    // 6 / 7 padded row / column layout sizes of the q <= 16 ADM
    unsigned long long *counters;
};

}  // namespace lmc

struct lmc_ctx {
    lmc_config cfg;
    cudaStream_t stream = nullptr;
    int state = 0;                 // 0 created, 1 sliced, 2 pass1, 3 coarsened, 4 pass2, 5 completed
    lmc_status sticky = LMC_OK;
    std::string err;
    // sizes
    int64_t M = 0;                 // valid rows
    int32_t W = 0, H = 0;
    int64_t NV = 0, NN = 0;
    double diag = 1.0;
    int32_t G = 0;                 // |global cut|
    int32_t S = 0;                 // slices (whole frame)
    std::vector<int32_t> h_slice_off;
    int32_t s0 = 0, s1 = 0, SL = 0;
    int64_t row0 = 0, ML = 0;
    // what the stage kernels index: the whole frame's slice offsets / rows from s0, row0
    // (contiguous shares), or this rank's gathered copy from 0 (interleaved); random draws use the
    // global slice id rs0 + ls * rss
    bool interleaved = false;
    const int32_t *soff_k = nullptr;
    int32_t *rows_k = nullptr;
    int32_t s0k = 0, lbase_k = 0, rs0 = 0, rss = 1;
    int64_t row0_k = 0;
    std::vector<int32_t> h_lrow;       // local row offset of each of this rank's slices (SL + 1), both modes
    int32_t mmax = 0;
    int32_t q = 0, nmax = 0;
    int64_t pool_cap = 0, ncap = 0, scap = 0;
    int64_t gcap = 0;              // groups per slice and phase of the q <= 16 ADM layout
    int32_t adm2_Tr = 64, adm2_Tc = 64;   // segment length caps (rows, columns)
    bool use_adm2 = false;         // complete2.cu kernels (q <= 16) instead of complete.cu
    // slicing level structure
    // rows [lo, lo + n); tiles relative to lo; fused: one CTA per tile (slice.cu)
    struct Level { int64_t lo, n; int32_t tile_off, tile_n, work_off, work_n, nslots; bool fused; };
    int32_t sub_k = -1;            // P = 2^k ranks: slicing levels >= k run in this rank's subtree only
    std::vector<int32_t> h_part_slice;   // [world + 1] first slice of every rank
    std::vector<int64_t> h_part_row;     // [world + 1] first row of every rank
    std::vector<Level> levels;
    int32_t max_tiles = 0;
    // scene + upper tree
    lmc::SceneConst scene;
    int scene_slot = -1;           // index into the __constant__ scene table
    lmc::Upper up;
    std::vector<int32_t> h_up_node;   // for getters
    int nsm = 0;                      // SMs of the device
    bool adm_ordered = false;         // d.adm_order holds this frame's completion launch order
    std::vector<int32_t> h_nnz, h_order;   // completion launch order (lmc_complete)
    lmc::Dev d;
    // timing
    int timing = 0;
    cudaEvent_t ev[12];   // [0, 7) stage boundaries, [8, 10) around the completion kernel, [10, 12) the pass-2 entry kernel
    float ms[6] = {0, 0, 0, 0, 0, 0};
    bool ev_ok = false;
    float *h_stage = nullptr;
    int32_t *h_pix = nullptr;      // pinned [ML] pixel ids of the host-buffer resolve
    int64_t launches = 0;          // kernels (and CUB dispatches, 1 each) issued by stage calls
    void *comm = nullptr;          // ncclComm_t of the image gather (world > 1 with an NCCL id)
    bool have_prev = false;        // warm start: a previous frame's completion exists
};

namespace lmc {
// exact.cu (fp64 decision precision, compiled with -fmad=false)
cudaError_t run_slicing(lmc_ctx *c);
cudaError_t run_pack_rows(lmc_ctx *c);
cudaError_t run_pass1(lmc_ctx *c);
cudaError_t run_coarsen(lmc_ctx *c);
cudaError_t run_pass2(lmc_ctx *c);
cudaError_t run_direct(lmc_ctx *c);
cudaError_t run_eval_entries(lmc_ctx *c, int64_t n, const int32_t *d_rows, const int32_t *d_vpls, double *d_out,
                             float4 *d_tmp_rows);
int64_t slicing_launches(const lmc_ctx *c);
cudaError_t run_rank_rows(lmc_ctx *c);   // interleaved partition: this rank's rows into rows_loc
cudaError_t run_pack_vpls(lmc_ctx *c);
int acquire_scene_slot();
void release_scene_slot(int slot);
cudaError_t upload_scene(int slot, const SceneConst &sc);
// complete.cu (fp32 completion + resolve)
cudaError_t run_layout(lmc_ctx *c);
cudaError_t run_adm(lmc_ctx *c, int nmax);
cudaError_t run_resolve(lmc_ctx *c, float *image, float *rows_rgb, float4 *tile4 = nullptr);
cudaError_t run_scatter4(lmc_ctx *c, const float4 *all4, int64_t n, float *image);
cudaError_t run_scatter(lmc_ctx *c, const float *all_rows, float *image);
cudaError_t run_rank_pixels(lmc_ctx *c, int32_t *out);
cudaError_t run_check_pixels(lmc_ctx *c, unsigned long long *flag);
cudaError_t launch_order_bytes(int32_t SL, size_t *bytes);
cudaError_t run_launch_order(lmc_ctx *c, int ntail);
cudaError_t run_warm_check(lmc_ctx *c);
cudaError_t run_warm_save(lmc_ctx *c);
size_t adm_smem_bytes(int q, int mmax, int nmax);
// complete2.cu (lane-per-segment ADM, q <= 16)
cudaError_t run_layout2(lmc_ctx *c);
cudaError_t run_adm2(lmc_ctx *c);
// mals.cu (fp64 masked ALS)
cudaError_t run_mals(lmc_ctx *c);
size_t mals_smem_bytes(int q, int mmax, int G);
}  // namespace lmc
