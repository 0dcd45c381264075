/*
 * lmc.h — C ABI of the B200-native lighting-matrix completion library (liblmc.so).
 *
 * Hot path of arXiv 2202.12567 ("many-light rendering by sparse sampling and low-rank
 * completion"): per matrix slice, pass-1 uniform sampling + light-cut coarsening
 * (PAPER.md:96-122), pass-2 pdf sampling, nonnegative low-rank completion by
 * ADM (App. A) or masked ALS (BASELINE north_star), and the image as
 * I(s) = X (Y e).  All per-slice work runs in hand-written sm_100a CUDA kernels.
 *
 * Conventions for every call:
 *   - Return value: lmc_status; no exceptions cross the ABI; out-params are untouched on
 *     failure.  lmc_last_error(ctx) gives a message valid until the next call on ctx.
 *   - Streams: every stage call enqueues on cfg->stream (a cudaStream_t, NULL = legacy
 *     default stream) and returns without synchronising.  Getters synchronise.
 *   - Order: create -> build_slices -> sample_pass1 -> coarsen_cut -> sample_pass2 ->
 *     complete -> resolve_image.  Calling a stage before its predecessor returns
 *     LMC_ESTATE; re-running from any earlier stage is allowed (a new frame on the same
 *     inputs re-runs from build_slices).
 *   - Errors: LMC_EINVAL null pointers / sizes / invariants (rep(f) in {rep(l), rep(r)}, the
 *     global cut is an antichain cover, rate in (0,1], gamma in (0,1.618), 1 <= q <= 32,
 *     slice_target <= 1024, |global cut| <= 1024, p1_nmax <= 32, G-buffer pixel indices in
 *     [0, width*height));  LMC_ENOMEM device allocation failed;  LMC_ECUDA a CUDA error (sticky:
 *     the ctx must be destroyed);  LMC_EOVERFLOW a per-slice capacity was exceeded (reported by
 *     the next getter);  LMC_ENCCL an NCCL call failed (sticky).
 *   - Thread safety: a ctx is not thread-safe; distinct ctxs are independent.  One ctx per
 *     GPU / rank; at most 16 live contexts per process (LMC_EINVAL beyond).
 */
#ifndef LMC_H
#define LMC_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    LMC_OK = 0,
    LMC_EINVAL = 1,
    LMC_ESTATE = 2,
    LMC_ENOMEM = 3,
    LMC_ECUDA = 4,
    LMC_EOVERFLOW = 5,
    LMC_ENCCL = 6
} lmc_status;

typedef enum { LMC_SOLVER_ADM = 0, LMC_SOLVER_MALS = 1 } lmc_solver;
typedef enum { LMC_MEM_DEVICE = 0, LMC_MEM_HOST = 1 } lmc_memory;
typedef enum { LMC_SLICE_DIRECT = 1, LMC_SLICE_DIVERGED = 2, LMC_SLICE_ZERO = 4 } lmc_slice_flags;

/* G-buffer: one row per valid (hit) pixel = one surface point = one matrix row.
 * SoA float32 arrays of length count; pixel[r] = image index (y*width + x) of row r;
 * (vx,vy,vz) = unit direction from the point to the camera; rho = diffuse/glossy albedo;
 * spec in [0,1] = glossy weight s; exponent = Phong exponent e (>= 0).
 * Memory: device or host per lmc_config.input_memory; read only during lmc_create. */
typedef struct {
    int32_t width, height;
    int64_t count;
    const int32_t *pixel;
    const float *px, *py, *pz, *nx, *ny, *nz, *vx, *vy, *vz, *rho_r, *rho_g, *rho_b, *spec;
    const int32_t *exponent;
} lmc_gbuffer;

/* VPLs: position, unit normal, RGB intensity I_j; SoA float32, length count. */
typedef struct {
    int64_t count;
    const float *px, *py, *pz, *nx, *ny, *nz, *ir, *ig, *ib;
} lmc_vpls;

/* Light tree: binary; left/right = -1 for leaves; rep[f] = representative
 * VPL id (leaves: their VPL; internal: rep of one child); I_f = (ir, ig, ib)[f].
 * global_cut: node ids of the conservative global cut g, an antichain covering every
 * leaf.  int32/float32 arrays; memory per lmc_config.input_memory. */
typedef struct {
    int64_t num_nodes;
    int32_t root;
    const int32_t *left, *right, *rep;
    const float *ir, *ig, *ib;
    int64_t cut_size;
    const int32_t *global_cut;
} lmc_light_tree;

/* Analytic occluders for the shadow-ray visibility test (BASELINE north_star "procedural
 * analytic scene").  HOST pointers, float32: sph[4*k] = (cx,cy,cz,r); box[6*k] = (lo3, hi3);
 * rect[12*k] = (p0, e1, e2, nrm = e1 x e2).  At most 32 of each.  clamp_dist = d_c of the
 * d^2 clamp (DESIGN R2); shadow_eps = segment shrink at both ends (R3); diag = scene
 * diagonal D used by the slicing keys (R26), in [1e-30, 1e30] (R43: the slicing orders 32-bit
 * encodings of the coordinates, exact in that range; LMC_EINVAL outside). */
typedef struct {
    int32_t n_sph, n_box, n_rect;
    const float *sph, *box, *rect;
    double clamp_dist, shadow_eps, diag;
    /* SURVEY §8(f1) triangle meshes: tri[9*k] = (v0, v1, v2), HOST float32, 0 <= n_tri <= 2^26.
     * lmc_create builds a BVH over them on the host (median split, <= 4 triangles per leaf) and
     * keeps nodes + triangles in device memory for the context's lifetime; traversal uses fp32
     * node boxes widened by 1e-3 D and the exact fp64 Moller-Trumbore test of DESIGN.md R39 at
     * the leaves, so each visibility decision equals the brute-force test over all triangles. */
    int32_t n_tri;
    const float *tri;
} lmc_scene;

typedef struct {
    int32_t slice_target;   /* max rows per slice ("about 800 pixels"), <= 1024 */
    double normal_weight;   /* w_n of the 6D slicing key (R26): 0 or in [1e-30, 1e30] (R43), else LMC_EINVAL */
    uint64_t seed;          /* Philox key for every random draw (R7) */
    int32_t p1_nmax, p1_nmin; /* pass-1 rows per pair: min(m, max(nmin, ceil(nmax lum I_f / l_max))) (R6) */
    double coarsen_tau;     /* coarsening bound: merge iff cost(L_f) < tau (R11) */
    double rate;            /* sampling rate of the coarsened slice matrix (R27) */
    int32_t rank_q;         /* q */
    int32_t solver;         /* lmc_solver */
    int32_t max_iter;       /* K (100) */
    double tol;             /* stop when ||P_Omega(M - XY)|| / ||P_Omega M|| < tol (0 = run K) */
    double alpha, beta, gamma; /* ADM penalties / step (R19) */
    double lambda;          /* MALS ridge */
    int32_t rank, world;    /* this process' share of the slices (lmc_get_partition): for world = 2^k the
                               rank-th subtree of depth k of the slicing (levels >= k are sliced by
                               that rank only), otherwise slices [S*rank/world, S*(rank+1)/world);
                               with partition = 1 (below) slices rank, rank + world, ...  Per-slice getters
                               take the global slice id */
    int32_t input_memory;   /* lmc_memory of the gbuffer / vpls / tree arrays */
    void *stream;           /* cudaStream_t */
    uint8_t nccl_id[128];   /* world > 1: the ncclUniqueId from lmc_nccl_unique_id() on rank 0, broadcast
                               to every rank by the caller; all zero = no NCCL communicator (then the
                               image is assembled with lmc_resolve_rows / lmc_scatter_rows) */
    /* SURVEY §8(f3) variants, 0 = the paper's method:
     *   row_importance 1: pass-2 rows drawn by f(i) = max - min of the row's carried observations
     *                     (integer weights as for g(j); P:145 sets f = 1; DESIGN R36)
     *   cost_mode 1:      Eq. (1) sensitivity, cost(L_f) = (eps(L_f) + cost(L_b)) + cost(L_a)
     *   resolve_mode 1:   Z-mode image, tint (<U_i, V w^k> + sum_{j in Omega_i} (M~_ij - <U_i, V_j>) w^k_j) */
    int32_t row_importance, cost_mode, resolve_mode;
    /* SURVEY §8(f4) temporal coherence: warm_start 1 starts the ADM of every slice whose rows and
     * cut equal the previous frame's (and whose previous result was regular) from the previous
     * frame's factors (U, V / sigma; multipliers 0) for warm_iters iterations (0: max_iter) */
    int32_t warm_start, warm_iters;
    /* SURVEY §8(f2) count-target coarsening (DESIGN R37): > 0 merges, per slice, the least-cost
     * pair of sibling cut nodes (ties: smallest node id) until the cut has coarsen_target nodes
     * (coarsen_tau unused); 0 = the threshold rule */
    int32_t coarsen_target;
    /* world > 1, how the slices are shared: 0 = slicing subtrees for P = 2^k ranks
     * (each rank slices the top k levels of the whole G-buffer, then its own subtree), contiguous
     * slice ranges otherwise; 1 = interleaved: every rank slices the whole G-buffer and takes
     * slices r, r + P, r + 2P, ... (neighbouring slices cost alike, so the ranks' loads balance;
     * random draws stay keyed by the global slice id, so the image is the same either way) */
    int32_t partition;
} lmc_config;

typedef struct {
    int64_t n_slices;          /* S, whole frame */
    int64_t slice_begin, slice_end; /* this rank's slices */
    int64_t rows;              /* rows of this rank's slices */
    int64_t sum_cols;          /* sum_s n_s (coarsened columns) */
    int64_t sum_samples;       /* sum_s |Omega_s| */
    int64_t sum_completed;     /* sum_s m_s * n_s: entries of the completed matrices */
    int64_t evals_pass1, evals_coarsen, evals_pass2; /* entry evaluations (shadow rays) */
    int64_t n_direct, n_zero, n_diverged;
    int64_t pool_used_max, pool_cap; /* coarsening sample pool per slice (entries) */
    int64_t launches;          /* kernel launches issued by the stage calls since lmc_create */
    float ms_slices, ms_pass1, ms_coarsen, ms_pass2, ms_complete, ms_resolve; /* last frame, if timed */
    float ms_solver;           /* last frame, if timed: the completion kernel alone (ADM or MALS) */
    int64_t layout_row_slots, layout_col_slots; /* q <= 16 ADM: padded sample slots of the row / column layouts */
    float ms_eval2;            /* last frame, if timed: the pass-2 entry-evaluation kernel alone */
    int64_t n_warm;            /* slices of the last frame whose completion started warm (warm_start) */
} lmc_stats;

typedef struct lmc_ctx lmc_ctx;

/* Creates a context on the current CUDA device: validates and copies all inputs into a
 * ctx-owned device arena (host->device when input_memory == LMC_MEM_HOST), builds the
 * upper light tree (global cut + ancestors) and allocates every per-frame buffer, so the
 * stage calls never allocate.  Synchronises cfg->stream before returning. */
lmc_status lmc_create(const lmc_gbuffer *g, const lmc_vpls *v, const lmc_light_tree *t, const lmc_scene *sc,
                      const lmc_config *cfg, lmc_ctx **out);

/* Re-upload the per-frame inputs (G-buffer, VPLs) of an existing context: same counts and
 * memory kind as at lmc_create; the light tree and global cut are those given at creation.
 * Synchronises cfg->stream.  Resets the stage state to "created".  LMC_EINVAL when a pixel index
 * lies outside [0, width * height) or a G-buffer position / normal is not finite (R43); the same
 * checks run inside lmc_create. */
lmc_status lmc_upload_inputs(lmc_ctx *ctx, const lmc_gbuffer *g, const lmc_vpls *v, const lmc_light_tree *t);

/* Matrix slicing: recursive binary split of the rows as 6D points
 * (x/D, w_n n) on the dimension of largest extent at the lower median of (key, row), the
 * left child taking ceil(n/2), until <= slice_target rows; slice ids in left-first DFS order,
 * rows ascending within a slice. */
lmc_status lmc_build_slices(lmc_ctx *ctx);

/* Pass 1: for every slice of this rank and every base pair f (both children in g),
 * n_f distinct rows drawn uniformly (Floyd + Philox keyed by (f, slice)) and the entries
 * T(i, rep a), T(i, rep b) evaluated in fp64 (decision precision, DESIGN R30). */
lmc_status lmc_sample_pass1(lmc_ctx *ctx);

/* Light coarsening (Eq. (1)): per slice, bottom-up merge of sibling cut nodes
 * while cost(L_f) = eps(L_f) + cost(L_b) < tau, reusing sample sets by union. */
lmc_status lmc_coarsen_cut(lmc_ctx *ctx);

/* Pass 2: carried observations, light importance g(j) = max C_j - min C_j,
 * integer pdf weights and CDF, column-then-row draws skipping observed entries until
 * ceil(rate m n) entries, one forced entry per empty column; CSR + CSC of Omega. */
lmc_status lmc_sample_pass2(lmc_ctx *ctx);

/* Completion (App. A): per slice M ~= U V with U, V >= 0 (ADM) or masked ALS;
 * slices with min(m, n) <= q, or a non-finite residual, are rendered directly (flagged). */
lmc_status lmc_complete(lmc_ctx *ctx);

/* Image: per slice out^k = tint^k * U (V w^k), written into image_rgb
 * (float32, height*width*3, row-major pixels, RGB interleaved) at the G-buffer's pixels only;
 * other pixels are untouched.  image_memory: LMC_MEM_DEVICE (enqueued, no synchronisation) or
 * LMC_MEM_HOST (the call synchronises).
 * world = 1: this rank's pixels.  world > 1 (needs the NCCL communicator of lmc_config.nccl_id):
 * every rank packs its rows, rank 0 receives the other ranks' tiles with ncclRecv (the others
 * ncclSend theirs; one NCCL group) and writes every pixel of the frame; image_rgb is ignored on
 * ranks != 0 (may be NULL there).  world > 1 without a communicator: this rank's pixels only. */
lmc_status lmc_resolve_image(lmc_ctx *ctx, float *image_rgb, int32_t image_memory);

/* Step 1 on the GPU (DESIGN R38): the light tree of v and its conservative
 * global cut.  Tree: median split on the axis of the largest bounding-box extent, (coordinate, VPL
 * index) order, left child ceil(n/2), breadth-first node ids; I_f = I_l + I_r (fp64, returned as
 * float32), rep(f) = rep of the brighter child (ties: left).  Cut: the internal nodes of largest
 * bound lum(I_f) |bbox diagonal| (ties: smaller id) split until the cut has cut_max nodes
 * (fewer if the tree has fewer leaves).  Inputs v and the outputs (2 count - 1 node arrays, a cut
 * array of cut_max ids in ascending order, any output may be NULL) are device or host memory per
 * `memory`; runs on `stream` (cudaStream_t) and synchronises it; *cut_size = |cut|.
 * LMC_EINVAL bad sizes / null inputs, LMC_ENOMEM, LMC_ECUDA. */
lmc_status lmc_build_light_tree(const lmc_vpls *v, int32_t cut_max, int32_t memory, void *stream, int32_t *left,
                                int32_t *right, int32_t *rep, float *ir, float *ig, float *ib, int32_t *global_cut,
                                int64_t *cut_size);

/* sizeof of the ABI structs (0 gbuffer, 1 vpls, 2 light tree, 3 scene, 4 config, 5 stats; -1 otherwise):
 * lets a binding check its struct layouts against the library */
int64_t lmc_sizeof_struct(int32_t which);

/* ncclGetUniqueId for lmc_config.nccl_id (call on rank 0 only; LMC_ENCCL on failure) */
lmc_status lmc_nccl_unique_id(uint8_t out[128]);

/* The ranks' shares: slice_first[r] / row_first[r] = first slice / first slice-ordered row of rank r
 * (world + 1 entries each, last = S / M).  Host buffers; either may be NULL. */
lmc_status lmc_get_partition(lmc_ctx *ctx, int32_t *slice_first, int64_t *row_first);
/* The triangle BVH lmc_create builds for lmc_scene.tri (host only, no GPU): nodes[8 k ..]
 * = (lo3, first, hi3, count) with first / count int32 bit patterns (count 0: internal node whose
 * children are nodes first and first + 1; else a leaf of count <= 4 triangles starting at
 * triangle `first` of the reordered list), tris[12 k ..] = (v0, v1, v2, 0, 0, 0) in leaf order, order[k]
 * = the input index of reordered triangle k.  Capacities: nodes 8 (2 n_tri - 1) floats, tris 12 n_tri
 * floats, order n_tri; *n_nodes = nodes written.  Any output may be NULL.  LMC_EINVAL on bad sizes
 * or non-finite vertices. */
lmc_status lmc_plan_bvh(const float *tri, int32_t n_tri, float *nodes, int32_t *n_nodes, float *tris, int32_t *order);

/* The same shares without a context or a GPU (host planning only, e.g. for tests): for `rows`
 * G-buffer rows and slice_target, world + 1 entries each and the frame's slice count. */
lmc_status lmc_plan_partition(int64_t rows, int32_t slice_target, int32_t world, int32_t *slice_first,
                              int64_t *row_first, int64_t *n_slices);

/* This rank's pixels as a packed tile for a cross-rank gather done by the caller (e.g. with
 * torch.distributed): tile = rows x 4 float32 (r, g, b, image pixel index as int32 bits) in this
 * rank's slice-row order (device buffer, lmc_get_stats().rows rows).  lmc_scatter_rows() writes n
 * such packed rows (any order, e.g. every rank's tile concatenated) into a device image.  Both
 * only enqueue. */
lmc_status lmc_resolve_rows(lmc_ctx *ctx, float *tile);
lmc_status lmc_scatter_rows(lmc_ctx *ctx, const float *tiles, int64_t n_rows, float *image_rgb);

void lmc_destroy(lmc_ctx *ctx);
const char *lmc_last_error(const lmc_ctx *ctx);
const char *lmc_status_str(lmc_status s);

/* ---- introspection (synchronous; HOST buffers; NULL buffers -> sizes only) ------------------ */
lmc_status lmc_get_slices(lmc_ctx *ctx, int32_t *off /* S+1 */, int32_t *rows /* count */, int64_t *n_slices);
/* pass-1 record of a slice: for base pair k (ascending node id): node[k], count[k], rows
 * (nmax per pair, local rows), Ta/Tb (fp64 T values, nmax per pair). */
lmc_status lmc_get_pass1(lmc_ctx *ctx, int32_t slice, int32_t *node, int32_t *count, int32_t *rows, double *Ta,
                         double *Tb, int32_t *n_pairs, int32_t *nmax);
/* per upper-tree node (ascending node id) of a slice: processed / merged flags, eps, cost */
lmc_status lmc_get_coarsen(lmc_ctx *ctx, int32_t slice, int32_t *node, int32_t *processed, int32_t *merged,
                           double *eps, double *cost, int32_t *n_nodes);
lmc_status lmc_get_cut(lmc_ctx *ctx, int32_t slice, int32_t *nodes, int32_t *n);
/* Omega of a slice in CSR order: local row, column, value M~ (float32 of the fp64 entry),
 * carried flag (1 = observed during pass 1 / coarsening) */
lmc_status lmc_get_samples(lmc_ctx *ctx, int32_t slice, int32_t *row, int32_t *col, float *val, int32_t *carried,
                           int64_t *n, int64_t *target_n);
/* factors of a slice: U (m*q row-major), V (q*n row-major, already times sigma) */
lmc_status lmc_get_factors(lmc_ctx *ctx, int32_t slice, float *U, float *V, int32_t *m, int32_t *n, int32_t *q,
                           int32_t *flags, int32_t *iters, float *resid);
lmc_status lmc_get_stats(lmc_ctx *ctx, lmc_stats *st);
/* enable CUDA-event stage timing (stats.ms_*); adds event records on the stream */
lmc_status lmc_set_timing(lmc_ctx *ctx, int32_t enabled);

/* Test hook: evaluate T(row, vpl) with the fp64 decision-precision entry kernel for n
 * arbitrary pairs (host arrays in, host array out).  Same device code as the stages. */
lmc_status lmc_eval_entries(lmc_ctx *ctx, int64_t n, const int32_t *rows, const int32_t *vpls, double *out);

#ifdef __cplusplus
}
#endif
#endif
