/*
 * oracle.h — plain, slow, fp64 CPU oracle of the hot path of arXiv 2202.12567
 * ("many-light rendering by sparse sampling and low-rank completion of the lighting matrix").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it.  It shares no code, header, table or
 * helper with the CUDA path (paper_2202_12567_b200/), and neither includes the other.
 *
 * Every function follows a passage of /root/reference/PAPER.md ("P:<line>") read as in
 * DESIGN.md §"Readings"; where the paper is silent the reading number (R<k>) is cited.
 * Arithmetic: IEEE binary64, round-to-nearest, compiled with -ffp-contract=off (no FMA),
 * products/sums in the written order.
 */
#ifndef LMC_ORACLE_H
#define LMC_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* one slice of the previous frame (warm start) */
typedef struct {
    int32_t slice, m, n, flags;
    const int32_t *rows;          /* m G-buffer rows */
    const int32_t *cut;           /* n cut nodes */
    const double *U, *V;          /* m*q, q*n (V times that frame's sigma) */
} orc_warm;

typedef struct {
    /* G-buffer rows (valid pixels), float32 promoted exactly to double */
    int64_t m;
    const float *px, *py, *pz, *nx, *ny, *nz, *vx, *vy, *vz, *rr, *rg, *rb, *spec;
    const int32_t *expo;
    /* VPLs */
    int64_t nv;
    const float *lx, *ly, *lz, *lnx, *lny, *lnz, *lir, *lig, *lib;
    /* light tree + global cut */
    int64_t nn;
    const int32_t *left, *right, *rep;
    const float *tir, *tig, *tib;
    int64_t ncut;
    const int32_t *cut;
    /* analytic occluders */
    int32_t nsph, nbox, nrect;
    const float *sph, *box, *rect;
    double clamp_dist, shadow_eps, diag;
    /* method parameters */
    double wn;
    int32_t target;
    uint64_t seed;
    int32_t nmax, nmin;
    double tau, rate;
    int32_t q, solver, K;
    double tol, alpha, beta, gamma, lam;
    uint64_t order_seed; /* 0: FIFO candidate order; else a seeded shuffle (order-independence pin) */
    /* SURVEY §8(f3) variants (0 = the paper's method) */
    int32_t row_importance; /* 1: rows drawn by f(i) = max - min of their carried observations (R36) */
    int32_t cost_mode;      /* 1: cost(L_f) = (eps + cost(L_b)) + cost(L_a) (Eq. (1) sensitivity) */
    int32_t resolve_mode;   /* 1: Z-mode image (factored + the observed entries' residuals, A24) */
    /* warm start: ADM slices found in warm[] (same slice, rows and cut, regular
     * result) start from those factors and run warm_iters iterations (0: K) */
    int32_t warm_iters, nwarm;
    /* SURVEY §8(f2) count-target coarsening (R37): > 0 merges the least-cost sibling pair
     * until the cut has this many nodes (tau unused); 0 = the threshold rule */
    int32_t coarsen_target;
    const orc_warm *warm;
    /* SURVEY §8(f1) triangle occluders, tri[9*k] = (v0, v1, v2), tested by brute force (R39) */
    int64_t ntri;
    const float *tri;
} orc_inputs;

enum { ORC_FLAG_DIRECT = 1, ORC_FLAG_DIVERGED = 2, ORC_FLAG_ZERO = 4 };

typedef struct {
    int32_t slice, m, n;          /* rows, final columns */
    int32_t *rows;                /* m G-buffer rows (ascending) */
    int32_t *cut_nodes;           /* n, ascending node id = column order */
    /* coarsening record, one entry per processed candidate, in processing order */
    int32_t n_proc;
    int32_t *proc_node, *proc_merged, *proc_zoff; /* zoff: n_proc+1 */
    double *proc_eps, *proc_cost;
    int32_t *proc_zrows;          /* concatenated zeta_f (sorted local rows) */
    double *proc_Va, *proc_Vb;    /* T values (not scaled) on zeta_f: T(i,rep a), T(i,rep b) */
    int64_t n_evals_coarsen;      /* unique (row, vpl) entry evaluations in pass 1 + coarsening */
    /* pass 2 */
    int64_t nnz, n_carried, n_new, n_forced, n_draws, target_N;
    int32_t *om_row, *om_col;     /* CSR order */
    double *om_val;               /* M~(i,c) */
    int32_t *om_carried;
    uint32_t *weights;            /* n */
    /* completion */
    int32_t q, iters, flags;
    double sigma, resid;
    double *U, *V;                /* m*q row-major, q*n row-major (V already times sigma) */
    double *obj;                  /* MALS: objective after each half step (2K) */
    int32_t n_obj;
    double *full;                 /* m*n full M~ for direct slices, else NULL */
    /* resolve */
    double *rgb;                  /* m*3 */
    int32_t warm;                 /* 1: the completion started from the previous frame's factors */
} orc_slice_result;

int64_t orc_sizeof_inputs(void);
int64_t orc_sizeof_result(void);
/* P:? — Philox4x32-10 (Salmon et al. SC'11), R-readings O3 */
void orc_philox(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
/* Floyd sampling of n distinct rows of [0,m) keyed by (a, slice); writes sorted rows, returns count */
int32_t orc_floyd(int32_t m, int32_t n, uint32_t a, int32_t slice, uint64_t seed, uint32_t tag, int32_t *out);
/* Lighting-matrix entry T(p, v) (geometry x BRDF x visibility), P:61 with readings R1-R3 */
double orc_entry_T(const orc_inputs *in, int64_t row, int64_t vpl);
void orc_entry_T_many(const orc_inputs *in, int64_t n, const int32_t *rows, const int32_t *vpls, double *out);
/* floating-point operations (+ - * / sqrt) orc_entry_T executes over n pairs (measurement only) */
int64_t orc_entry_flops(const orc_inputs *in, int64_t n, const int32_t *rows, const int32_t *vpls);
/* visibility only (1 visible, 0 occluded) of segment x -> y */
int32_t orc_visible(const orc_inputs *in, const double x[3], const double y[3]);
/* Matrix slicing, P:71-73 / P:172 with reading R26 */
int32_t orc_build_slices(const orc_inputs *in, int32_t *off, int32_t *rows, int64_t *nslices);
/* Pass-2 building blocks (readings R14, R29): light importance g(c) = max - min of
 * each column's observations, integer pdf weights, CDF inversion, one draw (t) of the pass */
void orc_light_importance(int32_t n, int64_t nobs, const int32_t *col, const double *val, double *g, int32_t *cnt);
void orc_pdf_weights(int32_t n, const double *g, const int32_t *cnt, uint32_t *w);
int32_t orc_cdf_pick(int32_t n, const uint64_t *cdf, uint64_t x);
void orc_pass2_draw(uint64_t seed, int32_t slice, uint32_t t, uint64_t W, const uint64_t *cdf, int32_t n, int32_t m,
                    int32_t *row, int32_t *col);
void orc_pass2_draw_f(uint64_t seed, int32_t slice, uint32_t t, uint64_t W, const uint64_t *cdf, int32_t n, uint64_t Wr,
                      const uint64_t *rcdf, int32_t m, int32_t *row, int32_t *col);
void orc_pass2_draws(uint64_t seed, int32_t slice, uint32_t t0, int64_t count, const uint32_t *w, int32_t n, int32_t m,
                     int32_t *rows, int32_t *cols);
/* Per-slice pipeline: coarsening, sampling, completion (App. A),
 * resolve.  stage: 1 = coarsen, 2 = + pass 2, 3 = + completion, 4 = + resolve */
orc_slice_result *orc_run_slice(const orc_inputs *in, const int32_t *rows, int32_t m, int32_t slice, int32_t stage);
void orc_run_slices(const orc_inputs *in, const int32_t *off, const int32_t *rows, int32_t nsel,
                    const int32_t *slice_ids, int32_t stage, orc_slice_result **out);
void orc_free_result(orc_slice_result *r);
/* ADM (App. A) on an explicit sample set; literal dense Z.  vals are M~ (unnormalised). */
int32_t orc_adm(int32_t m, int32_t n, int64_t nnz, const int32_t *row, const int32_t *col, const double *val,
                int32_t q, int32_t K, double tol, double alpha, double beta, double gamma, uint64_t seed,
                int32_t slice, double *U, double *V, int32_t *iters, double *resid, double *sigma);
/* ADM started from given factors X0 (m*q), Y0 (q*n, in units of val / sigma) -- warm start */
int32_t orc_adm_warm(int32_t m, int32_t n, int64_t nnz, const int32_t *row, const int32_t *col, const double *val,
                     int32_t q, int32_t K, double tol, double alpha, double beta, double gamma, const double *X0,
                     const double *Y0, double *U, double *V, int32_t *iters, double *resid, double *sigma);
/* Masked ALS (BASELINE north_star) on an explicit sample set. obj: 2K objective values (may be NULL). */
int32_t orc_mals(int32_t m, int32_t n, int64_t nnz, const int32_t *row, const int32_t *col, const double *val,
                 int32_t q, int32_t K, double lam, uint64_t seed, int32_t slice, double *X, double *Y,
                 double *obj, double *sigma);
/* full-cut rendering of a slice (every entry of M~, exact column sums), out m*3 */
void orc_fullcut_slice(const orc_inputs *in, const int32_t *rows, int32_t m, const int32_t *cut_nodes,
                       int32_t n, double *out);
/* brute force over all VPLs for the given rows, out nrows*3 */
void orc_bruteforce_rows(const orc_inputs *in, const int32_t *rows, int32_t nrows, double *out);

/* Light tree + conservative global lightcut (reading R38): arrays of 2 nv - 1
 * nodes, cut (<= cut_max nodes, ascending id); returns 0 */
int32_t orc_build_light_tree(int64_t nv, const float *px, const float *py, const float *pz, const float *ir,
                             const float *ig, const float *ib, int32_t cut_max, int32_t *left, int32_t *right,
                             int32_t *rep, float *tir, float *tig, float *tib, int32_t *cut, int64_t *ncut);

#ifdef __cplusplus
}
#endif
#endif
