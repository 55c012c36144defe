/*
 * oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, single-threaded fp64 CPU oracle for the AMG-PCG method of
 * arxiv 2006.16147 (§3.1-§3.3, §5).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  It shares no
 * code, header or helper with the product library under paper_2006_16147_b200/.
 *
 * Every function follows the paper (and SURVEY.md §8c's numbered readings) step by
 * step in the paper's order; see oracle.c for the per-function citations.
 * All integers are int64, all reals fp64; compiled with -O2 -ffp-contract=off.
 */
#ifndef AMG_ORACLE_H
#define AMG_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ocsr ocsr;      /* CSR matrix, sorted columns */
typedef struct ohier ohier;    /* AMG hierarchy */

/* status codes (mirror SPEC.md:632 exit semantics) */
enum { OR_OK = 0, OR_ERR_ARG = 1, OR_ERR_NOT_SPD = 2, OR_NOT_CONVERGED = 6, OR_BREAKDOWN = 7 };

/* --- sparse core --------------------------------------------------------- */
ocsr*   or_csr_new_copy(int64_t nrows, int64_t ncols, const int64_t* rp,
                        const int64_t* ci, const double* v);
void    or_csr_dims(const ocsr* A, int64_t out3[3]);          /* nrows, ncols, nnz */
void    or_csr_export(const ocsr* A, int64_t* rp, int64_t* ci, double* v);
void    or_csr_free(ocsr* A);
void    or_spmv(const ocsr* A, const double* x, double* y);
ocsr*   or_transpose(const ocsr* X);
ocsr*   or_matmul_canonical(const ocsr* A, const ocsr* Y);
ocsr*   or_rap(const ocsr* X, const ocsr* A, const ocsr* Y);  /* X^T A Y, no mirror */
void    or_mirror_drop(ocsr* C);                                /* C4 + C5 in place */

/* --- matching-based aggregation (§3.2) -------------------------- */
int64_t or_edge_weights(const ocsr* A, const double* w, int64_t* ei, int64_t* ej, double* c);
void    or_greedy_matching(int64_t n, int64_t ne, const int64_t* ei, const int64_t* ej,
                           const double* c, int64_t* mate);
int64_t or_aggregates(int64_t n, const int64_t* mate, int64_t* agg);
/* one pairwise sweep (O2.1-O2.5): returns A_{s+1}; fills w_next (nc), agg (n),
 * pval (n; NaN where P has no stored entry) and *nc */
ocsr*   or_pairwise_sweep(const ocsr* A, const double* w, double* w_next,
                          int64_t* agg, double* pval, int64_t* nc);
double  or_dinv_a_inf_norm(const ocsr* A);
ocsr*   or_prolongator_csr(int64_t n, int64_t nc, const int64_t* agg, const double* pval);
ocsr*   or_smooth_prolongator(const ocsr* A, const ocsr* P, double omega);
void    or_l1_jacobi_inv(const ocsr* A, double* m);

/* --- hierarchy ----------------------------------------------------------- */
ohier*  or_build(const ocsr* A0, const double* w0 /* NULL => ones */,
                 int32_t sweeps_per_level, int32_t smooth_prolongator,
                 double prol_omega_scale, int64_t max_coarse_size, int32_t max_levels,
                 double min_coarsening_ratio, int32_t pre_sweeps, int32_t post_sweeps,
                 int32_t* status);
void    or_free(ohier* h);
int32_t or_nlevels(const ohier* h);
const ocsr* or_level_A(const ohier* h, int32_t l);
const ocsr* or_level_P(const ohier* h, int32_t l);   /* smoothed P-bar (NULL at coarsest) */
int64_t or_level_n(const ohier* h, int32_t l);
void    or_level_agg(const ohier* h, int32_t l, int64_t* agg);
void    or_level_pval(const ohier* h, int32_t l, double* pval);  /* unsmoothed composite */
void    or_level_w(const ohier* h, int32_t l, double* w);
void    or_level_m(const ohier* h, int32_t l, double* m);
double  or_level_omega(const ohier* h, int32_t l);
int32_t or_level_sweeps(const ohier* h, int32_t l);
double  or_opc(const ohier* h);
double  or_avg_cr(const ohier* h);

/* --- apply / solve (Eq. 3.1) ---------------- */
void    or_vcycle(const ohier* h, const double* r, double* z);
int32_t or_pcg(const ohier* h, const double* b, double* x, double rtol, int32_t maxit,
               int32_t* iters, double* relres, double* true_relres, double* hist);
/* SURVEY §8f NEXT-2 (the paper's GPU method VA3S5CS1): FCG(1) outer
 * solver and the coarsest level solved by l1-Jacobi-preconditioned CG. */
int32_t or_fcg(const ohier* h, const double* b, double* x, double rtol, int32_t maxit,
               int32_t* iters, double* relres, double* true_relres, double* hist);
void    or_set_coarse_cg(ohier* h, int32_t on, double rtol, int32_t maxit);
/* cycle = 1 replaces the coarse correction of every level whose
 * coarse level is not the coarsest by two FCG(1) iterations (K-cycle);
 * or_vcycle / or_pcg / or_fcg then apply the K-cycle.  or_coarse_visits counts the
 * coarsest solves performed since the hierarchy was built. */
void    or_set_cycle(ohier* h, int32_t cycle);
/* smoother kind 1 = INVK: IC(0) = ILU(0) in
 * LDL^T form, W = L^{-1} truncated to `fill` levels of positional fill, smoothing
 * step x += W^T D^{-1} W (b - A x) on every non-coarsest level; 0 = l1-Jacobi.
 * Returns OR_ERR_NOT_SPD on a non-positive IC(0) pivot.  or_level_invk returns
 * D^{-1} W (which = 0) or Z = W^T (which = 1) of level l. */
int32_t or_set_smoother(ohier* h, int32_t kind, int32_t fill);
/* The paper's parallel block-Jacobi forms: the INVK factors of the
 * diagonal blocks A_pp (HINVK), or of A_pp + D_l1,p (l1 = 1, l1-INVK), with nblocks row
 * blocks [bounds0[p], bounds0[p+1]) at level 0 and coarse rows owned by the block of their
 * aggregate's minimum member (R18).  fill_per_level (NULL = `fill` everywhere) overrides
 * the fill of each level.  Also builds the coarsest level's factors when the coarse CG
 * uses them (or_set_coarse_prec, call it first). */
int32_t or_set_smoother_ex(ohier* h, int32_t kind, int32_t fill, int32_t nblocks, const int64_t* bounds0,
                           int32_t l1, const int32_t* fill_per_level);
/* coarse CG preconditioner: 0 = l1-Jacobi (VA3S5CS1), 1 = the INVK factors of A_L (VA3S3CS1,
 * PAPER.md:420) */
void    or_set_coarse_prec(ohier* h, int32_t kind);
const ocsr* or_level_invk(const ohier* h, int32_t l, int32_t which);
int64_t or_coarse_visits(const ohier* h);
/* cycle applications rooted at level l since the build (K-opc weights) */
int64_t or_level_visits(const ohier* h, int32_t l);
/* solve-phase threads: 1 = the sequential parity reference (default); > 1 = OpenMP row
 * loops and fixed-chunk dots (SURVEY §8d (ii) all-core timing only) */
void    or_set_threads(int32_t t);

#ifdef __cplusplus
}
#endif
#endif
