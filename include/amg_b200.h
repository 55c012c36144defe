/*
 * amg_b200.h — C ABI of the B200-native AMG-PCG solve path (arxiv 2006.16147).
 *
 * The library solves A x = b for a symmetric positive-definite sparse A
 * ("systems ... where A is symmetric and positive-definite")
 * with preconditioned CG (north_star) whose preconditioner is
 * one V-cycle (Eq. 3.1) over a hierarchy built by coarsening
 * based on compatible weighted matching (Eqs. 3.2-3.3) with a
 * Jacobi-smoothed prolongator and l1-Jacobi smoothing
 * (nb = 1).  The hierarchy is built once per matrix (host,
 * C++/OpenMP) and uploaded; the solve phase runs entirely in hand-written
 * sm_100a CUDA kernels launched from CUDA graphs.
 *
 * Conventions shared by every entry point:
 *  - Status codes only; no exception crosses the ABI.  amg_last_error() returns a
 *    thread-local message describing the last failing call.
 *  - Host arrays are BORROWED for the duration of the call; the hierarchy owns
 *    its device copies.  Device pointers (`*_dev`) are caller-owned fp64 buffers
 *    on the context's device (typically torch tensors' data_ptr()).
 *  - All calls are ordered on the context's CUDA stream.  amg_solve /
 *    amg_solve_host / amg_precond_apply return after the stream work they issued
 *    has completed (they synchronize the context stream).
 *  - Multi-rank: every rank passes its own contiguous row block; build, solve and
 *    apply are collective over the ranks of the context.
 *  - Indices: global int64 on input; rows are contiguous blocks [row_begin, row_end).
 *  - fp64 throughout (the paper never states precision).
 *  - Threads: a hierarchy owns per-solve state (its CUDA graphs, the PCG vectors, the
 *    staging buffers of the host-buffer calls).  amg_solve, amg_solve_host,
 *    amg_solve_host_batch, amg_precond_apply and amg_profile_vcycle take a per-hierarchy
 *    lock, so calls from several threads on ONE hierarchy are serialised, not concurrent
 *    (a divergence from SPEC.md's "concurrent solves on shared immutable hierarchies":
 *    for concurrency build one hierarchy per thread / stream).  Different hierarchies are
 *    independent.  amg_hierarchy_destroy must not race with calls on the same hierarchy.
 */
#ifndef AMG_B200_H
#define AMG_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    AMG_OK = 0,
    AMG_ERR_ARG = 1,          /* bad argument: shape, ordering, asymmetry, sizes */
    AMG_ERR_NOT_SPD = 2,      /* non-positive diagonal, w == 0, coarsest Cholesky failed */
    AMG_ERR_CUDA = 3,         /* CUDA runtime / launch failure */
    AMG_ERR_NCCL = 4,         /* NCCL failure (multi-rank contexts) */
    AMG_ERR_OOM = 5,          /* host or device allocation failure */
    AMG_NOT_CONVERGED = 6,    /* maxit reached; x and the report are valid */
    AMG_ERR_BREAKDOWN = 7     /* p^T A p <= 0 in PCG; x holds the last iterate */
} amg_status_t;

typedef struct amg_ctx_s* amg_ctx_t;    /* one per rank = one GPU */
typedef struct amg_hier_s* amg_hier_t;  /* a built hierarchy, owned device data */

/* Hierarchy / cycle configuration.  Defaults (amg_config_default) reproduce the
 * paper's VA3 hierarchy with the readings of SURVEY.md §8c. */
typedef struct {
    int32_t sweeps_per_level;     /* m pairwise-matching sweeps per level; aggregates <= 2^m
                                     (PAPER.md:134).  Default 3. */
    int32_t smooth_prolongator;   /* 1: P-bar = (I - omega D^-1 A) P; 0: P. */
    double  prol_omega_scale;     /* omega = scale / ||D^-1 A||_inf.  Default 4/3 (reading R3:
                                     reproduces Table SM1); 1.0 = text's
                                     reading. */
    int64_t max_coarse_size;      /* stop coarsening once n_l <= this.
                                     Default 200; use 200*np across np GPUs. */
    int32_t max_levels;           /* default 20 */
    double  min_coarsening_ratio; /* a level with n_l/n_{l+1} < this is discarded (default 1.2) */
    int32_t pre_sweeps;           /* l1-Jacobi pre-smoothing sweeps, >= 1 (default 1) */
    int32_t post_sweeps;          /* l1-Jacobi post-smoothing sweeps, >= 1 (default 1) */
    int64_t replicate_below_bytes;/* multi-rank: levels whose A_l + P-bar_l bytes are below
                                     this are held whole on every rank (default 128 MiB: at c4 np = 8 the
                                     4k-row level, ~0.1 GB, whose rows would otherwise be ~500 per rank) */
    int32_t setup_threads;        /* host OpenMP threads for setup; 0 = all available */
    int32_t use_graphs;           /* 1 (default): a solve is ONE CUDA graph (a device-side WHILE node over
                                     the iteration, on one or several ranks; NCCL contexts fall back,
                                     collectively, to one graph per iteration if the WHILE graph cannot be
                                     built); 0: eager launches with one status read per iteration (debug /
                                     per-kernel timing). */
    int32_t emulate_ranks;        /* single-rank contexts only: > 1 partitions the hierarchy into
                                     this many equal row blocks held by ONE process on one GPU and
                                     runs the multi-rank kernels with in-process halo copies
                                     ("loopback"); the caller's vectors stay global.  Default 1. */
    /* --- the paper's own GPU method VA3S5CS1 --- */
    int32_t krylov;               /* outer solver of amg_solve: 0 = PCG (default, north_star;
                                     reading R1), 1 = FCG(1) ("Flexible Conjugate
                                     Gradient"), required when the preconditioner is nonlinear */
    int32_t coarse_solver;        /* 0 = dense direct solve with the explicit inverse (default,
                                     reading R2); 1 = CG preconditioned by the l1-Jacobi diagonal
                                     of A_L, run as one thread-block-cluster
                                     kernel; makes the V-cycle nonlinear (use krylov = 1) */
    int32_t coarse_maxit;         /* coarse CG iteration cap (default 30) */
    double  coarse_rtol;          /* coarse CG stops when ||r||/||b|| < this (default 1e-4,
                                     PAPER.md:264) */
    int32_t cycle;                /* 0 = V-cycle (default, Eq. 3.1); 1 = K-cycle: the coarse
                                     correction of every level whose coarse level is not the
                                     coarsest is two FCG(1) iterations preconditioned by the cycle
                                     rooted there.  Nonlinear:
                                     use krylov = 1.  Several ranks: the inner FCG exchanges p halos
                                     and finishes its dots in rank order on every rank. */
    int32_t setup_device;         /* 1 = build the hierarchy on the context's GPU (default; SURVEY.md
                                     §8f NEXT-1: suitor matching, expand-sort-compress canonical
                                     SpGEMM), bit-identical to 0 = the host build (C++/OpenMP).
                                     When the device build's working set (~40 B per stored entry of
                                     A, x8) exceeds 70% of the free device memory the host build is
                                     used instead (same result).  amg_host_hierarchy_build honours it
                                     (current CUDA device) when a cfg is passed and builds on the
                                     host when cfg is NULL. */
    int64_t tail_rows;            /* single-process contexts with a direct coarsest solve: the cycle
                                     rooted at the first level l >= 1 with n_l <= tail_rows runs as
                                     ONE cooperative persistent kernel (grid barriers between its
                                     operations) instead of ~4 launches per level and visit.
                                     Default 0 = off: measured slower than the launched graph on
                                     B200 (grid barriers cost more than PDL launch overlap). */
    int32_t smoother;             /* 0 = l1-Jacobi (default); 1 = INVK (
                                     SURVEY.md §8f NEXT-3): IC(0) = ILU(0) in LDL^T form, W = L^{-1}
                                     with `invk_fill` levels of positional fill, a smoothing step is
                                     x += W^T D^{-1} W (b - A x) (two extra SpMVs), computed per
                                     diagonal block (HINVK / l1-INVK, see invk_l1 / invk_blocks).  With
                                     one block (one process) HINVK = INVK. */
    int32_t invk_fill;            /* fill levels admitted in the inversion (default 1, Table 1
                                     caption PAPER.md:207) */
    int64_t tail_bytes;           /* single-process, direct coarsest: the cycle rooted at the first
                                     level from which all coarser operators take <= tail_bytes runs
                                     as ONE thread-block-cluster kernel (<= 16 CTAs, hardware
                                     cluster barriers between its operations).  0 = off. */
    /* --- block-Jacobi INVK forms and the VA3S3CS1 coarse solver --- */
    int32_t invk_l1;              /* smoother == 1: 0 = HINVK, the INVK factors of every rank's
                                     diagonal block A_pp; 1 = l1-INVK, the factors of
                                     A_pp + D_l1,p (Eq. 3.5 weights of the couplings outside the block,
                                     PAPER.md:180-181).  With one block both are plain INVK. */
    int32_t invk_blocks;          /* number of diagonal blocks: 0 (default) = one per rank of the
                                     partition (nranks, or emulate_ranks); k > 0 = k equal level-0 row
                                     blocks with coarse rows in the block of their aggregate's minimum
                                     member (R18): the paper's k-process block-Jacobi setting on one GPU
                                     (single-rank contexts; multi-rank contexts need 0 or nranks) */
    int32_t invk_dense_cut;       /* 0 (default) = "a single level of fill-in in the inversion" on every
                                     level.  c > 0: levels with more than c stored entries
                                     per row of A_l keep only the pattern of L (fill 0) -- a NON-paper
                                     setup-cost knob (the level-1 fill of a dense coarse row fills most of
                                     the triangle), documented as a deviation in DESIGN.md §8e */
    int32_t coarse_prec;          /* coarse_solver == 1: preconditioner of the coarse CG; 0 = l1-Jacobi
                                     diagonal of A_L (VA3S5CS1, default); 1 = the (H)INVK factors of A_L
                                     with the smoother's blocks / l1 / fill (VA3S3CS1: "we apply HINVK also
                                     as preconditioner of the CG method at the coarsest level",
                                     PAPER.md:420) */
    int32_t setup_distributed;    /* several ranks: 1 = the DISTRIBUTED setup: every
                                     rank builds only its rows of every level and its own plan (cross-rank
                                     matching rounds, remote-row-gather Galerkin products, all-reduced
                                     omega), bit-identical to the single-process build; 0 = rank 0 gathers
                                     the matrix, builds the whole hierarchy and scatters the plans; -1
                                     (default) = 1 for NCCL contexts, 0 for emulate_ranks (loopback) */
} amg_config_t;

/* Solve report (SPEC.md:440-443 SolveReport). */
typedef struct {
    int32_t iterations;           /* PCG iterations performed */
    int32_t converged;            /* 1 iff final_relres <= rtol */
    int32_t nlevels;              /* levels in the hierarchy */
    int32_t status;               /* amg_status_t of the solve */
    double  final_relres;         /* ||r_k||_2 / ||b||_2 (recursive residual, reading R12) */
    double  setup_s;              /* wall seconds of amg_hierarchy_build (host + upload) */
    double  solve_s;              /* device seconds of the solve (CUDA events) */
    double  opc;                  /* operator complexity sum nnz(A_l)/nnz(A_0) */
    double  avg_cr;               /* average coarsening ratio */
    double  vcycle_bytes_model;   /* algorithmic bytes of one V-cycle */
    double  iteration_bytes_model;/* algorithmic bytes of one PCG iteration */
} amg_report_t;

/* Fills *cfg with the defaults listed above. */
void amg_config_default(amg_config_t* cfg);

/* Writes a fresh 128-byte ncclUniqueId to out128 (call on rank 0, then broadcast). */
int amg_nccl_unique_id(void* out128);

/* Creates a context bound to CUDA device `device` and stream `cuda_stream`
 * (a cudaStream_t; NULL = a non-blocking stream created and owned by the context —
 * CUDA graphs cannot be captured on the legacy default stream).  For nranks > 1,
 * `nccl_unique_id` points to the 128-byte ncclUniqueId produced by rank 0 and
 * broadcast by the caller (e.g. through torch.distributed).  With nranks == 1 a
 * non-NULL id creates a ONE-rank communicator: hierarchies built with emulate_ranks > 1
 * on that context then move every halo and dot slot by NCCL self send/recv instead of
 * device copies ("NCCL loopback"), taking the real ranks' code path -- graph capture of
 * the collectives and its collective fallback included -- on one GPU (testing aid; the
 * arithmetic is unchanged, results are bitwise those of the device-copy loopback).
 * Returns AMG_ERR_ARG for rank/nranks out of range, AMG_ERR_CUDA / AMG_ERR_NCCL when
 * the device or communicator cannot be initialised. */
int amg_ctx_create(int device, int rank, int nranks, const void* nccl_unique_id,
                   void* cuda_stream, amg_ctx_t* out);
/* Destroy the hierarchies built on a context before the context itself. */
int amg_ctx_destroy(amg_ctx_t ctx);

/* Builds the hierarchy for the s.p.d. matrix A.
 *  n_global            global order of A
 *  row_begin, row_end  this rank's contiguous row block; blocks of all ranks must
 *                      be in rank order and cover [0, n_global)
 *  rowptr   host, int64, (row_end-row_begin)+1 entries, 0-based offsets into colind
 *  colind   host, int64 GLOBAL column indices, strictly ascending within each row
 *  values   host, fp64; A must be exactly symmetric (pattern and values)
 *  w        host, fp64, local rows of the matching weight vector; NULL = all ones
 *           ("starting from a vector w of all ones")
 *  cfg      NULL = defaults
 * Errors: AMG_ERR_ARG (unsorted/out-of-range columns, asymmetry, bad block),
 * AMG_ERR_NOT_SPD (a_ii <= 0, w == 0, coarsest Cholesky failure), AMG_ERR_OOM. */
int amg_hierarchy_build(amg_ctx_t ctx, int64_t n_global, int64_t row_begin, int64_t row_end,
                        const int64_t* rowptr, const int64_t* colind, const double* values,
                        const double* w, const amg_config_t* cfg, amg_hier_t* out);
int amg_hierarchy_destroy(amg_hier_t h);

/* PCG with one V-cycle per iteration (north_star):
 * x0 = 0, stops when ||r_k||/||b|| <= rtol or after maxit iterations; rtol = 0
 * runs exactly maxit iterations.  b_dev (read) and x_dev (written) hold this
 * rank's local rows.  b = 0 returns x = 0 after 0 iterations.  `rep` may be NULL.
 * Returns AMG_OK, AMG_NOT_CONVERGED or AMG_ERR_BREAKDOWN (x valid in all three). */
int amg_solve(amg_hier_t h, const double* b_dev, double* x_dev, double rtol, int32_t maxit,
              amg_report_t* rep);

/* Same as amg_solve but b_host/x_host are HOST buffers (pinned or pageable):
 * the host->device copy of b and the device->host copy of x are part of the call. */
int amg_solve_host(amg_hier_t h, const double* b_host, double* x_host, double rtol,
                   int32_t maxit, amg_report_t* rep);

/* nrhs independent solves with the same hierarchy on HOST buffers: right-hand side k is
 * B_host[k*n .. k*n+n-1] (n = this rank's local rows), its solution goes to X_host at the
 * same offset.  The copies are pipelined with the solves (b_{k+1} travels host->device and
 * x_{k-1} device->host while solve k runs, two device buffer pairs, a copy stream); every
 * solve is exactly amg_solve's (bitwise the same x).  For the overlap B_host / X_host should
 * be pinned (cudaHostAlloc / cudaHostRegister); pageable buffers still give correct results.
 * `reps` may be NULL or hold nrhs reports (solve_s of each = the batch time / nrhs).  Returns
 * the first non-AMG_OK status of the batch (AMG_NOT_CONVERGED / AMG_ERR_BREAKDOWN: x valid).
 * NCCL contexts or use_graphs = 0: the solves run one after another (amg_solve_host). */
int amg_solve_host_batch(amg_hier_t h, int32_t nrhs, const double* B_host, double* X_host, double rtol,
                         int32_t maxit, amg_report_t* reps);

/* One application of the preconditioner z = B r, i.e. one V-cycle
 * (Eq. 3.1).  Device buffers, local rows. */
int amg_precond_apply(amg_hier_t h, const double* r_dev, double* z_dev);

/* Hierarchy inspection.
 * amg_level_info: global rows, global nnz of A_l and P-bar_l (0 at the coarsest),
 * this rank's row block of level l and the device storage format of A_l
 * (0 = SELL-32, 1 = CSR-vector, 2 = dense inverse (coarsest), 3 = SDIA-32: slices of 32
 * rows aligned by column offset, no per-entry column index, 4 = SELL-32-sigma: SELL-32
 * over rows sorted by length inside windows of 256 rows, with a slot -> row map). */
int amg_num_levels(amg_hier_t h, int32_t* nlevels);
/* Shape the solves of h currently take (use_graphs = 1): 0 = one CUDA graph per solve
 * with a device-side WHILE node over the iteration; 1 = one graph per iteration from a
 * host loop (NCCL transports fall back to it, collectively, when a collective cannot be
 * captured into the WHILE body; AMG_MULTI_GRAPH=iter forces it); 2 = eager launches
 * (use_graphs = 0, or no graph could be captured).  Set by the first solve. */
int amg_solve_graph_mode(amg_hier_t h, int32_t* mode);
/* How h moves halos and dot slots between ranks: 0 = one rank (nothing to move); 1 = device
 * copies (loopback without a communicator); 2 = NCCL send/recv + all-gather (the fallback);
 * 3 = peer memory over an NCCL symmetric window ("LSA": the sending kernel stores halo values
 * and dot slots straight into the receivers' windows over NVLink, then a flag barrier with
 * system-scope release/acquire; no NCCL call inside the solve, so it stays one WHILE graph).
 * NCCL contexts take 3 when the window can be registered, every rank is in one load/store
 * domain and an end-to-end check passes on every rank (decided collectively at build);
 * AMG_TRANSPORT=nccl forces 2.  A barrier that waits 60 s for a peer makes the solve return
 * AMG_ERR_NCCL instead of hanging. */
int amg_comm_transport(amg_hier_t h, int32_t* transport);
int amg_level_info(amg_hier_t h, int32_t lvl, int64_t* n_global, int64_t* nnzA_global,
                   int64_t* nnzP_global, int64_t* row_begin, int64_t* row_end, int32_t* format);
/* Aggregate map of level lvl (lvl < nlevels-1): for each local row of level lvl the
 * GLOBAL index of its aggregate on level lvl+1 (host int64 array of local length). */
int amg_level_aggregates(amg_hier_t h, int32_t lvl, int64_t* agg_out);
/* Report of the hierarchy alone (opc, avg_cr, byte models, setup_s). */
int amg_hierarchy_report(amg_hier_t h, amg_report_t* rep);

/* Kernel timing probe: runs `napply` V-cycles with CUDA events around every kernel
 * on the context stream (eager launches) and writes, for up to `cap` kernels of
 * one V-cycle in launch order, the average device milliseconds (ms_out), the
 * algorithmic bytes of one launch per SURVEY.md §8d (bytes_out: 12 B per stored
 * entry + 4 B per row for every operator), the bytes the chosen device format
 * actually has to move (stored_bytes_out; smaller than bytes_out for SDIA-32,
 * which stores no per-entry column index) and a static name (names_out).  Any
 * output pointer may be NULL.  *count receives the number of kernels per V-cycle. */
int amg_profile_vcycle(amg_hier_t h, int32_t napply, int32_t cap, double* ms_out,
                       double* bytes_out, double* stored_bytes_out, const char** names_out,
                       int32_t* count);

/* The same probe over whole solver iterations (the V-cycle, q = A p with its dots, the
 * vector updates): runs the solver's prologue on b_dev / x_dev (device, local rows; x_dev is
 * overwritten), one warm-up iteration, then `napply` iterations in fixed-count mode with CUDA
 * events around every kernel, and reports the kernels of one iteration in launch order.  Used
 * to name the dominant kernel of an iteration for the roofline. */
int amg_profile_iteration(amg_hier_t h, const double* b_dev, double* x_dev, int32_t napply, int32_t cap,
                          double* ms_out, double* bytes_out, double* stored_bytes_out, const char** names_out,
                          int32_t* count);

/* ---- Host-only view of the setup phase (no device needed with setup_device = 0) ----
 * Runs exactly the setup that amg_hierarchy_build runs (the same C++ code) on a
 * whole matrix held by one process and keeps the host hierarchy, so the
 * aggregate maps, coarse operators and prolongators can be inspected, e.g. for
 * bit-exact comparison with an independent implementation.  Arguments as in
 * amg_hierarchy_build with row_begin = 0, row_end = n. */
typedef struct amg_host_hier_s* amg_host_hier_t;
int amg_host_hierarchy_build(int64_t n, const int64_t* rowptr, const int64_t* colind,
                             const double* values, const double* w, const amg_config_t* cfg,
                             amg_host_hier_t* out);
int amg_host_hierarchy_destroy(amg_host_hier_t h);
int amg_host_num_levels(amg_host_hier_t h, int32_t* nlevels);
/* n, nnz(A_l), nnz(P-bar_l) (0 at the coarsest), omega_l (0 if unsmoothed/coarsest) */
int amg_host_level_sizes(amg_host_hier_t h, int32_t lvl, int64_t* n, int64_t* nnzA, int64_t* nnzP,
                         double* omega);
/* aggregate map of level lvl < nlevels-1, n_l int64 entries */
int amg_host_level_aggregates(amg_host_hier_t h, int32_t lvl, int64_t* agg_out);
/* which = 0: A_l (n_l x n_l); which = 1: P-bar_l (n_l x n_{l+1}).  Caller-allocated
 * int64 rowptr (n_l+1), int64 colind and fp64 values (nnz entries). */
int amg_host_level_matrix(amg_host_hier_t h, int32_t lvl, int32_t which, int64_t* rowptr,
                          int64_t* colind, double* values);

/* The DISTRIBUTED setup run by `nranks` ranks emulated as
 * threads of this process (an in-process transport): rank g owns level-0 rows
 * [n g/nranks, n (g+1)/nranks), builds only its rows of every level (cross-rank matching rounds,
 * remote-row-gather Galerkin products, all-reduced omega) and its own plan (windows, halos,
 * replicated levels all-gathered), with no rank ever holding the whole matrix of a distributed
 * level.  The result is inspected with the amg_host_level_* calls (levels concatenated in rank
 * order) and amg_host_plan_* (every rank's plan); it must equal amg_host_hierarchy_build +
 * amg_host_partition bit for bit.  Host only (no device needed). */
int amg_host_dist_build(int64_t n, const int64_t* rowptr, const int64_t* colind, const double* values,
                        const double* w, const amg_config_t* cfg, int32_t nranks, int64_t replicate_below_bytes,
                        amg_host_hier_t* out);

/* The same distributed setup for ONE rank of a caller-provided transport (e.g. torch.distributed over
 * gloo, one process per rank): `exchange` is called collectively; with phase 0 it exchanges byte
 * counts (send_counts[q] bytes go to rank q, recv_counts[q] receives rank q's count), with phase 1 the
 * payloads, concatenated in rank order (send_buf holds sum(send_counts) bytes, recv_buf has room for
 * sum(recv_counts)); it returns 0 on success (non-zero: AMG_ERR_NCCL).  rowptr / colind / values / w
 * hold this rank's rows [row_begin, row_end) (global column ids).  The result holds this rank's plan
 * (amg_host_plan_level / amg_host_plan_array with this rank) and level sizes.  Host only. */
typedef int (*amg_exchange_fn)(void* user, int32_t phase, const int64_t* send_counts, int64_t* recv_counts,
                               const void* send_buf, void* recv_buf);
int amg_host_dist_build_rank(int64_t n, int64_t row_begin, int64_t row_end, const int64_t* rowptr,
                             const int64_t* colind, const double* values, const double* w, const amg_config_t* cfg,
                             int32_t nranks, int32_t rank, int64_t replicate_below_bytes,
                             amg_exchange_fn exchange, void* user, amg_host_hier_t* out);

/* Partition plan of the host hierarchy over `nranks` ranks with level-0 row blocks
 * row_bounds[0..nranks] (coarse rows owned by the rank of their
 * aggregate's minimum member; levels whose operator bytes are <= replicate_below_bytes,
 * and the coarsest, replicated).  Host only; inspected with amg_host_plan_level /
 * amg_host_plan_array (used by the CPU multi-rank tests). */
int amg_host_partition(amg_host_hier_t h, int32_t nranks, const int64_t* row_bounds,
                       int64_t replicate_below_bytes);
/* info16 = {replicated, n_global, own_begin, own_end, comp_begin, comp_end, win_begin,
 * win_end, rst_begin, rst_end, n_recv, n_send, nnz(A_loc), nnz(P_loc), nnz(R_loc), 0} */
int amg_host_plan_level(amg_host_hier_t h, int32_t rank, int32_t lvl, int64_t* info16);
/* which: 0 recv_off (nranks+1, int64), 1 recv_ids, 2 send_off, 3 send_ids (global ids,
 * int64), 4/5/6 A_loc rowptr/colind (int64, window frame)/values, 7/8/9 P_loc, 10/11/12
 * R_loc, 13 l1 inverse diagonal over the window (fp64).  Caller-allocated. */
int amg_host_plan_array(amg_host_hier_t h, int32_t rank, int32_t lvl, int32_t which, void* out);

/* Thread-local message of the last failing call on this thread ("" if none). */
const char* amg_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* AMG_B200_H */
