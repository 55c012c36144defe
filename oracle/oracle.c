/*
 * oracle.c — TEST INFRASTRUCTURE ONLY (see oracle.h).  Never linked into, or
 * called from, the product path under paper_2006_16147_b200/.
 *
 * A plain, slow, obviously-correct fp64 implementation of the method of
 * arxiv 2006.16147 as the paper states it, with SURVEY.md §8c's readings where
 * the paper is silent:
 *
 *   hierarchy  PAPER.md:83-86 (Galerkin A_{l+1} = P^T A P),
 *              PAPER.md:106-110 (Eq. 3.2 weights), PAPER.md:111-131 (matching,
 *              pairs/singletons, Eq. 3.3 prolongator), PAPER.md:133-134 (recursion
 *              with restricted w, m sweeps), PAPER.md:138-139 (smoothed P-bar),
 *              PAPER.md:143-149 (half-approximate matching = locally dominant
 *              edges), PAPER.md:170 (l1-Jacobi, nb = 1), PAPER.md:264 (w = 1,
 *              maxsize stop rule).
 *   apply      PAPER.md:87-92 (Eq. 3.1 V-cycle, B_nl ~ A_nl^{-1}).
 *   solve      PCG (north_star; reading R1), x0 = 0, ||r||/||b|| <= rtol.
 *
 * Canonical arithmetic contract: no FMA (-ffp-contract=off),
 * expressions parenthesised exactly as written below, Galerkin products in the
 * fixed two-step order of C3, mirrored upper triangle (C4), exact zeros dropped (C5).
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

struct ocsr {
    int64_t nrows, ncols;
    int64_t* rp;
    int64_t* ci;
    double* v;
};

typedef struct {
    int64_t n;
    ocsr* A;          /* A_l */
    ocsr* P;          /* smoothed prolongator P-bar_l (n_l x n_{l+1}); NULL at coarsest */
    ocsr* R;          /* P-bar_l^T (restriction, ascending fine index per row) */
    int64_t* agg;     /* composite aggregate map, NULL at coarsest */
    double* pval;     /* composite unsmoothed P values (NaN if not stored) */
    double* w;        /* w_l */
    double* m;        /* l1-Jacobi inverse diagonal */
    double omega;
    int32_t sweeps;   /* pairwise sweeps actually performed */
    double* L;        /* coarsest: dense Cholesky factor (row-major, lower) */
    ocsr* Wd;         /* INVK smoother: D^{-1} W, W = truncated L^{-1} (lower, unit diagonal) */
    ocsr* Z;          /* INVK smoother: W^T */
} olevel;

struct ohier {
    int32_t nl;
    olevel* lv;
    int32_t pre, post;
    /* coarsest solver: 0 = dense Cholesky (reading R2); 1 = CG preconditioned by
     * l1-Jacobi, stopped at ||r||/||b|| < coarse_rtol or after coarse_maxit
     * iterations */
    int32_t coarse_cg;
    double coarse_rtol;
    int32_t coarse_maxit;
    /* cycle: 0 = V-cycle (Eq. 3.1); 1 = K-cycle */
    int32_t cycle;
    /* smoother: 0 = l1-Jacobi; 1 = INVK */
    int32_t smoother;
    /* coarse CG preconditioner: 0 = l1-Jacobi diagonal of A_L (VA3S5CS1); 1 = the INVK /
     * HINVK factors of A_L (VA3S3CS1: "we apply HINVK also as preconditioner of the CG
     * method at the coarsest level") */
    int32_t coarse_prec;
    int64_t coarse_visits;  /* coarsest solves performed (instrumentation) */
    int64_t visits[64];     /* cycle applications rooted at each level (instrumentation) */
};

/* Solve-phase threads (SURVEY §8d (ii) "OpenMP all-core" oracle timing).  1 (default) is
 * the parity reference: every loop sequential, every dot summed in index order.  With
 * g_threads > 1 the row loops run in parallel (same arithmetic per entry) and dots are
 * summed per fixed chunk in index order, then over the chunks in order: deterministic,
 * but rounded differently from the sequential sum.  Setup is always sequential. */
static int g_threads = 1;
#define OR_CHUNKS 256
void or_set_threads(int32_t t) { g_threads = t > 1 ? t : 1; }

/* ------------------------------------------------------------------ helpers */
static double dot(int64_t n, const double* a, const double* b);

static void* xmalloc(size_t n) {
    void* p = malloc(n ? n : 1);
    if (!p) abort();
    return p;
}
static void* xcalloc(size_t n, size_t s) {
    void* p = calloc(n ? n : 1, s ? s : 1);
    if (!p) abort();
    return p;
}

static ocsr* csr_alloc(int64_t nrows, int64_t ncols, int64_t nnz) {
    ocsr* A = (ocsr*)xmalloc(sizeof(ocsr));
    A->nrows = nrows;
    A->ncols = ncols;
    A->rp = (int64_t*)xcalloc((size_t)nrows + 1, sizeof(int64_t));
    A->ci = (int64_t*)xmalloc((size_t)nnz * sizeof(int64_t));
    A->v = (double*)xmalloc((size_t)nnz * sizeof(double));
    return A;
}

ocsr* or_csr_new_copy(int64_t nrows, int64_t ncols, const int64_t* rp, const int64_t* ci,
                      const double* v) {
    int64_t nnz = rp[nrows];
    ocsr* A = csr_alloc(nrows, ncols, nnz);
    memcpy(A->rp, rp, sizeof(int64_t) * (size_t)(nrows + 1));
    memcpy(A->ci, ci, sizeof(int64_t) * (size_t)nnz);
    memcpy(A->v, v, sizeof(double) * (size_t)nnz);
    return A;
}

void or_csr_dims(const ocsr* A, int64_t out3[3]) {
    out3[0] = A->nrows;
    out3[1] = A->ncols;
    out3[2] = A->rp[A->nrows];
}

void or_csr_export(const ocsr* A, int64_t* rp, int64_t* ci, double* v) {
    int64_t nnz = A->rp[A->nrows];
    memcpy(rp, A->rp, sizeof(int64_t) * (size_t)(A->nrows + 1));
    memcpy(ci, A->ci, sizeof(int64_t) * (size_t)nnz);
    memcpy(v, A->v, sizeof(double) * (size_t)nnz);
}

void or_csr_free(ocsr* A) {
    if (!A) return;
    free(A->rp);
    free(A->ci);
    free(A->v);
    free(A);
}

static double csr_get(const ocsr* A, int64_t i, int64_t j, int* found) {
    /* binary search of column j in row i */
    int64_t lo = A->rp[i], hi = A->rp[i + 1] - 1;
    while (lo <= hi) {
        int64_t mid = lo + (hi - lo) / 2;
        if (A->ci[mid] == j) {
            *found = 1;
            return A->v[mid];
        }
        if (A->ci[mid] < j) lo = mid + 1;
        else hi = mid - 1;
    }
    *found = 0;
    return 0.0;
}

static double diag_of(const ocsr* A, int64_t i) {
    int f;
    return csr_get(A, i, i, &f);
}

/* ---------------------------------------------------------------- sparse core */
/* y = A x, each row summed in ascending column order from +0.0. */
void or_spmv(const ocsr* A, const double* x, double* y) {
#pragma omp parallel for schedule(static) if (g_threads > 1) num_threads(g_threads)
    for (int64_t i = 0; i < A->nrows; ++i) {
        double s = 0.0;
        for (int64_t k = A->rp[i]; k < A->rp[i + 1]; ++k) s += A->v[k] * x[A->ci[k]];
        y[i] = s;
    }
}

/* X^T: row G lists (i, x_iG) for i ascending (C3). */
ocsr* or_transpose(const ocsr* X) {
    int64_t nnz = X->rp[X->nrows];
    ocsr* T = csr_alloc(X->ncols, X->nrows, nnz);
    for (int64_t k = 0; k < nnz; ++k) T->rp[X->ci[k] + 1]++;
    for (int64_t c = 0; c < X->ncols; ++c) T->rp[c + 1] += T->rp[c];
    int64_t* pos = (int64_t*)xmalloc(sizeof(int64_t) * (size_t)(X->ncols + 1));
    memcpy(pos, T->rp, sizeof(int64_t) * (size_t)(X->ncols + 1));
    for (int64_t i = 0; i < X->nrows; ++i)
        for (int64_t k = X->rp[i]; k < X->rp[i + 1]; ++k) {
            int64_t c = X->ci[k];
            T->ci[pos[c]] = i;
            T->v[pos[c]] = X->v[k];
            pos[c]++;
        }
    free(pos);
    return T;
}

static int cmp_i64(const void* a, const void* b) {
    int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
    return (x > y) - (x < y);
}

/* C = A * Y in the canonical order of C3: for row i, for each a_ij with j
 * ascending, for each y_jK with K ascending, acc[K] += a_ij*y_jK, every acc
 * starting from +0.0 and accumulating in arrival order.  Output columns ascending.
 * Exact zeros are kept here (dropped by the caller where the contract says so). */
ocsr* or_matmul_canonical(const ocsr* A, const ocsr* Y) {
    int64_t n = A->nrows, m = Y->ncols;
    double* acc = (double*)xcalloc((size_t)m, sizeof(double));
    char* mark = (char*)xcalloc((size_t)m, 1);
    int64_t* cols = (int64_t*)xmalloc(sizeof(int64_t) * (size_t)(m > 0 ? m : 1));
    int64_t cap = A->rp[n] + 16, nnz = 0;
    int64_t* ci = (int64_t*)xmalloc(sizeof(int64_t) * (size_t)cap);
    double* v = (double*)xmalloc(sizeof(double) * (size_t)cap);
    int64_t* rp = (int64_t*)xcalloc((size_t)n + 1, sizeof(int64_t));
    for (int64_t i = 0; i < n; ++i) {
        int64_t nc = 0;
        for (int64_t k = A->rp[i]; k < A->rp[i + 1]; ++k) {
            int64_t j = A->ci[k];
            double a = A->v[k];
            for (int64_t t = Y->rp[j]; t < Y->rp[j + 1]; ++t) {
                int64_t K = Y->ci[t];
                if (!mark[K]) {
                    mark[K] = 1;
                    acc[K] = 0.0;
                    cols[nc++] = K;
                }
                acc[K] += a * Y->v[t];
            }
        }
        qsort(cols, (size_t)nc, sizeof(int64_t), cmp_i64);
        if (nnz + nc > cap) {
            while (nnz + nc > cap) cap *= 2;
            ci = (int64_t*)realloc(ci, sizeof(int64_t) * (size_t)cap);
            v = (double*)realloc(v, sizeof(double) * (size_t)cap);
            if (!ci || !v) abort();
        }
        for (int64_t t = 0; t < nc; ++t) {
            ci[nnz] = cols[t];
            v[nnz] = acc[cols[t]];
            mark[cols[t]] = 0;
            nnz++;
        }
        rp[i + 1] = nnz;
    }
    free(acc);
    free(mark);
    free(cols);
    ocsr* C = (ocsr*)xmalloc(sizeof(ocsr));
    C->nrows = n;
    C->ncols = m;
    C->rp = rp;
    C->ci = ci;
    C->v = v;
    return C;
}

/* canonical_RAP(X^T, A, Y) of C3: T = A*Y, then C = X^T * T. */
ocsr* or_rap(const ocsr* X, const ocsr* A, const ocsr* Y) {
    ocsr* T = or_matmul_canonical(A, Y);
    ocsr* Xt = or_transpose(X);
    ocsr* C = or_matmul_canonical(Xt, T);
    or_csr_free(T);
    or_csr_free(Xt);
    return C;
}

/* C4: C[K,G] := C[G,K] for G < K (lower triangle copied from the upper one);
 * C5: drop entries that are exactly zero.  In place. */
void or_mirror_drop(ocsr* C) {
    int64_t n = C->nrows, nnz = 0;
    double* nv = (double*)xmalloc(sizeof(double) * (size_t)(C->rp[n] + 1));
    for (int64_t r = 0; r < n; ++r)
        for (int64_t k = C->rp[r]; k < C->rp[r + 1]; ++k) {
            int64_t c = C->ci[k];
            if (c < r) {
                int f;
                double u = csr_get(C, c, r, &f);
                nv[k] = f ? u : 0.0;
            } else {
                nv[k] = C->v[k];
            }
        }
    int64_t start = 0;
    for (int64_t r = 0; r < n; ++r) {
        int64_t end = C->rp[r + 1];
        for (int64_t k = start; k < end; ++k)
            if (nv[k] != 0.0) {
                C->ci[nnz] = C->ci[k];
                C->v[nnz] = nv[k];
                nnz++;
            }
        start = end;
        C->rp[r + 1] = nnz;
    }
    free(nv);
}

/* ------------------------------------------------------------ aggregation */
/* O2.1, Eq. 3.2: for every stored pair i < j of A (upper
 * triangle) c_ij = 1 - 2 a_ij w_i w_j / (a_ii w_i^2 + a_jj w_j^2), evaluated as
 *   den = (a_ii*w_i)*w_i + (a_jj*w_j)*w_j,  c = 1 - (((2*a_ij)*w_i)*w_j)/den.
 * Edges with den == 0 or c == 0 are dropped ("c_ij != 0").
 * Returns the number of edges; arrays must hold nnz(A) entries. */
int64_t or_edge_weights(const ocsr* A, const double* w, int64_t* ei, int64_t* ej, double* c) {
    int64_t ne = 0;
    for (int64_t i = 0; i < A->nrows; ++i) {
        double aii = diag_of(A, i);
        for (int64_t k = A->rp[i]; k < A->rp[i + 1]; ++k) {
            int64_t j = A->ci[k];
            if (j <= i) continue;
            double ajj = diag_of(A, j);
            double aij = A->v[k];
            double den = (aii * w[i]) * w[i] + (ajj * w[j]) * w[j];
            if (den == 0.0) continue;
            double cij = 1.0 - (((2.0 * aij) * w[i]) * w[j]) / den;
            if (cij == 0.0) continue;
            ei[ne] = i;
            ej[ne] = j;
            c[ne] = cij;
            ne++;
        }
    }
    return ne;
}

typedef struct {
    double key;
    int64_t i, j;
} oedge;

/* strict total order (R4, R5): |c| descending, then lo ascending, then hi ascending */
static int cmp_edge(const void* a, const void* b) {
    const oedge* x = (const oedge*)a;
    const oedge* y = (const oedge*)b;
    if (x->key > y->key) return -1;
    if (x->key < y->key) return 1;
    if (x->i != y->i) return (x->i < y->i) ? -1 : 1;
    if (x->j != y->j) return (x->j < y->j) ? -1 : 1;
    return 0;
}

/* O2.2: half-approximate maximum-weight matching.  The
 * additive weight -sum(log max|c| - log|c|) is a strictly monotone transform of
 * |c| (R4), so the edge order by |c| is the order of the transformed weights.
 * Greedy scan in that strict order; an edge is taken when both ends are free.
 * Under a strict total order this is the unique locally-dominant matching. */
void or_greedy_matching(int64_t n, int64_t ne, const int64_t* ei, const int64_t* ej,
                        const double* c, int64_t* mate) {
    oedge* E = (oedge*)xmalloc(sizeof(oedge) * (size_t)(ne > 0 ? ne : 1));
    for (int64_t e = 0; e < ne; ++e) {
        E[e].key = fabs(c[e]);
        E[e].i = ei[e] < ej[e] ? ei[e] : ej[e];
        E[e].j = ei[e] < ej[e] ? ej[e] : ei[e];
    }
    qsort(E, (size_t)ne, sizeof(oedge), cmp_edge);
    for (int64_t v = 0; v < n; ++v) mate[v] = -1;
    for (int64_t e = 0; e < ne; ++e)
        if (mate[E[e].i] < 0 && mate[E[e].j] < 0) {
            mate[E[e].i] = E[e].j;
            mate[E[e].j] = E[e].i;
        }
    free(E);
}

/* O2.3: matched pairs and unmatched singletons; aggregates
 * numbered by ascending minimum member (R5). Returns n_c = n_p + n_s. */
int64_t or_aggregates(int64_t n, const int64_t* mate, int64_t* agg) {
    int64_t nc = 0;
    for (int64_t i = 0; i < n; ++i) agg[i] = -1;
    for (int64_t i = 0; i < n; ++i) {
        if (agg[i] >= 0) continue;
        agg[i] = nc;
        if (mate[i] >= 0) agg[mate[i]] = nc;
        nc++;
    }
    return nc;
}

/* Eq. 3.3, O2.4: pair {i<j}: P[i,G] = w_i/nrm, P[j,G] = w_j/nrm,
 * nrm = sqrt((w_i*w_i)+(w_j*w_j)); nrm == 0 -> P[i,G] = 1, P[j,G] not stored.
 * Singleton s: P[s,G] = w_s/|w_s| (1.0 if w_s == 0).
 * pval[i] = NaN marks "no stored entry"; exact zeros are not stored (C5). */
static void pairwise_values(int64_t n, const int64_t* mate, const double* w, double* pval) {
    for (int64_t i = 0; i < n; ++i) {
        int64_t j = mate[i];
        if (j < 0) {
            pval[i] = (w[i] == 0.0) ? 1.0 : w[i] / fabs(w[i]);
            continue;
        }
        int64_t lo = i < j ? i : j, hi = i < j ? j : i;
        double nrm = sqrt((w[lo] * w[lo]) + (w[hi] * w[hi]));
        if (nrm == 0.0) {
            pval[i] = (i == lo) ? 1.0 : NAN;
        } else {
            double p = w[i] / nrm;
            pval[i] = (p == 0.0) ? NAN : p;
        }
    }
}

ocsr* or_prolongator_csr(int64_t n, int64_t nc, const int64_t* agg, const double* pval) {
    int64_t nnz = 0;
    for (int64_t i = 0; i < n; ++i) nnz += !isnan(pval[i]);
    ocsr* P = csr_alloc(n, nc, nnz);
    int64_t k = 0;
    for (int64_t i = 0; i < n; ++i) {
        if (!isnan(pval[i])) {
            P->ci[k] = agg[i];
            P->v[k] = pval[i];
            k++;
        }
        P->rp[i + 1] = k;
    }
    return P;
}

/* P^T w in canonical order: for each G, sum over i ascending from +0.0 (C3). */
static void restrict_weight(const ocsr* P, const double* w, double* wc) {
    ocsr* Pt = or_transpose(P);
    for (int64_t G = 0; G < Pt->nrows; ++G) {
        double s = 0.0;
        for (int64_t k = Pt->rp[G]; k < Pt->rp[G + 1]; ++k) s += Pt->v[k] * w[Pt->ci[k]];
        wc[G] = s;
    }
    or_csr_free(Pt);
}

/* One pairwise aggregation sweep, O2.1-O2.5: weights ->
 * matching -> aggregates -> pairwise P -> A_next = canonical_RAP(P, A, P),
 * mirrored and zero-dropped, w_next = P^T w. */
ocsr* or_pairwise_sweep(const ocsr* A, const double* w, double* w_next, int64_t* agg,
                        double* pval, int64_t* nc_out) {
    int64_t n = A->nrows, nnz = A->rp[n];
    int64_t* ei = (int64_t*)xmalloc(sizeof(int64_t) * (size_t)(nnz + 1));
    int64_t* ej = (int64_t*)xmalloc(sizeof(int64_t) * (size_t)(nnz + 1));
    double* c = (double*)xmalloc(sizeof(double) * (size_t)(nnz + 1));
    int64_t* mate = (int64_t*)xmalloc(sizeof(int64_t) * (size_t)(n + 1));
    int64_t ne = or_edge_weights(A, w, ei, ej, c);
    or_greedy_matching(n, ne, ei, ej, c, mate);
    int64_t nc = or_aggregates(n, mate, agg);
    pairwise_values(n, mate, w, pval);
    ocsr* P = or_prolongator_csr(n, nc, agg, pval);
    ocsr* An = or_rap(P, A, P);
    or_mirror_drop(An);
    restrict_weight(P, w, w_next);
    or_csr_free(P);
    free(ei);
    free(ej);
    free(c);
    free(mate);
    *nc_out = nc;
    return An;
}

/* ||D^{-1} A||_inf = max_i (sum_{j asc} |a_ij|) / a_ii. */
double or_dinv_a_inf_norm(const ocsr* A) {
    double mx = 0.0;
    for (int64_t i = 0; i < A->nrows; ++i) {
        double s = 0.0;
        for (int64_t k = A->rp[i]; k < A->rp[i + 1]; ++k) s += fabs(A->v[k]);
        double r = s / diag_of(A, i);
        if (r > mx) mx = r;
    }
    return mx;
}

/* O5: P-bar = (I - omega D^{-1} A) P, row by row:
 * t = (A P)_i in canonical order, P-bar[i,G] = P[i,G] - (omega/a_ii)*t_G,
 * exact zeros dropped. */
ocsr* or_smooth_prolongator(const ocsr* A, const ocsr* P, double omega) {
    ocsr* T = or_matmul_canonical(A, P);
    int64_t n = A->nrows, nnz = 0;
    ocsr* Pb = csr_alloc(n, P->ncols, T->rp[n]);
    for (int64_t i = 0; i < n; ++i) {
        double f = omega / diag_of(A, i);
        for (int64_t k = T->rp[i]; k < T->rp[i + 1]; ++k) {
            int64_t G = T->ci[k];
            int found;
            double p = csr_get(P, i, G, &found);
            double v = (found ? p : 0.0) - f * T->v[k];
            if (v != 0.0) {
                Pb->ci[nnz] = G;
                Pb->v[nnz] = v;
                nnz++;
            }
        }
        Pb->rp[i + 1] = nnz;
    }
    or_csr_free(T);
    return Pb;
}

/* O7, PAPER.md:165-170 with nb = 1: M = diag(a_ii + sum_{j != i}|a_ij|); the
 * oracle stores m_i = 1/(sum_{j asc} |a_ij|) (includes |a_ii| = a_ii > 0). */
void or_l1_jacobi_inv(const ocsr* A, double* m) {
    for (int64_t i = 0; i < A->nrows; ++i) {
        double s = 0.0;
        for (int64_t k = A->rp[i]; k < A->rp[i + 1]; ++k) s += fabs(A->v[k]);
        m[i] = 1.0 / s;
    }
}

/* --------------------------------------------------------------- hierarchy */
static int validate(const ocsr* A, const double* w) {
    if (A->nrows != A->ncols || A->nrows <= 0) return OR_ERR_ARG;
    int anyw = 0;
    for (int64_t i = 0; i < A->nrows; ++i) {
        for (int64_t k = A->rp[i]; k < A->rp[i + 1]; ++k) {
            if (k > A->rp[i] && A->ci[k] <= A->ci[k - 1]) return OR_ERR_ARG;
            if (A->ci[k] < 0 || A->ci[k] >= A->ncols) return OR_ERR_ARG;
            int f;
            double t = csr_get(A, A->ci[k], i, &f);
            if (!f || t != A->v[k]) return OR_ERR_ARG; /* exact symmetry */
        }
        if (!(diag_of(A, i) > 0.0)) return OR_ERR_NOT_SPD;
        if (w && w[i] != 0.0) anyw = 1;
    }
    if (w && !anyw) return OR_ERR_NOT_SPD;
    return OR_OK;
}

static ocsr* csr_clone(const ocsr* A) {
    return or_csr_new_copy(A->nrows, A->ncols, A->rp, A->ci, A->v);
}

/* O8 (reading R2): dense Cholesky of the coarsest matrix. */
static int dense_cholesky(const ocsr* A, double** Lout) {
    int64_t n = A->nrows;
    double* L = (double*)xcalloc((size_t)(n * n), sizeof(double));
    for (int64_t i = 0; i < n; ++i)
        for (int64_t k = A->rp[i]; k < A->rp[i + 1]; ++k) L[i * n + A->ci[k]] = A->v[k];
    for (int64_t j = 0; j < n; ++j) {
        double d = L[j * n + j];
        for (int64_t k = 0; k < j; ++k) d -= L[j * n + k] * L[j * n + k];
        if (!(d > 0.0)) {
            free(L);
            return OR_ERR_NOT_SPD;
        }
        double ljj = sqrt(d);
        L[j * n + j] = ljj;
        for (int64_t i = j + 1; i < n; ++i) {
            double s = L[i * n + j];
            for (int64_t k = 0; k < j; ++k) s -= L[i * n + k] * L[j * n + k];
            L[i * n + j] = s / ljj;
        }
    }
    for (int64_t i = 0; i < n; ++i)
        for (int64_t j = i + 1; j < n; ++j) L[i * n + j] = 0.0;
    *Lout = L;
    return OR_OK;
}

static void cholesky_solve(int64_t n, const double* L, const double* b, double* x) {
    for (int64_t i = 0; i < n; ++i) {
        double s = b[i];
        for (int64_t k = 0; k < i; ++k) s -= L[i * n + k] * x[k];
        x[i] = s / L[i * n + i];
    }
    for (int64_t i = n - 1; i >= 0; --i) {
        double s = x[i];
        for (int64_t k = i + 1; k < n; ++k) s -= L[k * n + i] * x[k];
        x[i] = s / L[i * n + i];
    }
}

static void level_free(olevel* L) {
    or_csr_free(L->A);
    or_csr_free(L->P);
    or_csr_free(L->R);
    free(L->agg);
    free(L->pval);
    free(L->w);
    free(L->m);
    free(L->L);
    or_csr_free(L->Wd);
    or_csr_free(L->Z);
}

/* Build the hierarchy, O1-O9. */
ohier* or_build(const ocsr* A0, const double* w0, int32_t sweeps_per_level,
                int32_t smooth_prolongator, double prol_omega_scale, int64_t max_coarse_size,
                int32_t max_levels, double min_coarsening_ratio, int32_t pre_sweeps,
                int32_t post_sweeps, int32_t* status) {
    *status = OR_OK;
    if (sweeps_per_level < 1 || max_coarse_size < 1 || max_levels < 1 || pre_sweeps < 1 ||
        post_sweeps < 1 || !(prol_omega_scale > 0.0)) {
        *status = OR_ERR_ARG;
        return NULL;
    }
    int64_t n0 = A0->nrows;
    double* w = (double*)xmalloc(sizeof(double) * (size_t)n0);
    for (int64_t i = 0; i < n0; ++i) w[i] = w0 ? w0[i] : 1.0; /* PAPER.md:264 w = 1 */
    int st = validate(A0, w);
    if (st != OR_OK) {
        free(w);
        *status = st;
        return NULL;
    }
    ohier* h = (ohier*)xcalloc(1, sizeof(ohier));
    h->lv = (olevel*)xcalloc((size_t)max_levels, sizeof(olevel));
    h->pre = pre_sweeps;
    h->post = post_sweeps;
    ocsr* A = csr_clone(A0);
    int32_t l = 0;
    for (;;) {
        olevel* L = &h->lv[l];
        L->n = A->nrows;
        L->A = A;
        L->w = w;
        L->m = (double*)xmalloc(sizeof(double) * (size_t)L->n);
        or_l1_jacobi_inv(A, L->m); /* O7 */
        /* O1 stop test: n_l <= maxsize or l = max_levels - 1 */
        if (L->n <= max_coarse_size || l == max_levels - 1) break;
        /* O2 sweeps s = 1..m on (A_s, w_s) */
        int64_t n = L->n;
        int64_t* comp_agg = (int64_t*)xmalloc(sizeof(int64_t) * (size_t)n);
        double* comp_val = (double*)xmalloc(sizeof(double) * (size_t)n);
        for (int64_t i = 0; i < n; ++i) {
            comp_agg[i] = i;
            comp_val[i] = 1.0;
        }
        const ocsr* As = A;
        ocsr* As_owned = NULL;
        double* ws = (double*)xmalloc(sizeof(double) * (size_t)n);
        memcpy(ws, w, sizeof(double) * (size_t)n);
        int64_t ns = n;
        int32_t done = 0;
        for (int32_t s = 0; s < sweeps_per_level; ++s) {
            int64_t* agg = (int64_t*)xmalloc(sizeof(int64_t) * (size_t)ns);
            double* pv = (double*)xmalloc(sizeof(double) * (size_t)ns);
            double* wn = (double*)xmalloc(sizeof(double) * (size_t)ns);
            int64_t nc;
            ocsr* An = or_pairwise_sweep(As, ws, wn, agg, pv, &nc);
            if (nc == ns) { /* no size reduction: stop the sweeps */
                or_csr_free(An);
                free(agg);
                free(pv);
                free(wn);
                break;
            }
            /* O3: composite P = P_1 P_2 ... P_m, value ((p1*p2)*p3) in sweep order
             * (comp_val starts at 1.0 and 1.0*p1 == p1 exactly; NaN = no entry) */
            for (int64_t i = 0; i < n; ++i) {
                int64_t a = comp_agg[i];
                comp_val[i] = comp_val[i] * pv[a];
                comp_agg[i] = agg[a];
            }
            free(agg);
            free(pv);
            or_csr_free(As_owned);
            As_owned = An;
            As = An;
            free(ws);
            ws = wn;
            ns = nc;
            done++;
        }
        or_csr_free(As_owned);
        free(ws);
        /* O1 second half: a level that does not coarsen by >= min ratio is dropped */
        if (done == 0 || (double)n / (double)ns < min_coarsening_ratio) {
            free(comp_agg);
            free(comp_val);
            break;
        }
        int64_t nc = ns;
        ocsr* P = or_prolongator_csr(n, nc, comp_agg, comp_val);
        /* O4 + O5: smoothed prolongator (R3) */
        ocsr* Pb;
        if (smooth_prolongator) {
            L->omega = prol_omega_scale / or_dinv_a_inf_norm(A);
            Pb = or_smooth_prolongator(A, P, L->omega);
        } else {
            L->omega = 0.0;
            Pb = csr_clone(P);
        }
        /* O6: Galerkin A_{l+1} = P-bar^T A P-bar, mirrored; w_{l+1} = P^T w (R6) */
        ocsr* Ac = or_rap(Pb, A, Pb);
        or_mirror_drop(Ac);
        double* wc = (double*)xmalloc(sizeof(double) * (size_t)nc);
        restrict_weight(P, w, wc);
        or_csr_free(P);
        L->P = Pb;
        L->R = or_transpose(Pb);
        L->agg = comp_agg;
        L->pval = comp_val;
        L->sweeps = done;
        A = Ac;
        w = wc;
        l++;
    }
    h->nl = l + 1;
    olevel* C = &h->lv[l];
    st = dense_cholesky(C->A, &C->L); /* O8 */
    if (st != OR_OK) {
        *status = st;
        or_free(h);
        return NULL;
    }
    return h;
}

void or_free(ohier* h) {
    if (!h) return;
    for (int32_t l = 0; l < h->nl; ++l) level_free(&h->lv[l]);
    free(h->lv);
    free(h);
}

int32_t or_nlevels(const ohier* h) { return h->nl; }
const ocsr* or_level_A(const ohier* h, int32_t l) { return h->lv[l].A; }
const ocsr* or_level_P(const ohier* h, int32_t l) { return h->lv[l].P; }
int64_t or_level_n(const ohier* h, int32_t l) { return h->lv[l].n; }
void or_level_agg(const ohier* h, int32_t l, int64_t* agg) {
    memcpy(agg, h->lv[l].agg, sizeof(int64_t) * (size_t)h->lv[l].n);
}
void or_level_pval(const ohier* h, int32_t l, double* pval) {
    memcpy(pval, h->lv[l].pval, sizeof(double) * (size_t)h->lv[l].n);
}
void or_level_w(const ohier* h, int32_t l, double* w) {
    memcpy(w, h->lv[l].w, sizeof(double) * (size_t)h->lv[l].n);
}
void or_level_m(const ohier* h, int32_t l, double* m) {
    memcpy(m, h->lv[l].m, sizeof(double) * (size_t)h->lv[l].n);
}
double or_level_omega(const ohier* h, int32_t l) { return h->lv[l].omega; }
int32_t or_level_sweeps(const ohier* h, int32_t l) { return h->lv[l].sweeps; }

/* O9: operator complexity and average coarsening ratio
 * ((1/nl) sum n_l/n_{l+1}, taken over the nl-1 coarsening steps). */
double or_opc(const ohier* h) {
    double s = 0.0;
    for (int32_t l = 0; l < h->nl; ++l) s += (double)h->lv[l].A->rp[h->lv[l].n];
    return s / (double)h->lv[0].A->rp[h->lv[0].n];
}
double or_avg_cr(const ohier* h) {
    if (h->nl < 2) return 1.0;
    double s = 0.0;
    for (int32_t l = 0; l + 1 < h->nl; ++l) s += (double)h->lv[l].n / (double)h->lv[l + 1].n;
    return s / (double)(h->nl - 1);
}

/* ------------------------------------------------------------------ V-cycle */
/* Coarsest iterative solve: CG from x0 = 0
 * preconditioned by the l1-Jacobi diagonal of A_L, stopped as soon as the
 * relative residual is less than rtol, or after maxit iterations. */
/* z = M^{-1} r of the coarse CG: the l1-Jacobi diagonal m, or (Wd != NULL) the INVK
 * factors z = Z (Wd r) (VA3S3CS1). */
static void coarse_prec_apply(const double* m, const ocsr* Wd, const ocsr* Z, int64_t n, const double* r,
                              double* z, double* t) {
    if (Wd) {
        or_spmv(Wd, r, t);
        or_spmv(Z, t, z);
    } else {
        for (int64_t i = 0; i < n; ++i) z[i] = m[i] * r[i];
    }
}

static void coarse_pcg(const ocsr* A, const double* m, const ocsr* Wd, const ocsr* Z, int64_t n, double rtol,
                       int32_t maxit, const double* b, double* x) {
    double* r = (double*)xmalloc(sizeof(double) * (size_t)n);
    double* z = (double*)xmalloc(sizeof(double) * (size_t)n);
    double* p = (double*)xmalloc(sizeof(double) * (size_t)n);
    double* q = (double*)xmalloc(sizeof(double) * (size_t)n);
    double* t = (double*)xmalloc(sizeof(double) * (size_t)n);
    for (int64_t i = 0; i < n; ++i) {
        x[i] = 0.0;
        r[i] = b[i];
    }
    coarse_prec_apply(m, Wd, Z, n, r, z, t);
    for (int64_t i = 0; i < n; ++i) p[i] = z[i];
    double bnorm = sqrt(dot(n, b, b));
    double rho = dot(n, r, z);
    if (bnorm > 0.0) {
        for (int32_t k = 1; k <= maxit; ++k) {
            or_spmv(A, p, q);
            double pq = dot(n, p, q);
            if (!(pq > 0.0)) break;
            double alpha = rho / pq;
            for (int64_t i = 0; i < n; ++i) {
                x[i] = x[i] + alpha * p[i];
                r[i] = r[i] - alpha * q[i];
            }
            if (sqrt(dot(n, r, r)) / bnorm < rtol) break;
            coarse_prec_apply(m, Wd, Z, n, r, z, t);
            double rho_new = dot(n, r, z);
            double beta = rho_new / rho;
            #pragma omp parallel for schedule(static) if (g_threads > 1) num_threads(g_threads)
            for (int64_t i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
            rho = rho_new;
        }
    }
    free(r);
    free(z);
    free(p);
    free(q);
    free(t);
}

void or_set_coarse_cg(ohier* h, int32_t on, double rtol, int32_t maxit) {
    h->coarse_cg = on;
    h->coarse_rtol = rtol;
    h->coarse_maxit = maxit;
}

static void vcycle_rec(const ohier* h, int32_t l, const double* b, double* x);

void or_set_cycle(ohier* h, int32_t cycle) { h->cycle = cycle; }

/* ------------------------------------------------------------------ INVK
 * "inversion and sparsification of an incomplete factorization
 * ... in the form M = L D L^T ... M^{-1} = L^{-T} D^{-1} L^{-1} = Z D^{-1} Z^T ...
 * positional dropping", Table 1 caption: "the incomplete LU factorization with 0
 * levels of fill-in, and admitting a single level of fill-in in the inversion".
 * Readings (I1-I3): ILU(0) of an s.p.d. matrix in LDL^T form is IC(0) on
 * the pattern of A; the inverse W = L^{-1} keeps the entries of level <= fill where
 * the diagonal and the pattern of L have level 0 and an entry first created through
 * l_ik w_kj has level lev(w_kj) + 1; the kept entries satisfy the truncated recurrence.
 * One block (the whole level) per process: with one process HINVK = INVK. */

/* IC(0): strict lower L (pattern of tril(A)) and pivots d.  Returns 0 on a non-positive pivot. */
static int ic0(const ocsr* A, ocsr** Lout, double* d) {
    int64_t n = A->nrows;
    int64_t* rp = (int64_t*)xcalloc((size_t)n + 1, sizeof(int64_t));
    for (int64_t i = 0; i < n; ++i) {
        int64_t c = 0;
        for (int64_t k = A->rp[i]; k < A->rp[i + 1]; ++k) c += (A->ci[k] < i);
        rp[i + 1] = rp[i] + c;
    }
    ocsr* L = (ocsr*)xcalloc(1, sizeof(ocsr));
    L->nrows = L->ncols = n;
    L->rp = rp;
    L->ci = (int64_t*)xmalloc(sizeof(int64_t) * (size_t)rp[n]);
    L->v = (double*)xmalloc(sizeof(double) * (size_t)rp[n]);
    for (int64_t i = 0; i < n; ++i) {
        int64_t o = rp[i];
        double aii = 0.0;
        for (int64_t k = A->rp[i]; k < A->rp[i + 1]; ++k) {
            if (A->ci[k] < i) {
                L->ci[o] = A->ci[k];
                L->v[o] = A->v[k];
                ++o;
            } else if (A->ci[k] == i) {
                aii = A->v[k];
            }
        }
        /* l_ij = (a_ij - sum_{k < j} (l_ik d_k) l_jk) / d_j, j ascending, k ascending */
        for (int64_t t = rp[i]; t < rp[i + 1]; ++t) {
            int64_t j = L->ci[t];
            double sv = L->v[t];
            int64_t q = L->rp[j];
            for (int64_t u = rp[i]; u < t; ++u) {
                int64_t k = L->ci[u];
                while (q < L->rp[j + 1] && L->ci[q] < k) ++q;
                if (q < L->rp[j + 1] && L->ci[q] == k) sv = sv - (L->v[u] * d[k]) * L->v[q];
            }
            L->v[t] = sv / d[j];
        }
        double di = aii;
        for (int64_t t = rp[i]; t < rp[i + 1]; ++t) di = di - (L->v[t] * L->v[t]) * d[L->ci[t]];
        if (!(di > 0.0)) {
            or_csr_free(L);
            return 0;
        }
        d[i] = di;
    }
    *Lout = L;
    return 1;
}

/* W = L^{-1} truncated to fill level <= fill, row by row:
 *   w_i = e_i - sum_{k in row i of L, ascending} l_ik w_k   (rows w_k already truncated),
 * each w_ij accumulated in arrival order (k ascending, then the columns of row k
 * ascending) and negated; lev(i,j) = 0 for j = i and the pattern of L, otherwise
 * min over the contributing k of lev(k,j) + 1.  W has a unit diagonal (last in row). */
static ocsr* invk_inverse(const ocsr* L, int32_t fill) {
    int64_t n = L->nrows;
    double* acc = (double*)xcalloc((size_t)n, sizeof(double));
    int32_t* lev = (int32_t*)xmalloc(sizeof(int32_t) * (size_t)n);
    int64_t* mark = (int64_t*)xmalloc(sizeof(int64_t) * (size_t)n);
    int64_t* cols = (int64_t*)xmalloc(sizeof(int64_t) * (size_t)n);
    for (int64_t j = 0; j < n; ++j) mark[j] = -1;
    int64_t cap = 16 * n + 16, nnz = 0;
    int64_t* rp = (int64_t*)xcalloc((size_t)n + 1, sizeof(int64_t));
    int64_t* ci = (int64_t*)xmalloc(sizeof(int64_t) * (size_t)cap);
    double* v = (double*)xmalloc(sizeof(double) * (size_t)cap);
    int32_t* lv = (int32_t*)xmalloc(sizeof(int32_t) * (size_t)cap);
    for (int64_t i = 0; i < n; ++i) {
        int64_t nc = 0;
        for (int64_t t = L->rp[i]; t < L->rp[i + 1]; ++t) {
            int64_t j = L->ci[t];
            mark[j] = i;
            acc[j] = 0.0;
            lev[j] = 0;
            cols[nc++] = j;
        }
        for (int64_t t = L->rp[i]; t < L->rp[i + 1]; ++t) {
            int64_t k = L->ci[t];
            double lik = L->v[t];
            for (int64_t q = rp[k]; q < rp[k + 1]; ++q) {
                int64_t j = ci[q];
                int32_t cl = lv[q] + 1;
                if (mark[j] != i) {
                    mark[j] = i;
                    acc[j] = 0.0;
                    lev[j] = cl;
                    cols[nc++] = j;
                } else if (cl < lev[j]) {
                    lev[j] = cl;
                }
                acc[j] = acc[j] + lik * v[q];
            }
        }
        /* keep level <= fill, ascending columns, then the unit diagonal */
        for (int64_t a = 1; a < nc; ++a) { /* insertion sort (rows are short) */
            int64_t x = cols[a], b = a - 1;
            while (b >= 0 && cols[b] > x) {
                cols[b + 1] = cols[b];
                --b;
            }
            cols[b + 1] = x;
        }
        if (nnz + nc + 1 > cap) {
            cap = 2 * (nnz + nc + 1);
            ci = (int64_t*)realloc(ci, sizeof(int64_t) * (size_t)cap);
            v = (double*)realloc(v, sizeof(double) * (size_t)cap);
            lv = (int32_t*)realloc(lv, sizeof(int32_t) * (size_t)cap);
            if (!ci || !v || !lv) abort();
        }
        for (int64_t a = 0; a < nc; ++a) {
            int64_t j = cols[a];
            if (lev[j] <= fill) {
                ci[nnz] = j;
                v[nnz] = -acc[j];
                lv[nnz] = lev[j];
                ++nnz;
            }
        }
        ci[nnz] = i;
        v[nnz] = 1.0;
        lv[nnz] = 0;
        ++nnz;
        rp[i + 1] = nnz;
    }
    ocsr* W = (ocsr*)xcalloc(1, sizeof(ocsr));
    W->nrows = W->ncols = n;
    W->rp = rp;
    W->ci = ci;
    W->v = v;
    free(lv);
    free(acc);
    free(lev);
    free(mark);
    free(cols);
    return W;
}

/* INVK factors of level l from the matrix B (A_l or its block-diagonal part):
 * Wd = D^{-1} W (row i scaled by 1/d_i) and Z = W^T, so that
 * M^{-1} r = W^T D^{-1} W r = Z (Wd r).  Returns 0 on an IC(0) breakdown. */
static int invk_level(olevel* Lv, const ocsr* B, int32_t fill) {
    int64_t n = Lv->n;
    double* d = (double*)xmalloc(sizeof(double) * (size_t)n);
    ocsr* L = NULL;
    if (!ic0(B, &L, d)) {
        free(d);
        return 0;
    }
    ocsr* W = invk_inverse(L, fill);
    or_csr_free(L);
    Lv->Z = or_transpose(W);
    for (int64_t i = 0; i < n; ++i)
        for (int64_t k = W->rp[i]; k < W->rp[i + 1]; ++k) W->v[k] = W->v[k] / d[i];
    Lv->Wd = W;
    free(d);
    return 1;
}

/* The matrix whose INVK factors the smoother uses, in the parallel block-Jacobi setting
 * of PAPER.md:165-170 and 178-181 ("we will always consider the case of computing the
 * decomposition M for the diagonal blocks A_pp of A"; "the l1-modification ... computing
 * the approximate inverse of the A_pp + D_l1,p blocks"): entries a_ij with owner(i) !=
 * owner(j) are dropped; with l1 = 1, row i's diagonal gains sum_{j: owner(j) != owner(i)}
 * |a_ij| (Eq. 3.5, the off-block l1 weights, summed in ascending column order).  One block
 * (owner == NULL) leaves A unchanged: HINVK = l1-INVK = INVK. */
static ocsr* block_diag_part(const ocsr* A, const int32_t* owner, int32_t l1) {
    int64_t n = A->nrows;
    ocsr* B = csr_alloc(n, n, A->rp[n]);
    int64_t o = 0;
    for (int64_t i = 0; i < n; ++i) {
        double off = 0.0;
        for (int64_t k = A->rp[i]; k < A->rp[i + 1]; ++k)
            if (owner && owner[A->ci[k]] != owner[i]) off = off + fabs(A->v[k]);
        for (int64_t k = A->rp[i]; k < A->rp[i + 1]; ++k) {
            int64_t j = A->ci[k];
            if (owner && owner[j] != owner[i]) continue;
            B->ci[o] = j;
            B->v[o] = (j == i && l1) ? A->v[k] + off : A->v[k];
            ++o;
        }
        B->rp[i + 1] = o;
    }
    return B;
}

/* Block owner of every row of every level (R18): level 0 rows belong to the blocks
 * [bounds0[p], bounds0[p+1]); a coarse row belongs to the block that owns the minimum
 * member of its aggregate. */
static int32_t** level_owners(const ohier* h, int32_t nblocks, const int64_t* bounds0) {
    int32_t** own = (int32_t**)xcalloc((size_t)h->nl, sizeof(int32_t*));
    for (int32_t l = 0; l < h->nl; ++l) {
        int64_t n = h->lv[l].n;
        own[l] = (int32_t*)xmalloc(sizeof(int32_t) * (size_t)n);
        if (l == 0) {
            for (int32_t p = 0; p < nblocks; ++p)
                for (int64_t i = bounds0[p]; i < bounds0[p + 1]; ++i) own[0][i] = p;
        } else {
            const olevel* F = &h->lv[l - 1];
            for (int64_t g = 0; g < n; ++g) own[l][g] = -1;
            for (int64_t i = 0; i < F->n; ++i) /* ascending i: the first member seen is the minimum */
                if (own[l][F->agg[i]] < 0) own[l][F->agg[i]] = own[l - 1][i];
        }
    }
    return own;
}

int32_t or_set_smoother_ex(ohier* h, int32_t kind, int32_t fill, int32_t nblocks, const int64_t* bounds0,
                           int32_t l1, const int32_t* fill_per_level) {
    h->smoother = kind;
    if (kind != 1 && !h->coarse_prec) return OR_OK;
    if (nblocks < 1 || (nblocks > 1 && (!bounds0 || bounds0[0] != 0 || bounds0[nblocks] != h->lv[0].n)))
        return OR_ERR_ARG;
    for (int32_t p = 0; nblocks > 1 && p < nblocks; ++p)
        if (bounds0[p + 1] < bounds0[p]) return OR_ERR_ARG;
    int32_t** own = nblocks > 1 ? level_owners(h, nblocks, bounds0) : NULL;
    int32_t st = OR_OK;
    /* every non-coarsest level (smoother), and the coarsest when it is the coarse CG's
     * preconditioner */
    for (int32_t l = 0; l < h->nl; ++l) {
        olevel* Lv = &h->lv[l];
        or_csr_free(Lv->Wd);
        or_csr_free(Lv->Z);
        Lv->Wd = Lv->Z = NULL;
        if (l == h->nl - 1 ? !h->coarse_prec : kind != 1) continue;
        /* "a single level of fill-in in the inversion" on every level; a
         * per-level override exists only to express the library's non-default knob */
        int32_t f = fill_per_level ? fill_per_level[l] : fill;
        ocsr* B = block_diag_part(Lv->A, own ? own[l] : NULL, l1);
        int ok = invk_level(Lv, B, f);
        or_csr_free(B);
        if (!ok) {
            st = OR_ERR_NOT_SPD;
            break;
        }
    }
    if (own) {
        for (int32_t l = 0; l < h->nl; ++l) free(own[l]);
        free(own);
    }
    return st;
}

int32_t or_set_smoother(ohier* h, int32_t kind, int32_t fill) {
    return or_set_smoother_ex(h, kind, fill, 1, NULL, 0, NULL);
}

void or_set_coarse_prec(ohier* h, int32_t kind) { h->coarse_prec = kind; }

const ocsr* or_level_invk(const ohier* h, int32_t l, int32_t which) {
    return which == 0 ? h->lv[l].Wd : h->lv[l].Z;
}

/* one smoothing step x = x + M^{-1}(b - A x) (or x = M^{-1} b from zero) with the
 * level's smoother: l1-Jacobi m o (.) or INVK Z (Wd (.)) */
static void smooth_apply(const ohier* h, const olevel* Lv, const double* res, double* out, double* tmp) {
    int64_t n = Lv->n;
    if (h->smoother == 1) {
        or_spmv(Lv->Wd, res, tmp);
        or_spmv(Lv->Z, tmp, out);
    } else {
        #pragma omp parallel for schedule(static) if (g_threads > 1) num_threads(g_threads)
        for (int64_t i = 0; i < n; ++i) out[i] = Lv->m[i] * res[i];
    }
}

int64_t or_coarse_visits(const ohier* h) { return h->coarse_visits; }
int64_t or_level_visits(const ohier* h, int32_t l) { return (l >= 0 && l < 64) ? h->visits[l] : 0; }

/* K-cycle coarse correction ("at each level except the fine and the
 * coarsest ones we apply two iterations of a Flexible Conjugate Gradient (FCG)
 * method with the already defined AMG method starting on the current level as
 * preconditioner"): two FCG(1) iterations on A_l x = b from x = 0, preconditioned
 * by the cycle rooted at level l, no residual test:
 *   z = B_l r; p = z; q = A p; alpha = p.r / p.q; x += alpha p; r -= alpha q;
 *   z = B_l r; beta = -(z.q)/(p.q); p = z + beta p; q = A p; alpha = p.r / p.q;
 *   x += alpha p.
 * If p.q <= 0 the iteration stops and returns the current x. */
static void kcycle_fcg2(const ohier* h, int32_t l, const double* b, double* x) {
    const olevel* L = &h->lv[l];
    int64_t n = L->n;
    double* r = (double*)xmalloc(sizeof(double) * (size_t)n);
    double* z = (double*)xmalloc(sizeof(double) * (size_t)n);
    double* p = (double*)xmalloc(sizeof(double) * (size_t)n);
    double* q = (double*)xmalloc(sizeof(double) * (size_t)n);
    for (int64_t i = 0; i < n; ++i) {
        x[i] = 0.0;
        r[i] = b[i];
    }
    double pq = 0.0;
    for (int32_t it = 0; it < 2; ++it) {
        vcycle_rec(h, l, r, z);
        if (it == 0) {
            memcpy(p, z, sizeof(double) * (size_t)n);
        } else {
            double beta = -dot(n, z, q) / pq;
            #pragma omp parallel for schedule(static) if (g_threads > 1) num_threads(g_threads)
            for (int64_t i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
        }
        or_spmv(L->A, p, q);
        pq = dot(n, p, q);
        if (!(pq > 0.0)) break;
        double alpha = dot(n, p, r) / pq;
#pragma omp parallel for schedule(static) if (g_threads > 1) num_threads(g_threads)
        for (int64_t i = 0; i < n; ++i) {
            x[i] = x[i] + alpha * p[i];
            r[i] = r[i] - alpha * q[i];
        }
    }
    free(r);
    free(z);
    free(p);
    free(q);
}

/* O10, Eq. 3.1: x = m.b; (s1-1) sweeps x += m.(b - A x);
 * e = V(l+1, P-bar^T (b - A x)); x += P-bar e; s2 sweeps; at l = L: A_L^{-1} b.
 * With the K-cycle (h->cycle == 1) the coarse correction e of every level l whose
 * coarse level l+1 is not the coarsest is kcycle_fcg2(l+1, P-bar^T (b - A x)). */
static void vcycle_rec(const ohier* h, int32_t l, const double* b, double* x) {
    const olevel* L = &h->lv[l];
    int64_t n = L->n;
    if (l < 64) ((ohier*)h)->visits[l] += 1;
    if (l == h->nl - 1) {
        ((ohier*)h)->coarse_visits += 1;
        if (h->coarse_cg)
            coarse_pcg(L->A, L->m, h->coarse_prec ? L->Wd : NULL, L->Z, n, h->coarse_rtol, h->coarse_maxit, b, x);
        else
            cholesky_solve(n, L->L, b, x);
        return;
    }
    double* t = (double*)xmalloc(sizeof(double) * (size_t)n);
    double* xn = (double*)xmalloc(sizeof(double) * (size_t)n);
    double* u = (double*)xmalloc(sizeof(double) * (size_t)n);
    double* tmp = (double*)xmalloc(sizeof(double) * (size_t)n);
    smooth_apply(h, L, b, x, tmp); /* first pre-sweep from x = 0: x = M^{-1} b */
    for (int32_t s = 1; s < h->pre; ++s) {
        or_spmv(L->A, x, t);
        #pragma omp parallel for schedule(static) if (g_threads > 1) num_threads(g_threads)
        for (int64_t i = 0; i < n; ++i) t[i] = b[i] - t[i];
        smooth_apply(h, L, t, u, tmp);
        #pragma omp parallel for schedule(static) if (g_threads > 1) num_threads(g_threads)
        for (int64_t i = 0; i < n; ++i) xn[i] = x[i] + u[i];
        memcpy(x, xn, sizeof(double) * (size_t)n);
    }
    or_spmv(L->A, x, t);
    #pragma omp parallel for schedule(static) if (g_threads > 1) num_threads(g_threads)
    for (int64_t i = 0; i < n; ++i) t[i] = b[i] - t[i];
    int64_t nc = h->lv[l + 1].n;
    double* bc = (double*)xmalloc(sizeof(double) * (size_t)nc);
    double* ec = (double*)xmalloc(sizeof(double) * (size_t)nc);
    or_spmv(L->R, t, bc); /* P-bar^T r, ascending fine index per coarse row */
    if (h->cycle == 1 && l + 1 < h->nl - 1)
        kcycle_fcg2(h, l + 1, bc, ec);
    else
        vcycle_rec(h, l + 1, bc, ec);
    or_spmv(L->P, ec, t);
    #pragma omp parallel for schedule(static) if (g_threads > 1) num_threads(g_threads)
    for (int64_t i = 0; i < n; ++i) x[i] = x[i] + t[i];
    for (int32_t s = 0; s < h->post; ++s) { /* post-smoothing with M^T = M */
        or_spmv(L->A, x, t);
        #pragma omp parallel for schedule(static) if (g_threads > 1) num_threads(g_threads)
        for (int64_t i = 0; i < n; ++i) t[i] = b[i] - t[i];
        smooth_apply(h, L, t, u, tmp);
        #pragma omp parallel for schedule(static) if (g_threads > 1) num_threads(g_threads)
        for (int64_t i = 0; i < n; ++i) xn[i] = x[i] + u[i];
        memcpy(x, xn, sizeof(double) * (size_t)n);
    }
    free(t);
    free(xn);
    free(u);
    free(tmp);
    free(bc);
    free(ec);
}

void or_vcycle(const ohier* h, const double* r, double* z) { vcycle_rec(h, 0, r, z); }

static double dot(int64_t n, const double* a, const double* b) {
    if (g_threads > 1 && n >= 4 * OR_CHUNKS) {
        double part[OR_CHUNKS];
#pragma omp parallel for schedule(static) num_threads(g_threads)
        for (int c = 0; c < OR_CHUNKS; ++c) {
            int64_t i0 = n * c / OR_CHUNKS, i1 = n * (c + 1) / OR_CHUNKS;
            double s = 0.0;
            for (int64_t i = i0; i < i1; ++i) s += a[i] * b[i];
            part[c] = s;
        }
        double s = 0.0;
        for (int c = 0; c < OR_CHUNKS; ++c) s += part[c];
        return s;
    }
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += a[i] * b[i];
    return s;
}

/* O11: PCG, x0 = 0, stop when ||r_k||/||b|| <= rtol (R12).
 * rtol = 0 runs exactly maxit iterations (fixed-count parity mode). */
int32_t or_pcg(const ohier* h, const double* b, double* x, double rtol, int32_t maxit,
               int32_t* iters, double* relres, double* true_relres, double* hist) {
    const ocsr* A = h->lv[0].A;
    int64_t n = h->lv[0].n;
    double* r = (double*)xmalloc(sizeof(double) * (size_t)n);
    double* z = (double*)xmalloc(sizeof(double) * (size_t)n);
    double* p = (double*)xmalloc(sizeof(double) * (size_t)n);
    double* q = (double*)xmalloc(sizeof(double) * (size_t)n);
    int32_t st = OR_NOT_CONVERGED;
    for (int64_t i = 0; i < n; ++i) {
        x[i] = 0.0;
        r[i] = b[i];
    }
    double bnorm = sqrt(dot(n, b, b));
    *iters = 0;
    *relres = 0.0;
    if (hist) hist[0] = 1.0;
    if (bnorm == 0.0) {
        *true_relres = 0.0;
        st = OR_OK;
        goto done;
    }
    *relres = 1.0;
    or_vcycle(h, r, z);
    memcpy(p, z, sizeof(double) * (size_t)n);
    double rho = dot(n, r, z);
    for (int32_t k = 1; k <= maxit; ++k) {
        or_spmv(A, p, q);
        double pq = dot(n, p, q);
        if (!(pq > 0.0)) {
            st = OR_BREAKDOWN;
            break;
        }
        double alpha = rho / pq;
#pragma omp parallel for schedule(static) if (g_threads > 1) num_threads(g_threads)
        for (int64_t i = 0; i < n; ++i) {
            x[i] = x[i] + alpha * p[i];
            r[i] = r[i] - alpha * q[i];
        }
        double rel = sqrt(dot(n, r, r)) / bnorm;
        *iters = k;
        *relres = rel;
        if (hist) hist[k] = rel;
        if (rel <= rtol) {
            st = OR_OK;
            break;
        }
        or_vcycle(h, r, z);
        double rho_new = dot(n, r, z);
        double beta = rho_new / rho;
        #pragma omp parallel for schedule(static) if (g_threads > 1) num_threads(g_threads)
        for (int64_t i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
        rho = rho_new;
    }
    or_spmv(A, x, q);
    for (int64_t i = 0; i < n; ++i) q[i] = b[i] - q[i];
    *true_relres = sqrt(dot(n, q, q)) / bnorm;
done:
    free(r);
    free(z);
    free(p);
    free(q);
    return st;
}

/* FCG(1): flexible CG with one-direction
 * orthogonalisation, x0 = 0, for a (possibly nonlinear) preconditioner B:
 *   z_k = B r_k; p_k = z_k - ((z_k^T q_{k-1}) / (p_{k-1}^T q_{k-1})) p_{k-1} (p_0 = z_0);
 *   q_k = A p_k; alpha = (p_k^T r_k) / (p_k^T q_k); x += alpha p_k; r -= alpha q_k;
 * stop when ||r_k||/||b|| <= rtol.  Returns as or_pcg. */
int32_t or_fcg(const ohier* h, const double* b, double* x, double rtol, int32_t maxit, int32_t* iters,
               double* relres, double* true_relres, double* hist) {
    const ocsr* A = h->lv[0].A;
    int64_t n = h->lv[0].n;
    double* r = (double*)xmalloc(sizeof(double) * (size_t)n);
    double* z = (double*)xmalloc(sizeof(double) * (size_t)n);
    double* p = (double*)xmalloc(sizeof(double) * (size_t)n);
    double* q = (double*)xmalloc(sizeof(double) * (size_t)n);
    int32_t st = OR_NOT_CONVERGED;
    for (int64_t i = 0; i < n; ++i) {
        x[i] = 0.0;
        r[i] = b[i];
    }
    double bnorm = sqrt(dot(n, b, b));
    *iters = 0;
    *relres = 0.0;
    if (hist) hist[0] = 1.0;
    if (bnorm == 0.0) {
        *true_relres = 0.0;
        st = OR_OK;
        goto done;
    }
    *relres = 1.0;
    double pq_prev = 0.0;
    for (int32_t k = 1; k <= maxit; ++k) {
        or_vcycle(h, r, z);
        if (k == 1) {
            memcpy(p, z, sizeof(double) * (size_t)n);
        } else {
            double beta = -dot(n, z, q) / pq_prev;
            #pragma omp parallel for schedule(static) if (g_threads > 1) num_threads(g_threads)
            for (int64_t i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
        }
        or_spmv(A, p, q);
        double pq = dot(n, p, q);
        if (!(pq > 0.0)) {
            st = OR_BREAKDOWN;
            break;
        }
        double alpha = dot(n, p, r) / pq;
#pragma omp parallel for schedule(static) if (g_threads > 1) num_threads(g_threads)
        for (int64_t i = 0; i < n; ++i) {
            x[i] = x[i] + alpha * p[i];
            r[i] = r[i] - alpha * q[i];
        }
        pq_prev = pq;
        double rel = sqrt(dot(n, r, r)) / bnorm;
        *iters = k;
        *relres = rel;
        if (hist) hist[k] = rel;
        if (rel <= rtol) {
            st = OR_OK;
            break;
        }
    }
    or_spmv(A, x, q);
    for (int64_t i = 0; i < n; ++i) q[i] = b[i] - q[i];
    *true_relres = sqrt(dot(n, q, q)) / bnorm;
done:
    free(r);
    free(z);
    free(p);
    free(q);
    return st;
}
