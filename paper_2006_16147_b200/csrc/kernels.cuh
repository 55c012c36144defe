// kernels.cuh — sm_100a device kernels of the AMG-PCG solve phase.
//
// Everything on the hot path is an fp64 sparse row reduction (~0.17 flop/B, HBM
// bound; no tensor-core contraction exists here).  One kernel
// family covers every step of the V-cycle (Eq. 3.1) and of PCG:
//
//   y_i = E( i, sum_k  a_ik * G(col_k) )
//
// with a Gather functor G (x_j, or m_j*b_j for the first sweep from x = 0) and an
// Epilogue functor E (residual, l1-Jacobi update, restriction store, prolongation
// update, SpMV + dot ...).  Two storage formats:
//   * SELL-32: slices of 32 consecutive rows stored column-major, one warp per
//     slice, so every lane's k-th entry is one coalesced 256 B (values) + 128 B
//     (indices) transaction; used for short rows with little padding (levels 0-1,
//     prolongators, restrictions).
//   * CSR-vector: VW lanes per row with a shuffle row reduction; used for the long
//     rows of the deep levels (hundreds to thousands of entries per row).
// Grids are persistent-style (a multiple of the SM count x resident blocks),
// rows are visited grid-stride.  Dot products are fused into the epilogue and
// reduced deterministically: per-block tree, then the last block to finish sums
// the block partials in a fixed order and runs a PCG "finisher" that computes
// alpha / beta / the convergence test on the device (and sets the CUDA-graph
// WHILE condition), so no host round trip happens inside a solve.
#pragma once
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

namespace cg = cooperative_groups;

namespace amgk {

constexpr int kBlock = 256;

// --------------------------------------------------------------- PCG state
enum PcgStatus : int32_t { ST_RUNNING = 0, ST_CONVERGED = 1, ST_MAXIT = 2, ST_BREAKDOWN = 3, ST_ZERO_RHS = 4 };

struct PcgState {
    double rho;     // r^T z of the current iterate
    double alpha, beta;
    double bnorm;   // ||b||_2
    double relres;  // ||r_k|| / ||b||
    double rtol;
    double pr;      // FCG: p_k^T r_k
    double pqprev;  // FCG: p_{k-1}^T q_{k-1}
    int32_t iter, maxit, status, pad;
};

// FIN_ZQ / FIN_PR / FIN_PQF are the FCG(1) finishers:
//   beta = -(z_k^T q_{k-1}) / (p_{k-1}^T q_{k-1}),  alpha = (p_k^T r_k) / (p_k^T q_k).
// FIN_K* drive the two inner FCG(1) iterations of the K-cycle on a
// per-level state k[] = {p^T r, p^T q, alpha, beta, stop}.
enum FinishKind : int32_t {
    FIN_NONE = 0, FIN_BNORM = 1, FIN_RZ = 2, FIN_PQ = 3, FIN_RR = 4, FIN_ZQ = 5, FIN_PR = 6, FIN_PQF = 7,
    FIN_KPR0 = 8, FIN_KPR = 9, FIN_KALPHA = 10, FIN_KBETA = 11, FIN_KALPHA2 = 12, FIN_KALPHA1 = 13, FIN_KPR0ALPHA1 = 14
};
// Multi-rank: a dot kernel only writes its local total (rc.out, kind FIN_NONE);
// the per-rank totals are all-gathered and k_finish sums them in rank order.

struct RedCtx {
    double* partials;     // >= gridDim.x doubles
    unsigned int* ticket; // zero-initialised counter, reset by the last block
    double* out;          // optional: total written here
    PcgState* st;
    unsigned long long cond;  // cudaGraphConditionalHandle of the PCG WHILE node (0 = none)
    int32_t kind;
    double* ks;               // K-cycle level state (FIN_K*), else nullptr
};

__device__ __forceinline__ void finish(const RedCtx& rc, double total) {
    if (rc.out) *rc.out = total;
    if (rc.ks) {
        double* k = rc.ks;
        switch (rc.kind) {
            case FIN_KPR0: k[4] = 0.0; k[0] = total; break;  // a new inner solve starts
            case FIN_KPR: k[0] = total; break;
            case FIN_KALPHA:  // alpha = p^T r / p^T q; p^T q <= 0 stops the inner solve (x kept)
                if (k[4] != 0.0 || !(total > 0.0)) {
                    k[2] = 0.0;
                    k[4] = 1.0;
                } else {
                    k[2] = k[0] / total;
                }
                k[1] = total;
                break;
            case FIN_KBETA: k[3] = (k[4] != 0.0) ? 0.0 : -total / k[1]; break;
            case FIN_KALPHA1:  // the first inner iteration's alpha, also kept as alpha_1 = k[5]
                if (k[4] != 0.0 || !(total > 0.0)) {
                    k[2] = 0.0;
                    k[4] = 1.0;
                } else {
                    k[2] = k[0] / total;
                }
                k[1] = total;
                k[5] = k[2];
                break;
            default: break;
        }
        return;
    }
    PcgState* st = rc.st;
    if (!st) return;
    switch (rc.kind) {
        case FIN_BNORM: {
            st->bnorm = sqrt(total);
            st->iter = 0;
            st->alpha = 0.0;
            st->beta = 0.0;
            st->rho = 0.0;
            if (total == 0.0) {
                st->status = ST_ZERO_RHS;
                st->relres = 0.0;
            } else {
                st->status = (st->maxit <= 0) ? ST_MAXIT : ST_RUNNING;
                st->relres = 1.0;
            }
            if (rc.cond) cudaGraphSetConditional(rc.cond, st->status == ST_RUNNING ? 1u : 0u);
            break;
        }
        case FIN_RZ: {  // rho' = r^T z ; beta = rho'/rho (0 on the first iteration)
            st->beta = (st->iter == 0) ? 0.0 : total / st->rho;
            st->rho = total;
            break;
        }
        case FIN_PQ: {  // alpha = rho / p^T q ; breakdown if p^T q <= 0
            if (!(total > 0.0)) {
                st->status = ST_BREAKDOWN;
                st->alpha = 0.0;
            } else {
                st->alpha = st->rho / total;
            }
            break;
        }
        case FIN_ZQ: {  // FCG: beta = -(z^T q_prev) / (p_prev^T q_prev) (0 on the first iteration)
            st->beta = (st->iter == 0) ? 0.0 : -total / st->pqprev;
            break;
        }
        case FIN_PR: {  // FCG: p^T r of the new direction
            st->pr = total;
            break;
        }
        case FIN_PQF: {  // FCG: alpha = p^T r / p^T q ; breakdown if p^T q <= 0
            if (!(total > 0.0)) {
                st->status = ST_BREAKDOWN;
                st->alpha = 0.0;
            } else {
                st->alpha = st->pr / total;
            }
            st->pqprev = total;
            break;
        }
        case FIN_RR: {  // convergence test on the recursive residual (reading R12)
            if (st->status == ST_RUNNING) {
                st->iter += 1;
                st->relres = sqrt(total) / st->bnorm;
                if (st->relres <= st->rtol) st->status = ST_CONVERGED;
                else if (st->iter >= st->maxit) st->status = ST_MAXIT;
            }
            if (rc.cond) cudaGraphSetConditional(rc.cond, st->status == ST_RUNNING ? 1u : 0u);
            break;
        }
        default:
            break;
    }
}

// FIN_KALPHA2 (K-cycle, fused direction update): t0 = p^T q, t1 = p^T r; then as FIN_KALPHA.
// FIN_KPR0ALPHA1 (K-cycle, collapsed inner level, first iteration): t0 = p^T q, t1 = p^T b;
// a new inner solve starts (as FIN_KPR0 with t1), then as FIN_KALPHA1 with t0.
__device__ __forceinline__ void finish2(const RedCtx& rc, double t0, double t1) {
    if (rc.ks && rc.kind == FIN_KALPHA2) {
        rc.ks[0] = t1;
        RedCtx r1 = rc;
        r1.kind = FIN_KALPHA;
        finish(r1, t0);
    } else if (rc.ks && rc.kind == FIN_KPR0ALPHA1) {
        rc.ks[4] = 0.0;
        rc.ks[0] = t1;
        RedCtx r1 = rc;
        r1.kind = FIN_KALPHA1;
        finish(r1, t0);
    }
}

// Deterministic grid reduction: fixed per-block tree, fixed-order sum of the
// block partials by the last block to arrive.
__device__ __forceinline__ void grid_reduce(double v, const RedCtx& rc) {
    __shared__ double wsum[kBlock / 32];
    __shared__ bool last;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) wsum[wid] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += wsum[w];
        rc.partials[blockIdx.x] = s;
        __threadfence();
        unsigned int t = atomicAdd(rc.ticket, 1u);
        last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    double s = 0.0;
    for (unsigned int b = threadIdx.x; b < gridDim.x; b += blockDim.x)
        s += ((volatile double*)rc.partials)[b];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) wsum[wid] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double tot = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += wsum[w];
        *rc.ticket = 0u;
        finish(rc, tot);
    }
}

// Two dots at once (same fixed trees, partials interleaved: 2 doubles per block).
__device__ __forceinline__ void finish2(const RedCtx& rc, double t0, double t1);
__device__ __forceinline__ void grid_reduce(double2 v, const RedCtx& rc) {
    __shared__ double wsum[2][kBlock / 32];
    __shared__ bool last;
    for (int o = 16; o > 0; o >>= 1) {
        v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
        v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) {
        wsum[0][wid] = v.x;
        wsum[1][wid] = v.y;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0, b = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
            a += wsum[0][w];
            b += wsum[1][w];
        }
        rc.partials[2 * blockIdx.x] = a;
        rc.partials[2 * blockIdx.x + 1] = b;
        __threadfence();
        unsigned int t = atomicAdd(rc.ticket, 1u);
        last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    double a = 0.0, b = 0.0;
    for (unsigned int q = threadIdx.x; q < gridDim.x; q += blockDim.x) {
        a += ((volatile double*)rc.partials)[2 * q];
        b += ((volatile double*)rc.partials)[2 * q + 1];
    }
    for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        b += __shfl_xor_sync(0xffffffffu, b, o);
    }
    if (lane == 0) {
        wsum[0][wid] = a;
        wsum[1][wid] = b;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double ta = 0.0, tb = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
            ta += wsum[0][w];
            tb += wsum[1][w];
        }
        *rc.ticket = 0u;
        finish2(rc, ta, tb);
    }
}

// ------------------------------------------------- programmatic dependent launch
// Every kernel is launched with programmatic stream serialization: it lets its
// dependents begin launching at once (their blocks take SM slots only as ours
// retire) and waits for its own prerequisites to complete and flush before it
// touches memory.  This overlaps launch latency and block ramp-up with the tail
// of the previous kernel — the deep levels are latency-bound.
__device__ __forceinline__ void pdl_begin() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
}

// ---------------------------------------------------------------- loads
__device__ __forceinline__ double ld_stream(const double* p) {
    double r;
    asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(r) : "l"(p));
    return r;
}
__device__ __forceinline__ int32_t ld_stream(const int32_t* p) {
    int32_t r;
    asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(r) : "l"(p));
    return r;
}
__device__ __forceinline__ int32_t ld_stream(const uint16_t* p) {
    unsigned short r;
    asm volatile("ld.global.nc.L1::no_allocate.u16 %0, [%1];" : "=h"(r) : "l"(p));
    return (int32_t)r;
}

// --------------------------------------------------------------- gathers
struct GVec {  // x_j
    static constexpr int kChunk = 8;
    const double* __restrict__ x;
    __device__ __forceinline__ double operator()(int32_t j) const { return __ldg(x + j); }
};
struct GMB {   // (m o b)_j : the first l1-Jacobi sweep from x = 0 (R9)
    static constexpr int kChunk = 4;
    const double* __restrict__ m;
    const double* __restrict__ b;
    __device__ __forceinline__ double operator()(int32_t j) const { return __ldg(m + j) * __ldg(b + j); }
};

// Functors whose operands depend on device-side PCG state (the p double buffer)
// resolve them once per thread at kernel start; every other functor is unchanged.
template <class T>
__device__ __forceinline__ void bind(T&) {}

// p_j = z_j + beta p_old_j (PCG direction update fused into q = A p; first
// iteration p = z).  p lives in two buffers that alternate every iteration:
// p_old = P[iter & 1], p_new = P[(iter + 1) & 1].
struct GPz {
    static constexpr int kChunk = 4;
    const double* __restrict__ z;
    const double* p0;
    const double* p1;
    const PcgState* st;
    const double* pold = nullptr;
    double beta = 0.0;
    bool first = true;
    __device__ __forceinline__ double operator()(int32_t j) const {
        return first ? __ldg(z + j) : __ldg(z + j) + beta * __ldg(pold + j);
    }
};
__device__ __forceinline__ void bind(GPz& g) {
    const int32_t it = g.st->iter;
    g.first = (it == 0);
    g.beta = g.st->beta;
    g.pold = (it & 1) ? g.p1 : g.p0;
}

// e_j = x_j + alpha p_j: the K-cycle inner FCG's final update, formed where its
// result is consumed (the prolongation); alpha = k[2] of the level's K state
struct GXap {
    static constexpr int kChunk = 4;
    const double* __restrict__ x;
    const double* __restrict__ p;
    const double* k;
    double alpha = 0.0;
    __device__ __forceinline__ double operator()(int32_t j) const { return __ldg(x + j) + alpha * __ldg(p + j); }
};
__device__ __forceinline__ void bind(GXap& g) { g.alpha = g.k[2]; }

// p_j = z_j + beta p_j: the K-cycle inner FCG's second direction formed in the
// gather of q = A p (beta = k[3] of the level's K state); cf. GPz for the outer PCG
struct GKpz {
    static constexpr int kChunk = 4;
    const double* __restrict__ z;
    const double* __restrict__ p;
    const double* k;
    double beta = 0.0;
    __device__ __forceinline__ double operator()(int32_t j) const { return __ldg(z + j) + beta * __ldg(p + j); }
};
__device__ __forceinline__ void bind(GKpz& g) { g.beta = g.k[3]; }

// e_j = alpha_1 p1_j + alpha_2 p2_j: the K-cycle inner FCG's result x = alpha_1 p_1 +
// alpha_2 p_2 (x_0 = 0), formed only where it is consumed (the prolongation)
struct GXap2 {
    static constexpr int kChunk = 4;
    const double* __restrict__ p1;
    const double* __restrict__ p2;
    const double* k;
    double a1 = 0.0, a2 = 0.0;
    __device__ __forceinline__ double operator()(int32_t j) const { return a1 * __ldg(p1 + j) + a2 * __ldg(p2 + j); }
};
__device__ __forceinline__ void bind(GXap2& g) {
    g.a1 = g.k[5];
    g.a2 = g.k[2];
}
// b_j - alpha q_j: the K-cycle inner residual r_1 = b - alpha_1 q_1, formed in the gather
// of the second cycle application's first kernel (alpha = k[2])
struct GBaq {
    static constexpr int kChunk = 4;
    const double* __restrict__ b;
    const double* __restrict__ q;
    const double* k;
    double alpha = 0.0;
    __device__ __forceinline__ double operator()(int32_t j) const { return __ldg(b + j) - alpha * __ldg(q + j); }
};
__device__ __forceinline__ void bind(GBaq& g) { g.alpha = g.k[2]; }

// m_j (b_j - alpha q_j): GMB over the K-cycle's second right-hand side (alpha = k[2])
struct GMBaq {
    static constexpr int kChunk = 4;
    const double* __restrict__ m;
    const double* __restrict__ b;
    const double* __restrict__ q;
    const double* k;
    double alpha = 0.0;
    __device__ __forceinline__ double operator()(int32_t j) const {
        return __ldg(m + j) * (__ldg(b + j) - alpha * __ldg(q + j));
    }
};
__device__ __forceinline__ void bind(GMBaq& g) { g.alpha = g.k[2]; }

// ------------------------------------------------------------- epilogues
// Epilogues that reduce two dot products at once declare `using dot_t = double2;`
// (the K-cycle's fused direction update: p^T q and p^T r in one pass).
__device__ __forceinline__ double2& operator+=(double2& a, const double2& b) {
    a.x += b.x;
    a.y += b.y;
    return a;
}
template <class E, class = void>
struct DotOf {
    using type = double;
};
template <class E>
struct DotOf<E, std::void_t<typename E::dot_t>> {
    using type = typename E::dot_t;
};

// An epilogue with `kAbs = true` also receives asum = sum_k |a_ik| of the row it
// streams, i.e. the l1-Jacobi diagonal 1/m_i (nb = 1), so m_i is
// recomputed in registers instead of being read from HBM.
template <class E>
__device__ __forceinline__ auto apply_epi(const E& e, int64_t i, double s, double asum) {
    if constexpr (E::kAbs) return e(i, s, asum);
    else return e(i, s);
}

// Epilogue operand prefetch: the row's own entries of the vectors an epilogue reads are
// requested into L2 before the row reduction starts, so the epilogue's loads (issued only once
// the reduction is done) do not add a serialised DRAM round trip per row (ncu on the 27-point
// post-sweep: warps stalled ~57 cycles per instruction on L1TEX scoreboards).  No registers are
// held across the reduction.  Default: nothing to prefetch.
__device__ __forceinline__ void pf_l2(const void* p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}
template <class E>
__device__ __forceinline__ void epi_prefetch(const E&, int64_t) {}

// r = b - s                                (residual; s = A x or A (m o b))
struct EResid {
    static constexpr bool kDot = false;
    static constexpr bool kAbs = false;
    const double* __restrict__ b;
    double* __restrict__ r;
    __device__ __forceinline__ double operator()(int64_t i, double s) const {
        r[i] = b[i] - s;
        return 0.0;
    }
};
// rhs = b - alpha q ; r = rhs - s            (EResid whose right-hand side is the K-cycle
// inner residual b - alpha_1 q_1, materialised here for the rest of the cycle)
struct EResidK {
    static constexpr bool kDot = false;
    static constexpr bool kAbs = false;
    const double* __restrict__ b;
    const double* __restrict__ q;
    const double* k;
    double* __restrict__ rhs;
    double* __restrict__ r;
    double alpha = 0.0;
    __device__ __forceinline__ double operator()(int64_t i, double s) const {
        const double bi = b[i] - alpha * q[i];
        rhs[i] = bi;
        r[i] = bi - s;
        return 0.0;
    }
};
__device__ __forceinline__ void bind(EResidK& e) { e.alpha = e.k[2]; }
// x' = x + m (b - s)                        (l1-Jacobi sweep, out of place)
// ABS = true: m_i = 1/asum from the streamed row (short rows); false: m_i read
// from `m` (long rows, where the extra per-entry |a| chain costs more than 8 B/row).
template <bool DOT, bool ABS = true>
struct ESweep {
    static constexpr bool kDot = DOT;
    static constexpr bool kAbs = ABS;
    const double* __restrict__ x;
    const double* __restrict__ b;
    double* __restrict__ xo;
    const double* __restrict__ m = nullptr;
    const double* __restrict__ dw = nullptr;  // dot weight: nullptr = b (PCG r^T z), q (FCG z^T q)
    __device__ __forceinline__ double f(int64_t i, double s, double mi) const {
        const double bi = b[i];
        const double v = x[i] + mi * (bi - s);
        xo[i] = v;
        return DOT ? (dw ? dw[i] : bi) * v : 0.0;  // r^T z (or q^T z) at the end of the level-0 V-cycle
    }
    __device__ __forceinline__ double operator()(int64_t i, double s, double asum) const { return f(i, s, 1.0 / asum); }
    __device__ __forceinline__ double operator()(int64_t i, double s) const { return f(i, s, m[i]); }
};
// First post-sweep after ONE pre-sweep from zero.  With x1 = m b, r = b - A x1 (kept
// from the down phase) and the prolongation u = P-bar e, the sweep on x = x1 + u is
//   x' = x1 + u + m (b - A x1 - A u) = m b + u + m (r - A u)        (Eq. 3.1, exact)
// so u is gathered instead of x and neither the prolongation nor this sweep reads m.
// MB: the rhs is given premultiplied (mb = m o b, levels >= 1) instead of b.
template <bool DOT, bool MB, bool ABS = true>
struct EPost1 {
    static constexpr bool kDot = DOT;
    static constexpr bool kAbs = ABS;
    const double* __restrict__ u;
    const double* __restrict__ r;
    const double* __restrict__ bmb;  // b (level 0) or m o b (MB)
    double* __restrict__ xo;
    const double* __restrict__ m = nullptr;
    const double* __restrict__ dw = nullptr;  // dot weight: nullptr = b (PCG r^T z), q (FCG z^T q)
    __device__ __forceinline__ double f(int64_t i, double s, double mi) const {
        const double bi = bmb[i];
        const double x1 = MB ? bi : mi * bi;
        const double v = x1 + u[i] + mi * (r[i] - s);
        xo[i] = v;
        return DOT ? (dw ? dw[i] : bi) * v : 0.0;  // DOT only at level 0 (b = r of PCG)
    }
    __device__ __forceinline__ double operator()(int64_t i, double s, double asum) const { return f(i, s, 1.0 / asum); }
    __device__ __forceinline__ double operator()(int64_t i, double s) const { return f(i, s, m[i]); }
};
// x' = m b + m (b - s)  with s = A (m o b)  (two sweeps from x = 0, s1 >= 2)
struct ESweep0 {
    static constexpr bool kDot = false;
    static constexpr bool kAbs = true;
    const double* __restrict__ b;
    double* __restrict__ xo;
    __device__ __forceinline__ double operator()(int64_t i, double s, double asum) const {
        const double mi = 1.0 / asum, bi = b[i];
        xo[i] = mi * bi + mi * (bi - s);
        return 0.0;
    }
};
// the compact level's smoothing term for the K-cycle's second application, whose rhs is
// b - alpha q: rhs_i = b_i - alpha q_i is stored, xo = m rhs + m (rhs - s), m from the row (ABS);
// s = A (m o rhs) comes from the GMBaq gather
struct ESweep0K {
    static constexpr bool kDot = false;
    static constexpr bool kAbs = true;
    const double* __restrict__ b;
    const double* __restrict__ q;
    const double* k;
    double* __restrict__ rhs;
    double* __restrict__ xo;
    double alpha = 0.0;
    __device__ __forceinline__ double operator()(int64_t i, double s, double asum) const {
        const double mi = 1.0 / asum, bi = b[i] - alpha * q[i];
        rhs[i] = bi;
        xo[i] = mi * bi + mi * (bi - s);
        return 0.0;
    }
};
__device__ __forceinline__ void bind(ESweep0K& e) { e.alpha = e.k[2]; }
// y = s                                     (restriction b_{l+1} = P-bar^T r)
struct EStore {
    static constexpr bool kDot = false;
    static constexpr bool kAbs = false;
    double* __restrict__ y;
    __device__ __forceinline__ double operator()(int64_t i, double s) const {
        y[i] = s;
        return 0.0;
    }
};
// y = s ; mb = m o y                         (restriction that also pre-multiplies the
//                                             coarse rhs by the coarse l1 diagonal)
struct EStoreMB {
    static constexpr bool kDot = false;
    static constexpr bool kAbs = false;
    double* __restrict__ y;
    const double* __restrict__ m;
    double* __restrict__ mb;
    __device__ __forceinline__ double operator()(int64_t i, double s) const {
        y[i] = s;
        mb[i] = m[i] * s;
        return 0.0;
    }
};
// x = mb + s                                (prolongation after one pre-sweep from 0, mb = m o b)
struct EProlongMB {
    static constexpr bool kDot = false;
    static constexpr bool kAbs = false;
    const double* __restrict__ mb;
    double* __restrict__ xo;
    __device__ __forceinline__ double operator()(int64_t i, double s) const {
        xo[i] = mb[i] + s;
        return 0.0;
    }
};
// x = m b + s                               (prolongation after one pre-sweep from 0)
struct EProlong0 {
    static constexpr bool kDot = false;
    static constexpr bool kAbs = false;
    const double* __restrict__ b;
    const double* __restrict__ m;
    double* __restrict__ xo;
    __device__ __forceinline__ double operator()(int64_t i, double s) const {
        xo[i] = m[i] * b[i] + s;
        return 0.0;
    }
};
// x' = x + s                                (prolongation, general)
struct EProlongAdd {
    static constexpr bool kDot = false;
    static constexpr bool kAbs = false;
    const double* x;
    double* xo;
    __device__ __forceinline__ double operator()(int64_t i, double s) const {
        xo[i] = x[i] + s;
        return 0.0;
    }
};
// q = s with p = z + beta p_old formed on the fly (GPz): writes p_new and q,
// applies the deferred x += alpha_prev p_old, returns p_i q_i
struct ESpmvDotPz {
    static constexpr bool kDot = true;
    static constexpr bool kAbs = false;
    const double* __restrict__ z;
    double* p0;
    double* p1;
    double* __restrict__ q;
    double* __restrict__ x;
    const PcgState* st;
    const double* pold = nullptr;
    double* pnew = nullptr;
    double beta = 0.0, alpha = 0.0;
    bool first = true;
    __device__ __forceinline__ double operator()(int64_t i, double s) const {
        double pi;
        if (first) {
            pi = z[i];
        } else {
            const double po = pold[i];
            x[i] = x[i] + alpha * po;
            pi = z[i] + beta * po;
        }
        pnew[i] = pi;
        q[i] = s;
        return pi * s;
    }
};
__device__ __forceinline__ void bind(ESpmvDotPz& e) {
    const int32_t it = e.st->iter;
    e.first = (it == 0);
    e.beta = e.st->beta;
    e.alpha = e.st->alpha;
    e.pold = (it & 1) ? e.p1 : e.p0;
    e.pnew = (it & 1) ? e.p0 : e.p1;
}

template <bool DOT, bool ABS>
__device__ __forceinline__ void epi_prefetch(const ESweep<DOT, ABS>& e, int64_t i) {
    pf_l2(e.x + i);
    pf_l2(e.b + i);
    if constexpr (!ABS) pf_l2(e.m + i);
}
template <bool DOT, bool MB, bool ABS>
__device__ __forceinline__ void epi_prefetch(const EPost1<DOT, MB, ABS>& e, int64_t i) {
    pf_l2(e.u + i);
    pf_l2(e.r + i);
    pf_l2(e.bmb + i);
    if constexpr (!ABS) pf_l2(e.m + i);
}
// (measured: prefetching for the residual and for q = A p with the fused direction update makes
// them 1-3 % slower -- their epilogues read one / three vectors the gathers already touch -- while the
// sweeps gain 1.5-4 % on c3; profiles/r02_ab_epi_prefetch.txt)
__device__ __forceinline__ void epi_prefetch(const EProlongAdd& e, int64_t i) { pf_l2(e.x + i); }

// x' = x + s, returns dw_i x'_i (DOT)       (INVK: x' = x + Z (D^-1 W r); the level-0
//                                            last post-sweep also reduces r^T z or q^T z)
template <bool DOT>
struct EAddDot {
    static constexpr bool kDot = DOT;
    static constexpr bool kAbs = false;
    const double* x;
    double* xo;
    const double* __restrict__ dw = nullptr;
    __device__ __forceinline__ double operator()(int64_t i, double s) const {
        const double v = x[i] + s;
        xo[i] = v;
        return DOT ? dw[i] * v : 0.0;
    }
};

// q = s, returns p_i q_i                    (PCG: q = A p fused with p^T q)
struct ESpmvDot {
    static constexpr bool kDot = true;
    static constexpr bool kAbs = false;
    const double* __restrict__ p;
    double* __restrict__ q;
    __device__ __forceinline__ double operator()(int64_t i, double s) const {
        q[i] = s;
        return p[i] * s;
    }
};

// q = A p with p = z + beta p_old formed per row (the owner writes p into pnew, a
// second buffer: neighbours still gather p_old), reducing p^T q and p^T r together
// (FIN_KALPHA2): the K-cycle's k_kpupd folded into its q = A p
struct EKSpmvPupd {
    static constexpr bool kDot = true;
    static constexpr bool kAbs = false;
    using dot_t = double2;
    const double* __restrict__ z;
    const double* __restrict__ pold;
    double* __restrict__ pnew;
    double* __restrict__ q;
    const double* __restrict__ r;
    const double* k;
    double beta = 0.0;
    __device__ __forceinline__ double2 operator()(int64_t i, double s) const {
        const double pi = z[i] + beta * pold[i];
        pnew[i] = pi;
        q[i] = s;
        return make_double2(pi * s, pi * r[i]);
    }
};
__device__ __forceinline__ void bind(EKSpmvPupd& e) { e.beta = e.k[3]; }

// ------------------------------------------------------------ SELL-32 kernel
struct SellView {
    const uint32_t* __restrict__ sptr;  // nslices+1, offsets in units of 32 entries
    const int32_t* __restrict__ col;
    const double* __restrict__ val;
    int64_t n;
    int64_t s0, s1;                     // slice range of this launch (multi-rank interior/boundary split)
    int64_t k0 = 0, kspan = 0;          // slices [k0, k0 + kspan) inside the range are skipped (boundary
                                        // launch of a split operator: head + tail in one launch)
    // SELL-32-sigma: slot (slice, lane) -> row (rows sorted by length inside windows of
    // sigma rows; -1 = padding slot); null for plain SELL-32 (slot = row)
    const int32_t* __restrict__ perm;
    // 16-bit columns (col null): column = cbase[slot] + c16[k]
    const uint16_t* __restrict__ c16 = nullptr;
    const int32_t* __restrict__ cbase = nullptr;
};

// Row-chunk of exactly W entries of one slice (lane = row): the W value loads are
// issued first, then the W column indices, then the W gathers, then the W FMAs in
// ascending order.  Fixed W (a full unroll with no predication) lets every load
// of the chunk be in flight at once; measured on B200 (tools/spmv_lab2.cu) this
// lifts the level-0 sweep from 5.45 to 6.65 TB/s of stored bytes (the pure read
// roofline of the part) and a 27-entry-per-row operator from 4.96 to 6.29 TB/s.
// The summation order is unchanged (ascending k), so results are bitwise equal
// to the one-entry-at-a-time loop.
template <int W, bool ABS, class G, class ColF>
__device__ __forceinline__ void row_chunk(const double* v, const ColF& colf, const G& g, double& acc, double& asum) {
    double a[W], x[W];
#pragma unroll
    for (int j = 0; j < W; ++j) a[j] = ld_stream(v + 32 * j);
    int32_t c[W];
#pragma unroll
    for (int j = 0; j < W; ++j) c[j] = colf(j);
#pragma unroll
    for (int j = 0; j < W; ++j) x[j] = g(c[j]);
#pragma unroll
    for (int j = 0; j < W; ++j) {
        acc += a[j] * x[j];
        if constexpr (ABS) asum += fabs(a[j]);
    }
}

// a slice row of width w: chunks of CH entries (SELL: G::kChunk = 8, or 4 for
// gathers that load two vectors, which keeps the kernels within 32 registers with
// no spills; SDIA: 8), then one exact-width remainder
template <int CH, bool ABS, class G, class ColAt>
__device__ __forceinline__ void slice_row(const double* v, uint32_t w, const ColAt& col_at, const G& g, double& acc,
                                          double& asum) {
    uint32_t k = 0;
    for (; k + CH <= w; k += CH)
        row_chunk<CH, ABS>(v + 32 * k, [&](int j) { return col_at(k + j); }, g, acc, asum);
    const double* vk = v + 32 * k;
    auto ck = [&](int j) { return col_at(k + j); };
    switch (w - k) {
        case 7: if constexpr (CH > 7) row_chunk<7, ABS>(vk, ck, g, acc, asum); break;
        case 6: if constexpr (CH > 6) row_chunk<6, ABS>(vk, ck, g, acc, asum); break;
        case 5: if constexpr (CH > 5) row_chunk<5, ABS>(vk, ck, g, acc, asum); break;
        case 4: if constexpr (CH > 4) row_chunk<4, ABS>(vk, ck, g, acc, asum); break;
        case 3: row_chunk<3, ABS>(vk, ck, g, acc, asum); break;
        case 2: row_chunk<2, ABS>(vk, ck, g, acc, asum); break;
        case 1: row_chunk<1, ABS>(vk, ck, g, acc, asum); break;
        default: break;
    }
}

// Resident 256-thread blocks per SM the SELL / SDIA kernels are compiled for: 8 (32 registers)
// keeps 64 warps in flight; the fused direction update of q = A p (two gathered vectors, three
// written) spills at 32 registers, so it may trade occupancy for no spills (AMG_PUPD_MINB).
#ifndef AMG_EPI_PREFETCH
#define AMG_EPI_PREFETCH 1
#endif
#ifndef AMG_PUPD_MINB
#define AMG_PUPD_MINB 8
#endif
// SDIA sweeps / updates that also reduce a dot (the level-0 last post-sweep r^T z, FCG's q^T z) over
// WIDE rows (> kDotWideEntries stored entries per row, the 27-point operators): the reduction's
// accumulator is one more live register across the row loop, and at 32 registers ptxas then
// serialises the chunk's loads (tools/tma_lab.cu, the EPost1 sweep on 256^3 27-point: 5.42 TB/s
// with the dot vs 6.38 without at 8 blocks/SM; 6 blocks at 40 registers: 6.30).  In the library the
// 7-point operators lose 0.3-2 % with 6 blocks (c4 / c2 / KA1 c2) while c5's post-sweep gains 15 %
// (0.82 -> 0.70 ms; profiles/r02_ab_dot_minb.txt), so launch_mat picks the 6-block instance for wide
// operators only.  AMG_DOT_MINB: an A/B knob.
#ifndef AMG_DOT_MINB
#define AMG_DOT_MINB 6
#endif
constexpr int kDotWideEntries = 16;
template <class G, class E>
struct MinBlocks {
    static constexpr int v = 8;
};
template <>
struct MinBlocks<GPz, ESpmvDotPz> {
    static constexpr int v = AMG_PUPD_MINB;
};

template <class G, class E>
__global__ void __launch_bounds__(kBlock, MinBlocks<G, E>::v) k_sell(SellView A, G g, E e, RedCtx rc) {
    pdl_begin();
    bind(g);
    bind(e);
    const int lane = threadIdx.x & 31;
    const int64_t w0 = ((int64_t)blockIdx.x * kBlock + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * kBlock) >> 5;
    typename DotOf<E>::type d{};
    for (int64_t vs = A.s0 + w0; vs < A.s1 - A.kspan; vs += nw) {
        const int64_t s = vs + (vs >= A.k0 ? A.kspan : 0);
        const uint32_t b0 = __ldg(A.sptr + s);
        const uint32_t w = __ldg(A.sptr + s + 1) - b0;
        const double* v = A.val + (int64_t)b0 * 32 + lane;
        double acc = 0.0, asum = 0.0;
        const int64_t row = A.perm ? (int64_t)__ldg(A.perm + (s << 5) + lane) : (s << 5) + lane;
        if (AMG_EPI_PREFETCH && row >= 0 && row < A.n) epi_prefetch(e, row);
        if (A.c16) {
            const int32_t cb = __ldg(A.cbase + (s << 5) + lane);
            const uint16_t* c = A.c16 + (int64_t)b0 * 32 + lane;
            slice_row<G::kChunk, E::kAbs>(v, w, [&](uint32_t k) { return cb + ld_stream(c + 32 * k); }, g, acc,
                                          asum);
        } else {
            const int32_t* c = A.col + (int64_t)b0 * 32 + lane;
            slice_row<G::kChunk, E::kAbs>(v, w, [&](uint32_t k) { return ld_stream(c + 32 * k); }, g, acc, asum);
        }
        if (row >= 0 && row < A.n) d += apply_epi(e, row, acc, asum);
    }
    if constexpr (E::kDot) grid_reduce(d, rc);
}

// ------------------------------------------------------------ SDIA-32 kernel
// Sliced-diagonal layout for square stencil-like operators: inside a slice of
// 32 rows the entries are aligned by their offset d = col - row (one int32 per
// slice column, shared by the 32 lanes), so no per-entry column index is
// stored.  Holes (a row without that offset) hold value 0; their column is
// clamped into range.  Entry order inside a row stays ascending in column.
struct SdiaView {
    const uint32_t* __restrict__ sptr;  // nslices+1, offsets in units of 32 entries
    const int32_t* __restrict__ offs;   // one offset per slice column (sptr units)
    const double* __restrict__ val;
    int64_t n;
    int32_t ncols;
    int32_t shift;  // row -> column frame: col = row + shift + offset (multi-rank windows)
    const int32_t* __restrict__ anchor;  // rectangular operators: col = anchor[row] + offset
    int64_t s0, s1;                      // slice range of this launch
    int64_t k0 = 0, kspan = 0;           // skipped slices [k0, k0 + kspan) (see SellView)
};

#ifndef AMG_SDIA_GPZ_CHUNK
#define AMG_SDIA_GPZ_CHUNK 8
#endif
template <class G>
struct SdiaChunk {
    static constexpr int v = 8;
};
template <>
struct SdiaChunk<GPz> {
    static constexpr int v = AMG_SDIA_GPZ_CHUNK;
};

template <class G, class E, int MB = MinBlocks<G, E>::v>
__global__ void __launch_bounds__(kBlock, MB) k_sdia(SdiaView A, G g, E e, RedCtx rc) {
    pdl_begin();
    bind(g);
    bind(e);
    const int lane = threadIdx.x & 31;
    const int64_t w0 = ((int64_t)blockIdx.x * kBlock + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * kBlock) >> 5;
    typename DotOf<E>::type d{};
    for (int64_t vs = A.s0 + w0; vs < A.s1 - A.kspan; vs += nw) {
        const int64_t s = vs + (vs >= A.k0 ? A.kspan : 0);
        const uint32_t b0 = __ldg(A.sptr + s);
        const uint32_t w = __ldg(A.sptr + s + 1) - b0;
        const int64_t row = (s << 5) + lane;
        const int32_t base =
            A.anchor ? (row < A.n ? __ldg(A.anchor + row) : 0) : (int32_t)row + A.shift;
        const int32_t* o = A.offs + b0;
        const double* v = A.val + (int64_t)b0 * 32 + lane;
        const int32_t rmax = A.ncols - 1;
        double acc = 0.0, asum = 0.0;
        // SDIA needs no registers for column indices: full chunks of 8 for every gather
        // (AMG_SDIA_GPZ_CHUNK: the chunk of the two-vector gather of q = A p, an A/B knob)
        if (AMG_EPI_PREFETCH && row < A.n) epi_prefetch(e, row);
        slice_row<SdiaChunk<G>::v, E::kAbs>(v, w, [&](uint32_t k) { return min(max(base + __ldg(o + k), 0), rmax); }, g, acc,
                              asum);
        if (row < A.n) d += apply_epi(e, row, acc, asum);
    }
    if constexpr (E::kDot) grid_reduce(d, rc);
}

// ---------------------------------------------------------- CSR-vector kernel
struct CsrView {
    const int32_t* __restrict__ rp;
    const int32_t* __restrict__ ci;
    const double* __restrict__ v;
    int64_t n;
    int64_t r0 = 0, r1 = 0;  // row range of this launch (k_csrv / k_csrb)
    int64_t k0 = 0, kspan = 0;  // skipped rows [k0, k0 + kspan) (see SellView)
    // 16-bit columns (ci null): column = cbase[row] + c16[k]
    const uint16_t* __restrict__ c16 = nullptr;
    const int32_t* __restrict__ cbase = nullptr;
};

// One lane's share of a CSR row: entries k, k+S, k+2S, ... < k1 (S lanes per row),
// in chunks of 4 whose loads are all issued before the FMAs (cf. row_chunk), then
// at most 3 single entries.  Ascending order per lane, as before.
template <int S, bool ABS, bool C16 = false, class G>
__device__ __forceinline__ void csr_lane_row(const CsrView& A, int32_t k, int32_t k1, const G& g, double& acc,
                                             double& asum, int32_t cb = 0) {
    auto col = [&](int32_t t) -> int32_t {
        if constexpr (C16) return cb + ld_stream(A.c16 + t);
        else return ld_stream(A.ci + t);
    };
    for (; k + 3 * S < k1; k += 4 * S) {
        double a[4], x[4];
        int32_t c[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) a[j] = ld_stream(A.v + k + j * S);
#pragma unroll
        for (int j = 0; j < 4; ++j) c[j] = col(k + j * S);
#pragma unroll
        for (int j = 0; j < 4; ++j) x[j] = g(c[j]);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            acc += a[j] * x[j];
            if constexpr (ABS) asum += fabs(a[j]);
        }
    }
    for (; k < k1; k += S) {
        const double a = ld_stream(A.v + k);
        acc += a * g(col(k));
        if constexpr (ABS) asum += fabs(a);
    }
}

template <int VW, class G, class E>
__global__ void __launch_bounds__(kBlock) k_csrv(CsrView A, G g, E e, RedCtx rc) {
    pdl_begin();
    bind(g);
    bind(e);
    const int64_t gid = (int64_t)blockIdx.x * kBlock + threadIdx.x;
    const int sub = threadIdx.x % VW;
    const int64_t g0 = gid / VW;
    const int64_t ng = ((int64_t)gridDim.x * kBlock) / VW;
    typename DotOf<E>::type d{};
    // every lane of a warp runs the same number of outer iterations (shuffles)
    const int64_t rend = A.r1 - A.kspan;
    const int64_t iters = (rend - A.r0 + ng - 1) / ng;
    for (int64_t it = 0; it < iters; ++it) {
        const int64_t vr = A.r0 + g0 + it * ng;
        const int64_t row = vr + (vr >= A.k0 ? A.kspan : 0);
        double acc = 0.0, asum = 0.0;
        if (vr < rend) {
            const int32_t k0 = __ldg(A.rp + row), k1 = __ldg(A.rp + row + 1);
            if (A.c16) csr_lane_row<VW, E::kAbs, true>(A, k0 + sub, k1, g, acc, asum, __ldg(A.cbase + row));
            else csr_lane_row<VW, E::kAbs>(A, k0 + sub, k1, g, acc, asum);
        }
#pragma unroll
        for (int o = VW / 2; o > 0; o >>= 1) {
            acc += __shfl_xor_sync(0xffffffffu, acc, o, VW);
            if constexpr (E::kAbs) asum += __shfl_xor_sync(0xffffffffu, asum, o, VW);
        }
        if (sub == 0 && vr < rend) d += apply_epi(e, row, acc, asum);
    }
    if constexpr (E::kDot) grid_reduce(d, rc);
}

// ------------------------------------------------------- CSR block-per-row
// For few, long rows (deep levels: hundreds to thousands of entries per row):
// one 256-thread block per row, fixed-order block reduction.
template <class G, class E>
__global__ void __launch_bounds__(kBlock) k_csrb(CsrView A, G g, E e, RedCtx rc) {
    pdl_begin();
    bind(g);
    bind(e);
    __shared__ double part[kBlock / 32], apart[kBlock / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    typename DotOf<E>::type d{};
    for (int64_t vr = A.r0 + blockIdx.x; vr < A.r1 - A.kspan; vr += gridDim.x) {
        const int64_t row = vr + (vr >= A.k0 ? A.kspan : 0);
        const int32_t k0 = __ldg(A.rp + row), k1 = __ldg(A.rp + row + 1);
        double acc = 0.0, asum = 0.0;
        if (A.c16)
            csr_lane_row<kBlock, E::kAbs, true>(A, k0 + (int32_t)threadIdx.x, k1, g, acc, asum, __ldg(A.cbase + row));
        else
            csr_lane_row<kBlock, E::kAbs>(A, k0 + (int32_t)threadIdx.x, k1, g, acc, asum);
        for (int o = 16; o > 0; o >>= 1) {
            acc += __shfl_xor_sync(0xffffffffu, acc, o);
            if constexpr (E::kAbs) asum += __shfl_xor_sync(0xffffffffu, asum, o);
        }
        if (lane == 0) {
            part[wid] = acc;
            apart[wid] = asum;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            double s = 0.0, as = 0.0;
            for (int w = 0; w < kBlock / 32; ++w) {
                s += part[w];
                as += apart[w];
            }
            d += apply_epi(e, row, s, as);
        }
        __syncthreads();
    }
    if constexpr (E::kDot) grid_reduce(d, rc);
}

// ------------------------------------------------------------ vector kernels
// PCG prologue: r = b, x = 0, ||b||^2 -> FIN_BNORM
__global__ void __launch_bounds__(kBlock) k_pcg_init(const double* __restrict__ b, double* __restrict__ r,
                                                     double* __restrict__ x, int64_t n, RedCtx rc) {
    pdl_begin();
    double d = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x; i < n; i += (int64_t)gridDim.x * kBlock) {
        const double bi = b[i];
        r[i] = bi;
        x[i] = 0.0;
        d += bi * bi;
    }
    grid_reduce(d, rc);
}

// a^T b -> finisher (single-level hierarchies: r^T z)
__global__ void __launch_bounds__(kBlock) k_dot(const double* __restrict__ a, const double* __restrict__ b,
                                                int64_t n, RedCtx rc) {
    pdl_begin();
    double d = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x; i < n; i += (int64_t)gridDim.x * kBlock)
        d += a[i] * b[i];
    grid_reduce(d, rc);
}

// p = z (first iteration) or p = z + beta p.  The previous iteration's
// x += alpha p is applied here, where the old p is read anyway (deferred from
// k_axpy_rr; the last one is applied by k_xfinal after the loop).
__global__ void __launch_bounds__(kBlock) k_pupdate(const double* __restrict__ z, double* __restrict__ p,
                                                    double* __restrict__ x, int64_t n,
                                                    const PcgState* __restrict__ st) {
    pdl_begin();
    const bool first = st->iter == 0;
    const double beta = st->beta, alpha = st->alpha;
    for (int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x; i < n; i += (int64_t)gridDim.x * kBlock) {
        if (first) {
            p[i] = z[i];
        } else {
            const double pi = p[i];
            x[i] = x[i] + alpha * pi;
            p[i] = z[i] + beta * pi;
        }
    }
}

// r -= alpha q ; ||r||^2 -> FIN_RR
__global__ void __launch_bounds__(kBlock) k_axpy_rr(double* __restrict__ r, const double* __restrict__ q, int64_t n,
                                                    const PcgState* __restrict__ st, RedCtx rc) {
    pdl_begin();
    const double alpha = st->alpha;
    double d = 0.0;
    const int64_t t0 = (int64_t)blockIdx.x * kBlock + threadIdx.x, nt = (int64_t)gridDim.x * kBlock;
    if (((reinterpret_cast<uintptr_t>(r) | reinterpret_cast<uintptr_t>(q)) & 15) == 0) {
        // 16-byte accesses, two pairs in flight per thread; the odd last element by thread 0
        double2* __restrict__ r2 = reinterpret_cast<double2*>(r);
        const double2* __restrict__ q2 = reinterpret_cast<const double2*>(q);
        const int64_t m = n >> 1;
        int64_t i = t0;
        for (; i + nt < m; i += 2 * nt) {
            const double2 a = r2[i], b = __ldg(q2 + i), c = r2[i + nt], e = __ldg(q2 + i + nt);
            const double2 u = make_double2(a.x - alpha * b.x, a.y - alpha * b.y);
            const double2 v = make_double2(c.x - alpha * e.x, c.y - alpha * e.y);
            r2[i] = u;
            r2[i + nt] = v;
            d += u.x * u.x;
            d += u.y * u.y;
            d += v.x * v.x;
            d += v.y * v.y;
        }
        if (i < m) {
            const double2 a = r2[i], b = __ldg(q2 + i);
            const double2 u = make_double2(a.x - alpha * b.x, a.y - alpha * b.y);
            r2[i] = u;
            d += u.x * u.x;
            d += u.y * u.y;
        }
        if ((n & 1) && t0 == 0) {
            const double ri = r[n - 1] - alpha * q[n - 1];
            r[n - 1] = ri;
            d += ri * ri;
        }
    } else {
        for (int64_t i = t0; i < n; i += nt) {
            const double ri = r[i] - alpha * q[i];
            r[i] = ri;
            d += ri * ri;
        }
    }
    grid_reduce(d, rc);
}

// After the loop: the pending x += alpha p of the last iteration (p1 != nullptr:
// p double-buffered, the last direction is P[iter & 1]).
__global__ void __launch_bounds__(kBlock) k_xfinal(double* __restrict__ x, const double* p0, const double* p1,
                                                   int64_t n, const PcgState* __restrict__ st) {
    pdl_begin();
    if (st->iter == 0) return;
    const double alpha = st->alpha;
    const double* __restrict__ p = (p1 && (st->iter & 1)) ? p1 : p0;
    for (int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x; i < n; i += (int64_t)gridDim.x * kBlock)
        x[i] = x[i] + alpha * p[i];
}

// Receive side of a peer-memory (LSA) barrier, fused into the kernel that consumes the data.
// Receive regions are double-buffered by the parity of the barrier that filled them; `seq` counts
// the barriers this rank has pushed (k_lsa_push advances it), so the data of the barrier just
// pushed sits at buf + ((seq - 1) & 1) * stride.  Every block's threads q < np wait (acquire, system
// scope) for rank q's flag to reach seq, bounded by timeout_ns of %globaltimer: a peer that never
// arrives sets *err and every later wait returns at once (the solve reports AMG_ERR_NCCL instead of
// hanging).  flags null: a plain buffer, no wait.
struct RxWait {
    const unsigned long long* flags = nullptr;
    const unsigned long long* seq = nullptr;
    int* err = nullptr;
    unsigned long long timeout_ns = 0;
    int np = 0;
    int64_t stride = 0;  // doubles between the two parities
};
__device__ __forceinline__ void rx_wait(const RxWait& w) {
    if (!w.flags) return;
    const unsigned long long e = *w.seq;
    const int q = threadIdx.x;
    if (q < w.np && !*(volatile int*)w.err) {
        unsigned long long t0, t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        for (;;) {
            unsigned long long v;
            asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(w.flags + q) : "memory");
            if (v >= e) break;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            if (t - t0 > w.timeout_ns) {
                atomicExch(w.err, 1);
                break;
            }
            __nanosleep(64);
        }
    }
    __syncthreads();
}
__device__ __forceinline__ const double* rx_buf(const double* buf, const RxWait& w) {
    return w.flags ? buf + (int64_t)(((*w.seq) - 1ull) & 1ull) * w.stride : buf;
}

// Multi-rank dot finisher: sum the all-gathered per-rank totals in rank order.
__global__ void k_finish(const double* __restrict__ totals, int np, RedCtx rc, RxWait w) {
    pdl_begin();
    rx_wait(w);
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        const double* t = rx_buf(totals, w);
        double s = 0.0;
        for (int g = 0; g < np; ++g) s += t[g];
        finish(rc, s);
    }
}

// Halo pack / unpack: buf[k] = v[idx[k]] ; v[idx[k]] = buf[k]
__global__ void __launch_bounds__(kBlock) k_pack(const double* __restrict__ v, const int32_t* __restrict__ idx,
                                                 double* __restrict__ buf, int64_t n) {
    pdl_begin();
    for (int64_t k = (int64_t)blockIdx.x * kBlock + threadIdx.x; k < n; k += (int64_t)gridDim.x * kBlock)
        buf[k] = v[idx[k]];
}
__global__ void __launch_bounds__(kBlock) k_unpack(double* __restrict__ v, const int32_t* __restrict__ idx,
                                                   const double* __restrict__ buf0, int64_t n, RxWait w) {
    pdl_begin();
    rx_wait(w);
    const double* __restrict__ buf = rx_buf(buf0, w);
    for (int64_t k = (int64_t)blockIdx.x * kBlock + threadIdx.x; k < n; k += (int64_t)gridDim.x * kBlock)
        v[idx[k]] = buf[k];
}

// ---------------------------------------------------------------- peer-memory (LSA) transport
// Every rank's receive buffers live in an NCCL symmetric window; peer_base[q] is rank q's window
// segment as this GPU addresses it over NVLink (ncclGetLsaPointer).  A halo exchange is: push
// and arrive (k_lsa_push: gather v at the send positions and STORE straight into each destination's
// receive region -- no send buffer, no copy engine -- then flag stores), wait (flag loads), unpack.
// The region is chosen by the parity of the barrier being pushed (see RxWait).
struct LsaPush {
    char* const* peer_base;           // np window segments
    const int64_t* send_off;          // np+1: entries for peer q are [send_off[q], send_off[q+1])
    const int64_t* dst_off;           // np: byte offset, inside q's segment, of my data in q's region 0
    int64_t stride;                   // bytes between a region's two parities
    unsigned long long* seq;          // barriers this rank has pushed (advanced by the last block)
    unsigned int* count;              // blocks done (last-block pattern; reset by the last block)
    int np, me;
    int64_t flag_off;                 // byte offset of the np barrier flags in every segment
    const double* dots;               // non-null: this rank's kdot dot slots, pushed to every rank
    int kdot;
    int64_t dot_off, dot_stride;      // dot region (slot me) and its parity stride, in bytes
};
// Push + arrive in one launch: every thread stores its halo entries straight into the destination
// ranks' receive regions; each block fences them once (system scope); the last block to finish
// (threadfence-reduction pattern) pushes the dot slots, if any, and release-stores the barrier epoch into flag
// `me` of every rank's segment.  n = 0 with one block: a dot gather / plain barrier arrival.
__global__ void __launch_bounds__(kBlock) k_lsa_push(const double* __restrict__ v, const int32_t* __restrict__ idx,
                                                     int64_t n, LsaPush P) {
    pdl_begin();
    const unsigned long long s = *P.seq;
    const int64_t par = (int64_t)(s & 1ull) * P.stride;
    for (int64_t k = (int64_t)blockIdx.x * kBlock + threadIdx.x; k < n; k += (int64_t)gridDim.x * kBlock) {
        int q = 0;
        while (k >= P.send_off[q + 1]) ++q;
        double* dst = (double*)(P.peer_base[q] + P.dst_off[q] + par) + (k - P.send_off[q]);
        *dst = v[idx[k]];
    }
    // the block's stores happen-before thread 0's fence and arrival count (bar.sync, then a cumulative
    // GPU-scope fence: the grid-sync pattern); the last block observes every block's count, and its
    // system-scope release stores below are cumulative over all of them
    __shared__ bool last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(P.count, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    const int q = threadIdx.x;
    if (q < P.np) {
        if (P.dots) {
            double* d = (double*)(P.peer_base[q] + P.dot_off + (int64_t)(s & 1ull) * P.dot_stride) + (int64_t)P.me * P.kdot;
            for (int j = 0; j < P.kdot; ++j) d[j] = P.dots[j];
        }
        unsigned long long* f = (unsigned long long*)(P.peer_base[q] + P.flag_off) + P.me;
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(f), "l"(s + 1ull) : "memory");
    }
    if (q == 0) {
        *P.count = 0u;
        *P.seq = s + 1ull;  // read by this rank's receive side (stream-ordered after this launch)
    }
}

// A rank with nothing to receive at an exchange still waits at its barrier (so no rank runs two
// barriers ahead of a peer still reading the other parity).
__global__ void k_lsa_wait(RxWait w) {
    pdl_begin();
    rx_wait(w);
}



// Halo unpack of z for the fused direction update (several ranks): z[idx] = buf and, at the
// same halo positions, p_new = z + beta p_old (p_new = z on the first iteration), with the p
// double buffer selected by the iteration parity exactly as GPz / ESpmvDotPz do.
__global__ void __launch_bounds__(kBlock) k_unpack_pz(double* __restrict__ z, double* p0, double* p1,
                                                      const int32_t* __restrict__ idx,
                                                      const double* __restrict__ buf0, int64_t n,
                                                      const PcgState* __restrict__ st, RxWait w) {
    pdl_begin();
    rx_wait(w);
    const double* __restrict__ buf = rx_buf(buf0, w);
    const int32_t it = st->iter;
    const bool first = (it == 0);
    const double beta = st->beta;
    const double* pold = (it & 1) ? p1 : p0;
    double* pnew = (it & 1) ? p0 : p1;
    for (int64_t k = (int64_t)blockIdx.x * kBlock + threadIdx.x; k < n; k += (int64_t)gridDim.x * kBlock) {
        const int32_t j = idx[k];
        const double zj = buf[k];
        z[j] = zj;
        pnew[j] = first ? zj : zj + beta * pold[j];
    }
}

// The level just above a direct coarsest solve, collapsed: the whole rest of the cycle from
// that level is a fixed linear map, out = B b with B dense (formed at setup), one 256-thread
// block per row; G gathers b (GVec, or GBaq for the K-cycle's b - alpha q, whose values are then
// stored in rhs); DOT reduces dw_i out_i (dw = nullptr: the rhs itself).
template <class G, bool DOT, bool STORE_RHS>
__global__ void __launch_bounds__(kBlock) k_collapsed(const double* __restrict__ B, int64_t n, G g,
                                                      double* __restrict__ rhs, double* __restrict__ out,
                                                      const double* __restrict__ dw, RedCtx rc) {
    pdl_begin();
    bind(g);
    __shared__ double part[kBlock / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    double d = 0.0;
    for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
        const double* Bi = B + i * n;
        double acc = 0.0;
        for (int64_t j = threadIdx.x; j < n; j += kBlock) acc += __ldg(Bi + j) * g((int32_t)j);
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) part[wid] = acc;
        __syncthreads();
        if (threadIdx.x == 0) {
            double v = 0.0;
            for (int w = 0; w < kBlock / 32; ++w) v += part[w];
            out[i] = v;
            const double bi = (STORE_RHS || (DOT && !dw)) ? g((int32_t)i) : 0.0;
            if constexpr (STORE_RHS) rhs[i] = bi;
            if constexpr (DOT) d += (dw ? dw[i] : bi) * v;
        }
        __syncthreads();
    }
    if constexpr (DOT) grid_reduce(d, rc);
}

// The K-cycle's first inner iteration on a collapsed level: p = z = B b and q = A p = (A B) b
// in one kernel (two dense rows per block), reducing p^T q and p^T b together (FIN_KPR0ALPHA1)
// — the cycle application and the inner FCG's first SpMV in one launch.
__global__ void __launch_bounds__(kBlock) k_collapsed_kq(const double* __restrict__ B,
                                                         const double* __restrict__ AB, int64_t n,
                                                         const double* __restrict__ b, double* __restrict__ p,
                                                         double* __restrict__ q, RedCtx rc) {
    pdl_begin();
    __shared__ double part[2][kBlock / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    double2 d = make_double2(0.0, 0.0);
    for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
        const double* Bi = B + i * n;
        const double* Ai = AB + i * n;
        double z = 0.0, w = 0.0;
        for (int64_t j = threadIdx.x; j < n; j += kBlock) {
            const double bj = __ldg(b + j);
            z += __ldg(Bi + j) * bj;
            w += __ldg(Ai + j) * bj;
        }
        for (int o = 16; o > 0; o >>= 1) {
            z += __shfl_xor_sync(0xffffffffu, z, o);
            w += __shfl_xor_sync(0xffffffffu, w, o);
        }
        if (lane == 0) {
            part[0][wid] = z;
            part[1][wid] = w;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            double zs = 0.0, ws = 0.0;
            for (int k = 0; k < kBlock / 32; ++k) {
                zs += part[0][k];
                ws += part[1][k];
            }
            p[i] = zs;
            q[i] = ws;
            d.x += zs * ws;
            d.y += zs * b[i];
        }
        __syncthreads();
    }
    grid_reduce(d, rc);
}

// The K-cycle's second inner iteration on a collapsed level: with rhs r1 = b - alpha_1 q1
// (stored), z = B r1 and w = (A B) r1 = A z in one kernel, reducing z^T q1 (FIN_KBETA).
__global__ void __launch_bounds__(kBlock) k_collapsed_kw(const double* __restrict__ B,
                                                         const double* __restrict__ AB, int64_t n, GBaq g,
                                                         double* __restrict__ rhs, double* __restrict__ z,
                                                         double* __restrict__ w, const double* __restrict__ q1,
                                                         RedCtx rc) {
    pdl_begin();
    bind(g);
    __shared__ double part[2][kBlock / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    double d = 0.0;
    for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
        const double* Bi = B + i * n;
        const double* Ai = AB + i * n;
        double zs = 0.0, ws = 0.0;
        for (int64_t j = threadIdx.x; j < n; j += kBlock) {
            const double gj = g((int32_t)j);
            zs += __ldg(Bi + j) * gj;
            ws += __ldg(Ai + j) * gj;
        }
        for (int o = 16; o > 0; o >>= 1) {
            zs += __shfl_xor_sync(0xffffffffu, zs, o);
            ws += __shfl_xor_sync(0xffffffffu, ws, o);
        }
        if (lane == 0) {
            part[0][wid] = zs;
            part[1][wid] = ws;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            double a = 0.0, c = 0.0;
            for (int k = 0; k < kBlock / 32; ++k) {
                a += part[0][k];
                c += part[1][k];
            }
            z[i] = a;
            w[i] = c;
            rhs[i] = g((int32_t)i);
            d += q1[i] * a;
        }
        __syncthreads();
    }
    grid_reduce(d, rc);
}
// ... then p2 = z + beta p1 (into p2), q2 = w + beta q1 (in place), p2^T q2 and p2^T r1 (FIN_KALPHA2)
__global__ void __launch_bounds__(kBlock) k_kpq2(const double* __restrict__ z, const double* __restrict__ p1,
                                                 double* __restrict__ p2, const double* __restrict__ w,
                                                 double* __restrict__ q, const double* __restrict__ r1, int64_t n,
                                                 const double* __restrict__ k, RedCtx rc) {
    pdl_begin();
    const double beta = k[3];
    double2 d = make_double2(0.0, 0.0);
    for (int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x; i < n; i += (int64_t)gridDim.x * kBlock) {
        const double pi = z[i] + beta * p1[i];
        const double qi = w[i] + beta * q[i];
        p2[i] = pi;
        q[i] = qi;
        d.x += pi * qi;
        d.y += pi * r1[i];
    }
    grid_reduce(d, rc);
}

// Coarsest level: z = A_L^{-1} b, dense row-major inverse, one warp per row.
__global__ void __launch_bounds__(kBlock) k_dense_gemv(const double* __restrict__ Ainv, const double* __restrict__ b,
                                                       double* __restrict__ z, int64_t n) {
    pdl_begin();
    const int64_t warp = ((int64_t)blockIdx.x * kBlock + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * kBlock) >> 5;
    for (int64_t row = warp; row < n; row += nw) {
        const double* a = Ainv + row * n;
        double s = 0.0;
        for (int64_t k = lane; k < n; k += 32) s += __ldg(a + k) * __ldg(b + k);
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) z[row] = s;
    }
}

// FCG(1) direction update: p = z (first iteration) or
// p = z + beta p with beta = -(z^T q_prev)/(p_prev^T q_prev); the deferred
// x += alpha p_old is applied here as in k_pupdate, and p^T r -> FIN_PR.
__global__ void __launch_bounds__(kBlock) k_pupdate_fcg(const double* __restrict__ z, double* __restrict__ p,
                                                        double* __restrict__ x, const double* __restrict__ r,
                                                        int64_t n, const PcgState* __restrict__ st, RedCtx rc) {
    pdl_begin();
    const bool first = st->iter == 0;
    const double beta = st->beta, alpha = st->alpha;
    double d = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x; i < n; i += (int64_t)gridDim.x * kBlock) {
        double pn;
        if (first) {
            pn = z[i];
        } else {
            const double pi = p[i];
            x[i] = x[i] + alpha * pi;
            pn = z[i] + beta * pi;
        }
        p[i] = pn;
        d += pn * r[i];
    }
    grid_reduce(d, rc);
}

// K-cycle inner FCG vector updates (k = {p^T r, p^T q, alpha, beta, stop})
// x = alpha p ; r = b - alpha q ; mb = m o r
__global__ void __launch_bounds__(kBlock) k_kupd1(double* __restrict__ x, double* __restrict__ r,
                                                  double* __restrict__ mb, const double* __restrict__ p,
                                                  const double* __restrict__ q, const double* __restrict__ b,
                                                  const double* __restrict__ m, int64_t n,
                                                  const double* __restrict__ k) {
    pdl_begin();
    const double alpha = k[2];
    for (int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x; i < n; i += (int64_t)gridDim.x * kBlock) {
        x[i] = alpha * p[i];
        const double ri = b[i] - alpha * q[i];
        r[i] = ri;
        mb[i] = m[i] * ri;
    }
}
// K-cycle inner FCG, several ranks (own rows): p = z + beta p, p^T r -> rc (the rank's dot
// slot; beta = k[3]); x += alpha p (alpha = k[2]), the inner solve's last update.
__global__ void __launch_bounds__(kBlock) k_kpupd(double* __restrict__ p, const double* __restrict__ z,
                                                  const double* __restrict__ r, int64_t n,
                                                  const double* __restrict__ k, RedCtx rc) {
    pdl_begin();
    const double beta = k[3];
    double d = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x; i < n; i += (int64_t)gridDim.x * kBlock) {
        const double pi = z[i] + beta * p[i];
        p[i] = pi;
        d += pi * r[i];
    }
    grid_reduce(d, rc);
}
__global__ void __launch_bounds__(kBlock) k_kupd2(double* __restrict__ x, const double* __restrict__ p, int64_t n,
                                                  const double* __restrict__ k) {
    pdl_begin();
    const double alpha = k[2];
    for (int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x; i < n; i += (int64_t)gridDim.x * kBlock)
        x[i] = x[i] + alpha * p[i];
}

// ------------------------------------------------------- coarsest iterative solve
// The paper's coarsest solver for the GPU runs: CG
// preconditioned by the l1-Jacobi diagonal of A_L, x0 = 0, stopped as soon as
// ||r||/||b|| < rtol or after maxit iterations (and on p^T A p <= 0).  A_L is
// small (n_L <= a few thousand rows) and the loop is latency-bound, so the
// whole solve is ONE kernel on ONE thread-block cluster: CTA c owns a contiguous
// row block (balanced by nnz) and keeps its rows of A_L in shared memory when
// they fit; every CTA holds the full direction vector p (its own slice is
// published to the peers through distributed shared memory after each update);
// dot products are reduced per CTA in a fixed tree and summed over the CTAs in
// rank order, so every CTA computes bitwise-identical alpha, beta and stop
// decisions.  Three cluster barriers per iteration.
struct CoarseCG {
    const int32_t* __restrict__ rp;    // CSR of A_L (n+1), int32
    const int32_t* __restrict__ ci;
    const double* __restrict__ v;
    const double* __restrict__ m;      // l1-Jacobi inverse diagonal of A_L
    const int32_t* __restrict__ split; // ncta+1 row boundaries
    int32_t n;
    int32_t ncta;
    int32_t smem_a;                    // 1: the CTA's rows of A_L are staged in shared memory
    int32_t maxit;
    double rtol;
    // VA3S3CS1: the preconditioner is z = Z (Wd r), the (H)INVK factors of A_L
    // (CSR, int32 row pointers); nullptr: the l1-Jacobi diagonal m
    const int32_t* __restrict__ wrp;
    const int32_t* __restrict__ wci;
    const double* __restrict__ wv;
    const int32_t* __restrict__ zrp;
    const int32_t* __restrict__ zci;
    const double* __restrict__ zv;
};

constexpr int kCgBlock = 512;

__device__ __forceinline__ void cg_sync(int ncta) {
    if (ncta > 1) {
        asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
        asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    } else {
        __syncthreads();
    }
}

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

// generic address of the same shared variable in cluster CTA `rank`
template <class T>
__device__ __forceinline__ T* peer_smem(T* p, uint32_t rank) {
    uint64_t out;
    asm volatile("mapa.u64 %0, %1, %2;" : "=l"(out) : "l"((uint64_t)p), "r"(rank));
    return (T*)out;
}

// block sum of NV values, then the fixed rank-order sum over the cluster
template <int NV>
__device__ __forceinline__ void cg_allreduce(double (&v)[NV], double* wsum /*[NV][32]*/, double* slots /*[NV]*/,
                                             int ncta) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
        for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
        if (lane == 0) wsum[k * 32 + wid] = v[k];
    }
    __syncthreads();
    if (threadIdx.x < NV) {
        double s = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += wsum[threadIdx.x * 32 + w];
        slots[threadIdx.x] = s;
    }
    cg_sync(ncta);
#pragma unroll
    for (int k = 0; k < NV; ++k) {
        double s = 0.0;
        for (int c = 0; c < ncta; ++c) s += (ncta > 1 ? peer_smem(slots, (uint32_t)c) : slots)[k];
        v[k] = s;
    }
}

// every CTA copies the peers' slices [split[c], split[c+1]) of the full-length shared vector
// `full` into its own copy (after a cluster barrier that published them)
__device__ __forceinline__ void cg_gather(double* full, const int32_t* split, int ncta, uint32_t me) {
    for (int c = 0; c < ncta; ++c) {
        if (c == (int)me) continue;
        const int32_t c0 = split[c], c1 = split[c + 1];
        const double* src = peer_smem(full, (uint32_t)c);
        for (int i = c0 + threadIdx.x; i < c1; i += blockDim.x) full[i] = src[i];
    }
}

// y_i = sum_k M_ik v_k on the own rows [r0, r0 + nown) (warp per row, ascending k per lane)
__device__ __forceinline__ void cg_rows(const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                        const double* __restrict__ v, const double* vfull, int32_t r0,
                                        int32_t nown, double* y) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
    for (int i = wid; i < nown; i += nwarp) {
        const int32_t a0 = rp[r0 + i], a1 = rp[r0 + i + 1];
        double s = 0.0;
        for (int k = a0 + lane; k < a1; k += 32) s += __ldg(v + k) * vfull[__ldg(ci + k)];
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) y[i] = s;
    }
}

__global__ void __launch_bounds__(kCgBlock, 1) k_coarse_cg(CoarseCG A, const double* __restrict__ b,
                                                           double* __restrict__ x) {
    pdl_begin();
    extern __shared__ __align__(16) unsigned char cg_smem[];
    __shared__ double wsum[2 * 32];
    __shared__ double slots[2][2];
    const int ncta = A.ncta;
    const uint32_t me = ncta > 1 ? cluster_rank() : 0u;
    const int32_t r0 = A.split[me], r1 = A.split[me + 1], nown = r1 - r0;
    const int n = A.n;
    const bool invk = A.wrp != nullptr;
    // shared layout: pfull[n] | (INVK: vfull[n] | tfull[n]) | r[nown] | x[nown] | q[nown] |
    // m[nown] (l1-Jacobi) or z[nown] (INVK) | (vals | cols)
    double* pfull = (double*)cg_smem;
    double* vfull = pfull + n;  // INVK: r of all rows, then t = Wd r of all rows in tfull
    double* tfull = vfull + n;
    double* rs = invk ? tfull + n : pfull + n;
    double* xs = rs + nown;
    double* qs = xs + nown;
    double* ms = qs + nown;
    const int32_t k0 = A.rp[r0], nnz_own = A.rp[r1] - k0;
    double* av = ms + nown;
    int32_t* ac = (int32_t*)(av + (A.smem_a ? nnz_own : 0));
    if (A.smem_a) {
        for (int k = threadIdx.x; k < nnz_own; k += blockDim.x) {
            av[k] = __ldg(A.v + k0 + k);
            ac[k] = __ldg(A.ci + k0 + k);
        }
    }
    const double* vals = A.smem_a ? av : A.v + k0;
    const int32_t* cols = A.smem_a ? ac : A.ci + k0;
    double* ps = pfull + r0;
    // INVK: z = Z (Wd r) into ms; Wd and Z couple rows of other CTAs, so r and t = Wd r are
    // published through distributed shared memory (two cluster barriers)
    auto precond = [&]() {
        for (int i = threadIdx.x; i < nown; i += blockDim.x) vfull[r0 + i] = rs[i];
        cg_sync(ncta);
        if (ncta > 1) cg_gather(vfull, A.split, ncta, me);
        __syncthreads();
        cg_rows(A.wrp, A.wci, A.wv, vfull, r0, nown, tfull + r0);
        cg_sync(ncta);
        if (ncta > 1) cg_gather(tfull, A.split, ncta, me);
        __syncthreads();
        cg_rows(A.zrp, A.zci, A.zv, tfull, r0, nown, ms);
        __syncthreads();
    };
    // x = 0, r = b, z = M^{-1} r, p = z; ||b||^2 and rho = r^T z
    double red[2] = {0.0, 0.0};
    if (invk) {
        for (int i = threadIdx.x; i < nown; i += blockDim.x) {
            rs[i] = b[r0 + i];
            xs[i] = 0.0;
        }
        __syncthreads();
        precond();
        for (int i = threadIdx.x; i < nown; i += blockDim.x) {
            const double bi = rs[i], zi = ms[i];
            ps[i] = zi;
            red[0] += bi * bi;
            red[1] += bi * zi;
        }
    } else {
        for (int i = threadIdx.x; i < nown; i += blockDim.x) {
            const double bi = b[r0 + i], mi = A.m[r0 + i];
            rs[i] = bi;
            xs[i] = 0.0;
            ms[i] = mi;
            const double zi = mi * bi;
            ps[i] = zi;
            red[0] += bi * bi;
            red[1] += bi * zi;
        }
    }
    cg_allreduce<2>(red, wsum, slots[1], ncta);
    const double bnorm = sqrt(red[0]);
    double rho = red[1];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
    if (bnorm > 0.0) {
        for (int it = 1; it <= A.maxit; ++it) {
            // (A) publish / gather p
            cg_sync(ncta);
            if (ncta > 1) {
                cg_gather(pfull, A.split, ncta, me);
                __syncthreads();
            }
            // q = A p on the own rows (warp per row), p^T q
            double pq[1] = {0.0};
            for (int i = wid; i < nown; i += nwarp) {
                const int32_t a0 = A.rp[r0 + i] - k0, a1 = A.rp[r0 + i + 1] - k0;
                double s = 0.0;
                for (int k = a0 + lane; k < a1; k += 32) s += vals[k] * pfull[cols[k]];
                for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
                if (lane == 0) {
                    qs[i] = s;
                    pq[0] += ps[i] * s;
                }
            }
            cg_allreduce<1>(pq, wsum, slots[0], ncta);  // (B)
            if (!(pq[0] > 0.0)) break;
            const double alpha = rho / pq[0];
            double rr[2] = {0.0, 0.0};
            if (invk) {  // z = M^{-1} r is formed before the stop test (discarded on the last step)
                for (int i = threadIdx.x; i < nown; i += blockDim.x) {
                    xs[i] = xs[i] + alpha * ps[i];
                    rs[i] = rs[i] - alpha * qs[i];
                }
                __syncthreads();
                precond();
                for (int i = threadIdx.x; i < nown; i += blockDim.x) {
                    const double ri = rs[i];
                    rr[0] += ri * ri;
                    rr[1] += ri * ms[i];
                }
            } else {
                for (int i = threadIdx.x; i < nown; i += blockDim.x) {
                    xs[i] = xs[i] + alpha * ps[i];
                    const double ri = rs[i] - alpha * qs[i];
                    rs[i] = ri;
                    rr[0] += ri * ri;
                    rr[1] += ri * (ms[i] * ri);
                }
            }
            cg_allreduce<2>(rr, wsum, slots[1], ncta);  // (C)
            if (sqrt(rr[0]) / bnorm < A.rtol) break;
            const double beta = rr[1] / rho;
            if (invk)
                for (int i = threadIdx.x; i < nown; i += blockDim.x) ps[i] = ms[i] + beta * ps[i];
            else
                for (int i = threadIdx.x; i < nown; i += blockDim.x) ps[i] = ms[i] * rs[i] + beta * ps[i];
            rho = rr[1];
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nown; i += blockDim.x) x[r0 + i] = xs[i];
    cg_sync(ncta);  // no CTA may exit while a peer can still read its shared memory
}


// ------------------------------------------------------- persistent deep-level tail
// The deep levels of a cycle (n_l <= a few ten thousand rows) are latency-bound:
// each of their ~4 kernels per level costs a launch and a ramp for a few us of
// work, and the K-cycle visits them 2^l times.  The whole cycle rooted at the
// first such level (V: one application; K: the level's two-iteration FCG solve)
// is compiled on the host into a flat program of operations and executed by ONE
// cooperative persistent kernel, with a grid barrier between operations.  Every
// operation is a warp-per-row CSR row reduction with an epilogue, a dense GEMV
// (coarsest), a dot product (fixed-order block partials -> one finisher) or a
// vector update.  Dots are deterministic; the program runs the same operations
// in the same order as the launched path (only the CSR row-sum lane split differs).
enum TailKind : int32_t { TK_SPMV = 0, TK_GEMV = 1, TK_DOT = 2, TK_KUPD1 = 3, TK_KPUPD = 4, TK_KUPD2 = 5 };
enum TailEpi : int32_t { TE_RESID = 0, TE_STORE = 1, TE_STOREMB = 2, TE_SWEEP0 = 3, TE_SWEEP = 4, TE_PROLADD = 5,
                         TE_POST1 = 6, TE_SPMVDOT = 7 };
// gather with a plain (coherent) load: inside k_tail the gathered vectors are
// written by earlier operations of the same launch, so the read-only path
// (ld.global.nc / __ldg) must not be used for them
struct GVecC {
    static constexpr int kChunk = 8;
    const double* x;
    __device__ __forceinline__ double operator()(int32_t j) const { return x[j]; }
};

struct TailOp {
    int32_t kind, epi;
    int32_t mb, abs;      // TE_POST1: rhs given as m o b; m from the streamed row
    int32_t fin;          // finisher kind (FIN_K*) of a reduction, FIN_NONE otherwise
    int32_t vw;           // TK_SPMV: lanes per row (4, 8, 16, 32, or 256 = one block per row)
    const int32_t* rp;    // CSR (TK_SPMV) / dense row-major matrix in v (TK_GEMV)
    const int32_t* ci;
    const double* v;
    int64_t n;            // rows (vector length)
    const double* g;      // gathered vector
    const double* b;      // rhs / first operand
    const double* r;      // residual / second operand
    const double* x;      // current iterate / u
    double* y;            // output
    double* y2;           // second output (m o y)
    const double* m;      // l1 inverse diagonal
    double* ks;           // K-cycle level state
};

__device__ __forceinline__ double tail_epi(const TailOp& o, int64_t i, double s, double asum) {
    switch (o.epi) {
        case TE_RESID: o.y[i] = o.b[i] - s; return 0.0;
        case TE_STORE: o.y[i] = s; return 0.0;
        case TE_STOREMB: o.y[i] = s; o.y2[i] = o.m[i] * s; return 0.0;
        case TE_SWEEP0: {
            const double mi = 1.0 / asum, bi = o.b[i];
            o.y[i] = mi * bi + mi * (bi - s);
            return 0.0;
        }
        case TE_SWEEP: {
            const double mi = o.abs ? 1.0 / asum : o.m[i];
            o.y[i] = o.x[i] + mi * (o.b[i] - s);
            return 0.0;
        }
        case TE_PROLADD: o.y[i] = o.x[i] + s; return 0.0;
        case TE_POST1: {
            const double mi = o.abs ? 1.0 / asum : o.m[i];
            const double bi = o.b[i];
            const double x1 = o.mb ? bi : mi * bi;
            o.y[i] = x1 + o.x[i] + mi * (o.r[i] - s);
            return 0.0;
        }
        case TE_SPMVDOT: o.y[i] = s; return o.x[i] * s;
        default: return 0.0;
    }
}

__device__ __forceinline__ void tail_finish(const TailOp& o, double total) {
    RedCtx rc{nullptr, nullptr, nullptr, nullptr, 0ull, o.fin, o.ks};
    finish(rc, total);
}

// rows of one TK_SPMV operation, VW lanes per row (VW = 256: a whole block per row)
template <int VW>
__device__ __forceinline__ double tail_spmv(const TailOp& o, double* wpart) {
    const CsrView A{o.rp, o.ci, o.v, o.n};
    double d = 0.0;
    if constexpr (VW == kBlock) {
        const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
        for (int64_t row = blockIdx.x; row < o.n; row += gridDim.x) {
            const int32_t k0 = __ldg(o.rp + row), k1 = __ldg(o.rp + row + 1);
            double acc = 0.0, asum = 0.0;
            if (o.abs) csr_lane_row<kBlock, true>(A, k0 + (int32_t)threadIdx.x, k1, GVecC{o.g}, acc, asum);
            else csr_lane_row<kBlock, false>(A, k0 + (int32_t)threadIdx.x, k1, GVecC{o.g}, acc, asum);
            for (int off = 16; off > 0; off >>= 1) {
                acc += __shfl_xor_sync(0xffffffffu, acc, off);
                asum += __shfl_xor_sync(0xffffffffu, asum, off);
            }
            if (lane == 0) {
                wpart[wid] = acc;
                wpart[kBlock / 32 + wid] = asum;
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                double sa = 0.0, sb = 0.0;
                for (int w = 0; w < kBlock / 32; ++w) {
                    sa += wpart[w];
                    sb += wpart[kBlock / 32 + w];
                }
                d += tail_epi(o, row, sa, sb);
            }
            __syncthreads();
        }
    } else {
        const int sub = threadIdx.x % VW;
        const int64_t g0 = ((int64_t)blockIdx.x * kBlock + threadIdx.x) / VW;
        const int64_t ng = ((int64_t)gridDim.x * kBlock) / VW;
        const int64_t iters = (o.n + ng - 1) / ng;
        for (int64_t it = 0; it < iters; ++it) {
            const int64_t row = g0 + it * ng;
            double acc = 0.0, asum = 0.0;
            if (row < o.n) {
                const int32_t k0 = __ldg(o.rp + row), k1 = __ldg(o.rp + row + 1);
                if (o.abs) csr_lane_row<VW, true>(A, k0 + sub, k1, GVecC{o.g}, acc, asum);
                else csr_lane_row<VW, false>(A, k0 + sub, k1, GVecC{o.g}, acc, asum);
            }
#pragma unroll
            for (int off = VW / 2; off > 0; off >>= 1) {
                acc += __shfl_xor_sync(0xffffffffu, acc, off, VW);
                asum += __shfl_xor_sync(0xffffffffu, asum, off, VW);
            }
            if (sub == 0 && row < o.n) d += tail_epi(o, row, acc, asum);
        }
    }
    return d;
}

// CL = false: a cooperative grid over the whole GPU (grid barriers); CL = true: ONE
// thread-block cluster (<= 16 CTAs, hardware cluster barriers) for deep levels whose
// operators are a few MB — the same program interpreter either way.
template <bool CL>
__device__ __forceinline__ void tail_barrier() {
    if constexpr (CL) {
        asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
        asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    } else {
        cg::this_grid().sync();
    }
}

template <bool CL>
__global__ void __launch_bounds__(kBlock, 6) k_tail(const TailOp* __restrict__ prog, int32_t nops, double* partials) {
    __shared__ double wsum[kBlock / 32];
    __shared__ double wpart[2 * (kBlock / 32)];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t gw = ((int64_t)blockIdx.x * kBlock + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * kBlock) >> 5;
    const int64_t gt = (int64_t)blockIdx.x * kBlock + threadIdx.x;
    const int64_t nt = (int64_t)gridDim.x * kBlock;
    for (int32_t k = 0; k < nops; ++k) {
        const TailOp& o = prog[k];
        double d = 0.0;
        if (o.kind == TK_SPMV) {
            switch (o.vw) {
                case 4: d = tail_spmv<4>(o, wpart); break;
                case 8: d = tail_spmv<8>(o, wpart); break;
                case 16: d = tail_spmv<16>(o, wpart); break;
                case kBlock: d = tail_spmv<kBlock>(o, wpart); break;
                default: d = tail_spmv<32>(o, wpart); break;
            }
        } else if (o.kind == TK_GEMV) {
            for (int64_t row = gw; row < o.n; row += nw) {
                const double* a = o.v + row * o.n;
                double sacc = 0.0;
                for (int64_t c = lane; c < o.n; c += 32) sacc += __ldg(a + c) * o.g[c];
                for (int off = 16; off > 0; off >>= 1) sacc += __shfl_xor_sync(0xffffffffu, sacc, off);
                if (lane == 0) o.y[row] = sacc;
            }
        } else if (o.kind == TK_DOT) {
            for (int64_t i = gt; i < o.n; i += nt) d += o.b[i] * o.r[i];
        } else if (o.kind == TK_KUPD1) {  // y = alpha p (x = p) ; y2 = b - alpha q (r = q)
            const double alpha = o.ks[2];
            for (int64_t i = gt; i < o.n; i += nt) {
                o.y[i] = alpha * o.x[i];
                o.y2[i] = o.b[i] - alpha * o.r[i];
            }
        } else if (o.kind == TK_KPUPD) {  // p = z + beta p ; p^T r
            const double beta = o.ks[3];
            for (int64_t i = gt; i < o.n; i += nt) {
                const double pn = o.b[i] + beta * o.y[i];
                o.y[i] = pn;
                d += pn * o.r[i];
            }
        } else if (o.kind == TK_KUPD2) {  // x += alpha p
            const double alpha = o.ks[2];
            for (int64_t i = gt; i < o.n; i += nt) o.y[i] = o.y[i] + alpha * o.x[i];
        }
        if (o.fin != FIN_NONE) {  // deterministic reduction: warp tree, block partial, fixed-order total
            for (int off = 16; off > 0; off >>= 1) d += __shfl_xor_sync(0xffffffffu, d, off);
            if (lane == 0) wsum[wid] = d;
            __syncthreads();
            if (threadIdx.x == 0) {
                double sb = 0.0;
                for (int w = 0; w < kBlock / 32; ++w) sb += wsum[w];
                partials[blockIdx.x] = sb;
            }
            tail_barrier<CL>();
            if (blockIdx.x == 0 && threadIdx.x == 0) {
                double tot = 0.0;
                for (unsigned int bb = 0; bb < gridDim.x; ++bb) tot += ((volatile double*)partials)[bb];
                tail_finish(o, tot);
                __threadfence();
            }
        }
        tail_barrier<CL>();
    }
}

}  // namespace amgk
