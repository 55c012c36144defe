// setup_gpu.cu — GPU-resident hierarchy construction.
//
// The same construction as setup.cpp (§3.2) run
// on the device, bit-identical to it: this file is compiled with --fmad=false
// and every product / sum that can round is an explicit __dmul_rn / __dadd_rn /
// __dsub_rn / __ddiv_rn in the parenthesisation of the canonical arithmetic
// contract C1-C5.  Different algorithms from both the host setup and the oracle:
//  * matching: the "suitor" algorithm (Manne & Halappanavar) — every vertex
//    proposes to its best neighbour whose current suitor it beats (64-bit
//    atomicMax on a packed (key rank, ~index) word); displaced suitors re-propose.
//    Under the strict edge order (|c| desc, lo asc, hi asc) its result is the
//    unique greedy = locally-dominant matching (reading R5);
//  * SpGEMM: expand-sort-compress for wide outputs.  Products are generated in
//    the canonical arrival order of C3 (row i of X, j ascending, K ascending),
//    stably radix-sorted by (i, K), and each output entry is summed sequentially
//    over its run, starting from +0.0 — the accumulation order of C3 exactly.
//    Narrow outputs (<= 16384 columns: the deep, dense-ish levels) use one block
//    per row with a shared-memory dense accumulator and a barrier between the
//    row's X entries, which gives every acc[K] the same arrival order;
//  * transpose: stable radix sort by column (row order kept inside a column).
// The coarsest dense inverse is computed on the host from the copied-back A_L
// (n_L <= a few thousand).
#include <cuda_runtime.h>

#include <cub/cub.cuh>
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <string>
#include <vector>

#include "setup.hpp"

namespace amgsetup {

void tmark(const char* what);
bool dense_inverse_host(const Csr& A, std::vector<double>& inv);

namespace {

#define GCK(call)                                                            \
    do {                                                                     \
        cudaError_t e_ = (call);                                             \
        if (e_ != cudaSuccess) throw std::string(#call) + ": " + cudaGetErrorString(e_); \
    } while (0)

constexpr int TB = 256;

inline int grid_for(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + TB - 1) / TB, 148 * 16)); }

// stream-ordered device buffer
template <class T>
struct Buf {
    T* p = nullptr;
    size_t n = 0;
    cudaStream_t s = nullptr;
    Buf() = default;
    Buf(size_t count, cudaStream_t st) { alloc(count, st); }
    void alloc(size_t count, cudaStream_t st) {
        release();
        s = st;
        n = count;
        GCK(cudaMallocAsync((void**)&p, std::max<size_t>(1, count) * sizeof(T), s));
    }
    void release() {
        if (p) cudaFreeAsync(p, s);
        p = nullptr;
        n = 0;
    }
    T* hand_over() {  // ownership leaves the buffer (freed later with cudaFree)
        T* q = p;
        p = nullptr;
        n = 0;
        return q;
    }
    ~Buf() { release(); }
    Buf(const Buf&) = delete;
    Buf& operator=(const Buf&) = delete;
    Buf(Buf&& o) noexcept : p(o.p), n(o.n), s(o.s) { o.p = nullptr; o.n = 0; }
    Buf& operator=(Buf&& o) noexcept {
        release();
        p = o.p;
        n = o.n;
        s = o.s;
        o.p = nullptr;
        o.n = 0;
        return *this;
    }
};

struct DCsr {
    int64_t nrows = 0, ncols = 0, nnz = 0;
    Buf<int64_t> rp;
    Buf<int32_t> ci;
    Buf<double> v;
};

// ------------------------------------------------------------------ cub helpers
template <class T>
void excl_scan(const T* in, T* out, int64_t n, cudaStream_t s) {
    size_t tb = 0;
    GCK(cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, n, s));
    Buf<char> tmp(tb, s);
    GCK(cub::DeviceScan::ExclusiveSum(tmp.p, tb, in, out, n, s));
}
template <class T>
void incl_scan(const T* in, T* out, int64_t n, cudaStream_t s) {
    size_t tb = 0;
    GCK(cub::DeviceScan::InclusiveSum(nullptr, tb, in, out, n, s));
    Buf<char> tmp(tb, s);
    GCK(cub::DeviceScan::InclusiveSum(tmp.p, tb, in, out, n, s));
}
template <class K, class V>
void sort_pairs(Buf<K>& k, Buf<V>& v, int64_t n, int end_bit, cudaStream_t s) {
    Buf<K> k2(n, s);
    Buf<V> v2(n, s);
    cub::DoubleBuffer<K> dk(k.p, k2.p);
    cub::DoubleBuffer<V> dv(v.p, v2.p);
    size_t tb = 0;
    GCK(cub::DeviceRadixSort::SortPairs(nullptr, tb, dk, dv, n, 0, end_bit, s));
    Buf<char> tmp(tb, s);
    GCK(cub::DeviceRadixSort::SortPairs(tmp.p, tb, dk, dv, n, 0, end_bit, s));
    if (dk.Current() != k.p) std::swap(k.p, k2.p);
    if (dv.Current() != v.p) std::swap(v.p, v2.p);
}
template <class T>
T dev_get(const T* p, cudaStream_t s) {
    T h;
    GCK(cudaMemcpyAsync(&h, p, sizeof(T), cudaMemcpyDeviceToHost, s));
    GCK(cudaStreamSynchronize(s));
    return h;
}
int bits_for(uint64_t maxval) {
    int b = 1;
    while (b < 64 && (maxval >> b) != 0) ++b;
    return b;
}

// ------------------------------------------------------------------ kernels
__global__ void k_diag(const int64_t* rp, const int32_t* ci, const double* v, int64_t n, double* d) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        int64_t lo = rp[i], hi = rp[i + 1];
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (ci[mid] < i) lo = mid + 1;
            else hi = mid;
        }
        d[i] = (lo < rp[i + 1] && ci[lo] == i) ? v[lo] : 0.0;
    }
}

// l1-Jacobi inverse diagonal m_i = 1/sum_j |a_ij| (O7, ascending j); rowabs_over_diag
// (O4) = (sum_j |a_ij|) / a_ii when d != nullptr
__global__ void k_rowabs(const int64_t* rp, const double* v, int64_t n, const double* d, double* m, double* q) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int64_t k = rp[i]; k < rp[i + 1]; ++k) s = __dadd_rn(s, fabs(v[k]));
        if (m) m[i] = __ddiv_rn(1.0, s);
        if (q) q[i] = __ddiv_rn(s, d[i]);
    }
}

// Eq. 3.2 key |c_ij| of every stored entry, (lo, hi) orientation (O2.1, C2);
// invalid (diagonal, den == 0, c == 0) -> 0 (as a bit pattern), valid keys are
// positive doubles whose bit patterns order like their values.
__global__ void k_keys(const int64_t* rp, const int32_t* ci, const double* v, const double* d, const double* w,
                       int64_t n, uint64_t* key) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        for (int64_t k = rp[i]; k < rp[i + 1]; ++k) {
            const int64_t j = ci[k];
            uint64_t out = 0;
            if (j != i) {
                const int64_t lo = min(i, j), hi = max(i, j);
                const double a = v[k];
                const double den =
                    __dadd_rn(__dmul_rn(__dmul_rn(d[lo], w[lo]), w[lo]), __dmul_rn(__dmul_rn(d[hi], w[hi]), w[hi]));
                if (den != 0.0) {
                    const double c =
                        __dsub_rn(1.0, __ddiv_rn(__dmul_rn(__dmul_rn(__dmul_rn(2.0, a), w[lo]), w[hi]), den));
                    if (c != 0.0) out = (uint64_t)__double_as_longlong(fabs(c));
                }
            }
            key[k] = out;
        }
    }
}

// rank of every key among the distinct valid keys (1-based, ascending); 0 = invalid
__global__ void k_rank(const uint64_t* key, int64_t nnz, const uint64_t* uniq, int64_t nu, uint32_t* rank) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t x = key[k];
        if (x == 0) {
            rank[k] = 0;
            continue;
        }
        int64_t lo = 0, hi = nu;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (uniq[mid] < x) lo = mid + 1;
            else hi = mid;
        }
        rank[k] = (uint32_t)(lo + (uniq[0] == 0 ? 0 : 1));  // uniq[0] is the invalid 0 when present
    }
}

__device__ __forceinline__ uint64_t pack(uint32_t rank, int32_t u) {
    return ((uint64_t)rank << 32) | (uint64_t)(0xFFFFFFFFu - (uint32_t)u);
}
__device__ __forceinline__ int32_t unpack(uint64_t x) { return (int32_t)(0xFFFFFFFFu - (uint32_t)(x & 0xFFFFFFFFu)); }

// Suitor matching.  sv[v] = best proposal received by v so far (0 = none).
__global__ void k_suitor(const int64_t* rp, const int32_t* ci, const uint32_t* rank, int64_t n,
                         unsigned long long* sv) {
    for (int64_t u0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u0 < n; u0 += (int64_t)gridDim.x * blockDim.x) {
        int32_t cur = (int32_t)u0;
        while (cur >= 0) {
            uint32_t br = 0;
            int32_t bv = -1;
            for (int64_t k = rp[cur]; k < rp[cur + 1]; ++k) {
                const uint32_t r = rank[k];
                if (r == 0) continue;
                const int32_t v = ci[k];
                if (r < br || (r == br && v > bv)) continue;  // not better than the best found
                const uint64_t cand = pack(r, cur);
                const uint64_t now = *((volatile unsigned long long*)&sv[v]);
                if (cand > now) {
                    br = r;
                    bv = v;
                }
            }
            if (bv < 0) break;
            const uint64_t cand = pack(br, cur);
            const uint64_t old = atomicMax(&sv[bv], (unsigned long long)cand);
            if (old < cand) cur = (old == 0) ? -1 : unpack(old);  // displaced suitor re-proposes
            // else: lost the race, cur searches again
        }
    }
}

__global__ void k_mates(const unsigned long long* sv, int64_t n, int32_t* mate) {
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n; u += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t a = sv[u];
        int32_t m = -1;
        if (a) {
            const int32_t v = unpack(a);
            const uint64_t b = sv[v];
            if (b && unpack(b) == (int32_t)u) m = v;
        }
        mate[u] = m;
    }
}

__global__ void k_heads(const int32_t* mate, int64_t n, int64_t* head) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
        head[v] = (mate[v] < 0 || mate[v] > v) ? 1 : 0;
}

// aggregates by ascending minimum member and the pairwise values of Eq. 3.3 (O2.3-O2.4)
__global__ void k_pairwise(const int32_t* mate, const int64_t* id, const double* w, int64_t n, int32_t* agg,
                           double* pval) {
    const double nan = __longlong_as_double(0x7ff8000000000000ll);
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = mate[v];
        if (j < 0) {
            agg[v] = (int32_t)id[v];
            pval[v] = (w[v] == 0.0) ? 1.0 : __ddiv_rn(w[v], fabs(w[v]));
            continue;
        }
        const int64_t lo = min(v, j), hi = max(v, j);
        agg[v] = (int32_t)id[lo];
        const double nrm = __dsqrt_rn(__dadd_rn(__dmul_rn(w[lo], w[lo]), __dmul_rn(w[hi], w[hi])));
        if (nrm == 0.0) {
            pval[v] = (v == lo) ? 1.0 : nan;
        } else {
            const double p = __ddiv_rn(w[v], nrm);
            pval[v] = (p == 0.0) ? nan : p;
        }
    }
}

// composite map and values over the sweeps (O3): val_i = val_i * pval_s[agg_i]
__global__ void k_compose(int32_t* cagg, double* cval, const int32_t* sagg, const double* spval, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t a = cagg[i];
        cval[i] = __dmul_rn(cval[i], spval[a]);
        cagg[i] = sagg[a];
    }
}

__global__ void k_iota(int32_t* a, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        a[i] = (int32_t)i;
}
__global__ void k_fill(double* a, int64_t n, double x) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) a[i] = x;
}

// one entry per row from (agg, val), NaN = not stored
__global__ void k_opr_count(const double* val, int64_t n, int64_t* cnt) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        cnt[i] = isnan(val[i]) ? 0 : 1;
}
__global__ void k_opr_fill(const int32_t* agg, const double* val, const int64_t* rp, int64_t n, int32_t* ci, double* v) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        if (!isnan(val[i])) {
            ci[rp[i]] = agg[i];
            v[rp[i]] = val[i];
        }
}

// ---- SpGEMM (expand-sort-compress, canonical order)
// products contributed by each entry of X: nnz of row ci[k] of Y
__global__ void k_prod_count(const int32_t* xci, int64_t xnnz, const int64_t* yrp, int64_t* cnt) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < xnnz; k += (int64_t)gridDim.x * blockDim.x)
        cnt[k] = yrp[xci[k] + 1] - yrp[xci[k]];
}
__global__ void k_rowof(const int64_t* rp, int64_t n, int32_t* row) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        for (int64_t k = rp[i]; k < rp[i + 1]; ++k) row[k] = (int32_t)i;
}
__global__ void k_runflag(const uint64_t* key, int64_t n, int64_t* flag) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
        flag[t] = (t == 0 || key[t] != key[t - 1]) ? 1 : 0;
}
__global__ void k_runstart(const int64_t* flag, const int64_t* pos, int64_t n, int64_t* start) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
        if (flag[t]) start[pos[t]] = t;
}
// one output entry per run: sequential sum from +0.0 in arrival order (C3)
__global__ void k_runsum(const uint64_t* key, const double* val, const int64_t* start, int64_t nruns, int64_t n,
                         uint64_t ncols, int32_t* ci, double* v, unsigned long long* rowcnt) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nruns; r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t a = start[r], b = (r + 1 < nruns) ? start[r + 1] : n;
        double acc = 0.0;
        for (int64_t t = a; t < b; ++t) acc = __dadd_rn(acc, val[t]);
        const uint64_t kk = key[a];
        ci[r] = (int32_t)(kk % ncols);
        v[r] = acc;
        atomicAdd(&rowcnt[kk / ncols], 1ull);
    }
}

// ---- SpGEMM with a dense per-row accumulator (outputs of <= kDenseBlocks x kDenseMax
// columns, processed in column blocks of <= kDenseMax):
// one block per output row; for each entry j of row i of X in ascending order the
// block's threads add x_ij*y_jK into acc[K] for the (distinct) K of row j of Y, with
// a barrier between entries — so every acc[K] receives its products in exactly the
// arrival order of C3.  Touched columns are emitted in ascending order with a block
// scan.  VALUES = false: count only.
constexpr int kDenseMax = 16384;
// outputs up to kDenseBlocks x kDenseMax columns use the column-blocked dense accumulator
constexpr int kDenseBlocks = 4;
constexpr int DB = 256;

template <bool VALUES>
__global__ void __launch_bounds__(DB) k_spgemm_dense(const int64_t* xrp, const int32_t* xci, const double* xv,
                                                     int64_t nrows, const int64_t* yrp, const int32_t* yci,
                                                     const double* yv, int32_t ncols, int32_t cb, int64_t* cnt,
                                                     const int64_t* crp, int32_t* cci, double* cv) {
    // output columns in blocks of cb (<= kDenseMax): the row is traversed once per block,
    // so every output entry still sums its products in ascending X-entry order (C3)
    extern __shared__ __align__(16) unsigned char sm[];
    double* acc = (double*)sm;
    unsigned char* flag = (unsigned char*)(acc + (VALUES ? cb : 0));
    typedef cub::BlockScan<int, DB> Scan;
    __shared__ typename Scan::TempStorage tmp;
    for (int64_t i = blockIdx.x; i < nrows; i += gridDim.x) {
        int64_t out = VALUES ? crp[i] : 0;
        for (int32_t c0 = 0; c0 < ncols; c0 += cb) {
            const int32_t w = min(cb, ncols - c0);
            for (int c = threadIdx.x; c < w; c += DB) {
                if (VALUES) acc[c] = 0.0;
                flag[c] = 0;
            }
            __syncthreads();
            for (int64_t e = xrp[i]; e < xrp[i + 1]; ++e) {
                const int32_t j = xci[e];
                const double x = xv[e];
                for (int64_t t = yrp[j] + threadIdx.x; t < yrp[j + 1]; t += DB) {
                    const int32_t K = yci[t] - c0;
                    if (K >= 0 && K < w) {
                        if (VALUES) acc[K] = __dadd_rn(acc[K], __dmul_rn(x, yv[t]));
                        flag[K] = 1;
                    }
                }
                __syncthreads();
            }
            for (int cc = 0; cc < w; cc += DB) {
                const int c = cc + threadIdx.x;
                const int f = (c < w) ? flag[c] : 0;
                int pos, agg;
                Scan(tmp).ExclusiveSum(f, pos, agg);
                if (VALUES && f) {
                    cci[out + pos] = c0 + c;
                    cv[out + pos] = acc[c];
                }
                out += agg;
                __syncthreads();
            }
        }
        if (!VALUES && threadIdx.x == 0) cnt[i] = out;
        __syncthreads();
    }
}

// ---- transpose (stable)
__global__ void k_colkey(const int32_t* ci, int64_t nnz, uint32_t* ck, int64_t* idx) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x) {
        ck[k] = (uint32_t)ci[k];
        idx[k] = k;
    }
}
__global__ void k_tr_gather(const int64_t* idx, const int32_t* row, const double* v, int64_t nnz, int32_t* tci,
                            double* tv, unsigned long long* cnt, const uint32_t* ck) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nnz; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = idx[t];
        tci[t] = row[k];
        tv[t] = v[k];
        atomicAdd(&cnt[ck[t]], 1ull);
    }
}

// ---- mirror (C4) + exact-zero drop (C5)
__global__ void k_mirror(const int64_t* rp, const int32_t* ci, const double* v, int64_t n, double* nv, int64_t* keep) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
        for (int64_t k = rp[r]; k < rp[r + 1]; ++k) {
            const int32_t c = ci[k];
            double val = v[k];
            if (c < r) {
                int64_t lo = rp[c], hi = rp[c + 1];
                while (lo < hi) {
                    const int64_t mid = (lo + hi) >> 1;
                    if (ci[mid] < r) lo = mid + 1;
                    else hi = mid;
                }
                val = (lo < rp[c + 1] && ci[lo] == r) ? v[lo] : 0.0;
            }
            nv[k] = val;
            keep[k] = (val != 0.0) ? 1 : 0;
        }
}
__global__ void k_compact(const int64_t* rp, const int32_t* ci, const double* nv, const int64_t* keep,
                          const int64_t* pos, int64_t n, int32_t* oci, double* ov, int64_t* orow) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
        orow[r] = pos[rp[r]];  // new row start
        for (int64_t k = rp[r]; k < rp[r + 1]; ++k)
            if (keep[k]) {
                oci[pos[k]] = ci[k];
                ov[pos[k]] = nv[k];
            }
    }
}

// ---- restriction of w: w_c[G] = sum_{i asc} p_iG w_i over the transposed P (C3)
__global__ void k_restrict_w(const int64_t* trp, const int32_t* tci, const double* tv, const double* w, int64_t nc,
                             double* out) {
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < nc; g += (int64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int64_t k = trp[g]; k < trp[g + 1]; ++k) s = __dadd_rn(s, __dmul_rn(tv[k], w[tci[k]]));
        out[g] = s;
    }
}

// ---- smoothed prolongator (O5): P-bar[i,G] = P[i,G] - (omega/a_ii) * T[i,G], zeros dropped
__global__ void k_pbar(const int64_t* trp, const int32_t* tci, const double* tv, const int64_t* prp,
                       const int32_t* pci, const double* pv, const double* d, double omega, int64_t n, double* nv,
                       int64_t* keep) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double f = __ddiv_rn(omega, d[i]);
        const bool has = prp[i + 1] > prp[i];
        for (int64_t k = trp[i]; k < trp[i + 1]; ++k) {
            const bool own = has && tci[k] == pci[prp[i]];
            const double p = own ? pv[prp[i]] : 0.0;
            const double x = __dsub_rn(p, __dmul_rn(f, tv[k]));
            nv[k] = x;
            keep[k] = (x != 0.0) ? 1 : 0;
        }
    }
}

#define LAUNCH(kern, n, s, ...) kern<<<grid_for(n), TB, 0, s>>>(__VA_ARGS__)

// ------------------------------------------------------------------ host-side primitives
DCsr upload(const Csr& A, cudaStream_t s) {
    DCsr D;
    D.nrows = A.nrows;
    D.ncols = A.ncols;
    D.nnz = A.nnz();
    D.rp.alloc(A.nrows + 1, s);
    D.ci.alloc(D.nnz, s);
    D.v.alloc(D.nnz, s);
    GCK(cudaMemcpyAsync(D.rp.p, A.rp.data(), (A.nrows + 1) * 8, cudaMemcpyHostToDevice, s));
    if (D.nnz) {
        GCK(cudaMemcpyAsync(D.ci.p, A.ci.data(), D.nnz * 4, cudaMemcpyHostToDevice, s));
        GCK(cudaMemcpyAsync(D.v.p, A.v.data(), D.nnz * 8, cudaMemcpyHostToDevice, s));
    }
    return D;
}

Csr download(const DCsr& D, cudaStream_t s) {
    Csr A;
    A.nrows = D.nrows;
    A.ncols = D.ncols;
    A.rp.resize(D.nrows + 1);
    A.ci.resize(D.nnz);
    A.v.resize(D.nnz);
    GCK(cudaMemcpyAsync(A.rp.data(), D.rp.p, (D.nrows + 1) * 8, cudaMemcpyDeviceToHost, s));
    if (D.nnz) {
        GCK(cudaMemcpyAsync(A.ci.data(), D.ci.p, D.nnz * 4, cudaMemcpyDeviceToHost, s));
        GCK(cudaMemcpyAsync(A.v.data(), D.v.p, D.nnz * 8, cudaMemcpyDeviceToHost, s));
    }
    GCK(cudaStreamSynchronize(s));
    return A;
}

template <class T>
std::vector<T> download_vec(const Buf<T>& b, int64_t n, cudaStream_t s) {
    std::vector<T> h(n);
    if (n) GCK(cudaMemcpyAsync(h.data(), b.p, n * sizeof(T), cudaMemcpyDeviceToHost, s));
    GCK(cudaStreamSynchronize(s));
    return h;
}

// rows of entries -> rp by counts (counts per row given)
void rp_from_counts(const unsigned long long* cnt, int64_t n, Buf<int64_t>& rp, cudaStream_t s) {
    rp.alloc(n + 1, s);
    GCK(cudaMemsetAsync(rp.p, 0, 8, s));
    incl_scan((const int64_t*)cnt, rp.p + 1, n, s);
}

// C = X Y in the canonical order of C3: a dense per-row accumulator in shared
// memory for narrow outputs, expand-sort-compress otherwise
DCsr spgemm_dense(const DCsr& X, const DCsr& Y, cudaStream_t s) {
    DCsr C;
    C.nrows = X.nrows;
    C.ncols = Y.ncols;
    const int nc = (int)Y.ncols;
    const int nb = (nc + kDenseMax - 1) / kDenseMax;  // column blocks
    const int cb = (nc + nb - 1) / nb;
    const size_t sm_cnt = (size_t)cb, sm_val = (size_t)cb * 9;
    // function attributes are per device: set on every call (cheap, thread-safe)
    GCK(cudaFuncSetAttribute(k_spgemm_dense<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kDenseMax * 9));
    GCK(cudaFuncSetAttribute(k_spgemm_dense<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kDenseMax * 9));
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(X.nrows, 148 * 8));
    Buf<int64_t> cnt(X.nrows + 1, s);
    GCK(cudaMemsetAsync(cnt.p + X.nrows, 0, 8, s));
    k_spgemm_dense<false><<<grid, DB, sm_cnt, s>>>(X.rp.p, X.ci.p, X.v.p, X.nrows, Y.rp.p, Y.ci.p, Y.v.p, nc, cb,
                                                   cnt.p, nullptr, nullptr, nullptr);
    GCK(cudaGetLastError());
    C.rp.alloc(X.nrows + 1, s);
    excl_scan(cnt.p, C.rp.p, X.nrows + 1, s);
    C.nnz = dev_get(C.rp.p + X.nrows, s);
    C.ci.alloc(C.nnz, s);
    C.v.alloc(C.nnz, s);
    k_spgemm_dense<true><<<grid, DB, sm_val, s>>>(X.rp.p, X.ci.p, X.v.p, X.nrows, Y.rp.p, Y.ci.p, Y.v.p, nc, cb,
                                                  nullptr, C.rp.p, C.ci.p, C.v.p);
    GCK(cudaGetLastError());
    return C;
}

// X entries [k0, k1) of rows [r0, r1): key = (row - r0) * ncols + col
__global__ void k_expand_rows(const int32_t* xrow, const int32_t* xci, const double* xv, int64_t k0, int64_t k1,
                              int32_t r0, const int64_t* yrp, const int32_t* yci, const double* yv, const int64_t* off,
                              int64_t off0, uint64_t ncols, uint64_t* key, double* val) {
    for (int64_t k = k0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < k1; k += (int64_t)gridDim.x * blockDim.x) {
        const int32_t j = xci[k];
        const double x = xv[k];
        const uint64_t base = (uint64_t)(xrow[k] - r0) * ncols;
        int64_t o = off[k] - off0;
        for (int64_t t = yrp[j]; t < yrp[j + 1]; ++t, ++o) {
            key[o] = base + (uint64_t)yci[t];
            val[o] = __dmul_rn(x, yv[t]);
        }
    }
}
__global__ void k_row_off(const int64_t* xrp, const int64_t* off, int64_t n, int64_t* rowoff) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n; i += (int64_t)gridDim.x * blockDim.x)
        rowoff[i] = off[xrp[i]];
}

// Products per chunk of the expand-sort-compress SpGEMM: bounds the transient
// memory (key + value, double-buffered sort, run flags: ~48 B per product) so
// that large operators (27-point, multi-GPU-sized level 0) build on one device.
// AMG_SPGEMM_CHUNK overrides (tests force many chunks on small inputs).
int64_t spgemm_chunk_products() {
    if (const char* e = std::getenv("AMG_SPGEMM_CHUNK")) {
        const long long v = std::atoll(e);
        if (v > 0) return (int64_t)v;
    }
    size_t fr = 0, tot = 0;
    int64_t cap = (int64_t)1 << 28;
    if (cudaMemGetInfo(&fr, &tot) == cudaSuccess) cap = std::min<int64_t>(cap, (int64_t)(fr / 4 / 48));
    return std::max<int64_t>(cap, (int64_t)1 << 20);
}

// C = X Y, rows in chunks of at most spgemm_chunk_products() products (a row is
// never split).  Within a chunk the stable radix sort keeps the products of an
// output entry in expansion order (ascending X entry, then ascending Y entry), so
// the result is independent of the chunking and equal to the one-pass result (C3).
DCsr spgemm(const DCsr& X, const DCsr& Y, cudaStream_t s) {
    if (Y.ncols <= kDenseBlocks * kDenseMax && Y.ncols > 0) return spgemm_dense(X, Y, s);
    DCsr C;
    C.nrows = X.nrows;
    C.ncols = Y.ncols;
    Buf<int64_t> cnt(X.nnz + 1, s), off(X.nnz + 1, s);
    GCK(cudaMemsetAsync(cnt.p + X.nnz, 0, 8, s));
    LAUNCH(k_prod_count, X.nnz, s, X.ci.p, X.nnz, Y.rp.p, cnt.p);
    excl_scan(cnt.p, off.p, X.nnz + 1, s);
    cnt.release();
    std::vector<int64_t> rowoff, xrp;
    {
        Buf<int64_t> ro(X.nrows + 1, s);
        LAUNCH(k_row_off, X.nrows + 1, s, X.rp.p, off.p, X.nrows, ro.p);
        rowoff = download_vec(ro, X.nrows + 1, s);
        xrp = download_vec(X.rp, X.nrows + 1, s);
    }
    Buf<int32_t> xrow(X.nnz, s);
    LAUNCH(k_rowof, X.nrows, s, X.rp.p, X.nrows, xrow.p);
    const uint64_t ncols = (uint64_t)std::max<int64_t>(1, Y.ncols);
    const int64_t budget = spgemm_chunk_products();
    Buf<unsigned long long> rc(C.nrows, s);
    GCK(cudaMemsetAsync(rc.p, 0, std::max<int64_t>(1, C.nrows) * 8, s));
    std::vector<Buf<int32_t>> pci;
    std::vector<Buf<double>> pv;
    std::vector<int64_t> pn;
    for (int64_t r0 = 0; r0 < X.nrows;) {
        int64_t r1 = r0 + 1;
        {  // the longest run of rows within the budget (at least one row)
            int64_t lo = r0 + 1, hi = X.nrows;
            while (lo < hi) {
                const int64_t mid = (lo + hi + 1) / 2;
                if (rowoff[mid] - rowoff[r0] <= budget) lo = mid;
                else hi = mid - 1;
            }
            r1 = lo;
        }
        const int64_t np = rowoff[r1] - rowoff[r0];
        const int64_t k0 = xrp[r0], k1 = xrp[r1];
        Buf<int32_t> cci;
        Buf<double> cv;
        int64_t nr = 0;
        if (np > 0) {
            Buf<uint64_t> key(np, s);
            Buf<double> val(np, s);
            LAUNCH(k_expand_rows, k1 - k0, s, xrow.p, X.ci.p, X.v.p, k0, k1, (int32_t)r0, Y.rp.p, Y.ci.p, Y.v.p, off.p,
                   rowoff[r0], ncols, key.p, val.p);
            sort_pairs(key, val, np, bits_for((uint64_t)(r1 - r0) * ncols), s);
            Buf<int64_t> flag(np + 1, s), pos(np + 1, s);
            GCK(cudaMemsetAsync(flag.p + np, 0, 8, s));
            LAUNCH(k_runflag, np, s, key.p, np, flag.p);
            excl_scan(flag.p, pos.p, np + 1, s);
            nr = dev_get(pos.p + np, s);
            Buf<int64_t> start(nr, s);
            LAUNCH(k_runstart, np, s, flag.p, pos.p, np, start.p);
            flag.release();
            pos.release();
            cci.alloc(nr, s);
            cv.alloc(nr, s);
            LAUNCH(k_runsum, nr, s, key.p, val.p, start.p, nr, np, ncols, cci.p, cv.p, rc.p + r0);
        }
        pci.push_back(std::move(cci));
        pv.push_back(std::move(cv));
        pn.push_back(nr);
        r0 = r1;
    }
    xrow.release();
    off.release();
    int64_t tot = 0;
    for (int64_t x : pn) tot += x;
    C.nnz = tot;
    if (pci.size() == 1) {
        C.ci = std::move(pci[0]);
        C.v = std::move(pv[0]);
    } else {
        C.ci.alloc(tot, s);
        C.v.alloc(tot, s);
        int64_t o = 0;
        for (size_t c = 0; c < pci.size(); ++c) {
            if (pn[c]) {
                GCK(cudaMemcpyAsync(C.ci.p + o, pci[c].p, pn[c] * 4, cudaMemcpyDeviceToDevice, s));
                GCK(cudaMemcpyAsync(C.v.p + o, pv[c].p, pn[c] * 8, cudaMemcpyDeviceToDevice, s));
            }
            o += pn[c];
            pci[c].release();
            pv[c].release();
        }
    }
    rp_from_counts(rc.p, C.nrows, C.rp, s);
    return C;
}

DCsr transpose(const DCsr& X, cudaStream_t s) {
    DCsr T;
    T.nrows = X.ncols;
    T.ncols = X.nrows;
    T.nnz = X.nnz;
    Buf<uint32_t> ck(X.nnz, s);
    Buf<int64_t> idx(X.nnz, s);
    LAUNCH(k_colkey, X.nnz, s, X.ci.p, X.nnz, ck.p, idx.p);
    sort_pairs(ck, idx, X.nnz, bits_for((uint64_t)std::max<int64_t>(1, X.ncols)), s);
    Buf<int32_t> row(X.nnz, s);
    LAUNCH(k_rowof, X.nrows, s, X.rp.p, X.nrows, row.p);
    T.ci.alloc(X.nnz, s);
    T.v.alloc(X.nnz, s);
    Buf<unsigned long long> cnt(T.nrows, s);
    GCK(cudaMemsetAsync(cnt.p, 0, T.nrows * 8, s));
    LAUNCH(k_tr_gather, X.nnz, s, idx.p, row.p, X.v.p, X.nnz, T.ci.p, T.v.p, cnt.p, ck.p);
    rp_from_counts(cnt.p, T.nrows, T.rp, s);
    return T;
}

// keep the entries flagged in keep[] (values nv), rows unchanged
DCsr compact(const DCsr& X, const Buf<double>& nv, const Buf<int64_t>& keep, cudaStream_t s) {
    DCsr C;
    C.nrows = X.nrows;
    C.ncols = X.ncols;
    Buf<int64_t> pos(X.nnz + 1, s);
    excl_scan(keep.p, pos.p, X.nnz + 1, s);
    C.nnz = dev_get(pos.p + X.nnz, s);
    C.ci.alloc(C.nnz, s);
    C.v.alloc(C.nnz, s);
    C.rp.alloc(C.nrows + 1, s);
    LAUNCH(k_compact, X.nrows, s, X.rp.p, X.ci.p, nv.p, keep.p, pos.p, X.nrows, C.ci.p, C.v.p, C.rp.p);
    GCK(cudaMemcpyAsync(C.rp.p + C.nrows, pos.p + X.nnz, 8, cudaMemcpyDeviceToDevice, s));
    return C;
}

void mirror_drop(DCsr& C, cudaStream_t s) {
    Buf<double> nv(C.nnz, s);
    Buf<int64_t> keep(C.nnz + 1, s);
    GCK(cudaMemsetAsync(keep.p + C.nnz, 0, 8, s));
    LAUNCH(k_mirror, C.nrows, s, C.rp.p, C.ci.p, C.v.p, C.nrows, nv.p, keep.p);
    C = compact(C, nv, keep, s);
}

DCsr galerkin(const DCsr& P, const DCsr& A, cudaStream_t s) {
    DCsr T = spgemm(A, P, s);
    DCsr Pt = transpose(P, s);
    DCsr C = spgemm(Pt, T, s);
    mirror_drop(C, s);
    return C;
}

DCsr one_per_row(const Buf<int32_t>& agg, const Buf<double>& val, int64_t n, int64_t nc, cudaStream_t s) {
    DCsr P;
    P.nrows = n;
    P.ncols = nc;
    Buf<int64_t> cnt(n + 1, s);
    GCK(cudaMemsetAsync(cnt.p + n, 0, 8, s));
    LAUNCH(k_opr_count, n, s, val.p, n, cnt.p);
    P.rp.alloc(n + 1, s);
    excl_scan(cnt.p, P.rp.p, n + 1, s);
    P.nnz = dev_get(P.rp.p + n, s);
    P.ci.alloc(P.nnz, s);
    P.v.alloc(P.nnz, s);
    LAUNCH(k_opr_fill, n, s, agg.p, val.p, P.rp.p, n, P.ci.p, P.v.p);
    return P;
}

Buf<double> restrict_vec(const DCsr& P, const Buf<double>& w, cudaStream_t s) {
    DCsr Pt = transpose(P, s);
    Buf<double> out(Pt.nrows, s);
    LAUNCH(k_restrict_w, Pt.nrows, s, Pt.rp.p, Pt.ci.p, Pt.v.p, w.p, Pt.nrows, out.p);
    return out;
}

// suitor matching on A with weights w -> mate (device)
void matching(const DCsr& A, const Buf<double>& w, Buf<int32_t>& mate, cudaStream_t s) {
    const int64_t n = A.nrows;
    Buf<double> d(n, s);
    LAUNCH(k_diag, n, s, A.rp.p, A.ci.p, A.v.p, n, d.p);
    Buf<uint64_t> key(A.nnz, s);
    LAUNCH(k_keys, n, s, A.rp.p, A.ci.p, A.v.p, d.p, w.p, n, key.p);
    // distinct key values (ascending) -> 32-bit ranks
    Buf<uint64_t> sorted(A.nnz, s), uniq(A.nnz, s);
    Buf<int64_t> nu(1, s);
    {
        size_t tb = 0;
        GCK(cub::DeviceRadixSort::SortKeys(nullptr, tb, key.p, sorted.p, A.nnz, 0, 64, s));
        Buf<char> tmp(tb, s);
        GCK(cub::DeviceRadixSort::SortKeys(tmp.p, tb, key.p, sorted.p, A.nnz, 0, 64, s));
    }
    {
        size_t tb = 0;
        GCK(cub::DeviceSelect::Unique(nullptr, tb, sorted.p, uniq.p, nu.p, A.nnz, s));
        Buf<char> tmp(tb, s);
        GCK(cub::DeviceSelect::Unique(tmp.p, tb, sorted.p, uniq.p, nu.p, A.nnz, s));
    }
    const int64_t nuniq = dev_get(nu.p, s);
    sorted.release();
    Buf<uint32_t> rank(A.nnz, s);
    LAUNCH(k_rank, A.nnz, s, key.p, A.nnz, uniq.p, nuniq, rank.p);
    key.release();
    uniq.release();
    Buf<unsigned long long> sv(n, s);
    GCK(cudaMemsetAsync(sv.p, 0, n * 8, s));
    LAUNCH(k_suitor, n, s, A.rp.p, A.ci.p, rank.p, n, sv.p);
    mate.alloc(n, s);
    LAUNCH(k_mates, n, s, sv.p, n, mate.p);
}


DevCsrRaw hand_over(DCsr& D) {
    DevCsrRaw r;
    r.nrows = D.nrows;
    r.ncols = D.ncols;
    r.nnz = D.nnz;
    r.rp = D.rp.hand_over();
    r.ci = D.ci.hand_over();
    r.v = D.v.hand_over();
    return r;
}

// host Csr carrying only the shape and the row pointers of a device matrix
Csr rp_only(const DCsr& D, cudaStream_t s) {
    Csr A;
    A.nrows = D.nrows;
    A.ncols = D.ncols;
    A.rp.resize(D.nrows + 1);
    GCK(cudaMemcpyAsync(A.rp.data(), D.rp.p, (D.nrows + 1) * 8, cudaMemcpyDeviceToHost, s));
    GCK(cudaStreamSynchronize(s));
    return A;
}

}  // namespace

void DeviceKeep::free_all() {
    for (auto* M : {&A, &P, &R})
        for (auto& x : *M) {
            cudaFree(x.rp);
            cudaFree(x.ci);
            cudaFree(x.v);
        }
    for (double* x : m) cudaFree(x);
    A.clear();
    P.clear();
    R.clear();
    m.clear();
}


// Full GPU build with the same results as amgsetup::build (validated input A0 on the
// host; the hierarchy is copied back into `out` for partitioning / format upload).
int build_gpu(Csr&& A0, std::vector<double>&& w0, const Config& cfg, Hierarchy& out, std::string& err) {
    // a non-sticky error left by an unrelated earlier runtime call of this thread would be
    // reported by the first CUB call below (CUB peeks at the last error): clear it first
    cudaGetLastError();
    cudaStream_t s;
    if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) {
        err = "build_gpu: cudaStreamCreate failed";
        return SETUP_ERR_ARG;
    }
    int code = SETUP_OK;
    // keep freed blocks in the stream-ordered pool for the whole build (the default
    // threshold 0 returns them to the driver at every synchronisation, and the next
    // allocation maps fresh memory); trimmed again at the end
    int dev = 0;
    cudaGetDevice(&dev);
    cudaMemPool_t pool = nullptr;
    cudaDeviceGetDefaultMemPool(&pool, dev);
    uint64_t keep_all = UINT64_MAX, old_thr = 0;
    if (pool) {
        cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &old_thr);
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep_all);
    }
    try {
        out.lv.clear();
        out.lv.emplace_back();
        DCsr A = upload(A0, s);
        Buf<double> w(A0.nrows, s);
        GCK(cudaMemcpyAsync(w.p, w0.data(), A0.nrows * 8, cudaMemcpyHostToDevice, s));
        out.lv[0].A = std::move(A0);
        out.lv[0].w = std::move(w0);
        tmark("(gpu upload)");
        for (int l = 0;; ++l) {
            const int64_t n = A.nrows;
            {
                Buf<double> m(n, s);
                LAUNCH(k_rowabs, n, s, A.rp.p, A.v.p, n, (const double*)nullptr, m.p, (double*)nullptr);
                out.lv[l].m = download_vec(m, n, s);  // O7
                if (out.keep_device) out.dev.m.push_back(m.hand_over());
            }
            if (n <= cfg.max_coarse_size || l == cfg.max_levels - 1) break;  // O1
            Buf<int32_t> cagg(n, s);
            Buf<double> cval(n, s);
            LAUNCH(k_iota, n, s, cagg.p, n);
            LAUNCH(k_fill, n, s, cval.p, n, 1.0);
            DCsr As_store;
            const DCsr* As = &A;
            Buf<double> ws(n, s);
            GCK(cudaMemcpyAsync(ws.p, w.p, n * 8, cudaMemcpyDeviceToDevice, s));
            int64_t ns = n;
            int done = 0;
            for (int sw = 0; sw < cfg.sweeps_per_level; ++sw) {
                Buf<int32_t> mate;
                matching(*As, ws, mate, s);
                Buf<int64_t> head(ns + 1, s), id(ns + 1, s);
                GCK(cudaMemsetAsync(head.p + ns, 0, 8, s));
                LAUNCH(k_heads, ns, s, mate.p, ns, head.p);
                excl_scan(head.p, id.p, ns + 1, s);
                const int64_t nc = dev_get(id.p + ns, s);
                if (nc == ns) break;  // no size reduction
                Buf<int32_t> sagg(ns, s);
                Buf<double> spval(ns, s);
                LAUNCH(k_pairwise, ns, s, mate.p, id.p, ws.p, ns, sagg.p, spval.p);
                DCsr Ps = one_per_row(sagg, spval, ns, nc, s);
                DCsr An = galerkin(Ps, *As, s);
                Buf<double> wn = restrict_vec(Ps, ws, s);
                LAUNCH(k_compose, n, s, cagg.p, cval.p, sagg.p, spval.p, n);
                As_store = std::move(An);
                As = &As_store;
                ws = std::move(wn);
                ns = nc;
                ++done;
            }
            As_store = DCsr();
            tmark("(gpu sweeps)");
            if (done == 0 || (double)n / (double)ns < cfg.min_coarsening_ratio) break;  // O1
            const int64_t nc = ns;
            DCsr P = one_per_row(cagg, cval, n, nc, s);
            DCsr Pb;
            Level& L = out.lv[l];
            if (cfg.smooth_prolongator) {
                Buf<double> d(n, s), q(n, s);
                LAUNCH(k_diag, n, s, A.rp.p, A.ci.p, A.v.p, n, d.p);
                LAUNCH(k_rowabs, n, s, A.rp.p, A.v.p, n, (const double*)d.p, (double*)nullptr, q.p);
                Buf<double> mx(1, s);
                {
                    size_t tb = 0;
                    GCK(cub::DeviceReduce::Max(nullptr, tb, q.p, mx.p, n, s));
                    Buf<char> tmp(tb, s);
                    GCK(cub::DeviceReduce::Max(tmp.p, tb, q.p, mx.p, n, s));
                }
                L.omega = cfg.prol_omega_scale / dev_get(mx.p, s);  // O4 (host division, correctly rounded)
                DCsr T = spgemm(A, P, s);
                Buf<double> nv(T.nnz, s);
                Buf<int64_t> keep(T.nnz + 1, s);
                GCK(cudaMemsetAsync(keep.p + T.nnz, 0, 8, s));
                LAUNCH(k_pbar, n, s, T.rp.p, T.ci.p, T.v.p, P.rp.p, P.ci.p, P.v.p, d.p, L.omega, n, nv.p, keep.p);
                Pb = compact(T, nv, keep, s);
            } else {
                L.omega = 0.0;
                Pb = std::move(P);
                P = DCsr();
            }
            DCsr Ac = galerkin(Pb, A, s);  // O6
            Buf<double> wc = restrict_vec(cfg.smooth_prolongator ? P : Pb, w, s);
            DCsr R = transpose(Pb, s);
            tmark("(gpu P-bar, galerkin)");
            L.agg = download_vec(cagg, n, s);
            L.sweeps = done;
            Level next;
            next.w = download_vec(wc, nc, s);
            if (out.keep_device) {  // operators stay on the device; the host keeps shapes + row pointers
                L.P = rp_only(Pb, s);
                L.R = rp_only(R, s);
                next.A = rp_only(Ac, s);
                GCK(cudaStreamSynchronize(s));
                out.dev.P.push_back(hand_over(Pb));
                out.dev.R.push_back(hand_over(R));
                out.dev.A.push_back(hand_over(A));
            } else {
                L.P = download(Pb, s);
                L.R = download(R, s);
                next.A = download(Ac, s);
            }
            out.lv.push_back(std::move(next));
            A = std::move(Ac);
            w = std::move(wc);
            tmark("(gpu download)");
        }
        if (out.keep_device) {  // the coarsest: device copy kept, full host copy for the dense inverse
            out.lv.back().A = download(A, s);
            out.dev.A.push_back(hand_over(A));
        }
        GCK(cudaStreamSynchronize(s));
    } catch (const std::string& e) {
        err = "build_gpu: " + e;
        code = SETUP_ERR_ARG;
        out.dev.free_all();
    }
    cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
    if (pool) {
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &old_thr);
        cudaMemPoolTrimTo(pool, 0);
    }
    if (code != SETUP_OK) return code;
    if (!dense_inverse_host(out.lv.back().A, out.coarse_inv)) {  // O8
        err = "coarsest-level Cholesky failed (matrix not s.p.d.)";
        return SETUP_ERR_NOT_SPD;
    }
    return SETUP_OK;
}

}  // namespace amgsetup
