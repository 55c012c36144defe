// amg_api.cu — implementation of include/amg_b200.h.
//
// Host side: validates/copies the caller's CSR, runs the C++ setup
// (csrc/setup), chooses a device format per operator, uploads, and drives the
// solve phase.  Device side: kernels.cuh.  A PCG solve is ONE graph launch: a
// prologue kernel followed by a CUDA-graph WHILE node whose body is
//   V-cycle(r -> z) [fused r^T z -> beta]   -> p = z + beta p
//   q = A p [fused p^T q -> alpha]          -> x += alpha p, r -= alpha q [fused
//   ||r||^2 -> convergence test -> cudaGraphSetConditional]
// so the iteration count is decided on the device (no host round trip).
#include <cuda_runtime.h>
#include <omp.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/amg_b200.h"
#include "kernels.cuh"
#include "setup/setup.hpp"

using namespace amgk;

namespace {

thread_local std::string g_err;
void set_err(const std::string& s) { g_err = s; }

#define CK(call)                                                                 \
    do {                                                                         \
        cudaError_t e_ = (call);                                                 \
        if (e_ != cudaSuccess) {                                                 \
            set_err(std::string(#call) + ": " + cudaGetErrorString(e_));         \
            return e_ == cudaErrorMemoryAllocation ? AMG_ERR_OOM : AMG_ERR_CUDA; \
        }                                                                        \
    } while (0)

enum { FMT_SELL = 0, FMT_CSRV = 1, FMT_DENSE = 2, FMT_SDIA = 3 };
constexpr int kVWBlock = 256;  // CSR-vector "VW" value meaning one block per row

struct DevMat {
    int fmt = FMT_SELL;
    int vw = 32;
    int64_t nrows = 0, ncols = 0, nnz = 0, stored = 0;
    uint32_t* sptr = nullptr;  // SELL / SDIA
    int32_t* offs = nullptr;   // SDIA: one column offset per slice column
    int32_t* rp = nullptr;     // CSR
    int32_t* col = nullptr;
    double* val = nullptr;
    // algorithmic bytes of one pass over the operator: 12 nnz + 4 (n+1)
    double model_bytes() const { return 12.0 * (double)nnz + 4.0 * (double)(nrows + 1); }
    // bytes the chosen device format actually stores for one pass
    double stored_bytes() const {
        const double nsl = (double)((nrows + 31) / 32);
        switch (fmt) {
            case FMT_SELL: return 12.0 * (double)stored + 4.0 * (nsl + 1);
            case FMT_SDIA: return 8.0 * (double)stored + 4.0 * (double)stored / 32.0 + 4.0 * (nsl + 1);
            default: return 12.0 * (double)nnz + 4.0 * (double)(nrows + 1);
        }
    }
    void release() {
        cudaFree(sptr);
        cudaFree(offs);
        cudaFree(rp);
        cudaFree(col);
        cudaFree(val);
        sptr = nullptr;
        offs = nullptr;
        rp = col = nullptr;
        val = nullptr;
    }
};

struct DevLevel {
    int64_t n = 0;
    DevMat A, P, R;
    double* m = nullptr;
    double* b = nullptr;   // rhs of the level (unused at level 0: the caller's vector)
    double* mb = nullptr;  // m o b, written by the restriction into this level (levels >= 1)
    double* r = nullptr;   // residual
    double* xa = nullptr;  // the level's x (output of its V-cycle)
    double* xb = nullptr;  // ping-pong partner
    std::vector<int32_t> agg;
    int sweeps = 0;
    double omega = 0.0;
};

struct KernelRec {
    const char* name;
    double bytes;         // algorithmic
    double stored_bytes;  // what the device format actually moves (compulsory)
    cudaEvent_t e0, e1;
};

}  // namespace

struct amg_ctx_s {
    int device = 0, rank = 0, nranks = 1;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    int nsm = 148;
};

struct amg_hier_s {
    amg_ctx_s* ctx = nullptr;
    amg_config_t cfg{};
    std::vector<DevLevel> lv;   // non-coarsest levels
    DevMat A0;                  // level-0 operator when the hierarchy has one level
    int64_t n0 = 0, nnz0 = 0, nL = 0;
    int64_t nnzL = 0;
    double* cinv = nullptr;     // dense A_L^{-1}, row-major
    double* cb = nullptr;       // coarsest rhs
    double* cx = nullptr;       // coarsest solution
    double *pr = nullptr, *pz = nullptr, *pp = nullptr, *pq = nullptr;  // PCG vectors
    double *hb = nullptr, *hx = nullptr;  // staging for amg_solve_host
    PcgState* st = nullptr;
    PcgState* st_host = nullptr;
    double* partials = nullptr;
    unsigned int* ticket = nullptr;
    double setup_s = 0, opc = 0, avg_cr = 0, bytes_v = 0, bytes_it = 0;
    cudaGraphExec_t solve_exec = nullptr;
    const double* solve_b = nullptr;
    double* solve_x = nullptr;
    cudaGraphExec_t apply_exec = nullptr;
    const double* apply_r = nullptr;
    double* apply_z = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    std::vector<KernelRec>* prof = nullptr;

    const DevMat& Afine() const { return lv.empty() ? A0 : lv[0].A; }
    ~amg_hier_s() {
        if (solve_exec) cudaGraphExecDestroy(solve_exec);
        if (apply_exec) cudaGraphExecDestroy(apply_exec);
        for (auto& D : lv) {
            D.A.release();
            D.P.release();
            D.R.release();
            cudaFree(D.m);
            cudaFree(D.b);
            cudaFree(D.mb);
            cudaFree(D.r);
            cudaFree(D.xa);
            cudaFree(D.xb);
        }
        A0.release();
        cudaFree(cinv);
        cudaFree(cb);
        cudaFree(cx);
        cudaFree(pr);
        cudaFree(pz);
        cudaFree(pp);
        cudaFree(pq);
        cudaFree(hb);
        cudaFree(hx);
        cudaFree(st);
        cudaFreeHost(st_host);
        cudaFree(partials);
        cudaFree(ticket);
        if (ev0) cudaEventDestroy(ev0);
        if (ev1) cudaEventDestroy(ev1);
    }
};

namespace {

constexpr int kMaxPartials = 8192;

int max_grid(const void* fn, int nsm) {
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, kBlock, 0);
    if (nb < 1) nb = 1;
    return std::min(nb * nsm, kMaxPartials);
}

int vec_grid(int64_t n, int nsm) {
    const int64_t need = (n + kBlock - 1) / kBlock;
    return (int)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)nsm * 8));
}

// Optional per-launch CUDA-event timing (amg_profile_vcycle).
struct Launch {
    amg_hier_s* h;
    cudaStream_t s;
    void begin(const char* name, double bytes, double stored = -1.0) {
        if (!h->prof) return;
        KernelRec r{name, bytes, stored < 0.0 ? bytes : stored, nullptr, nullptr};
        cudaEventCreate(&r.e0);
        cudaEventCreate(&r.e1);
        cudaEventRecord(r.e0, s);
        h->prof->push_back(r);
    }
    void end() {
        if (h->prof) cudaEventRecord(h->prof->back().e1, s);
    }
};

template <class G, class E>
void launch_mat(Launch& L, const DevMat& M, G g, E e, RedCtx rc, const char* name, double vec_bytes) {
    const int nsm = L.h->ctx->nsm;
    L.begin(name, M.model_bytes() + vec_bytes, M.stored_bytes() + vec_bytes);
    if (M.fmt == FMT_SDIA) {
        static const int cap = max_grid((const void*)k_sdia<G, E>, nsm);
        const int64_t need = (M.nrows + kBlock - 1) / kBlock;
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(need, cap));
        k_sdia<G, E><<<grid, kBlock, 0, L.s>>>(SdiaView{M.sptr, M.offs, M.val, M.nrows, (int32_t)M.ncols}, g, e, rc);
    } else if (M.fmt == FMT_SELL) {
        static const int cap = max_grid((const void*)k_sell<G, E>, nsm);
        const int64_t need = (M.nrows + kBlock - 1) / kBlock;
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(need, cap));
        k_sell<G, E><<<grid, kBlock, 0, L.s>>>(SellView{M.sptr, M.col, M.val, M.nrows}, g, e, rc);
    } else {
        const CsrView v{M.rp, M.col, M.val, M.nrows};
        const int64_t need = (M.nrows * M.vw + kBlock - 1) / kBlock;
        if (M.vw == kVWBlock) {
            static const int cap = max_grid((const void*)k_csrb<G, E>, nsm);
            const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(M.nrows, cap));
            k_csrb<G, E><<<grid, kBlock, 0, L.s>>>(v, g, e, rc);
            L.end();
            return;
        }
        switch (M.vw) {
#define VWCASE(W)                                                                 \
    case W: {                                                                     \
        static const int cap = max_grid((const void*)k_csrv<W, G, E>, nsm);       \
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(need, cap)); \
        k_csrv<W, G, E><<<grid, kBlock, 0, L.s>>>(v, g, e, rc);                   \
        break;                                                                    \
    }
            VWCASE(2)
            VWCASE(4)
            VWCASE(8)
            VWCASE(16)
            VWCASE(32)
#undef VWCASE
            default:
                break;
        }
    }
    L.end();
}

RedCtx no_red() { return RedCtx{nullptr, nullptr, nullptr, nullptr, 0ull, FIN_NONE}; }
RedCtx red(amg_hier_s* h, int kind, unsigned long long cond) {
    return RedCtx{h->partials, h->ticket, nullptr, h->st, cond, kind};
}

// z0 = A_L^{-1} b0 on the coarsest level.
void enqueue_coarse(amg_hier_s* h, Launch& L, const double* b, double* z) {
    L.begin("coarse_gemv", 8.0 * (double)h->nL * (double)h->nL + 16.0 * (double)h->nL);
    k_dense_gemv<<<vec_grid(h->nL * 32, h->ctx->nsm), kBlock, 0, L.s>>>(h->cinv, b, z, h->nL);
    L.end();
}

// One V-cycle z0 = B b0 (Eq. 3.1) enqueued on
// L.s.  If `rz` is given, the last level-0 post-sweep also reduces b0^T z0.
void enqueue_vcycle(amg_hier_s* h, Launch& L, const double* b0, double* z0, const RedCtx* rz) {
    const int nlev = (int)h->lv.size();
    const int s1 = h->cfg.pre_sweeps, s2 = h->cfg.post_sweeps;
    if (nlev == 0) {  // single-level hierarchy: B = A^{-1}
        enqueue_coarse(h, L, b0, z0);
        return;
    }
    std::vector<double*> xpre(nlev, nullptr);  // pre-smoothed x of each level (s1 >= 2)
    // ---- down: pre-smoothing, residual, restriction
    for (int l = 0; l < nlev; ++l) {
        DevLevel& D = h->lv[l];
        const double* b = (l == 0) ? b0 : D.b;
        const double n8 = 8.0 * (double)D.n;
        if (s1 == 1) {
            // x = m o b is never stored: r = b - A (m o b)
            if (l == 0)
                launch_mat(L, D.A, GMB{D.m, b}, EResid{b, D.r}, no_red(), "resid0", 3 * n8);
            else
                launch_mat(L, D.A, GVec{D.mb}, EResid{b, D.r}, no_red(), "resid0", 3 * n8);
        } else {
            // x2 = m b + m (b - A (m b)): the first two sweeps from x = 0 in one pass
            double* xi = D.xa;
            double* xo = D.xb;
            if (l == 0)
                launch_mat(L, D.A, GMB{D.m, b}, ESweep0{b, D.m, xi}, no_red(), "sweep0", 3 * n8);
            else
                launch_mat(L, D.A, GVec{D.mb}, ESweep0{b, D.m, xi}, no_red(), "sweep0", 3 * n8);
            for (int s = 2; s < s1; ++s) {
                launch_mat(L, D.A, GVec{xi}, ESweep<false>{xi, b, D.m, xo}, no_red(), "presweep", 4 * n8);
                std::swap(xi, xo);
            }
            launch_mat(L, D.A, GVec{xi}, EResid{b, D.r}, no_red(), "resid", 3 * n8);
            xpre[l] = xi;
        }
        if (l + 1 < nlev) {
            DevLevel& C = h->lv[l + 1];
            launch_mat(L, D.R, GVec{D.r}, EStoreMB{C.b, C.m, C.mb}, no_red(), "restrict",
                       n8 + 24.0 * (double)C.n);
        } else {
            launch_mat(L, D.R, GVec{D.r}, EStore{h->cb}, no_red(), "restrict", n8 + 8.0 * (double)h->nL);
        }
    }
    enqueue_coarse(h, L, h->cb, h->cx);  // z_L = A_L^{-1} b_L (reading R2)
    // ---- up: prolongation, post-smoothing
    for (int l = nlev - 1; l >= 0; --l) {
        DevLevel& D = h->lv[l];
        const double* b = (l == 0) ? b0 : D.b;
        const double* e = (l + 1 < nlev) ? h->lv[l + 1].xa : h->cx;
        const int64_t nc = (l + 1 < nlev) ? h->lv[l + 1].n : h->nL;
        const double n8 = 8.0 * (double)D.n;
        double* fin = (l == 0) ? z0 : D.xa;  // the level's result (read by level l-1)
        double* tmp = D.xb;                  // the prolongation update is row-local, so it
                                             // may run in place on xpre
        double* dst = (s2 % 2 == 1) ? tmp : fin;
        if (s1 == 1) {
            if (l == 0)
                launch_mat(L, D.P, GVec{e}, EProlong0{b, D.m, dst}, no_red(), "prolong0", 3 * n8 + 8.0 * nc);
            else
                launch_mat(L, D.P, GVec{e}, EProlongMB{D.mb, dst}, no_red(), "prolong0", 2 * n8 + 8.0 * nc);
        } else {
            launch_mat(L, D.P, GVec{e}, EProlongAdd{xpre[l], dst}, no_red(), "prolong", 2 * n8 + 8.0 * nc);
        }
        double* xi = dst;
        for (int s = 0; s < s2; ++s) {
            double* xo = (xi == tmp) ? fin : tmp;
            if (l == 0 && s == s2 - 1 && rz)
                launch_mat(L, D.A, GVec{xi}, ESweep<true>{xi, b, D.m, xo}, *rz, "postsweep_dot", 4 * n8);
            else
                launch_mat(L, D.A, GVec{xi}, ESweep<false>{xi, b, D.m, xo}, no_red(), "postsweep", 4 * n8);
            xi = xo;
        }
    }
}

// PCG loop body, rotated so that the convergence test is the last node:
//   z = V(r), rho' = r^T z, beta ; p = z + beta p ; q = A p, alpha ; x, r update, test.
void enqueue_pcg_body(amg_hier_s* h, Launch& L, double* x, unsigned long long cond) {
    const int64_t n = h->n0;
    const int nsm = h->ctx->nsm;
    RedCtx rz = red(h, FIN_RZ, 0);
    if (!h->lv.empty()) {
        enqueue_vcycle(h, L, h->pr, h->pz, &rz);
    } else {
        enqueue_coarse(h, L, h->pr, h->pz);
        L.begin("dot_rz", 16.0 * n);
        k_dot<<<vec_grid(n, nsm), kBlock, 0, L.s>>>(h->pr, h->pz, n, rz);
        L.end();
    }
    L.begin("pupdate", 24.0 * n);
    k_pupdate<<<vec_grid(n, nsm), kBlock, 0, L.s>>>(h->pz, h->pp, n, h->st);
    L.end();
    launch_mat(L, h->Afine(), GVec{h->pp}, ESpmvDot{h->pp, h->pq}, red(h, FIN_PQ, 0), "spmv_dot", 16.0 * n);
    L.begin("axpy_rr", 48.0 * n);
    k_axpy_rr<<<vec_grid(n, nsm), kBlock, 0, L.s>>>(x, h->pr, h->pp, h->pq, n, red(h, FIN_RR, cond));
    L.end();
}

void enqueue_pcg_init(amg_hier_s* h, Launch& L, const double* b, double* x, unsigned long long cond) {
    L.begin("pcg_init", 24.0 * h->n0);
    k_pcg_init<<<vec_grid(h->n0, h->ctx->nsm), kBlock, 0, L.s>>>(b, h->pr, x, h->n0, red(h, FIN_BNORM, cond));
    L.end();
}

// ------------------------------------------------------------- upload
template <class T>
int dev_copy(T** dst, const T* src, size_t count) {
    CK(cudaMalloc((void**)dst, std::max<size_t>(1, count) * sizeof(T)));
    if (count) CK(cudaMemcpy(*dst, src, count * sizeof(T), cudaMemcpyHostToDevice));
    return AMG_OK;
}

template <class T>
int dev_alloc(T** dst, size_t count) {
    CK(cudaMalloc((void**)dst, std::max<size_t>(1, count) * sizeof(T)));
    CK(cudaMemset(*dst, 0, std::max<size_t>(1, count) * sizeof(T)));
    return AMG_OK;
}

// Per-operator storage choice (north_star (1): "CSR/sliced-ELL storage chosen per
// level"): SELL-32 when rows are short and padding is small, CSR-vector with
// VW lanes per row otherwise.
int upload_mat(const amgsetup::Csr& M, DevMat& D) {
    const int64_t n = M.nrows, nnz = M.nnz();
    D.nrows = n;
    D.ncols = M.ncols;
    D.nnz = nnz;
    const int64_t nsl = (n + 31) / 32;
    std::vector<uint32_t> width(nsl, 0);
#pragma omp parallel for schedule(static)
    for (int64_t s = 0; s < nsl; ++s) {
        int64_t w = 0;
        for (int64_t r = s * 32; r < std::min(n, s * 32 + 32); ++r) w = std::max(w, M.rp[r + 1] - M.rp[r]);
        width[s] = (uint32_t)w;
    }
    int64_t padded = 0;
    for (int64_t s = 0; s < nsl; ++s) padded += 32 * (int64_t)width[s];
    const double mean = n ? (double)nnz / (double)n : 0.0;
    // SDIA-32 candidate: per slice, the sorted distinct offsets col - row
    if (M.nrows == M.ncols && nsl >= 148 * 16 && mean <= 64.0) {
        std::vector<uint32_t> dw(nsl, 0);
        std::vector<std::vector<int32_t>> soffs(nsl);
#pragma omp parallel for schedule(static)
        for (int64_t s = 0; s < nsl; ++s) {
            auto& o = soffs[s];
            for (int64_t r = s * 32; r < std::min(n, s * 32 + 32); ++r)
                for (int64_t t = M.rp[r]; t < M.rp[r + 1]; ++t) o.push_back((int32_t)((int64_t)M.ci[t] - r));
            std::sort(o.begin(), o.end());
            o.erase(std::unique(o.begin(), o.end()), o.end());
            dw[s] = (uint32_t)o.size();
        }
        int64_t dpad = 0;
        for (int64_t s = 0; s < nsl; ++s) dpad += 32 * (int64_t)dw[s];
        if ((double)dpad <= 1.02 * (double)padded + 64.0 && dpad / 32 < (int64_t)UINT32_MAX) {
            D.fmt = FMT_SDIA;
            D.stored = dpad;
            std::vector<uint32_t> sptr(nsl + 1, 0);
            for (int64_t s = 0; s < nsl; ++s) sptr[s + 1] = sptr[s] + dw[s];
            std::vector<int32_t> offs(dpad / 32);
            std::vector<double> val(dpad, 0.0);
#pragma omp parallel for schedule(static)
            for (int64_t s = 0; s < nsl; ++s) {
                const auto& o = soffs[s];
                std::copy(o.begin(), o.end(), offs.begin() + sptr[s]);
                const int64_t base = (int64_t)sptr[s] * 32;
                for (int64_t r = s * 32; r < std::min(n, s * 32 + 32); ++r) {
                    const int64_t lane = r - s * 32;
                    size_t k = 0;
                    for (int64_t t = M.rp[r]; t < M.rp[r + 1]; ++t) {
                        const int32_t d = (int32_t)((int64_t)M.ci[t] - r);
                        while (o[k] != d) ++k;  // both ascending
                        val[base + (int64_t)k * 32 + lane] = M.v[t];
                    }
                }
            }
            int st;
            if ((st = dev_copy(&D.sptr, sptr.data(), sptr.size()))) return st;
            if ((st = dev_copy(&D.offs, offs.data(), offs.size()))) return st;
            if ((st = dev_copy(&D.val, val.data(), val.size()))) return st;
            return AMG_OK;
        }
    }
    // SELL-32 (one thread per row, coalesced column-major slices) needs little padding and
    // enough slices to fill the GPU (>= ~16 warps per SM); long rows are fine there because
    // every lane streams its own row with many loads in flight.
    const bool sell = (double)padded <= 1.10 * (double)nnz + 64.0 && nsl >= 148 * 16 &&
                      padded / 32 < (int64_t)UINT32_MAX;
    if (sell) {
        D.fmt = FMT_SELL;
        D.stored = padded;
        std::vector<uint32_t> sptr(nsl + 1, 0);
        for (int64_t s = 0; s < nsl; ++s) sptr[s + 1] = sptr[s] + width[s];
        std::vector<int32_t> col(padded, 0);
        std::vector<double> val(padded, 0.0);
#pragma omp parallel for schedule(static)
        for (int64_t s = 0; s < nsl; ++s) {
            const int64_t base = (int64_t)sptr[s] * 32;
            for (int64_t r = s * 32; r < std::min(n, s * 32 + 32); ++r) {
                const int64_t lane = r - s * 32;
                int64_t k = 0;
                for (int64_t t = M.rp[r]; t < M.rp[r + 1]; ++t, ++k) {
                    col[base + k * 32 + lane] = M.ci[t];
                    val[base + k * 32 + lane] = M.v[t];
                }
                for (; k < width[s]; ++k) col[base + k * 32 + lane] = (int32_t)std::min<int64_t>(r, M.ncols - 1);
            }
        }
        int st;
        if ((st = dev_copy(&D.sptr, sptr.data(), sptr.size()))) return st;
        if ((st = dev_copy(&D.col, col.data(), col.size()))) return st;
        if ((st = dev_copy(&D.val, val.data(), val.size()))) return st;
    } else {
        if (nnz >= (int64_t)INT32_MAX) {
            set_err("operator too large for 32-bit CSR row pointers on one rank");
            return AMG_ERR_ARG;
        }
        D.fmt = FMT_CSRV;
        D.stored = nnz;
        // lanes per row: enough threads to fill 148 SMs x 2048 threads, 2..32 lanes per
        // row inside a warp, or a whole block per row for few very long rows
        const double want = 148.0 * 2048.0 / (double)std::max<int64_t>(n, 1);
        int vw = 2;
        while (vw < 32 && (vw < want || vw * 8 < mean) && vw * 2 <= std::max(2.0, mean)) vw *= 2;
        static const double block_mean = std::getenv("AMG_BLOCK_MEAN") ? std::atof(std::getenv("AMG_BLOCK_MEAN")) : 256.0;
        static const double block_rows = std::getenv("AMG_BLOCK_ROWS") ? std::atof(std::getenv("AMG_BLOCK_ROWS")) : 18944.0;
        if (mean >= block_mean && (double)n < block_rows) vw = kVWBlock;
        D.vw = vw;
        std::vector<int32_t> rp(n + 1);
        for (int64_t i = 0; i <= n; ++i) rp[i] = (int32_t)M.rp[i];
        int st;
        if ((st = dev_copy(&D.rp, rp.data(), rp.size()))) return st;
        if ((st = dev_copy(&D.col, M.ci.data(), M.ci.size()))) return st;
        if ((st = dev_copy(&D.val, M.v.data(), M.v.size()))) return st;
    }
    return AMG_OK;
}

// SURVEY.md §8d byte model.
void byte_model(amg_hier_s* h, const amgsetup::Hierarchy& H) {
    const double s1 = h->cfg.pre_sweeps, s2 = h->cfg.post_sweeps;
    double bv = 0.0;
    const size_t nl = H.lv.size();
    for (size_t l = 0; l + 1 < nl; ++l) {
        const double n = (double)H.lv[l].A.nrows, nc = (double)H.lv[l + 1].A.nrows;
        const double MA = 12.0 * (double)H.lv[l].A.nnz() + 4.0 * (n + 1);
        const double MP = 12.0 * (double)H.lv[l].P.nnz() + 4.0 * (n + 1);
        bv += (s1 + s2) * MA + 2 * MP + 8 * n * ((s1 + s2) + 2 + 3 * (s1 - 1) + 2 + 2 + 3 * s2) + 16 * nc;
    }
    const double nL = (double)H.lv.back().A.nrows;
    bv += 8 * nL * nL + 16 * nL;
    h->bytes_v = bv;
    const double n0 = (double)H.lv[0].A.nrows;
    h->bytes_it = bv + 12.0 * (double)H.lv[0].A.nnz() + 4.0 * (n0 + 1) + 88.0 * n0;
}

int ensure_solve_graph(amg_hier_s* h, const double* b, double* x) {
    if (h->solve_exec && h->solve_b == b && h->solve_x == x) return AMG_OK;
    if (h->solve_exec) {
        cudaGraphExecDestroy(h->solve_exec);
        h->solve_exec = nullptr;
    }
    cudaStream_t s = h->ctx->stream;
    cudaGraph_t g;
    CK(cudaGraphCreate(&g, 0));
    cudaGraphConditionalHandle cond;
    CK(cudaGraphConditionalHandleCreate(&cond, g, 1, cudaGraphCondAssignDefault));
    Launch L{h, s};
    CK(cudaStreamBeginCaptureToGraph(s, g, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    enqueue_pcg_init(h, L, b, x, (unsigned long long)cond);
    CK(cudaStreamEndCapture(s, &g));
    size_t nn = 0;
    CK(cudaGraphGetNodes(g, nullptr, &nn));
    std::vector<cudaGraphNode_t> nodes(nn);
    CK(cudaGraphGetNodes(g, nodes.data(), &nn));
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = cond;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t wnode;
    CK(cudaGraphAddNode(&wnode, g, nodes.data(), nn, &cp));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    CK(cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    enqueue_pcg_body(h, L, x, (unsigned long long)cond);
    CK(cudaStreamEndCapture(s, &body));
    CK(cudaGraphInstantiate(&h->solve_exec, g, 0));
    CK(cudaGraphDestroy(g));
    h->solve_b = b;
    h->solve_x = x;
    return AMG_OK;
}

int ensure_apply_graph(amg_hier_s* h, const double* r, double* z) {
    if (h->apply_exec && h->apply_r == r && h->apply_z == z) return AMG_OK;
    if (h->apply_exec) {
        cudaGraphExecDestroy(h->apply_exec);
        h->apply_exec = nullptr;
    }
    cudaStream_t s = h->ctx->stream;
    Launch L{h, s};
    cudaGraph_t g;
    CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    enqueue_vcycle(h, L, r, z, nullptr);
    CK(cudaStreamEndCapture(s, &g));
    CK(cudaGraphInstantiate(&h->apply_exec, g, 0));
    CK(cudaGraphDestroy(g));
    h->apply_r = r;
    h->apply_z = z;
    return AMG_OK;
}

void fill_report(amg_hier_s* h, amg_report_t* rep) {
    rep->nlevels = (int32_t)h->lv.size() + 1;
    rep->setup_s = h->setup_s;
    rep->opc = h->opc;
    rep->avg_cr = h->avg_cr;
    rep->vcycle_bytes_model = h->bytes_v;
    rep->iteration_bytes_model = h->bytes_it;
}

// Copies the caller's CSR into the setup's form and runs the host setup.
int host_setup(int64_t n, const int64_t* rowptr, const int64_t* colind, const double* values,
               const double* w, const amg_config_t& cfg, amgsetup::Hierarchy& H) {
    if (!rowptr || !colind || !values || n <= 0) {
        set_err("null argument or empty matrix");
        return AMG_ERR_ARG;
    }
    if (n >= (int64_t)INT32_MAX) {
        set_err("n_global must be < 2^31");
        return AMG_ERR_ARG;
    }
    if (cfg.setup_threads > 0) omp_set_num_threads(cfg.setup_threads);
    if (rowptr[0] != 0) {
        set_err("rowptr[0] must be 0");
        return AMG_ERR_ARG;
    }
    for (int64_t i = 0; i < n; ++i)
        if (rowptr[i + 1] < rowptr[i]) {
            set_err("rowptr must be non-decreasing");
            return AMG_ERR_ARG;
        }
    const int64_t nnz = rowptr[n];
    amgsetup::Csr A;
    A.nrows = A.ncols = n;
    A.rp.assign(rowptr, rowptr + n + 1);
    A.ci.resize(nnz);
    A.v.assign(values, values + nnz);
    int bad = 0;
#pragma omp parallel for schedule(static) reduction(max : bad)
    for (int64_t k = 0; k < nnz; ++k) {
        const int64_t c = colind[k];
        if (c < 0 || c >= n) bad = 1;
        A.ci[k] = (int32_t)c;
    }
    if (bad) {
        set_err("column index out of range");
        return AMG_ERR_ARG;
    }
    std::vector<double> wv(n, 1.0);
    if (w) std::copy(w, w + n, wv.begin());
    amgsetup::Config sc;
    sc.sweeps_per_level = cfg.sweeps_per_level;
    sc.smooth_prolongator = cfg.smooth_prolongator;
    sc.prol_omega_scale = cfg.prol_omega_scale;
    sc.max_coarse_size = cfg.max_coarse_size;
    sc.max_levels = cfg.max_levels;
    sc.min_coarsening_ratio = cfg.min_coarsening_ratio;
    sc.pre_sweeps = cfg.pre_sweeps;
    sc.post_sweeps = cfg.post_sweeps;
    sc.threads = cfg.setup_threads;
    std::string err;
    const int sst = amgsetup::build(std::move(A), std::move(wv), sc, H, err);
    if (sst != amgsetup::SETUP_OK) {
        set_err(err);
        return sst == amgsetup::SETUP_ERR_ARG ? AMG_ERR_ARG : AMG_ERR_NOT_SPD;
    }
    return AMG_OK;
}

}  // namespace

// ===================================================================== ABI
extern "C" {

const char* amg_last_error(void) { return g_err.c_str(); }

void amg_config_default(amg_config_t* c) {
    if (!c) return;
    c->sweeps_per_level = 3;
    c->smooth_prolongator = 1;
    c->prol_omega_scale = 4.0 / 3.0;
    c->max_coarse_size = 200;
    c->max_levels = 20;
    c->min_coarsening_ratio = 1.2;
    c->pre_sweeps = 1;
    c->post_sweeps = 1;
    c->replicate_below_bytes = 64ll << 20;
    c->setup_threads = 0;
    c->use_graphs = 1;
}

int amg_ctx_create(int device, int rank, int nranks, const void* nccl_unique_id, void* cuda_stream,
                   amg_ctx_t* out) {
    (void)nccl_unique_id;
    if (!out || nranks < 1 || rank < 0 || rank >= nranks) {
        set_err("amg_ctx_create: bad rank/nranks or null out");
        return AMG_ERR_ARG;
    }
    if (nranks > 1) {
        set_err("amg_ctx_create: multi-rank contexts are not built in this version");
        return AMG_ERR_ARG;
    }
    *out = nullptr;
    CK(cudaSetDevice(device));
    auto* c = new amg_ctx_s();
    c->device = device;
    c->rank = rank;
    c->nranks = nranks;
    cudaDeviceGetAttribute(&c->nsm, cudaDevAttrMultiProcessorCount, device);
    if (cuda_stream) {
        c->stream = (cudaStream_t)cuda_stream;
    } else {
        cudaError_t e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
        if (e != cudaSuccess) {
            delete c;
            set_err(std::string("cudaStreamCreate: ") + cudaGetErrorString(e));
            return AMG_ERR_CUDA;
        }
        c->own_stream = true;
    }
    *out = c;
    return AMG_OK;
}

int amg_ctx_destroy(amg_ctx_t c) {
    if (!c) return AMG_OK;
    if (c->own_stream) cudaStreamDestroy(c->stream);
    delete c;
    return AMG_OK;
}

int amg_hierarchy_build(amg_ctx_t ctx, int64_t n_global, int64_t row_begin, int64_t row_end,
                        const int64_t* rowptr, const int64_t* colind, const double* values, const double* w,
                        const amg_config_t* cfg_in, amg_hier_t* out) {
    auto t0 = std::chrono::steady_clock::now();
    if (!ctx || !out || !rowptr || !colind || !values || n_global <= 0) {
        set_err("amg_hierarchy_build: null argument or empty matrix");
        return AMG_ERR_ARG;
    }
    *out = nullptr;
    if (row_begin != 0 || row_end != n_global) {
        set_err("amg_hierarchy_build: a single-rank context must own all rows");
        return AMG_ERR_ARG;
    }
    amg_config_t cfg;
    amg_config_default(&cfg);
    if (cfg_in) cfg = *cfg_in;
    // AMG_EAGER=1 forces eager launches (ncu cannot profile kernels inside graphs
    // that contain conditional nodes)
    if (const char* ev = std::getenv("AMG_EAGER")) cfg.use_graphs = (ev[0] == '1') ? 0 : cfg.use_graphs;
    CK(cudaSetDevice(ctx->device));

    amgsetup::Hierarchy H;
    {
        const int hs = host_setup(n_global, rowptr, colind, values, w, cfg, H);
        if (hs != AMG_OK) {
            set_err("amg_hierarchy_build: " + g_err);
            return hs;
        }
    }
    // ---- upload
    auto* h = new amg_hier_s();
    h->ctx = ctx;
    h->cfg = cfg;
    const size_t nl = H.lv.size();
    h->n0 = H.lv[0].A.nrows;
    h->nnz0 = H.lv[0].A.nnz();
    int st = AMG_OK;
    auto fail = [&](int code) {
        delete h;
        return code;
    };
    h->lv.resize(nl - 1);
    for (size_t l = 0; l + 1 < nl; ++l) {
        DevLevel& D = h->lv[l];
        const amgsetup::Level& S = H.lv[l];
        D.n = S.A.nrows;
        if ((st = upload_mat(S.A, D.A))) return fail(st);
        if ((st = upload_mat(S.P, D.P))) return fail(st);
        if ((st = upload_mat(S.R, D.R))) return fail(st);
        if ((st = dev_copy(&D.m, S.m.data(), S.m.size()))) return fail(st);
        if (l > 0 && (st = dev_alloc(&D.b, D.n))) return fail(st);
        if (l > 0 && (st = dev_alloc(&D.mb, D.n))) return fail(st);
        if ((st = dev_alloc(&D.r, D.n))) return fail(st);
        if ((st = dev_alloc(&D.xa, D.n))) return fail(st);
        if ((st = dev_alloc(&D.xb, D.n))) return fail(st);
        D.agg = S.agg;
        D.sweeps = S.sweeps;
        D.omega = S.omega;
    }
    if (nl == 1 && (st = upload_mat(H.lv[0].A, h->A0))) return fail(st);
    h->nL = H.lv.back().A.nrows;
    h->nnzL = H.lv.back().A.nnz();
    if ((st = dev_copy(&h->cinv, H.coarse_inv.data(), H.coarse_inv.size()))) return fail(st);
    if ((st = dev_alloc(&h->cb, h->nL))) return fail(st);
    if ((st = dev_alloc(&h->cx, h->nL))) return fail(st);
    if ((st = dev_alloc(&h->pr, h->n0))) return fail(st);
    if ((st = dev_alloc(&h->pz, h->n0))) return fail(st);
    if ((st = dev_alloc(&h->pp, h->n0))) return fail(st);
    if ((st = dev_alloc(&h->pq, h->n0))) return fail(st);
    if ((st = dev_alloc(&h->st, 1))) return fail(st);
    if ((st = dev_alloc(&h->partials, kMaxPartials))) return fail(st);
    if ((st = dev_alloc(&h->ticket, 1))) return fail(st);
    if (cudaMallocHost((void**)&h->st_host, sizeof(PcgState)) != cudaSuccess) {
        set_err("cudaMallocHost failed");
        return fail(AMG_ERR_OOM);
    }
    cudaEventCreate(&h->ev0);
    cudaEventCreate(&h->ev1);
    // ---- statistics and the §8d byte model
    double s = 0.0;
    for (auto& L : H.lv) s += (double)L.A.nnz();
    h->opc = s / (double)H.lv[0].A.nnz();
    double cr = 0.0;
    for (size_t l = 0; l + 1 < nl; ++l) cr += (double)H.lv[l].A.nrows / (double)H.lv[l + 1].A.nrows;
    h->avg_cr = nl > 1 ? cr / (double)(nl - 1) : 1.0;
    byte_model(h, H);
    CK(cudaDeviceSynchronize());
    h->setup_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    *out = h;
    return AMG_OK;
}

int amg_hierarchy_destroy(amg_hier_t h) {
    if (h) {
        cudaSetDevice(h->ctx->device);
        delete h;
    }
    return AMG_OK;
}

int amg_solve(amg_hier_t h, const double* b_dev, double* x_dev, double rtol, int32_t maxit, amg_report_t* rep) {
    if (!h || !b_dev || !x_dev || rtol < 0.0 || maxit < 0) {
        set_err("amg_solve: bad argument");
        return AMG_ERR_ARG;
    }
    CK(cudaSetDevice(h->ctx->device));
    cudaStream_t s = h->ctx->stream;
    PcgState init{};
    init.rtol = rtol;
    init.maxit = maxit;
    *h->st_host = init;
    CK(cudaMemcpyAsync(h->st, h->st_host, sizeof(PcgState), cudaMemcpyHostToDevice, s));
    CK(cudaEventRecord(h->ev0, s));
    if (h->cfg.use_graphs) {
        int e = ensure_solve_graph(h, b_dev, x_dev);
        if (e) return e;
        CK(cudaGraphLaunch(h->solve_exec, s));
        CK(cudaEventRecord(h->ev1, s));
        CK(cudaMemcpyAsync(h->st_host, h->st, sizeof(PcgState), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
    } else {
        Launch L{h, s};
        enqueue_pcg_init(h, L, b_dev, x_dev, 0);
        for (;;) {
            CK(cudaMemcpyAsync(h->st_host, h->st, sizeof(PcgState), cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            if (h->st_host->status != ST_RUNNING) break;
            enqueue_pcg_body(h, L, x_dev, 0);
        }
        CK(cudaEventRecord(h->ev1, s));
        CK(cudaStreamSynchronize(s));
    }
    CK(cudaGetLastError());
    float ms = 0.f;
    cudaEventElapsedTime(&ms, h->ev0, h->ev1);
    const PcgState& S = *h->st_host;
    if (rep) {
        fill_report(h, rep);
        rep->iterations = S.iter;
        rep->final_relres = S.relres;
        rep->converged = (S.status == ST_CONVERGED || S.status == ST_ZERO_RHS) ? 1 : 0;
        rep->solve_s = ms * 1e-3;
    }
    int code = AMG_OK;
    if (S.status == ST_MAXIT) code = AMG_NOT_CONVERGED;
    if (S.status == ST_BREAKDOWN) {
        code = AMG_ERR_BREAKDOWN;
        set_err("amg_solve: breakdown, p^T A p <= 0");
    }
    if (rep) rep->status = code;
    return code;
}

int amg_solve_host(amg_hier_t h, const double* b_host, double* x_host, double rtol, int32_t maxit,
                   amg_report_t* rep) {
    if (!h || !b_host || !x_host) {
        set_err("amg_solve_host: bad argument");
        return AMG_ERR_ARG;
    }
    CK(cudaSetDevice(h->ctx->device));
    int st;
    if (!h->hb && (st = dev_alloc(&h->hb, h->n0))) return st;
    if (!h->hx && (st = dev_alloc(&h->hx, h->n0))) return st;
    cudaStream_t s = h->ctx->stream;
    CK(cudaMemcpyAsync(h->hb, b_host, sizeof(double) * h->n0, cudaMemcpyHostToDevice, s));
    const int code = amg_solve(h, h->hb, h->hx, rtol, maxit, rep);
    if (code != AMG_OK && code != AMG_NOT_CONVERGED && code != AMG_ERR_BREAKDOWN) return code;
    CK(cudaMemcpyAsync(x_host, h->hx, sizeof(double) * h->n0, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return code;
}

int amg_precond_apply(amg_hier_t h, const double* r_dev, double* z_dev) {
    if (!h || !r_dev || !z_dev) {
        set_err("amg_precond_apply: bad argument");
        return AMG_ERR_ARG;
    }
    CK(cudaSetDevice(h->ctx->device));
    cudaStream_t s = h->ctx->stream;
    if (h->cfg.use_graphs) {
        int e = ensure_apply_graph(h, r_dev, z_dev);
        if (e) return e;
        CK(cudaGraphLaunch(h->apply_exec, s));
    } else {
        Launch L{h, s};
        enqueue_vcycle(h, L, r_dev, z_dev, nullptr);
    }
    CK(cudaStreamSynchronize(s));
    CK(cudaGetLastError());
    return AMG_OK;
}

int amg_num_levels(amg_hier_t h, int32_t* nl) {
    if (!h || !nl) return AMG_ERR_ARG;
    *nl = (int32_t)h->lv.size() + 1;
    return AMG_OK;
}

int amg_level_info(amg_hier_t h, int32_t l, int64_t* n_global, int64_t* nnzA, int64_t* nnzP, int64_t* rb,
                   int64_t* re, int32_t* format) {
    if (!h || l < 0 || l > (int32_t)h->lv.size()) {
        set_err("amg_level_info: bad level");
        return AMG_ERR_ARG;
    }
    int64_t n, a, p;
    int32_t f;
    if (l < (int32_t)h->lv.size()) {
        n = h->lv[l].n;
        a = h->lv[l].A.nnz;
        p = h->lv[l].P.nnz;
        f = h->lv[l].A.fmt;
    } else {
        n = h->nL;
        a = h->nnzL;
        p = 0;
        f = FMT_DENSE;
    }
    if (n_global) *n_global = n;
    if (nnzA) *nnzA = a;
    if (nnzP) *nnzP = p;
    if (rb) *rb = 0;
    if (re) *re = n;
    if (format) *format = f;
    return AMG_OK;
}

int amg_level_aggregates(amg_hier_t h, int32_t l, int64_t* agg) {
    if (!h || !agg || l < 0 || l >= (int32_t)h->lv.size()) {
        set_err("amg_level_aggregates: bad level");
        return AMG_ERR_ARG;
    }
    const auto& a = h->lv[l].agg;
    for (size_t i = 0; i < a.size(); ++i) agg[i] = a[i];
    return AMG_OK;
}

int amg_hierarchy_report(amg_hier_t h, amg_report_t* rep) {
    if (!h || !rep) return AMG_ERR_ARG;
    std::memset(rep, 0, sizeof(*rep));
    fill_report(h, rep);
    return AMG_OK;
}

int amg_profile_vcycle(amg_hier_t h, int32_t napply, int32_t cap, double* ms_out, double* bytes_out,
                       double* stored_bytes_out, const char** names_out, int32_t* count) {
    if (!h || napply < 1 || !count) {
        set_err("amg_profile_vcycle: bad argument");
        return AMG_ERR_ARG;
    }
    CK(cudaSetDevice(h->ctx->device));
    cudaStream_t s = h->ctx->stream;
    CK(cudaMemsetAsync(h->pr, 0, sizeof(double) * h->n0, s));
    std::vector<KernelRec> recs;
    Launch L{h, s};
    enqueue_vcycle(h, L, h->pr, h->pz, nullptr);  // warm-up
    CK(cudaStreamSynchronize(s));
    h->prof = &recs;
    for (int a = 0; a < napply; ++a) enqueue_vcycle(h, L, h->pr, h->pz, nullptr);
    h->prof = nullptr;
    CK(cudaStreamSynchronize(s));
    CK(cudaGetLastError());
    const int per = (int)(recs.size() / napply);
    *count = per;
    for (int k = 0; k < per && k < cap; ++k) {
        double tot = 0.0;
        for (int a = 0; a < napply; ++a) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, recs[a * per + k].e0, recs[a * per + k].e1);
            tot += ms;
        }
        if (ms_out) ms_out[k] = tot / napply;
        if (bytes_out) bytes_out[k] = recs[k].bytes;
        if (stored_bytes_out) stored_bytes_out[k] = recs[k].stored_bytes;
        if (names_out) names_out[k] = recs[k].name;
    }
    for (auto& r : recs) {
        cudaEventDestroy(r.e0);
        cudaEventDestroy(r.e1);
    }
    return AMG_OK;
}

struct amg_host_hier_s {
    amgsetup::Hierarchy H;
};

int amg_host_hierarchy_build(int64_t n, const int64_t* rowptr, const int64_t* colind, const double* values,
                             const double* w, const amg_config_t* cfg_in, amg_host_hier_t* out) {
    if (!out) {
        set_err("amg_host_hierarchy_build: null out");
        return AMG_ERR_ARG;
    }
    *out = nullptr;
    amg_config_t cfg;
    amg_config_default(&cfg);
    if (cfg_in) cfg = *cfg_in;
    auto* h = new amg_host_hier_s();
    const int st = host_setup(n, rowptr, colind, values, w, cfg, h->H);
    if (st != AMG_OK) {
        delete h;
        set_err("amg_host_hierarchy_build: " + g_err);
        return st;
    }
    *out = h;
    return AMG_OK;
}

int amg_host_hierarchy_destroy(amg_host_hier_t h) {
    delete h;
    return AMG_OK;
}

int amg_host_num_levels(amg_host_hier_t h, int32_t* nl) {
    if (!h || !nl) return AMG_ERR_ARG;
    *nl = (int32_t)h->H.lv.size();
    return AMG_OK;
}

int amg_host_level_sizes(amg_host_hier_t h, int32_t l, int64_t* n, int64_t* nnzA, int64_t* nnzP, double* omega) {
    if (!h || l < 0 || l >= (int32_t)h->H.lv.size()) {
        set_err("amg_host_level_sizes: bad level");
        return AMG_ERR_ARG;
    }
    const auto& L = h->H.lv[l];
    if (n) *n = L.A.nrows;
    if (nnzA) *nnzA = L.A.nnz();
    if (nnzP) *nnzP = L.P.nnz();
    if (omega) *omega = L.omega;
    return AMG_OK;
}

int amg_host_level_aggregates(amg_host_hier_t h, int32_t l, int64_t* agg) {
    if (!h || !agg || l < 0 || l + 1 >= (int32_t)h->H.lv.size()) {
        set_err("amg_host_level_aggregates: bad level");
        return AMG_ERR_ARG;
    }
    const auto& a = h->H.lv[l].agg;
    for (size_t i = 0; i < a.size(); ++i) agg[i] = a[i];
    return AMG_OK;
}

int amg_host_level_matrix(amg_host_hier_t h, int32_t l, int32_t which, int64_t* rowptr, int64_t* colind,
                          double* values) {
    if (!h || l < 0 || l >= (int32_t)h->H.lv.size() || which < 0 || which > 1 ||
        (which == 1 && l + 1 >= (int32_t)h->H.lv.size())) {
        set_err("amg_host_level_matrix: bad level/which");
        return AMG_ERR_ARG;
    }
    const amgsetup::Csr& M = which == 0 ? h->H.lv[l].A : h->H.lv[l].P;
    for (int64_t i = 0; i <= M.nrows; ++i) rowptr[i] = M.rp[i];
    for (int64_t k = 0; k < M.nnz(); ++k) {
        colind[k] = M.ci[k];
        values[k] = M.v[k];
    }
    return AMG_OK;
}

}  // extern "C"
