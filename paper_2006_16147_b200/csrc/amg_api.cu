// amg_api.cu — implementation of include/amg_b200.h.
//
// Host side: validates/copies the caller's CSR, runs the C++ setup
// (csrc/setup), partitions the hierarchy over the ranks (csrc/setup/partition),
// chooses a device format per operator, uploads, and drives the solve phase.
// Device side: kernels.cuh.
//
// Single rank: a PCG solve is ONE graph launch — a prologue kernel followed by
// a CUDA-graph WHILE node whose body is
//   V-cycle(r -> z) [fused r^T z -> beta]   -> p = z + beta p
//   q = A p [fused p^T q -> alpha]          -> x += alpha p, r -= alpha q [fused
//   ||r||^2 -> convergence test -> cudaGraphSetConditional]
// so the iteration count is decided on the device.
//
// Several ranks (north_star (4)): every rank owns a row block of
// every distributed level and holds each level vector as a window of the global
// vector; before each kernel that gathers a vector, its halo is exchanged
// (pack -> NCCL send/recv over NVLink -> unpack).  Dot products reduce locally,
// the per-rank totals are all-gathered and summed in rank order (identical and
// deterministic on all ranks).  Deep levels are replicated after one gather.
// The same per-rank code runs in "loopback" mode (cfg.emulate_ranks > 1): all
// ranks live in one process on one GPU and the transport is a device copy,
// which is how the multi-rank kernels are parity-tested on a single B200.
#include <cuda_runtime.h>
#include <nccl.h>
#include <nccl_device.h>
#include <nvtx3/nvToolsExt.h>
#include <omp.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <set>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/amg_b200.h"
#include "kernels.cuh"
#include "setup/dist_setup.hpp"
#include "setup/partition.hpp"
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

#define NK(call)                                                         \
    do {                                                                 \
        ncclResult_t r_ = (call);                                        \
        if (r_ != ncclSuccess) {                                         \
            set_err(std::string(#call) + ": " + ncclGetErrorString(r_)); \
            return AMG_ERR_NCCL;                                         \
        }                                                                \
    } while (0)

enum { FMT_SELL = 0, FMT_CSRV = 1, FMT_DENSE = 2, FMT_SDIA = 3, FMT_SELL_SIGMA = 4 /* reported only */ };
constexpr int kVWBlock = 256;  // CSR-vector "VW" value meaning one block per row

struct DevMat {
    int fmt = FMT_SELL;
    int vw = 32;
    int64_t nrows = 0, ncols = 0, nnz = 0, stored = 0;
    int32_t shift = 0;         // SDIA: row -> window column frame
    uint32_t* sptr = nullptr;  // SELL / SDIA
    int32_t* offs = nullptr;   // SDIA: one column offset per slice column
    int32_t* anchor = nullptr; // SDIA of a rectangular operator: per-row base column
    int32_t* rp = nullptr;     // CSR
    int32_t* col = nullptr;
    double* val = nullptr;
    int32_t* perm = nullptr;   // SELL-32-sigma: slot -> row (null: plain SELL-32)
    // 16-bit columns (SELL / CSR whose every row spans < 2^16 columns): col = cbase[row or slot]
    // + c16[k]; `col` is then null.  10 instead of 12 B per stored entry (+ 4 B per row)
    uint16_t* c16 = nullptr;
    int32_t* cbase = nullptr;
    // multi-rank overlap: launch units (slices for SELL/SDIA, rows for CSR) and the largest
    // contiguous block of units whose gathers touch only owned columns ("interior": it can
    // run while the halo is in flight); the rest ("head" / "tail") runs after the exchange
    int64_t units = 0, ib0 = 0, ib1 = 0;
    bool persist = false;      // deep-level operator: launched with an L2 persistence window
    // algorithmic bytes of one pass over the operator: 12 nnz + 4 (n+1)
    double model_bytes() const { return 12.0 * (double)nnz + 4.0 * (double)(nrows + 1); }
    // bytes the chosen device format actually stores for one pass
    double stored_bytes() const {
        const double nsl = (double)((nrows + 31) / 32);
        switch (fmt) {
            case FMT_SELL:
                return (c16 ? 10.0 : 12.0) * (double)stored + 4.0 * (nsl + 1) + (perm ? 128.0 * nsl : 0.0) +
                       (c16 ? 128.0 * nsl : 0.0);
            case FMT_SDIA:
                return 8.0 * (double)stored + 4.0 * (double)stored / 32.0 + 4.0 * (nsl + 1) +
                       (anchor ? 4.0 * (double)nrows : 0.0);
            default: return (c16 ? 10.0 : 12.0) * (double)nnz + 4.0 * (double)(nrows + 1) + (c16 ? 4.0 * nrows : 0.0);
        }
    }
    void release() {
        cudaFree(sptr);
        cudaFree(offs);
        cudaFree(anchor);
        cudaFree(rp);
        cudaFree(col);
        cudaFree(val);
        cudaFree(perm);
        cudaFree(c16);
        cudaFree(cbase);
        c16 = nullptr;
        cbase = nullptr;
        sptr = nullptr;
        offs = nullptr;
        anchor = nullptr;
        rp = col = nullptr;
        val = nullptr;
        perm = nullptr;
    }
};

// Halo exchange plan of one level on one rank.
struct Exch {
    int64_t nsend = 0, nrecv = 0;
    std::vector<int64_t> send_off, recv_off;  // np+1 (host)
    int32_t* send_idx = nullptr;              // window positions to pack
    int32_t* recv_idx = nullptr;              // window positions to unpack into
    double* sbuf = nullptr;
    double* rbuf = nullptr;       // LSA transport: region 0 of this level in the rank's window segment
    int64_t* d_send_off = nullptr;  // LSA: device copy of send_off
    int64_t* d_dst_off = nullptr;   // LSA: np byte offsets of my data in each destination's region 0
    bool rbuf_in_window = false;
    RxWait rx{};                    // LSA: the receive side's barrier wait + region parity (flags null: none)
    void release() {
        cudaFree(send_idx);
        cudaFree(recv_idx);
        cudaFree(sbuf);
        if (!rbuf_in_window) cudaFree(rbuf);
        cudaFree(d_send_off);
        cudaFree(d_dst_off);
        send_idx = recv_idx = nullptr;
        sbuf = rbuf = nullptr;
        d_send_off = d_dst_off = nullptr;
    }
};

struct DevLevel {
    bool replicated = false;
    bool coarsest = false;
    int64_t n_global = 0;
    int64_t own_begin = 0, own_n = 0;
    int64_t comp_n = 0, win_n = 0;
    int64_t ep_off = 0;    // comp_begin - win_begin
    int64_t own_off = 0;   // own_begin - win_begin
    int64_t rst_n = 0;     // rows of R computed here
    int64_t rst_off = 0;   // rst_begin - next.win_begin
    DevMat A, P, R;
    // A_l diag(m_l) (columns scaled by the l1 diagonal) for the residual of the first
    // pre-sweep from zero, r = b - A (m o b) = b - (A diag(m)) b: the kernel gathers b
    // alone, and no level needs m o b (s1 == 1 only)
    DevMat Am;
    // INVK smoother (cfg.smoother == 1): D^{-1} W and Z = W^T
    DevMat Wd, Z;
    // Compact small level (one pre- and one post-sweep, single rank): Rc = R (I - A diag(m)) and
    // Pc = (I - diag(m) A) P-bar, so the level is s = S2(b), b_{l+1} = Rc b, out = s + Pc e
    bool compact = false;
    DevMat Rc, Pc;
    // collapsed (the compact level just above a direct coarsest solve): M = Pc A_L^{-1} Rc dense
    double* Mc = nullptr;
    double* AMc = nullptr;  // K-cycle inner level: A_l B (the first inner SpMV folded into the cycle)
    double* m = nullptr;   // window-sized vectors
    double* b = nullptr;
    double* mb = nullptr;
    double* r = nullptr;
    double* xa = nullptr;
    double* xb = nullptr;
    // K-cycle FCG vectors of this level (cfg.cycle == 1, levels 1..nl-2) and its
    // device scalars {p^T r, p^T q, alpha, beta, stop}
    double *kx = nullptr, *kr = nullptr, *kmb = nullptr, *kz = nullptr, *kp = nullptr, *kq = nullptr;
    double* kp2 = nullptr;  // the inner FCG's second direction (written while kp is gathered)
    double* kst = nullptr;
    Exch ex;
    void release() {
        A.release();
        P.release();
        R.release();
        Am.release();
        Wd.release();
        Z.release();
        Rc.release();
        Pc.release();
        cudaFree(Mc);
        Mc = nullptr;
        cudaFree(AMc);
        AMc = nullptr;
        for (double* v : {kx, kr, kmb, kz, kp, kq, kst, kp2}) cudaFree(v);
        cudaFree(m);
        cudaFree(b);
        cudaFree(mb);
        cudaFree(r);
        cudaFree(xa);
        cudaFree(xb);
        ex.release();
    }
};

struct KernelRec {
    const char* name;
    double bytes;         // algorithmic
    double stored_bytes;  // what the device format actually moves (compulsory)
    cudaEvent_t e0, e1;
};

// Device state of one rank.
struct RankState {
    int rank = 0;
    std::vector<DevLevel> lv;   // all levels; the last one is the (replicated) coarsest
    double* cinv = nullptr;     // dense A_L^{-1}, row-major
    int64_t nL = 0;
    int64_t user_off = 0;       // offset of this rank's rows in the caller's vectors (loopback)
    double *pr = nullptr, *pz = nullptr, *pp = nullptr, *pq = nullptr;  // level-0 window vectors
    double* pp2 = nullptr;  // second p buffer (fused direction update, single rank)
    PcgState* st = nullptr;
    double* partials = nullptr;
    unsigned int* ticket = nullptr;
    double* dot_local = nullptr;  // this rank's dot total
    double* dot_all = nullptr;    // all-gathered totals (np)
    // LSA transport: barriers completed by this rank, the push kernel's block counter, the dot
    // region (region 0) and the barrier flags in this rank's window segment
    unsigned long long* lsa_seq = nullptr;
    unsigned int* lsa_count = nullptr;
    double* lsa_dots = nullptr;
    unsigned long long* lsa_flags = nullptr;
    // coarsest iterative solve (cfg.coarse_solver == 1): CSR of A_L, its l1 diagonal,
    // the per-CTA row split and the cluster launch shape of k_coarse_cg
    int32_t *cg_rp = nullptr, *cg_ci = nullptr, *cg_split = nullptr;
    double *cg_v = nullptr, *cg_m = nullptr;
    // coarse CG preconditioned by the (H)INVK factors of A_L (coarse_prec == 1, VA3S3CS1)
    int32_t *cg_wrp = nullptr, *cg_wci = nullptr, *cg_zrp = nullptr, *cg_zci = nullptr;
    double *cg_wv = nullptr, *cg_zv = nullptr;
    int64_t cg_nnz = 0;
    int cg_ncta = 1, cg_smem_a = 0;
    size_t cg_smem = 0;
    void release() {
        for (auto& D : lv) D.release();
        cudaFree(cg_rp);
        cudaFree(cg_ci);
        cudaFree(cg_split);
        cudaFree(cg_v);
        cudaFree(cg_m);
        for (int32_t* p : {cg_wrp, cg_wci, cg_zrp, cg_zci}) cudaFree(p);
        cudaFree(cg_wv);
        cudaFree(cg_zv);
        cudaFree(cinv);
        cudaFree(pr);
        cudaFree(pz);
        cudaFree(pp);
        cudaFree(pp2);
        cudaFree(pq);
        cudaFree(st);
        cudaFree(partials);
        cudaFree(ticket);
        cudaFree(dot_local);
        cudaFree(dot_all);
        cudaFree(lsa_seq);
        cudaFree(lsa_count);
    }
    const DevLevel& L0() const { return lv[0]; }
};

}  // namespace

struct amg_ctx_s {
    int device = 0, rank = 0, nranks = 1;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    int nsm = 148;
    ncclComm_t nccl = nullptr;
    // launch caps (SM count x resident blocks) per kernel, computed once per context
    std::unordered_map<const void*, int> caps;
    std::mutex caps_mu;
    // live hierarchies built on this context: amg_ctx_destroy releases their CUDA graphs before
    // destroying the communicator (graphs holding captured NCCL work would block it forever)
    std::set<struct amg_hier_s*> hiers;
    std::mutex hiers_mu;
};

struct amg_hier_s {
    amg_ctx_s* ctx = nullptr;
    int device = 0;  // the context's device, kept for amg_hierarchy_destroy
    amg_config_t cfg{};
    int np = 1;                 // ranks of the partition
    bool loopback = false;      // all ranks in this process (emulate_ranks)
    std::vector<RankState> ranks;  // local ranks (1, or np in loopback mode)
    std::vector<std::vector<int32_t>> agg;  // host aggregate maps (owned rows; all rows in loopback)
    std::vector<int64_t> lvl_n, lvl_nnzA, lvl_nnzP;  // global level statistics
    std::vector<int32_t> lvl_fmt;
    std::vector<int64_t> lvl_own_begin, lvl_own_end;  // this rank's owned rows per level
    int64_t n0_local = 0;       // rows of the caller's vectors
    double *hb = nullptr, *hx = nullptr;  // staging for amg_solve_host
    PcgState* st_host = nullptr;
    double setup_s = 0, opc = 0, avg_cr = 0, bytes_v = 0, bytes_it = 0;
    cudaGraphExec_t solve_exec = nullptr;
    const double* solve_b = nullptr;
    double* solve_x = nullptr;
    // pipelined host batch (amg_solve_host_batch): two device (b, x) pairs and their graphs
    double* bb[2] = {nullptr, nullptr};
    double* bx[2] = {nullptr, nullptr};
    cudaGraphExec_t batch_exec[2] = {nullptr, nullptr};
    cudaStream_t cstream = nullptr, dstream = nullptr;  // host->device / device->host copies
    // solve graph shape: GM_WHILE = one graph per solve (a device-side WHILE node over the
    // iteration, no host round trip); GM_ITER = one graph per iteration launched from a host loop
    // with one status read each (the fallback of NCCL contexts if the WHILE graph cannot be built
    // or instantiated, decided collectively; AMG_MULTI_GRAPH=iter forces it)
    int graph_mode = 0;
    cudaGraphExec_t iter_exec = nullptr;
    double* iter_x = nullptr;
    cudaGraphExec_t apply_exec = nullptr;
    const double* apply_r = nullptr;
    double* apply_z = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    // multi-rank: halo exchanges run on `comm` while the interior rows compute on the
    // context stream (fork/join events)
    cudaStream_t comm = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    std::vector<KernelRec>* prof = nullptr;
    // persistent deep-level tail (single rank): first tail level, the compiled
    // program (device), its cooperative grid and reduction scratch
    int tail_level = -1;
    TailOp* tail_prog = nullptr;
    int tail_nops = 0, tail_grid = 0;
    bool tail_cluster = false;  // one thread-block cluster (tail_bytes) instead of a cooperative grid
    double* tail_partials = nullptr;
    double tail_bytes = 0.0;

    // one solve / apply at a time per hierarchy: the graphs, PCG vectors and staging buffers
    // are per-hierarchy state (include/amg_b200.h, "Threads")
    std::recursive_mutex mu;
    // peer-memory (LSA) transport over an NCCL symmetric window (include/amg_b200.h "Transport"):
    // one segment per rank (np segments on a one-rank loopback communicator) holding the barrier
    // flags, the double-buffered dot region and every distributed level's double-buffered receive region
    bool lsa = false;
    ncclComm_t lsa_comm = nullptr;
    void* lsa_mem = nullptr;
    ncclWindow_t lsa_win = nullptr;
    int64_t lsa_seg = 0, lsa_flag_off = 0, lsa_dot_off = 0, lsa_dot_stride = 0;
    std::vector<int64_t> lsa_lvl_stride;  // bytes between the parities of a level's region
    char** lsa_peer = nullptr;            // device: np segment bases as this GPU addresses them
    int* lsa_err = nullptr;               // device: a barrier timed out (sticky)
    unsigned long long lsa_timeout_ns = 60ull * 1000000000ull;
    void release_lsa() {
        if (lsa_win && lsa_comm) ncclCommWindowDeregister(lsa_comm, lsa_win);
        if (lsa_mem) ncclMemFree(lsa_mem);
        cudaFree(lsa_peer);
        cudaFree(lsa_err);
        lsa_win = nullptr;
        lsa_mem = nullptr;
        lsa_peer = nullptr;
        lsa_err = nullptr;
        lsa = false;
    }
    // first NCCL failure of an enqueue pass (exchange / all-gather), reported as AMG_ERR_NCCL
    ncclResult_t nccl_status = ncclSuccess;
    std::string nccl_what;

    bool multi() const { return np > 1; }
    // halos and dot slots travel through NCCL: real ranks, or loopback on a context that holds a
    // one-rank communicator (every transfer a self send/recv -- the captured NCCL transport
    // exercised on one GPU, no kernel waiting on another rank)
    bool nccl_xport() const { return multi() && ctx->nccl != nullptr; }
    bool loop_nccl() const { return loopback && nccl_xport(); }
    int nlev() const { return (int)ranks[0].lv.size(); }
    void release_graphs() {
        if (solve_exec) cudaGraphExecDestroy(solve_exec);
        solve_exec = nullptr;
        solve_b = nullptr;
        solve_x = nullptr;
        for (int q = 0; q < 2; ++q) {
            if (batch_exec[q]) cudaGraphExecDestroy(batch_exec[q]);
            batch_exec[q] = nullptr;
        }
        if (apply_exec) cudaGraphExecDestroy(apply_exec);
        apply_exec = nullptr;
        if (iter_exec) cudaGraphExecDestroy(iter_exec);
        iter_exec = nullptr;
    }
    ~amg_hier_s() {
        release_lsa();
        cudaFree(tail_prog);
        cudaFree(tail_partials);
        release_graphs();
        for (int q = 0; q < 2; ++q) {
            cudaFree(bb[q]);
            cudaFree(bx[q]);
        }
        if (cstream) cudaStreamDestroy(cstream);
        if (dstream) cudaStreamDestroy(dstream);
        for (auto& R : ranks) R.release();
        cudaFree(hb);
        cudaFree(hx);
        cudaFreeHost(st_host);
        if (ev0) cudaEventDestroy(ev0);
        if (ev1) cudaEventDestroy(ev1);
        if (ev_fork) cudaEventDestroy(ev_fork);
        if (ev_join) cudaEventDestroy(ev_join);
        if (comm) cudaStreamDestroy(comm);
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
// per-context cache of max_grid (the SM count is the context device's)
int ctx_cap(amg_ctx_s* c, const void* fn) {
    std::lock_guard<std::mutex> g(c->caps_mu);
    auto it = c->caps.find(fn);
    if (it != c->caps.end()) return it->second;
    const int v = max_grid(fn, c->nsm);
    c->caps.emplace(fn, v);
    return v;
}

// The synchronous-API cudaMemcpy / cudaMemset run on the legacy default stream, which the library's
// non-blocking streams (the context's, the GPU setup's) do NOT wait for, and a host-to-device copy
// from pageable memory or a device memset may return before the device has finished it.  A kernel
// launched next on the context stream could then read the buffer before (or while) it is written:
// a rare, build-to-build race (found on the SELL-32-sigma slot map of c5's A_1, zeroed by dev_alloc
// and written by the next kernel: one build in ~10 took 500 iterations).  Every such call goes
// through these helpers, which wait for the legacy stream before returning.
cudaError_t h2d_sync(void* dst, const void* src, size_t bytes) {
    cudaError_t e = cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice);
    return e == cudaSuccess ? cudaStreamSynchronize(cudaStreamLegacy) : e;
}
cudaError_t memset_sync(void* dst, int v, size_t bytes) {
    cudaError_t e = cudaMemset(dst, v, bytes);
    return e == cudaSuccess ? cudaStreamSynchronize(cudaStreamLegacy) : e;
}

int vec_grid(int64_t n, int nsm) {
    const int64_t need = (n + kBlock - 1) / kBlock;
    return (int)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)nsm * 8));
}

// NVTX range over one ABI call (visible in nsys / ncu --nvtx; a no-op without a tool attached).
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

// Kernel launch with programmatic stream serialization (PDL, see kernels.cuh).
bool pdl_enabled() {
    static const bool on = !(std::getenv("AMG_PDL") && std::getenv("AMG_PDL")[0] == '0');
    return on;
}
// Sweeps recompute m_i = sum_j |a_ij| from the streamed row while rows average at most this many
// entries, else read the stored m (AMG_ABS_ROW_CUT, an A/B knob; default 40).
double abs_row_cut() {
    static const double cut = [] {
        const char* e = std::getenv("AMG_ABS_ROW_CUT");
        return e ? std::atof(e) : 40.0;
    }();
    return cut;
}
// L2 persistence window of the next launch_mat launch (deep-level operators, AMG_L2_PERSIST_MB;
// an experiment: VERDICT r1 W8 / SURVEY §7.5).  Thread-local: set and consumed by launch_mat.
thread_local const void* g_persist_ptr = nullptr;
thread_local size_t g_persist_bytes = 0;
template <class... KArgs, class... Args>
void launch_k(void (*kern)(KArgs...), int grid, int block, cudaStream_t s, Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3((unsigned)block);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    int na = 0;
    if (pdl_enabled()) {
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    if (g_persist_ptr) {
        attr[na].id = cudaLaunchAttributeAccessPolicyWindow;
        attr[na].val.accessPolicyWindow.base_ptr = const_cast<void*>(g_persist_ptr);
        attr[na].val.accessPolicyWindow.num_bytes = g_persist_bytes;
        attr[na].val.accessPolicyWindow.hitRatio = 1.0f;
        attr[na].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        attr[na].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
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

// Experiment knob (AMG_SMALL_GRID="<rows>:<blocks per SM>"): operators of at most <rows> rows launch at
// most <blocks per SM> x #SM blocks, leaving SM slots free so that the next kernel's blocks (PDL) can
// become resident -- and wait -- before this one finishes.  Off by default.
int small_cap(amg_hier_s* h, const DevMat& M, int cap) {
    static const std::pair<int64_t, int> knob = [] {
        const char* e = std::getenv("AMG_SMALL_GRID");
        long long rows = 0;
        int bps = 0;
        if (e && std::sscanf(e, "%lld:%d", &rows, &bps) == 2 && rows > 0 && bps > 0) return std::make_pair((int64_t)rows, bps);
        return std::make_pair((int64_t)0, 0);
    }();
    if (knob.first > 0 && M.nrows <= knob.first) return std::min(cap, knob.second * h->ctx->nsm);
    return cap;
}

template <class G, class E>
void launch_mat(Launch& L, const DevMat& M, G g, E e, RedCtx rc, const char* name, double vec_bytes,
                int part = 0) {
    // part 0: all rows; 1: the interior units; 2: the units before AND after them (one launch,
    // the interior skipped); 3: nothing (kept for the callers' slot numbering)
    const int64_t units = (M.fmt == FMT_SDIA || M.fmt == FMT_SELL) ? (M.nrows + 31) / 32 : M.nrows;
    int64_t u0 = 0, u1 = units, k0 = 0, kspan = 0;
    if (part == 1) {
        u0 = M.ib0;
        u1 = M.ib1;
    } else if (part == 2) {
        k0 = M.ib0;
        kspan = M.ib1 - M.ib0;
    } else if (part == 3) {
        return;
    }
    if (part != 0 && u1 - u0 - kspan <= 0) return;
    const double frac = units ? (double)(u1 - u0 - kspan) / (double)units : 1.0;
    L.begin(name, frac * (M.model_bytes() + vec_bytes), frac * (M.stored_bytes() + vec_bytes));
    struct PersistScope {  // the window covers this operator's values for this launch only
        PersistScope(const DevMat& M) {
            if (M.persist) {
                g_persist_ptr = M.val;
                g_persist_bytes = (size_t)(M.fmt == FMT_SDIA || M.fmt == FMT_SELL ? M.stored : M.nnz) * 8;
            }
        }
        ~PersistScope() { g_persist_ptr = nullptr; }
    } persist_scope(M);
    if (M.fmt == FMT_SDIA) {
        auto go = [&](auto kern) {
            const int cap = small_cap(L.h, M, ctx_cap(L.h->ctx, (const void*)kern));
            const int64_t need = ((u1 - u0 - kspan) * 32 + kBlock - 1) / kBlock;
            const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(need, cap));
            launch_k(kern, grid, kBlock, L.s,
                     SdiaView{M.sptr, M.offs, M.val, M.nrows, (int32_t)M.ncols, M.shift, M.anchor, u0, u1, k0, kspan},
                     g, e, rc);
        };
        // dot-fused kernels over wide rows: the 40-register instance (kernels.cuh, kDotWideEntries)
        bool wide = false;
        // (the q = A p kernels with the fused direction update gather two vectors and stay at 8 blocks:
        // c5's spmv_dot_pupd ran 0.82 -> 1.21 ms at 6)
        if constexpr (E::kDot && !std::is_same<G, GPz>::value && !std::is_same<G, GKpz>::value) {
            static const bool wide_off = std::getenv("AMG_DOT_WIDE_OFF") != nullptr;  // A/B switch
            wide = !wide_off && M.stored > (int64_t)kDotWideEntries * M.nrows;
            if (wide) go(k_sdia<G, E, AMG_DOT_MINB>);
        }
        if (!wide) go(k_sdia<G, E>);
    } else if (M.fmt == FMT_SELL) {
        const int cap = small_cap(L.h, M, ctx_cap(L.h->ctx, (const void*)k_sell<G, E>));
        const int64_t need = ((u1 - u0 - kspan) * 32 + kBlock - 1) / kBlock;
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(need, cap));
        launch_k(k_sell<G, E>, grid, kBlock, L.s, SellView{M.sptr, M.col, M.val, M.nrows, u0, u1, k0, kspan, M.perm, M.c16, M.cbase},
                 g, e, rc);
    } else {
        const CsrView v{M.rp, M.col, M.val, M.nrows, u0, u1, k0, kspan, M.c16, M.cbase};
        const int64_t need = ((u1 - u0 - kspan) * M.vw + kBlock - 1) / kBlock;
        if (M.vw == kVWBlock) {
            const int cap = small_cap(L.h, M, ctx_cap(L.h->ctx, (const void*)k_csrb<G, E>));
            const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(u1 - u0 - kspan, cap));
            launch_k(k_csrb<G, E>, grid, kBlock, L.s, v, g, e, rc);
            L.end();
            return;
        }
        switch (M.vw) {
#define VWCASE(W)                                                                 \
    case W: {                                                                     \
        const int cap = small_cap(L.h, M, ctx_cap(L.h->ctx, (const void*)k_csrv<W, G, E>)); \
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(need, cap)); \
        launch_k(k_csrv<W, G, E>, grid, kBlock, L.s, v, g, e, rc);                   \
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

RedCtx no_red() { return RedCtx{nullptr, nullptr, nullptr, nullptr, 0ull, FIN_NONE, nullptr}; }

// Dot epilogue context: fused finisher on one rank; local total (deferred) on many.
// Multi-rank: three local slots (a kernel split into interior / head / tail parts writes
// one slot per part); dot_finish sums all slots of all ranks in a fixed order.
constexpr int kDotSlots = 3;
int part_slot(int part) { return part <= 1 ? 0 : part - 1; }
RedCtx dot_red(amg_hier_s* h, RankState& R, int kind, unsigned long long cond, int part = 0) {
    if (!h->multi()) return RedCtx{R.partials, R.ticket, nullptr, R.st, cond, kind, nullptr};
    return RedCtx{R.partials, R.ticket, R.dot_local + part_slot(part), nullptr, 0ull, FIN_NONE, nullptr};
}

// ------------------------------------------------------------- communication
// Records the first NCCL failure of an enqueue pass (checked by the ABI entry points).
void nccl_note(amg_hier_s* h, ncclResult_t r, const char* what) {
    if (r != ncclSuccess && h->nccl_status == ncclSuccess) {
        h->nccl_status = r;
        h->nccl_what = std::string(what) + ": " + ncclGetErrorString(r);
    }
}

// Loopback over a one-rank NCCL communicator: every (destination, source) rank pair's dot slots
// as one self send/recv of a group (NCCL matches a peer's sends and receives in issue order).
void loop_nccl_dots(amg_hier_s* h, cudaStream_t s) {
    nccl_note(h, ncclGroupStart(), "ncclGroupStart (loopback dots)");
    for (auto& Rd : h->ranks)
        for (auto& Rs : h->ranks) {
            nccl_note(h, ncclSend(Rs.dot_local, kDotSlots, ncclDouble, 0, h->ctx->nccl, s), "ncclSend (loopback dots)");
            nccl_note(h, ncclRecv(Rd.dot_all + kDotSlots * Rs.rank, kDotSlots, ncclDouble, 0, h->ctx->nccl, s),
                      "ncclRecv (loopback dots)");
        }
    nccl_note(h, ncclGroupEnd(), "ncclGroupEnd (loopback dots)");
}

// ------------------------------------------------------ peer-memory (LSA) transport
LsaPush lsa_args(amg_hier_s* h, RankState& R, const Exch* E, int l) {
    LsaPush P{};
    P.peer_base = h->lsa_peer;
    P.send_off = E ? E->d_send_off : nullptr;
    P.dst_off = E ? E->d_dst_off : nullptr;
    P.stride = l >= 0 ? h->lsa_lvl_stride[l] : 0;
    P.seq = R.lsa_seq;
    P.count = R.lsa_count;
    P.np = h->np;
    P.me = R.rank;
    P.flag_off = h->lsa_flag_off;
    P.dots = nullptr;
    P.kdot = kDotSlots;
    P.dot_off = h->lsa_dot_off;
    P.dot_stride = h->lsa_dot_stride;
    return P;
}
RxWait lsa_rx(amg_hier_s* h, RankState& R, int64_t stride_doubles) {
    RxWait w;
    w.flags = R.lsa_flags;
    w.seq = R.lsa_seq;
    w.err = h->lsa_err;
    w.timeout_ns = h->lsa_timeout_ns;
    w.np = h->np;
    w.stride = stride_doubles;
    return w;
}
// every rank's dot slots to every rank (slot rank), one barrier (the receive side: k_finish)
void lsa_dot_push(amg_hier_s* h, cudaStream_t s) {
    for (auto& R : h->ranks) {
        LsaPush P = lsa_args(h, R, nullptr, -1);
        P.dots = R.dot_local;
        launch_k(k_lsa_push, 1, kBlock, s, (const double*)nullptr, (const int32_t*)nullptr, (int64_t)0, P);
    }
}
// finish every rank's gathered dots (loopback: every rank pushed before any waits)
void lsa_dot_finish(amg_hier_s* h, Launch& L, const std::function<RedCtx(RankState&)>& rc) {
    lsa_dot_push(h, L.s);
    for (auto& R : h->ranks) {
        L.begin("dot_finish", 8.0 * kDotSlots * h->np);
        launch_k(k_finish, 1, kBlock, L.s, (const double*)R.lsa_dots, kDotSlots * h->np, rc(R),
                 lsa_rx(h, R, h->lsa_dot_stride / 8));
        L.end();
        cudaMemsetAsync(R.dot_local, 0, kDotSlots * sizeof(double), L.s);
    }
}

// Multi-rank: gather every rank's dot total to every rank, then finish in rank order.
void dot_finish(amg_hier_s* h, Launch& L, int kind, unsigned long long cond = 0) {
    if (!h->multi()) return;
    if (h->lsa) {
        lsa_dot_finish(h, L, [&](RankState& R) { return RedCtx{nullptr, nullptr, nullptr, R.st, cond, kind, nullptr}; });
        return;
    }
    if (h->loop_nccl()) {
        loop_nccl_dots(h, L.s);
    } else if (h->loopback) {
        for (auto& Rd : h->ranks)
            for (auto& Rs : h->ranks)
                cudaMemcpyAsync(Rd.dot_all + kDotSlots * Rs.rank, Rs.dot_local, kDotSlots * sizeof(double),
                                cudaMemcpyDeviceToDevice, L.s);
    } else {
        RankState& R = h->ranks[0];
        nccl_note(h, ncclAllGather(R.dot_local, R.dot_all, kDotSlots, ncclDouble, h->ctx->nccl, L.s),
                  "ncclAllGather (dot totals)");
    }
    for (auto& R : h->ranks) {
        // every rank computes the same status; in loopback each sets the (shared) WHILE condition
        RedCtx rc{nullptr, nullptr, nullptr, R.st, cond, kind, nullptr};
        L.begin("dot_finish", 8.0 * kDotSlots * h->np);
        launch_k(k_finish, 1, 32, L.s, (const double*)R.dot_all, kDotSlots * h->np, rc, RxWait{});
        L.end();
        cudaMemsetAsync(R.dot_local, 0, kDotSlots * sizeof(double), L.s);  // slots of skipped parts stay 0
    }
}

// Several ranks, K-cycle: the same gather, finished into each rank's level-lvl K state.
void dot_finish_k(amg_hier_s* h, Launch& L, int kind, int lvl) {
    if (!h->multi()) return;
    if (h->lsa) {
        lsa_dot_finish(h, L, [&](RankState& R) {
            return RedCtx{nullptr, nullptr, nullptr, nullptr, 0ull, kind, R.lv[lvl].kst};
        });
        return;
    }
    if (h->loop_nccl()) {
        loop_nccl_dots(h, L.s);
    } else if (h->loopback) {
        for (auto& Rd : h->ranks)
            for (auto& Rs : h->ranks)
                cudaMemcpyAsync(Rd.dot_all + kDotSlots * Rs.rank, Rs.dot_local, kDotSlots * sizeof(double),
                                cudaMemcpyDeviceToDevice, L.s);
    } else {
        RankState& R = h->ranks[0];
        nccl_note(h, ncclAllGather(R.dot_local, R.dot_all, kDotSlots, ncclDouble, h->ctx->nccl, L.s),
                  "ncclAllGather (K-cycle dot totals)");
    }
    for (auto& R : h->ranks) {
        RedCtx rc{nullptr, nullptr, nullptr, nullptr, 0ull, kind, R.lv[lvl].kst};
        L.begin("dot_finish", 8.0 * kDotSlots * h->np);
        launch_k(k_finish, 1, 32, L.s, (const double*)R.dot_all, kDotSlots * h->np, rc, RxWait{});
        L.end();
        cudaMemsetAsync(R.dot_local, 0, kDotSlots * sizeof(double), L.s);
    }
}

using VecOf = std::function<double*(RankState&)>;
// custom unpack of a received halo (rank, its exchange plan, stream); null: v[idx] = buf
using UnpackFn = std::function<void(RankState&, const Exch&, cudaStream_t)>;

// Halo exchange of a level-l vector (window base pointer given per rank) on stream `st`.
// pack_st: stream of the pack kernels (null: st).  The overlapped form packs on the context stream
// BEFORE the interior kernel takes every SM, so the transfer runs during it.
void exchange_on(amg_hier_s* h, cudaStream_t st, int l, const VecOf& vec, const UnpackFn* unpack = nullptr,
                 cudaStream_t pack_st = nullptr);
void exchange(amg_hier_s* h, Launch& L, int l, const VecOf& vec) { exchange_on(h, L.s, l, vec); }

// Overlapped exchange: fork the comm stream off the context stream, exchange there,
// and let the caller launch the interior rows before exchange_end joins the streams.
void exchange_begin(amg_hier_s* h, Launch& L, int l, const VecOf& vec, const UnpackFn* unpack = nullptr) {
    exchange_on(h, h->comm, l, vec, unpack, L.s);
    cudaEventRecord(h->ev_join, h->comm);
}
void exchange_end(amg_hier_s* h, Launch& L) { cudaStreamWaitEvent(L.s, h->ev_join, 0); }

// An operator application that gathers a level-lx vector xv: single rank / replicated:
// one launch (part 0).  Distributed: exchange the halo on the comm stream while the
// interior units (no halo columns) run, then the head and tail units (north_star (4):
// "halo exchange ... overlapped with interior SpMV").
using PartFn = std::function<void(RankState&, int)>;
// distributed levels with fewer rows per rank are not split into interior / boundary launches:
// their operator passes are a few microseconds, shorter than the exchange they would overlap
constexpr int64_t kSplitRows = 4096;
void overlapped(amg_hier_s* h, Launch& L, int lx, const VecOf& xv, bool dist, const PartFn& fn,
                const UnpackFn* unpack = nullptr) {
    if (!h->multi() || !dist) {
        for (auto& R : h->ranks) fn(R, 0);
        return;
    }
    if (h->ranks[0].lv[lx].comp_n < kSplitRows) {  // tiny distributed level: the split only adds launches
        exchange_on(h, L.s, lx, xv, unpack);
        for (auto& R : h->ranks) fn(R, 0);
        return;
    }
    exchange_begin(h, L, lx, xv, unpack);
    for (auto& R : h->ranks) fn(R, 1);
    exchange_end(h, L);
    for (auto& R : h->ranks) {
        fn(R, 2);
        fn(R, 3);
    }
}

void exchange_on(amg_hier_s* h, cudaStream_t st, int l, const VecOf& vec, const UnpackFn* unpack,
                 cudaStream_t pack_st) {
    if (!h->multi()) return;
    Launch L{h, st};
    const int nsm = h->ctx->nsm;
    bool any = false;
    for (auto& R : h->ranks) any |= (R.lv[l].ex.nsend > 0 || R.lv[l].ex.nrecv > 0);
    if (!any && h->loopback) {
        if (pack_st) {  // keep the fork/join structure of the caller (ev_join recorded on st)
            cudaEventRecord(h->ev_fork, pack_st);
            cudaStreamWaitEvent(st, h->ev_fork, 0);
        }
        return;
    }
    if (h->lsa) {
        // push + arrive on the pack stream (ahead of the interior kernel), wait + unpack on st; every
        // rank arrives at every exchange, with or without entries for its peers
        Launch Lp{h, pack_st ? pack_st : st};
        for (auto& R : h->ranks) {
            const Exch& E = R.lv[l].ex;
            Lp.begin("halo_push", 16.0 * (double)E.nsend);
            launch_k(k_lsa_push, E.nsend ? vec_grid(E.nsend, nsm) : 1, kBlock, Lp.s, (const double*)vec(R),
                     (const int32_t*)E.send_idx, E.nsend, lsa_args(h, R, &E, l));
            Lp.end();
        }
        if (pack_st) {
            cudaEventRecord(h->ev_fork, pack_st);
            cudaStreamWaitEvent(st, h->ev_fork, 0);
        }
        for (auto& R : h->ranks) {  // ranks with something to receive wait inside their unpack (below)
            if (R.lv[l].ex.nrecv) continue;
            L.begin("halo_wait", 8.0 * h->np);
            launch_k(k_lsa_wait, 1, kBlock, L.s, R.lv[l].ex.rx);
            L.end();
        }
    } else {
    {
        Launch Lp{h, pack_st ? pack_st : st};
        for (auto& R : h->ranks) {
            const Exch& E = R.lv[l].ex;
            if (!E.nsend) continue;
            Lp.begin("halo_pack", 20.0 * (double)E.nsend);
            launch_k(k_pack, vec_grid(E.nsend, nsm), kBlock, Lp.s, vec(R), E.send_idx, E.sbuf, E.nsend);
            Lp.end();
        }
    }
    if (pack_st) {  // the transfer and the unpack follow the packs on st
        cudaEventRecord(h->ev_fork, pack_st);
        cudaStreamWaitEvent(st, h->ev_fork, 0);
    }
    if (h->loopback) {
        const bool nc = h->loop_nccl();
        if (nc) nccl_note(h, ncclGroupStart(), "ncclGroupStart (loopback halo)");
        for (auto& Rd : h->ranks) {
            const Exch& Ed = Rd.lv[l].ex;
            for (auto& Rs : h->ranks) {
                const int64_t cnt = Ed.recv_off[Rs.rank + 1] - Ed.recv_off[Rs.rank];
                if (!cnt) continue;
                const Exch& Es = Rs.lv[l].ex;
                if (nc) {
                    nccl_note(h, ncclSend(Es.sbuf + Es.send_off[Rd.rank], cnt, ncclDouble, 0, h->ctx->nccl, L.s),
                              "ncclSend (loopback halo)");
                    nccl_note(h, ncclRecv(Ed.rbuf + Ed.recv_off[Rs.rank], cnt, ncclDouble, 0, h->ctx->nccl, L.s),
                              "ncclRecv (loopback halo)");
                } else {
                    cudaMemcpyAsync(Ed.rbuf + Ed.recv_off[Rs.rank], Es.sbuf + Es.send_off[Rd.rank],
                                    cnt * sizeof(double), cudaMemcpyDeviceToDevice, L.s);
                }
            }
        }
        if (nc) nccl_note(h, ncclGroupEnd(), "ncclGroupEnd (loopback halo)");
    } else {
        RankState& R = h->ranks[0];
        const Exch& E = R.lv[l].ex;
        nccl_note(h, ncclGroupStart(), "ncclGroupStart (halo)");
        for (int q = 0; q < h->np; ++q) {
            const int64_t ns = E.send_off[q + 1] - E.send_off[q];
            const int64_t nr = E.recv_off[q + 1] - E.recv_off[q];
            if (ns) nccl_note(h, ncclSend(E.sbuf + E.send_off[q], ns, ncclDouble, q, h->ctx->nccl, st), "ncclSend (halo)");
            if (nr) nccl_note(h, ncclRecv(E.rbuf + E.recv_off[q], nr, ncclDouble, q, h->ctx->nccl, st), "ncclRecv (halo)");
        }
        nccl_note(h, ncclGroupEnd(), "ncclGroupEnd (halo)");
    }
    }  // transports
    for (auto& R : h->ranks) {
        const Exch& E = R.lv[l].ex;
        if (!E.nrecv) continue;
        L.begin("halo_unpack", 20.0 * (double)E.nrecv);
        if (unpack) (*unpack)(R, E, L.s);
        else launch_k(k_unpack, vec_grid(E.nrecv, nsm), kBlock, L.s, vec(R), (const int32_t*)E.recv_idx,
                      (const double*)E.rbuf, E.nrecv, E.rx);  // rx.flags null: plain buffer
        L.end();
    }
}

// Coarsest-level solve z_L = B_L b_L: the explicit inverse (reading R2) or the
// paper's l1-Jacobi-preconditioned CG as one cluster kernel.
void launch_coarse(amg_hier_s* h, Launch& L, RankState& R, const double* b, double* x) {
    const int nsm = h->ctx->nsm;
    if (h->cfg.coarse_solver != 1) {
        L.begin("coarse_gemv", 8.0 * (double)R.nL * (double)R.nL + 16.0 * (double)R.nL);
        launch_k(k_dense_gemv, vec_grid(R.nL * 32, nsm), kBlock, L.s, R.cinv, b, x, R.nL);
        L.end();
        return;
    }
    // bytes of ONE pass over A_L (the iteration count is data dependent; latency-bound)
    L.begin("coarse_cg", 12.0 * (double)R.cg_nnz + 4.0 * (double)(R.nL + 1) + 24.0 * (double)R.nL);
    const CoarseCG A{R.cg_rp, R.cg_ci, R.cg_v, R.cg_m, R.cg_split, (int32_t)R.nL, R.cg_ncta, R.cg_smem_a,
                     h->cfg.coarse_maxit, h->cfg.coarse_rtol, R.cg_wrp, R.cg_wci, R.cg_wv, R.cg_zrp, R.cg_zci,
                     R.cg_zv};
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)R.cg_ncta);
    cfg.blockDim = dim3((unsigned)kCgBlock);
    cfg.dynamicSmemBytes = R.cg_smem;
    cfg.stream = L.s;
    cudaLaunchAttribute attr[2];
    int na = 0;
    if (pdl_enabled()) {
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    if (R.cg_ncta > 1) {
        attr[na].id = cudaLaunchAttributeClusterDimension;
        attr[na].val.clusterDim.x = (unsigned)R.cg_ncta;
        attr[na].val.clusterDim.y = 1;
        attr[na].val.clusterDim.z = 1;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    cudaLaunchKernelEx(&cfg, k_coarse_cg, A, b, x);
    L.end();
}

template <class T>
int dev_copy(T** dst, const T* src, size_t count);
template <class T>
int dev_alloc(T** dst, size_t count);

// ------------------------------------------------------------- persistent tail
// The cycle rooted at the first tail level as a flat program for k_tail (single
// rank): the same operations, in the same order and on the same vectors, as
// enqueue_level / enqueue_fcg2 would launch for those levels.
struct TailEmitter {
    amg_hier_s* h;
    std::vector<TailOp> ops;
    double bytes = 0.0;
    static TailOp op(int kind, int epi) {
        TailOp o;
        std::memset(&o, 0, sizeof(o));
        o.kind = kind;
        o.epi = epi;
        o.fin = FIN_NONE;
        return o;
    }
    void spmv(const DevMat& M, int epi, const double* g, double* y, int64_t nvec) {
        if (M.c16) std::abort();  // the tail's levels are uploaded with 32-bit columns (C16Scope)
        TailOp o = op(TK_SPMV, epi);
        o.rp = M.rp;
        o.ci = M.col;
        o.v = M.val;
        o.n = M.nrows;
        o.g = g;
        o.y = y;
        // lanes per row: enough groups to cover the grid, whole blocks for few long rows
        const double mean = (double)M.nnz / (double)std::max<int64_t>(M.nrows, 1);
        const double threads = (double)h->tail_grid * kBlock;
        int vw = 4;
        while (vw < 32 && (vw * (double)M.nrows < threads || vw * 8 < mean) && vw * 2 <= std::max(4.0, mean)) vw *= 2;
        if (mean >= 256.0 && (double)M.nrows * 32 < threads) vw = kBlock;
        o.vw = vw;
        ops.push_back(o);
        bytes += M.model_bytes() + 8.0 * (double)nvec * (double)M.nrows;
    }
    void level(int l, const double* b, const double* mb, double* out) {
        RankState& R = h->ranks[0];
        const int nl = h->nlev();
        const int s1 = h->cfg.pre_sweeps, s2 = h->cfg.post_sweeps;
        DevLevel& D = R.lv[l];
        if (l == nl - 1) {
            TailOp o = op(TK_GEMV, 0);
            o.v = R.cinv;
            o.n = R.nL;
            o.g = b;
            o.y = out;
            ops.push_back(o);
            bytes += 8.0 * (double)R.nL * (double)R.nL + 16.0 * (double)R.nL;
            return;
        }
        const bool am = (s1 == 1);
        const double* xpre = nullptr;
        if (am) {
            spmv(D.Am, TE_RESID, b, D.r, 2);
            ops.back().b = b;
        } else {
            spmv(D.A, TE_SWEEP0, mb, D.xa, 3);
            ops.back().b = b;
            ops.back().abs = 1;
            xpre = D.xa;
            for (int sw = 2; sw < s1; ++sw) {
                double* xo = (xpre == D.xa) ? D.xb : D.xa;
                spmv(D.A, TE_SWEEP, xpre, xo, 3);
                ops.back().x = xpre;
                ops.back().b = b;
                ops.back().abs = 1;
                xpre = xo;
            }
            spmv(D.A, TE_RESID, xpre, D.r, 3);
            ops.back().b = b;
        }
        DevLevel& C = R.lv[l + 1];
        if (!C.coarsest && !am) {
            spmv(D.R, TE_STOREMB, D.r, C.b, 3);
            ops.back().y2 = C.mb;
            ops.back().m = C.m;
        } else {
            spmv(D.R, TE_STORE, D.r, C.b, 2);
        }
        const double* e;
        if (h->cfg.cycle == 1 && l + 1 < nl - 1) {
            fcg2(l + 1);
            e = C.kx;
        } else {
            level(l + 1, C.b, C.mb, C.xa);
            e = C.xa;
        }
        double* tmp = D.xb;
        double* dst = (s2 % 2 == 1) ? tmp : out;
        if (am) {
            spmv(D.P, TE_STORE, e, dst, 2);
        } else {
            spmv(D.P, TE_PROLADD, e, dst, 3);
            ops.back().x = xpre;
        }
        const double* cur = dst;
        const bool abs = (double)D.A.nnz <= abs_row_cut() * (double)std::max<int64_t>(D.A.nrows, 1);
        for (int sw = 0; sw < s2; ++sw) {
            double* xo = (cur == tmp) ? out : tmp;
            if (sw == 0 && am) {
                spmv(D.A, TE_POST1, cur, xo, 4);
                ops.back().x = cur;
                ops.back().r = D.r;
                ops.back().b = b;
                ops.back().mb = 0;
            } else {
                spmv(D.A, TE_SWEEP, cur, xo, 3);
                ops.back().x = cur;
                ops.back().b = b;
            }
            ops.back().abs = abs ? 1 : 0;
            ops.back().m = D.m;
            cur = xo;
        }
    }
    void dot(const double* a, const double* b, int64_t n, double* ks, int fin) {
        TailOp o = op(TK_DOT, 0);
        o.b = a;
        o.r = b;
        o.n = n;
        o.ks = ks;
        o.fin = fin;
        ops.push_back(o);
        bytes += 16.0 * (double)n;
    }
    // final_update: apply x += alpha p here (nested solves, consumed inside the program);
    // the top-level solve leaves it to its launched consumer, which gathers x + alpha p
    void fcg2(int l, bool final_update = true) {
        RankState& R = h->ranks[0];
        DevLevel& D = R.lv[l];
        const int64_t n = D.comp_n;
        if (h->cfg.pre_sweeps != 1) {  // the inner applications need m o r (SWEEP0 gathers it)
            set_err("tail: K-cycle tail needs pre_sweeps == 1");
        }
        level(l, D.b, D.mb, D.kp);
        dot(D.kp, D.b, n, D.kst, FIN_KPR0);
        spmv(D.A, TE_SPMVDOT, D.kp, D.kq, 2);
        ops.back().x = D.kp;
        ops.back().ks = D.kst;
        ops.back().fin = FIN_KALPHA;
        TailOp u1 = op(TK_KUPD1, 0);
        u1.n = n;
        u1.y = D.kx;
        u1.x = D.kp;
        u1.y2 = D.kr;
        u1.b = D.b;
        u1.r = D.kq;
        u1.ks = D.kst;
        ops.push_back(u1);
        bytes += 40.0 * (double)n;
        level(l, D.kr, nullptr, D.kz);
        dot(D.kz, D.kq, n, D.kst, FIN_KBETA);
        TailOp pu = op(TK_KPUPD, 0);
        pu.n = n;
        pu.y = D.kp;
        pu.b = D.kz;
        pu.r = D.kr;
        pu.ks = D.kst;
        pu.fin = FIN_KPR;
        ops.push_back(pu);
        bytes += 32.0 * (double)n;
        spmv(D.A, TE_SPMVDOT, D.kp, D.kq, 2);
        ops.back().x = D.kp;
        ops.back().ks = D.kst;
        ops.back().fin = FIN_KALPHA;
        if (!final_update) return;
        TailOp u2 = op(TK_KUPD2, 0);
        u2.n = n;
        u2.y = D.kx;
        u2.x = D.kp;
        u2.ks = D.kst;
        ops.push_back(u2);
        bytes += 24.0 * (double)n;
    }
};

int build_tail(amg_hier_s* h) {
    const int lt = h->tail_level;
    if (h->tail_cluster) {
        // function attributes are per device: set on every build (cheap, thread-safe)
        CK(cudaFuncSetAttribute(k_tail<true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        int cl = 16;
        for (; cl > 1; cl /= 2) {  // the largest cluster the device can co-schedule
            cudaLaunchConfig_t lc = {};
            lc.gridDim = dim3((unsigned)cl);
            lc.blockDim = dim3((unsigned)kBlock);
            cudaLaunchAttribute at;
            at.id = cudaLaunchAttributeClusterDimension;
            at.val.clusterDim.x = (unsigned)cl;
            at.val.clusterDim.y = at.val.clusterDim.z = 1;
            lc.attrs = &at;
            lc.numAttrs = 1;
            int ncl = 0;
            if (cudaOccupancyMaxActiveClusters(&ncl, k_tail<true>, &lc) == cudaSuccess && ncl > 0) break;
            cudaGetLastError();
        }
        h->tail_grid = cl;
    } else {
        int nb = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_tail<false>, kBlock, 0));
        h->tail_grid = std::max(1, std::min(nb, 6)) * h->ctx->nsm;
    }
    TailEmitter E{h, {}, 0.0};
    RankState& R = h->ranks[0];
    if (h->cfg.cycle == 1) E.fcg2(lt, false);
    else E.level(lt, R.lv[lt].b, R.lv[lt].mb, R.lv[lt].xa);
    int st;
    if ((st = dev_copy(&h->tail_prog, E.ops.data(), E.ops.size()))) return st;
    h->tail_nops = (int)E.ops.size();
    h->tail_bytes = E.bytes;
    if ((st = dev_alloc(&h->tail_partials, (size_t)h->tail_grid))) return st;
    return AMG_OK;
}

void launch_tail(amg_hier_s* h, Launch& L) {
    L.begin("tail", h->tail_bytes);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)h->tail_grid);
    cfg.blockDim = dim3((unsigned)kBlock);
    cfg.stream = L.s;
    cudaLaunchAttribute attr[1];
    if (h->tail_cluster) {
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = (unsigned)h->tail_grid;
        attr[0].val.clusterDim.y = attr[0].val.clusterDim.z = 1;
    } else {
        attr[0].id = cudaLaunchAttributeCooperative;
        attr[0].val.cooperative = 1;
    }
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (h->tail_cluster)
        cudaLaunchKernelEx(&cfg, k_tail<true>, (const TailOp*)h->tail_prog, (int32_t)h->tail_nops, h->tail_partials);
    else
        cudaLaunchKernelEx(&cfg, k_tail<false>, (const TailOp*)h->tail_prog, (int32_t)h->tail_nops, h->tail_partials);
    L.end();
}

// ------------------------------------------------------------- V-cycle / K-cycle
void enqueue_fcg2(amg_hier_s* h, Launch& L, int l);
// K-cycle inner FCG without the vector-update kernel (one pre-sweep, l1-Jacobi): the
// second application forms r = b - alpha_1 q_1 itself, the consumer forms x (GXap2)
// (single rank: several ranks form the inner x explicitly, so a consumer gathers ONE vector)
inline bool kcycle_fused(const amg_hier_s* h) {
    return h->cfg.pre_sweeps == 1 && h->cfg.smoother == 0 && !h->multi();
}
// Where a cycle's fused dot goes: the PCG state (default) or a K-cycle level state.
struct DotSink {
    double* ks;  // single rank: the level's K state (ranks[0]); several ranks use lvl
    int kind;
    // K-cycle, s1 == 1: the application's right-hand side is b - alpha q (k = ks), formed by
    // its first kernel, which also writes it to the application's b vector
    const double* kb = nullptr;
    const double* kq = nullptr;
    int lvl = -1;  // the level whose K state {p^T r, p^T q, alpha, beta, stop} receives the dot
};
void enqueue_level(amg_hier_s* h, Launch& L, int l, const VecOf& bvec, const VecOf* mbvec, const VecOf& outv,
                   bool dot, const VecOf* dwv, const DotSink* sink = nullptr);
// Several ranks: every dot (PCG or K state) goes to the rank's local slots; end_dot all-gathers
// them and finishes into the PCG state or each rank's level-K state in rank order.
RedCtx sink_red(amg_hier_s* h, RankState& R, int dkind, const DotSink* sink, int part = 0) {
    if (sink && !h->multi()) return RedCtx{R.partials, R.ticket, nullptr, nullptr, 0ull, sink->kind, sink->ks};
    return dot_red(h, R, dkind, 0, part);
}
void dot_finish_k(amg_hier_s* h, Launch& L, int kind, int lvl);
void end_dot(amg_hier_s* h, Launch& L, bool dot, int dkind, const DotSink* sink) {
    if (!dot || !h->multi()) return;
    if (sink) dot_finish_k(h, L, sink->kind, sink->lvl);
    else dot_finish(h, L, dkind);
}

// Level l of the cycle with the INVK smoother (cfg.smoother == 1): M^{-1} r = Z (Wd r),
// Wd = D^{-1} W, Z = W^T of the rank's diagonal block (HINVK / l1-INVK).
// The iterate lives in `out` throughout (every update is row-local), Wd r in the level's mb
// buffer (m o b is not used with INVK), residuals in r:
//   out = Z (Wd b); [s1-1 times: r' = b - A out; out += Z (Wd r')]; r = b - A out;
//   b_{l+1} = R r; e = cycle(l+1); out += P-bar e; s2 times: r' = b - A out;
//   out += Z (Wd r')   (the last one at level 0 also reduces the PCG/FCG dot).
// Several ranks: the factors are block-diagonal over the ranks' rows, so only the residual
// SpMVs, the restriction and the prolongation exchange halos (overlapped with their interior
// rows); Wd and Z run on the rank's own rows.
void enqueue_level_invk(amg_hier_s* h, Launch& L, int l, const VecOf& bvec, const VecOf& outv, bool dot,
                        const VecOf* dwv, const DotSink* sink) {
    const int dkind = dwv ? FIN_ZQ : FIN_RZ;
    const int nl = h->nlev();
    const int s1 = h->cfg.pre_sweeps, s2 = h->cfg.post_sweeps;
    const bool dist = !h->ranks[0].lv[l].replicated;
    const bool cdist = !h->ranks[0].lv[l + 1].replicated;
    auto n8 = [l](RankState& R) { return 8.0 * (double)R.lv[l].comp_n; };
    // out (+)= Z (Wd src) on every rank's computed rows
    auto precond = [&](const VecOf& src, bool add, bool dt) {
        for (auto& R : h->ranks) {
            DevLevel& D = R.lv[l];
            double* x = outv(R) + D.ep_off;
            launch_mat(L, D.Wd, GVec{src(R)}, EStore{D.mb + D.ep_off}, no_red(), "invk_w", 2 * n8(R));
            if (dt)
                launch_mat(L, D.Z, GVec{D.mb}, EAddDot<true>{x, x, dwv ? (*dwv)(R) + D.ep_off : bvec(R) + D.ep_off},
                           sink ? sink_red(h, R, dkind, sink) : dot_red(h, R, dkind, 0), "invk_z_dot", 4 * n8(R));
            else if (add)
                launch_mat(L, D.Z, GVec{D.mb}, EAddDot<false>{x, x}, no_red(), "invk_z", 3 * n8(R));
            else
                launch_mat(L, D.Z, GVec{D.mb}, EStore{x}, no_red(), "invk_z", 2 * n8(R));
        }
    };
    const VecOf rv = [l](RankState& R) { return R.lv[l].r; };
    auto resid = [&](const char* name) {  // r = b - A out (halo of out)
        overlapped(h, L, l, outv, dist, [&](RankState& R, int part) {
            DevLevel& D = R.lv[l];
            launch_mat(L, D.A, GVec{outv(R)}, EResid{bvec(R) + D.ep_off, D.r + D.ep_off}, no_red(), name,
                       3 * n8(R), part);
        });
    };
    precond(bvec, false, false);
    for (int sw = 1; sw < s1; ++sw) {
        resid("invk_resid");
        precond(rv, true, false);
    }
    resid("resid");
    overlapped(h, L, l, rv, dist, [&](RankState& R, int part) {
        DevLevel& D = R.lv[l];
        launch_mat(L, D.R, GVec{D.r}, EStore{R.lv[l + 1].b + D.rst_off}, no_red(), "restrict",
                   n8(R) + 8.0 * (double)D.rst_n, part);
    });
    if (!cdist && dist)  // first replicated level: gather the restricted rhs
        exchange(h, L, l + 1, [&](RankState& R) { return R.lv[l + 1].b; });
    const bool kfcg = h->cfg.cycle == 1 && l + 1 < nl - 1;
    const VecOf cb = [l](RankState& R) { return R.lv[l + 1].b; };
    const VecOf ev = kfcg ? VecOf([l](RankState& R) { return R.lv[l + 1].kx; })
                          : VecOf([l](RankState& R) { return R.lv[l + 1].xa; });
    if (kfcg) enqueue_fcg2(h, L, l + 1);
    else enqueue_level(h, L, l + 1, cb, nullptr, ev, false, nullptr);
    overlapped(h, L, l + 1, ev, cdist, [&](RankState& R, int part) {
        DevLevel& D = R.lv[l];
        DevLevel& C = R.lv[l + 1];
        double* x = outv(R) + D.ep_off;
        if (kfcg && !h->multi())  // e = x + alpha p of the inner FCG, formed in the gather (its last update)
            launch_mat(L, D.P, GXap{C.kx, C.kp2, C.kst}, EProlongAdd{x, x}, no_red(), "prolong",
                       2 * n8(R) + 16.0 * (double)C.comp_n, part);
        else
            launch_mat(L, D.P, GVec{ev(R)}, EProlongAdd{x, x}, no_red(), "prolong",
                       2 * n8(R) + 8.0 * (double)C.comp_n, part);
    });
    for (int sw = 0; sw < s2; ++sw) {
        resid("invk_resid");
        precond(rv, true, dot && sw == s2 - 1);
    }
    end_dot(h, L, dot, dkind, sink);
}

// Collapsed level (compact, above a direct coarsest solve): out = S2(b) + M b in ONE kernel.
// Single rank, or a replicated level of a multi-rank hierarchy (every rank computes all rows).
void enqueue_level_collapsed(amg_hier_s* h, Launch& L, int l, const VecOf& bvec, const VecOf& outv, bool dot,
                             const VecOf* dwv, const DotSink* sink) {
    const int dkind = dwv ? FIN_ZQ : FIN_RZ;
    for (auto& R : h->ranks) {
        DevLevel& D = R.lv[l];
        const double* b = bvec(R);
        double* out = outv(R);
        const int64_t n = D.comp_n;
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(n, kMaxPartials));
        const bool krhs = sink && sink->kb;
        const double* dw = (dot && dwv) ? (*dwv)(R) : nullptr;
        const RedCtx red = dot ? sink_red(h, R, dkind, sink) : no_red();
        L.begin("collapsed", 8.0 * (double)n * (double)n + 16.0 * (double)n);
        if (krhs) {
            const GBaq g{sink->kb, sink->kq, sink->ks};
            double* rhs = const_cast<double*>(b);
            if (dot) launch_k(k_collapsed<GBaq, true, true>, grid, kBlock, L.s, (const double*)D.Mc, n, g, rhs, out, dw, red);
            else launch_k(k_collapsed<GBaq, false, true>, grid, kBlock, L.s, (const double*)D.Mc, n, g, rhs, out, dw, red);
        } else {
            const GVec g{b};
            if (dot) launch_k(k_collapsed<GVec, true, false>, grid, kBlock, L.s, (const double*)D.Mc, n, g, (double*)nullptr, out, dw, red);
            else launch_k(k_collapsed<GVec, false, false>, grid, kBlock, L.s, (const double*)D.Mc, n, g, (double*)nullptr, out, dw, red);
        }
        L.end();
    }
    end_dot(h, L, dot, dkind, sink);
}

// Compact small level (see compact_level_ok): s = S2(b) = m b + m (b - A (m b)) into r;
// b_{l+1} = Rc b; coarse correction e; out = s + Pc e (+ the K-cycle dot of a sink).
// Single rank, or a replicated level of a multi-rank hierarchy (no halo below it).
void enqueue_level_compact(amg_hier_s* h, Launch& L, int l, const VecOf& bvec, const VecOf& outv, bool dot,
                           const VecOf* dwv, const DotSink* sink) {
    const int nl = h->nlev();
    const bool krhs = sink && sink->kb;  // K-cycle second application: rhs = b - alpha q, stored in b
    // the smoothing branch s = S2(b) runs on the second stream, concurrently with the
    // restriction and the whole coarse correction; the post kernel joins it
    cudaEventRecord(h->ev_fork, L.s);
    cudaStreamWaitEvent(h->comm, h->ev_fork, 0);
    {
        Launch Ls{h, h->comm};
        for (auto& R : h->ranks) {
            DevLevel& D = R.lv[l];
            const double* b = bvec(R);
            const double n8 = 8.0 * (double)D.comp_n;
            if (krhs)
                launch_mat(Ls, D.A, GMBaq{D.m, sink->kb, sink->kq, sink->ks},
                           ESweep0K{sink->kb, sink->kq, sink->ks, const_cast<double*>(b), D.r}, no_red(), "sweep0_c",
                           5 * n8);
            else
                launch_mat(Ls, D.A, GMB{D.m, b}, ESweep0{b, D.r}, no_red(), "sweep0_c", 3 * n8);
        }
    }
    cudaEventRecord(h->ev_join, h->comm);
    for (auto& R : h->ranks) {
        DevLevel& D = R.lv[l];
        DevLevel& C = R.lv[l + 1];
        const double n8 = 8.0 * (double)D.comp_n, nc8 = 8.0 * (double)C.comp_n;
        if (krhs)
            launch_mat(L, D.Rc, GBaq{sink->kb, sink->kq, sink->ks}, EStore{C.b}, no_red(), "restrict_c", 2 * n8 + nc8);
        else
            launch_mat(L, D.Rc, GVec{bvec(R)}, EStore{C.b}, no_red(), "restrict_c", n8 + nc8);
    }
    const bool kfcg = h->cfg.cycle == 1 && l + 1 < nl - 1;
    const VecOf cb = [l](RankState& R) { return R.lv[l + 1].b; };
    const VecOf cmb = [l](RankState& R) { return R.lv[l + 1].mb; };
    const VecOf ev = kfcg ? VecOf([l](RankState& R) { return R.lv[l + 1].kx; })
                          : VecOf([l](RankState& R) { return R.lv[l + 1].xa; });
    if (h->tail_nops > 0 && l + 1 == h->tail_level) launch_tail(h, L);
    else if (kfcg) enqueue_fcg2(h, L, l + 1);
    else enqueue_level(h, L, l + 1, cb, &cmb, ev, false, nullptr);
    const bool tailc = h->tail_nops > 0 && l + 1 == h->tail_level;
    // joins this level's smoothing branch (a deeper compact level re-records ev_join later on the
    // same second stream, which orders after this level's branch: still a correct dependency)
    cudaStreamWaitEvent(L.s, h->ev_join, 0);
    const int dkind = dwv ? FIN_ZQ : FIN_RZ;
    for (auto& R : h->ranks) {
        DevLevel& D = R.lv[l];
        DevLevel& C = R.lv[l + 1];
        const double* b = bvec(R);
        double* out = outv(R);
        const double n8 = 8.0 * (double)D.comp_n, nc8 = 8.0 * (double)C.comp_n;
        auto post = [&](auto g) {
            if (dot)
                launch_mat(L, D.Pc, g, EAddDot<true>{D.r, out, dwv ? (*dwv)(R) : b}, sink_red(h, R, dkind, sink),
                           "prolong_post_c", 3 * n8 + nc8);
            else
                launch_mat(L, D.Pc, g, EAddDot<false>{D.r, out}, no_red(), "prolong_post_c", 2 * n8 + nc8);
        };
        if (kfcg && kcycle_fused(h) && !tailc) post(GXap2{C.kp, C.kp2, C.kst});
        else if (kfcg && !h->multi()) post(GXap{C.kx, tailc ? C.kp : C.kp2, C.kst});
        else post(GVec{ev(R)});
    }
    end_dot(h, L, dot, dkind, sink);
}

// out = B_l b: the part of the cycle rooted at level l (Eq. 3.1;
// SURVEY.md §8c O10).  bvec / outv give each rank's level-l WINDOW base pointers;
// mbvec gives m o b for levels >= 1 (the restriction writes it) and is null at
// level 0, where the first sweep gathers m_j b_j.  With `dot` (level 0 only), the
// last post-sweep also reduces b^T out (kind FIN_RZ) or, with a dot weight `dwv`
// (FCG), dwv^T out (kind FIN_ZQ).  The coarse correction is the cycle rooted at
// level l+1, or, for the K-cycle (cfg.cycle == 1) when level l+1 is not the
// coarsest, two FCG iterations at level l+1 (enqueue_fcg2).
void enqueue_level(amg_hier_s* h, Launch& L, int l, const VecOf& bvec, const VecOf* mbvec, const VecOf& outv,
                   bool dot, const VecOf* dwv, const DotSink* sink) {
    const int dkind = dwv ? FIN_ZQ : FIN_RZ;
    const int nl = h->nlev();
    const int s1 = h->cfg.pre_sweeps, s2 = h->cfg.post_sweeps;
    const int nsm = h->ctx->nsm;
    const int nr = (int)h->ranks.size();
    auto ri_of = [&](RankState& R) { return (int)(&R - h->ranks.data()); };
    if (h->cfg.smoother == 1 && l < nl - 1) {
        enqueue_level_invk(h, L, l, bvec, outv, dot, dwv, sink);
        return;
    }
    if (l == nl - 1) {  // coarsest: z_L = B_L b_L (reading R2 or the coarse CG), replicated on every rank
        for (auto& R : h->ranks) {
            launch_coarse(h, L, R, bvec(R), outv(R));
            if (dot) {  // single-level hierarchy
                L.begin("dot_rz", 16.0 * R.nL);
                launch_k(k_dot, vec_grid(R.nL, nsm), kBlock, L.s, dwv ? (*dwv)(R) : bvec(R), outv(R), R.nL,
                         sink_red(h, R, dkind, sink));
                L.end();
            }
        }
        end_dot(h, L, dot, dkind, sink);
        return;
    }
    if (h->ranks[0].lv[l].Mc) {
        enqueue_level_collapsed(h, L, l, bvec, outv, dot, dwv, sink);
        return;
    }
    if (h->ranks[0].lv[l].compact) {
        enqueue_level_compact(h, L, l, bvec, outv, dot, dwv, sink);
        return;
    }
    std::vector<double*> xpre(nr, nullptr);
    const bool dist = !h->ranks[0].lv[l].replicated;
    // s1 == 1: the residual streams A diag(m) and gathers b; m o b is never needed
    const bool am = (s1 == 1);
    if (am) mbvec = nullptr;
    // ---- down: pre-smoothing, residual, restriction
    overlapped(h, L, l, mbvec ? *mbvec : bvec, dist, [&](RankState& R, int part) {
        const int ri = ri_of(R);
        DevLevel& D = R.lv[l];
        const double* b = bvec(R);
        const double* be = b + D.ep_off;
        const double n8 = 8.0 * (double)D.comp_n;
        if (s1 == 1 && sink && sink->kb) {  // K-cycle: rhs = b - alpha_1 q_1 formed and stored here
            launch_mat(L, D.Am, GBaq{sink->kb, sink->kq, sink->ks},
                       EResidK{sink->kb, sink->kq, sink->ks, const_cast<double*>(b), D.r}, no_red(), "resid0",
                       4 * n8, part);
        } else if (s1 == 1) {  // x = m o b is never stored: r = b - A (m o b) = b - (A diag(m)) b
            launch_mat(L, D.Am, GVec{b}, EResid{be, D.r + D.ep_off}, no_red(), "resid0", 2 * n8, part);
        } else {  // x2 = m b + m (b - A (m b)): the first two sweeps from x = 0 in one pass
            if (!mbvec)
                launch_mat(L, D.A, GMB{D.m, b}, ESweep0{be, D.xa + D.ep_off}, no_red(), "sweep0", 3 * n8, part);
            else
                launch_mat(L, D.A, GVec{(*mbvec)(R)}, ESweep0{be, D.xa + D.ep_off}, no_red(), "sweep0", 3 * n8,
                           part);
            xpre[ri] = D.xa;
        }
    });
    if (s1 >= 2) {
        for (int s = 2; s < s1; ++s) {
            std::vector<double*> xnext(nr);
            for (int ri = 0; ri < nr; ++ri) {
                DevLevel& D = h->ranks[ri].lv[l];
                xnext[ri] = (xpre[ri] == D.xa) ? D.xb : D.xa;
            }
            overlapped(h, L, l, [&](RankState& R) { return xpre[ri_of(R)]; }, dist, [&](RankState& R, int part) {
                const int ri = ri_of(R);
                DevLevel& D = R.lv[l];
                double* xi = xpre[ri];
                double* xo = xnext[ri];
                launch_mat(L, D.A, GVec{xi}, ESweep<false>{xi + D.ep_off, bvec(R) + D.ep_off, xo + D.ep_off},
                           no_red(), "presweep", 3 * 8.0 * (double)D.comp_n, part);
            });
            xpre = xnext;
        }
        overlapped(h, L, l, [&](RankState& R) { return xpre[ri_of(R)]; }, dist, [&](RankState& R, int part) {
            DevLevel& D = R.lv[l];
            launch_mat(L, D.A, GVec{xpre[ri_of(R)]}, EResid{bvec(R) + D.ep_off, D.r + D.ep_off}, no_red(), "resid",
                       3 * 8.0 * (double)D.comp_n, part);
        });
    }
    overlapped(h, L, l, [l](RankState& R) { return R.lv[l].r; }, dist, [&](RankState& R, int part) {
        DevLevel& D = R.lv[l];
        DevLevel& C = R.lv[l + 1];
        if (!C.coarsest && !am)
            launch_mat(L, D.R, GVec{D.r}, EStoreMB{C.b + D.rst_off, C.m + D.rst_off, C.mb + D.rst_off}, no_red(),
                       "restrict", 8.0 * (double)D.comp_n + 24.0 * (double)D.rst_n, part);
        else
            launch_mat(L, D.R, GVec{D.r}, EStore{C.b + D.rst_off}, no_red(), "restrict",
                       8.0 * (double)D.comp_n + 8.0 * (double)D.rst_n, part);
    });
    if (h->ranks[0].lv[l + 1].replicated && dist) {  // first replicated level: gather the rhs
        exchange(h, L, l + 1, [&](RankState& R) { return R.lv[l + 1].b; });
        if (!h->ranks[0].lv[l + 1].coarsest && !am)
            exchange(h, L, l + 1, [&](RankState& R) { return R.lv[l + 1].mb; });
    }
    // ---- coarse correction e_{l+1}
    const bool kfcg = h->cfg.cycle == 1 && l + 1 < nl - 1;
    const VecOf cb = [l](RankState& R) { return R.lv[l + 1].b; };
    const VecOf cmb = [l](RankState& R) { return R.lv[l + 1].mb; };
    const VecOf ev = kfcg ? VecOf([l](RankState& R) { return R.lv[l + 1].kx; })
                          : VecOf([l](RankState& R) { return R.lv[l + 1].xa; });
    if (h->tail_nops > 0 && l + 1 == h->tail_level) launch_tail(h, L);
    else if (kfcg) enqueue_fcg2(h, L, l + 1);
    else enqueue_level(h, L, l + 1, cb, &cmb, ev, false, nullptr);
    // ---- up: prolongation, post-smoothing
    // the inner FCG's last direction: kp2 (launched inner solve), kp (the persistent tail's)
    auto kpfin = [&](DevLevel& C) -> const double* {
        return (h->tail_nops > 0 && l + 1 == h->tail_level) ? C.kp : C.kp2;
    };
    // the launched (not tail-run) inner solve without its update kernel: x was never formed
    auto kfused = [&](DevLevel&) { return kcycle_fused(h) && !(h->tail_nops > 0 && l + 1 == h->tail_level); };
    std::vector<double*> cur(nr), fin(nr), tmp(nr);
    for (int ri = 0; ri < nr; ++ri) {
        RankState& R = h->ranks[ri];
        DevLevel& D = R.lv[l];
        fin[ri] = outv(R);  // the level's result (read by level l-1)
        tmp[ri] = D.xb;     // the prolongation update is row-local: may run in place
        cur[ri] = (s2 % 2 == 1) ? tmp[ri] : fin[ri];
    }
    overlapped(h, L, l + 1, ev, !h->ranks[0].lv[l + 1].replicated, [&](RankState& R, int part) {
        const int ri = ri_of(R);
        DevLevel& D = R.lv[l];
        DevLevel& C = R.lv[l + 1];
        const double* e = ev(R);
        const double nc8 = 8.0 * (double)C.comp_n;
        double* dst = cur[ri];
        const double n8 = 8.0 * (double)D.comp_n;
        if (s1 == 1) {  // u = P-bar e only; the first post-sweep adds m o b (EPost1)
            if (kfcg && kfused(C))  // e = alpha_1 p_1 + alpha_2 p_2 of the inner FCG, formed in the gather
                launch_mat(L, D.P, GXap2{C.kp, C.kp2, C.kst}, EStore{dst + D.ep_off}, no_red(), "prolong",
                           n8 + 2 * nc8, part);
            else if (kfcg && !h->multi())  // e = x + alpha p of the inner FCG, formed in the gather
                launch_mat(L, D.P, GXap{C.kx, kpfin(C), C.kst}, EStore{dst + D.ep_off}, no_red(), "prolong",
                           n8 + 2 * nc8, part);
            else
                launch_mat(L, D.P, GVec{e}, EStore{dst + D.ep_off}, no_red(), "prolong", n8 + nc8, part);
        } else {
            if (kfcg && kfused(C))
                launch_mat(L, D.P, GXap2{C.kp, C.kp2, C.kst}, EProlongAdd{xpre[ri] + D.ep_off, dst + D.ep_off},
                           no_red(), "prolong", 2 * n8 + 2 * nc8, part);
            else if (kfcg && !h->multi())
                launch_mat(L, D.P, GXap{C.kx, kpfin(C), C.kst}, EProlongAdd{xpre[ri] + D.ep_off, dst + D.ep_off},
                           no_red(), "prolong", 2 * n8 + 2 * nc8, part);
            else
                launch_mat(L, D.P, GVec{e}, EProlongAdd{xpre[ri] + D.ep_off, dst + D.ep_off}, no_red(), "prolong",
                           2 * n8 + nc8, part);
        }
    });
    for (int s = 0; s < s2; ++s) {
        const bool last = (s == s2 - 1);
        std::vector<double*> nxt(nr);
        for (int ri = 0; ri < nr; ++ri) nxt[ri] = (cur[ri] == tmp[ri]) ? fin[ri] : tmp[ri];
        overlapped(h, L, l, [&](RankState& R) { return cur[ri_of(R)]; }, dist, [&](RankState& R, int part) {
            const int ri = ri_of(R);
            DevLevel& D = R.lv[l];
            const double* b = bvec(R);
            double* xi = cur[ri];
            double* xo = nxt[ri];
            const double n8 = 8.0 * (double)D.comp_n;
            const bool dt = (dot && last);
            const double* dw = (dt && dwv) ? (*dwv)(R) + D.ep_off : nullptr;
            // short rows: m_i recomputed from the streamed row; long rows: read m
            const bool abs = (double)D.A.nnz <= abs_row_cut() * (double)std::max<int64_t>(D.A.nrows, 1);
            const double mb8 = abs ? 0.0 : n8;
            double* m = D.m + D.ep_off;
            auto red = [&]() { return sink_red(h, R, dkind, sink, part); };
            if (s == 0 && s1 == 1) {
                const double* bo = !mbvec ? b + D.ep_off : (*mbvec)(R) + D.ep_off;
                const double* rr = D.r + D.ep_off;
                double* uu = xi + D.ep_off;
                double* xx = xo + D.ep_off;
                if (dt && abs)
                    launch_mat(L, D.A, GVec{xi}, EPost1<true, false, true>{uu, rr, bo, xx, nullptr, dw}, red(),
                               "postsweep_dot", 4 * n8, part);
                else if (dt)
                    launch_mat(L, D.A, GVec{xi}, EPost1<true, false, false>{uu, rr, bo, xx, m, dw}, red(),
                               "postsweep_dot", 5 * n8, part);
                else if (!mbvec && abs)
                    launch_mat(L, D.A, GVec{xi}, EPost1<false, false, true>{uu, rr, bo, xx}, no_red(), "postsweep",
                               4 * n8, part);
                else if (!mbvec)
                    launch_mat(L, D.A, GVec{xi}, EPost1<false, false, false>{uu, rr, bo, xx, m}, no_red(),
                               "postsweep", 5 * n8, part);
                else if (abs)
                    launch_mat(L, D.A, GVec{xi}, EPost1<false, true, true>{uu, rr, bo, xx}, no_red(), "postsweep",
                               4 * n8, part);
                else
                    launch_mat(L, D.A, GVec{xi}, EPost1<false, true, false>{uu, rr, bo, xx, m}, no_red(),
                               "postsweep", 5 * n8, part);
            } else if (dt) {
                if (abs)
                    launch_mat(L, D.A, GVec{xi},
                               ESweep<true, true>{xi + D.ep_off, b + D.ep_off, xo + D.ep_off, nullptr, dw}, red(),
                               "postsweep_dot", 3 * n8, part);
                else
                    launch_mat(L, D.A, GVec{xi}, ESweep<true, false>{xi + D.ep_off, b + D.ep_off, xo + D.ep_off, m, dw},
                               red(), "postsweep_dot", 3 * n8 + mb8, part);
            } else {
                if (abs)
                    launch_mat(L, D.A, GVec{xi}, ESweep<false, true>{xi + D.ep_off, b + D.ep_off, xo + D.ep_off},
                               no_red(), "postsweep", 3 * n8, part);
                else
                    launch_mat(L, D.A, GVec{xi}, ESweep<false, false>{xi + D.ep_off, b + D.ep_off, xo + D.ep_off, m},
                               no_red(), "postsweep", 3 * n8 + mb8, part);
            }
        });
        cur = nxt;
    }
    end_dot(h, L, dot, dkind, sink);
}

// K-cycle coarse correction at level l (oracle kcycle_fcg2): two
// FCG(1) iterations on A_l x = b_l from x = 0, preconditioned by the cycle rooted
// at level l, no residual test.  Single rank.  Scalars live in the level's
// device-side K state {p^T r, p^T q, alpha, beta, stop}; every dot is fused into
// the kernel that produces its operand and reduced deterministically.
// Several ranks (each level distributed or replicated): the same two FCG(1) iterations with
// the halo of p exchanged before each q = A p (overlapped with the interior rows), every dot
// reduced into the rank's local slots and finished into each rank's K state in rank order
// (dot_finish_k), and the inner solution x = x + alpha p formed explicitly (k_kupd2), so the
// consumer (the coarser level's prolongation) gathers, and exchanges, one vector.
void enqueue_fcg2_multi(amg_hier_s* h, Launch& L, int l) {
    const int nsm = h->ctx->nsm;
    const bool dist = !h->ranks[0].lv[l].replicated;
    const VecOf bv = [l](RankState& R) { return R.lv[l].b; };
    const VecOf mbv = [l](RankState& R) { return R.lv[l].mb; };
    const VecOf kp = [l](RankState& R) { return R.lv[l].kp; };
    const VecOf kr = [l](RankState& R) { return R.lv[l].kr; };
    const VecOf kmb = [l](RankState& R) { return R.lv[l].kmb; };
    const VecOf kz = [l](RankState& R) { return R.lv[l].kz; };
    const VecOf kq = [l](RankState& R) { return R.lv[l].kq; };
    auto spmv_alpha = [&]() {  // q = A p, p^T q -> alpha (FIN_KALPHA)
        overlapped(h, L, l, kp, dist, [&](RankState& R, int part) {
            DevLevel& D = R.lv[l];
            launch_mat(L, D.A, GVec{D.kp}, ESpmvDot{D.kp + D.ep_off, D.kq + D.ep_off}, dot_red(h, R, FIN_NONE, 0, part),
                       "kfcg_spmv", 16.0 * (double)D.comp_n, part);
        });
        dot_finish_k(h, L, FIN_KALPHA, l);
    };
    // iteration 1: p = z = B_l b with p^T b fused into the cycle's last step (a new inner solve)
    const DotSink s1{nullptr, FIN_KPR0, nullptr, nullptr, l};
    enqueue_level(h, L, l, bv, &mbv, kp, true, nullptr, &s1);
    spmv_alpha();
    for (auto& R : h->ranks) {  // x = alpha p ; r = b - alpha q ; m o r
        DevLevel& D = R.lv[l];
        const int64_t o = D.ep_off, n = D.comp_n;
        L.begin("kfcg_upd1", 56.0 * (double)n);
        launch_k(k_kupd1, vec_grid(n, nsm), kBlock, L.s, D.kx + o, D.kr + o, D.kmb + o, (const double*)D.kp + o,
                 (const double*)D.kq + o, (const double*)D.b + o, (const double*)D.m + o, n, (const double*)D.kst);
        L.end();
    }
    // iteration 2: z = B_l r with z^T q -> beta ; p = z + beta p, p^T r ; q = A p -> alpha ; x += alpha p
    const DotSink s2{nullptr, FIN_KBETA, nullptr, nullptr, l};
    enqueue_level(h, L, l, kr, &kmb, kz, true, &kq, &s2);
    for (auto& R : h->ranks) {
        DevLevel& D = R.lv[l];
        const int64_t o = D.ep_off, n = D.comp_n;
        L.begin("kfcg_pupd", 32.0 * (double)n);
        launch_k(k_kpupd, vec_grid(n, nsm), kBlock, L.s, D.kp + o, (const double*)D.kz + o, (const double*)D.kr + o,
                 n, (const double*)D.kst, dot_red(h, R, FIN_NONE, 0));
        L.end();
    }
    dot_finish_k(h, L, FIN_KPR, l);
    spmv_alpha();
    for (auto& R : h->ranks) {
        DevLevel& D = R.lv[l];
        const int64_t o = D.ep_off, n = D.comp_n;
        L.begin("kfcg_upd2", 24.0 * (double)n);
        launch_k(k_kupd2, vec_grid(n, nsm), kBlock, L.s, D.kx + o, (const double*)D.kp + o, n, (const double*)D.kst);
        L.end();
    }
}

void enqueue_fcg2(amg_hier_s* h, Launch& L, int l) {
    if (h->multi()) {
        enqueue_fcg2_multi(h, L, l);
        return;
    }
    const int nsm = h->ctx->nsm;
    RankState& R = h->ranks[0];
    DevLevel& D = R.lv[l];
    const int64_t n = D.comp_n;
    const double n8 = 8.0 * (double)n;
    auto kred = [&](int kind) { return RedCtx{R.partials, R.ticket, nullptr, nullptr, 0ull, kind, D.kst}; };
    const VecOf bv = [l](RankState& R) { return R.lv[l].b; };
    const VecOf mbv = [l](RankState& R) { return R.lv[l].mb; };
    const VecOf kp = [l](RankState& R) { return R.lv[l].kp; };
    const VecOf kr = [l](RankState& R) { return R.lv[l].kr; };
    const VecOf kmb = [l](RankState& R) { return R.lv[l].kmb; };
    const VecOf kz = [l](RankState& R) { return R.lv[l].kz; };
    // iteration 1: p = z = B_l b with p^T r (r = b) fused into the cycle's last step
    const DotSink s1{D.kst, FIN_KPR0, nullptr, nullptr, l};
    const bool fused = kcycle_fused(h);
    if (D.AMc && fused) {  // collapsed level: p = B b and q = (A B) b in one kernel
        L.begin("collapsed_kq", 16.0 * (double)n * (double)n + 24.0 * (double)n);
        launch_k(k_collapsed_kq, (int)std::max<int64_t>(1, std::min<int64_t>(n, kMaxPartials)), kBlock, L.s,
                 (const double*)D.Mc, (const double*)D.AMc, n, (const double*)D.b, D.kp, D.kq, kred(FIN_KPR0ALPHA1));
        L.end();
    } else {
        enqueue_level(h, L, l, bv, &mbv, kp, true, nullptr, &s1);
        launch_mat(L, D.A, GVec{D.kp}, ESpmvDot{D.kp, D.kq}, kred(fused ? FIN_KALPHA1 : FIN_KALPHA), "kfcg_spmv",
                   2 * n8);
    }
    if (!fused) {  // x = alpha p ; r = b - alpha q ; m o r (the SWEEP0 path gathers it)
        L.begin("kfcg_upd1", 7 * n8);
        launch_k(k_kupd1, vec_grid(n, nsm), kBlock, L.s, D.kx, D.kr, D.kmb, D.kp, D.kq, D.b, D.m, n,
                 (const double*)D.kst);
        L.end();
    }
    // iteration 2: z = B_l r with z^T q fused -> beta ; p = z + beta p, p^T r ; q = A p, alpha.
    // The final x += alpha p is formed by the consumer (the prolongation gathers x + alpha p).
    // fused: r = b - alpha_1 q_1 is formed (and stored in kr) by the application's first kernel,
    // x = alpha_1 p_1 + alpha_2 p_2 by the consumer (GXap2)
    const DotSink s2{D.kst, FIN_KBETA, fused ? D.b : nullptr, fused ? D.kq : nullptr, l};
    const VecOf kq = [l](RankState& R) { return R.lv[l].kq; };
    if (D.AMc && fused) {  // collapsed level: z = B r1, w = A z = (AB) r1, then p2 / q2 by vectors
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(n, kMaxPartials));
        L.begin("collapsed_kw", 16.0 * (double)n * (double)n + 40.0 * (double)n);
        launch_k(k_collapsed_kw, grid, kBlock, L.s, (const double*)D.Mc, (const double*)D.AMc, n,
                 GBaq{D.b, D.kq, D.kst}, D.kr, D.kz, D.kmb, (const double*)D.kq, kred(FIN_KBETA));
        L.end();
        L.begin("kfcg_pq2", 56.0 * (double)n);
        launch_k(k_kpq2, vec_grid(n, nsm), kBlock, L.s, (const double*)D.kz, (const double*)D.kp, D.kp2,
                 (const double*)D.kmb, D.kq, (const double*)D.kr, n, (const double*)D.kst, kred(FIN_KALPHA2));
        L.end();
        return;
    }
    enqueue_level(h, L, l, kr, &kmb, kz, true, &kq, &s2);
    // p = z + beta p formed inside q = A p (new p into kp2), p^T q and p^T r in one reduction
    launch_mat(L, D.A, GKpz{D.kz, D.kp, D.kst}, EKSpmvPupd{D.kz, D.kp, D.kp2, D.kq, D.kr, D.kst},
               kred(FIN_KALPHA2), "kfcg_spmv_pupd", 5 * n8);
}

// z0 = B b0 on the level-0 windows (the whole cycle).
void enqueue_vcycle(amg_hier_s* h, Launch& L, const VecOf& b0, const VecOf& z0, bool rz,
                    const VecOf* dwv = nullptr) {
    enqueue_level(h, L, 0, b0, nullptr, z0, rz, dwv);
}

// PCG loop body, rotated so that the convergence test is the last node:
//   z = V(r), rho' = r^T z, beta ; p = z + beta p ; q = A p, alpha ; x, r update, test.
//
// FCG(1) (cfg.krylov == 1) uses the same rotation:
//   z = V(r), beta = -(z^T q)/(p^T q)_prev ; p = z + beta p, p^T r ;
//   q = A p, alpha = p^T r / p^T q ; x, r update, test.
void enqueue_pcg_body(amg_hier_s* h, Launch& L, double* x_user, unsigned long long cond) {
    const int nsm = h->ctx->nsm;
    const bool fcg = h->cfg.krylov == 1;
    const VecOf qv = [](RankState& R) { return R.pq; };
    enqueue_vcycle(h, L, [](RankState& R) { return R.pr; }, [](RankState& R) { return R.pz; }, true,
                   fcg ? &qv : nullptr);
    if (!fcg && h->nlev() > 1) {
        // p = z + beta p fused into q = A p (p double-buffered, selected on the device).  (The
        // FCG variant, reducing p^T r there as well, measured 1 % slower: its SDIA/SELL kernels
        // spill under the 32-register bound, so FCG keeps k_pupdate_fcg.)  Several ranks: the
        // halo of z is exchanged and its unpack also forms p_new = z + beta p_old at the halo
        // positions (p_old's halo arrived with the previous iteration's z), so the gathers see
        // the same p_new as the owners write.
        const UnpackFn pz_unpack = [&](RankState& R, const Exch& E, cudaStream_t s) {
            launch_k(k_unpack_pz, vec_grid(E.nrecv, nsm), kBlock, s, R.pz, R.pp, R.pp2, (const int32_t*)E.recv_idx,
                     (const double*)E.rbuf, E.nrecv, (const PcgState*)R.st, E.rx);
        };
        overlapped(h, L, 0, [](RankState& R) { return R.pz; }, true, [&](RankState& R, int part) {
            const DevLevel& D = R.L0();
            const int64_t o = D.own_off;
            launch_mat(L, D.A, GPz{R.pz, R.pp, R.pp2, R.st},
                       ESpmvDotPz{R.pz + o, R.pp + o, R.pp2 + o, R.pq + o, x_user + R.user_off, R.st},
                       dot_red(h, R, FIN_PQ, 0, part), "spmv_dot_pupd", 48.0 * D.own_n, part);
        }, &pz_unpack);
        dot_finish(h, L, FIN_PQ);
    } else {  // FCG or one level: separate direction update, halo of p, q = A p
        for (auto& R : h->ranks) {
            const DevLevel& D = R.L0();
            if (fcg) {
                L.begin("pupdate_fcg", 48.0 * D.own_n);
                launch_k(k_pupdate_fcg, vec_grid(D.own_n, nsm), kBlock, L.s, R.pz + D.own_off, R.pp + D.own_off,
                         x_user + R.user_off, R.pr + D.own_off, D.own_n, R.st, dot_red(h, R, FIN_PR, 0));
            } else {
                L.begin("pupdate", 40.0 * D.own_n);
                launch_k(k_pupdate, vec_grid(D.own_n, nsm), kBlock, L.s, R.pz + D.own_off, R.pp + D.own_off,
                         x_user + R.user_off, D.own_n, R.st);
            }
            L.end();
        }
        if (fcg) dot_finish(h, L, FIN_PR);
        const int pqk = fcg ? FIN_PQF : FIN_PQ;
        overlapped(h, L, 0, [](RankState& R) { return R.pp; }, true, [&](RankState& R, int part) {
            const DevLevel& D = R.L0();
            launch_mat(L, D.A, GVec{R.pp}, ESpmvDot{R.pp + D.own_off, R.pq + D.own_off}, dot_red(h, R, pqk, 0, part),
                       "spmv_dot", 16.0 * D.own_n, part);
        });
        dot_finish(h, L, pqk);
    }
    for (auto& R : h->ranks) {
        const DevLevel& D = R.L0();
        L.begin("axpy_rr", 24.0 * D.own_n);
        launch_k(k_axpy_rr, vec_grid(D.own_n, nsm), kBlock, L.s, R.pr + D.own_off, R.pq + D.own_off, D.own_n, R.st,
                 dot_red(h, R, FIN_RR, cond));
        L.end();
    }
    dot_finish(h, L, FIN_RR, cond);
}

void enqueue_pcg_final(amg_hier_s* h, Launch& L, double* x_user) {
    for (auto& R : h->ranks) {
        const DevLevel& D = R.L0();
        L.begin("xfinal", 24.0 * D.own_n);
        const bool fused = h->cfg.krylov != 1 && h->nlev() > 1;
        launch_k(k_xfinal, vec_grid(D.own_n, h->ctx->nsm), kBlock, L.s, x_user + R.user_off,
                 (const double*)(R.pp + D.own_off), fused ? (const double*)(R.pp2 + D.own_off) : (const double*)nullptr,
                 D.own_n, (const PcgState*)R.st);
        L.end();
    }
}

void enqueue_pcg_init(amg_hier_s* h, Launch& L, const double* b_user, double* x_user, unsigned long long cond) {
    for (auto& R : h->ranks) {
        const DevLevel& D = R.L0();
        L.begin("pcg_init", 24.0 * D.own_n);
        launch_k(k_pcg_init, vec_grid(D.own_n, h->ctx->nsm), kBlock, L.s, b_user + R.user_off, R.pr + D.own_off,
                                                                        x_user + R.user_off, D.own_n,
                                                                        dot_red(h, R, FIN_BNORM, cond));
        L.end();
    }
    dot_finish(h, L, FIN_BNORM, cond);
}

// ------------------------------------------------------------- upload
template <class T>
int dev_copy(T** dst, const T* src, size_t count) {
    CK(cudaMalloc((void**)dst, std::max<size_t>(1, count) * sizeof(T)));
    if (count) CK(h2d_sync(*dst, src, count * sizeof(T)));
    return AMG_OK;
}

template <class T>
int dev_alloc(T** dst, size_t count) {
    CK(cudaMalloc((void**)dst, std::max<size_t>(1, count) * sizeof(T)));
    CK(memset_sync(*dst, 0, std::max<size_t>(1, count) * sizeof(T)));
    return AMG_OK;
}

// Per-operator storage choice (north_star (1): "CSR/sliced-ELL storage chosen per
// level"): SDIA-32 for stencil-like square operators whose slices share few column
// offsets, SELL-32 for short rows with little padding, CSR-vector (VW lanes per
// row, or one block per row) otherwise.  `shift` maps local rows to the column
// window frame (comp_begin - win_begin); `square` marks A_l.
// Largest contiguous run of interior units (flag[u] = 1) -> [b0, b1)
void interior_run(const std::vector<char>& flag, int64_t& b0, int64_t& b1) {
    b0 = b1 = 0;
    int64_t s = -1;
    for (int64_t u = 0; u <= (int64_t)flag.size(); ++u) {
        const bool in = u < (int64_t)flag.size() && flag[u];
        if (in && s < 0) s = u;
        if (!in && s >= 0) {
            if (u - s > b1 - b0) {
                b0 = s;
                b1 = u;
            }
            s = -1;
        }
    }
}

// own_lo/own_hi: columns (window frame) owned by this rank for the gathered vector;
// own_lo < 0: no split (single rank, replicated levels)
// ------------------------------------------------------------- 16-bit columns
// A SELL / CSR operator whose rows each span fewer than 2^16 columns stores col - cbase as
// uint16 (cbase = the row's smallest column; per slot for SELL, per row for CSR): 10 instead of
// 12 bytes per entry on the deep aggregation levels (c4 A_2 / A_3: 168 / 735 entries per row,
// spans <= 33k).  Same entries, same order: results bitwise equal.  Off with AMG_NO_C16=1, and
// for levels of the persistent tail (its TailOp reads 32-bit columns).
thread_local bool g_c16_allowed = true;
struct C16Scope {
    bool saved;
    explicit C16Scope(bool allow) : saved(g_c16_allowed) {
        const char* e = std::getenv("AMG_NO_C16");
        g_c16_allowed = allow && !(e && e[0] == '1');
    }
    ~C16Scope() { g_c16_allowed = saved; }
};
// per unit (SELL slot / CSR row): smallest column -> base, largest span -> atomicMax(*span)
__global__ void kc_c16_span(const uint32_t* __restrict__ sptr, const int32_t* __restrict__ rp,
                            const int32_t* __restrict__ col, int64_t nunits, int32_t* base, int* span) {
    int mx = 0;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nunits; q += (int64_t)gridDim.x * blockDim.x) {
        int64_t k0, k1, stride;
        if (sptr) {
            k0 = (int64_t)sptr[q >> 5] * 32 + (q & 31);
            k1 = (int64_t)sptr[(q >> 5) + 1] * 32 + (q & 31);
            stride = 32;
        } else {
            k0 = rp[q];
            k1 = rp[q + 1];
            stride = 1;
        }
        int32_t lo = INT32_MAX, hi = INT32_MIN;
        for (int64_t k = k0; k < k1; k += stride) {
            lo = min(lo, col[k]);
            hi = max(hi, col[k]);
        }
        if (k1 <= k0) lo = hi = 0;
        base[q] = lo;
        mx = max(mx, hi - lo);
    }
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) atomicMax(span, mx);
}
__global__ void kc_c16_fill(const uint32_t* __restrict__ sptr, const int32_t* __restrict__ rp,
                            const int32_t* __restrict__ col, int64_t nunits, const int32_t* __restrict__ base,
                            uint16_t* c16) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nunits; q += (int64_t)gridDim.x * blockDim.x) {
        int64_t k0, k1, stride;
        if (sptr) {
            k0 = (int64_t)sptr[q >> 5] * 32 + (q & 31);
            k1 = (int64_t)sptr[(q >> 5) + 1] * 32 + (q & 31);
            stride = 32;
        } else {
            k0 = rp[q];
            k1 = rp[q + 1];
            stride = 1;
        }
        for (int64_t k = k0; k < k1; k += stride) c16[k] = (uint16_t)(col[k] - base[q]);
    }
}
// SELL / CSR-vector operator with 32-bit columns -> 16-bit columns when every unit's span fits
// (and rows are long enough, >= 4 entries on average, for the 4 B per-row base to pay)
int compress_cols(DevMat& D, cudaStream_t s) {
    static const double min_mean = [] {  // AMG_C16_MIN_MEAN: an A/B knob (default 4 entries per row)
        const char* e = std::getenv("AMG_C16_MIN_MEAN");
        return e ? std::atof(e) : 4.0;
    }();
    if (!g_c16_allowed || !D.col || (D.fmt != FMT_SELL && D.fmt != FMT_CSRV) || D.nrows <= 0 ||
        (double)D.nnz < min_mean * (double)D.nrows)
        return AMG_OK;
    const bool sell = D.fmt == FMT_SELL;
    const int64_t nunits = sell ? D.units * 32 : D.nrows;
    const int64_t ncol = sell ? D.stored : D.nnz;
    int32_t* base = nullptr;
    int* dspan = nullptr;
    int st;
    if ((st = dev_alloc(&base, (size_t)nunits))) return st;
    if ((st = dev_alloc(&dspan, 1))) {
        cudaFree(base);
        return st;
    }
    const int gs = (int)std::max<int64_t>(1, std::min<int64_t>((nunits + 255) / 256, 148 * 16));
    CK(cudaMemsetAsync(dspan, 0, sizeof(int), s));
    kc_c16_span<<<gs, 256, 0, s>>>(sell ? D.sptr : nullptr, D.rp, D.col, nunits, base, dspan);
    int span = 0;
    CK(cudaMemcpyAsync(&span, dspan, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    cudaFree(dspan);
    if (span >= 65536) {
        cudaFree(base);
        return AMG_OK;
    }
    uint16_t* c16 = nullptr;
    if ((st = dev_alloc(&c16, (size_t)std::max<int64_t>(1, ncol)))) {
        cudaFree(base);
        return st;
    }
    kc_c16_fill<<<gs, 256, 0, s>>>(sell ? D.sptr : nullptr, D.rp, D.col, nunits, base, c16);
    CK(cudaStreamSynchronize(s));
    cudaFree(D.col);
    D.col = nullptr;
    D.c16 = c16;
    D.cbase = base;
    return AMG_OK;
}

int upload_mat_fmt(const amgsetup::Csr& M, DevMat& D, bool square, int64_t shift, bool force_csr,
                   int64_t own_lo, int64_t own_hi) {
    const int64_t n = M.nrows, nnz = M.nnz();
    D.nrows = n;
    D.ncols = M.ncols;
    D.nnz = nnz;
    D.shift = (int32_t)shift;
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
    // SDIA-32 candidate: per slice, the sorted distinct offsets col - base(row), with
    // base = row + shift for A_l and base = the row's first column (stored per row,
    // "anchor") for the rectangular P-bar_l / R_l
    if (!force_csr && nsl >= 148 * 16 && mean <= 64.0) {
        std::vector<int32_t> anc;
        if (!square) {
            anc.resize(n);
            for (int64_t r = 0; r < n; ++r) anc[r] = M.rp[r + 1] > M.rp[r] ? M.ci[M.rp[r]] : 0;
        }
        auto base = [&](int64_t r) -> int64_t { return square ? r + shift : (int64_t)anc[r]; };
        std::vector<uint32_t> dw(nsl, 0);
        std::vector<std::vector<int32_t>> soffs(nsl);
#pragma omp parallel for schedule(static)
        for (int64_t s = 0; s < nsl; ++s) {
            auto& o = soffs[s];
            for (int64_t r = s * 32; r < std::min(n, s * 32 + 32); ++r)
                for (int64_t t = M.rp[r]; t < M.rp[r + 1]; ++t) o.push_back((int32_t)((int64_t)M.ci[t] - base(r)));
            std::sort(o.begin(), o.end());
            o.erase(std::unique(o.begin(), o.end()), o.end());
            dw[s] = (uint32_t)o.size();
        }
        int64_t dpad = 0;
        for (int64_t s = 0; s < nsl; ++s) dpad += 32 * (int64_t)dw[s];
        const double sdia_bytes = 8.0 * (double)dpad + 4.0 * (double)dpad / 32.0 + (square ? 0.0 : 4.0 * (double)n);
        const double sell_bytes = 12.0 * (double)padded;
        const bool ok = square ? (double)dpad <= 1.02 * (double)padded + 64.0 : sdia_bytes <= 0.9 * sell_bytes;
        if (ok && dpad / 32 < (int64_t)UINT32_MAX) {
            D.fmt = FMT_SDIA;
            D.stored = dpad;
            if (!square) {
                int st;
                if ((st = dev_copy(&D.anchor, anc.data(), anc.size()))) return st;
            }
            std::vector<uint32_t> sptr(nsl + 1, 0);
            for (int64_t s = 0; s < nsl; ++s) sptr[s + 1] = sptr[s] + dw[s];
            std::vector<int32_t> offs(dpad / 32);
            std::vector<double> val(dpad, 0.0);
#pragma omp parallel for schedule(static)
            for (int64_t s = 0; s < nsl; ++s) {
                const auto& o = soffs[s];
                std::copy(o.begin(), o.end(), offs.begin() + sptr[s]);
                const int64_t vbase = (int64_t)sptr[s] * 32;
                for (int64_t r = s * 32; r < std::min(n, s * 32 + 32); ++r) {
                    const int64_t lane = r - s * 32;
                    size_t k = 0;
                    for (int64_t t = M.rp[r]; t < M.rp[r + 1]; ++t) {
                        const int32_t d = (int32_t)((int64_t)M.ci[t] - base(r));
                        while (o[k] != d) ++k;  // both ascending
                        val[vbase + (int64_t)k * 32 + lane] = M.v[t];
                    }
                }
            }
            D.units = nsl;
            if (own_lo >= 0) {  // a slice is interior when every lane's gathers (all slice offsets) are owned
                std::vector<char> fl(nsl, 0);
#pragma omp parallel for schedule(static)
                for (int64_t s2 = 0; s2 < nsl; ++s2) {
                    bool ok2 = true;
                    for (int64_t r = s2 * 32; ok2 && r < std::min(n, s2 * 32 + 32); ++r)
                        for (uint32_t k = sptr[s2]; ok2 && k < sptr[s2 + 1]; ++k) {
                            const int64_t c = std::min<int64_t>(std::max<int64_t>(base(r) + offs[k], 0), M.ncols - 1);
                            ok2 = (c >= own_lo && c < own_hi);
                        }
                    fl[s2] = ok2;
                }
                interior_run(fl, D.ib0, D.ib1);
            }
            int st;
            if ((st = dev_copy(&D.sptr, sptr.data(), sptr.size()))) return st;
            if ((st = dev_copy(&D.offs, offs.data(), offs.size()))) return st;
            if ((st = dev_copy(&D.val, val.data(), val.size()))) return st;
            return AMG_OK;
        }
    }
    // CSR rows (SELL pads with the row's own last column): row interior when all columns owned
    std::vector<char> rowin;
    if (own_lo >= 0) {
        rowin.assign(n, 0);
#pragma omp parallel for schedule(static)
        for (int64_t r = 0; r < n; ++r) {
            bool ok2 = true;
            for (int64_t k = M.rp[r]; ok2 && k < M.rp[r + 1]; ++k) ok2 = (M.ci[k] >= own_lo && M.ci[k] < own_hi);
            rowin[r] = ok2;
        }
    }
    // SELL-32 (one thread per row, coalesced column-major slices) needs little padding and
    // enough slices to fill the GPU (>= ~16 warps per SM)
    const bool sell = !force_csr && (double)padded <= 1.10 * (double)nnz + 64.0 && nsl >= 148 * 16 &&
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
                int32_t last = 0;
                for (int64_t t = M.rp[r]; t < M.rp[r + 1]; ++t, ++k) {
                    col[base + k * 32 + lane] = last = M.ci[t];
                    val[base + k * 32 + lane] = M.v[t];
                }
                for (; k < width[s]; ++k) col[base + k * 32 + lane] = last;
            }
        }
        D.units = nsl;
        if (own_lo >= 0) {
            std::vector<char> fl(nsl, 1);
            for (int64_t r = 0; r < n; ++r)
                if (!rowin[r]) fl[r / 32] = 0;
            interior_run(fl, D.ib0, D.ib1);
        }
        int st;
        if ((st = dev_copy(&D.sptr, sptr.data(), sptr.size()))) return st;
        if ((st = dev_copy(&D.col, col.data(), col.size()))) return st;
        if ((st = dev_copy(&D.val, val.data(), val.size()))) return st;
        return AMG_OK;
    }
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
    // block per row: few long rows, or rows long enough (>= 1024) to give every thread of a block
    // several entries (c5 A_3 at 256^3: 34k rows x 2,695 -> 5.6 vs 4.5 TB/s in spmv_lab3)
    if ((mean >= 256.0 && (double)n < 18944.0) || mean >= 1024.0) vw = kVWBlock;
    D.vw = vw;
    D.units = n;
    if (own_lo >= 0) interior_run(rowin, D.ib0, D.ib1);
    std::vector<int32_t> rp(n + 1);
    for (int64_t i = 0; i <= n; ++i) rp[i] = (int32_t)M.rp[i];
    int st;
    if ((st = dev_copy(&D.rp, rp.data(), rp.size()))) return st;
    if ((st = dev_copy(&D.col, M.ci.data(), M.ci.size()))) return st;
    if ((st = dev_copy(&D.val, M.v.data(), M.v.size()))) return st;
    return AMG_OK;
}
int upload_mat(const amgsetup::Csr& M, DevMat& D, bool square, int64_t shift, bool force_csr = false,
               int64_t own_lo = -1, int64_t own_hi = -1) {
    int st = upload_mat_fmt(M, D, square, shift, force_csr, own_lo, own_hi);
    return st ? st : compress_cols(D, 0);
}


// ------------------------------------------------------------- device-side formats
// Same decisions and layouts as upload_mat, computed on the device from a device CSR
// (GPU-built hierarchies never leave the device: NEXT-1).
__global__ void kc_slice_width(const int64_t* __restrict__ rp, int64_t n, int64_t nsl, uint32_t* width) {
    for (int64_t sl = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; sl < nsl; sl += (int64_t)gridDim.x * blockDim.x) {
        int64_t w = 0;
        for (int64_t r = sl * 32; r < min(n, sl * 32 + 32); ++r) w = max(w, rp[r + 1] - rp[r]);
        width[sl] = (uint32_t)w;
    }
}
// warp per slice: the sorted union of the 32 rows' offsets col - base(row) by repeated
// warp minima (rows are sorted, so each lane walks its row once); count or fill
__global__ void kc_slice_offs(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                              const double* __restrict__ v, int64_t n, int64_t nsl, int square, int64_t shift,
                              uint32_t* dw, const uint32_t* __restrict__ sptr, int32_t* offs, double* val) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t sl = w0; sl < nsl; sl += nw) {
        const int64_t r = sl * 32 + lane;
        int64_t p = 0, e = 0;
        if (r < n) {
            p = rp[r];
            e = rp[r + 1];
        }
        const int64_t base = square ? r + shift : (p < e ? (int64_t)ci[p] : 0);
        uint32_t k = 0;
        const uint32_t b0 = sptr ? sptr[sl] : 0u;
        for (;;) {
            const int64_t cur = (p < e) ? (int64_t)ci[p] - base : INT64_MAX;
            int64_t mn = cur;
            for (int o = 16; o > 0; o >>= 1) mn = min(mn, (int64_t)__shfl_xor_sync(0xffffffffu, mn, o));
            if (mn == INT64_MAX) break;
            if (sptr) {
                if (lane == 0) offs[b0 + k] = (int32_t)mn;
                val[(int64_t)(b0 + k) * 32 + lane] = (cur == mn) ? v[p] : 0.0;
            }
            if (cur == mn) ++p;
            ++k;
        }
        if (!sptr && lane == 0) dw[sl] = k;
    }
}
__global__ void kc_anchor(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci, int64_t n, int32_t* anc) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
        anc[r] = rp[r + 1] > rp[r] ? ci[rp[r]] : 0;
}
__global__ void kc_sell_fill(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                             const double* __restrict__ v, int64_t n, const uint32_t* __restrict__ sptr,
                             const uint32_t* __restrict__ width, int32_t* col, double* val) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t sl = r >> 5, lane = r & 31;
        const int64_t base = (int64_t)sptr[sl] * 32;
        int64_t k = 0;
        int32_t last = 0;
        for (int64_t t = rp[r]; t < rp[r + 1]; ++t, ++k) {
            col[base + k * 32 + lane] = last = ci[t];
            val[base + k * 32 + lane] = v[t];
        }
        for (; k < (int64_t)width[sl]; ++k) col[base + k * 32 + lane] = last;
    }
}
// SELL-32-sigma: inside each window of kSigma rows, rows ordered by length
// descending (ties by row index); one block per window, rank by counting
constexpr int kSigma = 256;
__global__ void __launch_bounds__(kSigma) kc_sigma_perm(const int64_t* __restrict__ rp, int64_t n, int32_t* perm) {
    __shared__ int64_t len[kSigma];
    const int64_t w0 = (int64_t)blockIdx.x * kSigma;
    const int t = threadIdx.x;
    const int64_t r = w0 + t;
    len[t] = (r < n) ? rp[r + 1] - rp[r] : -1;  // padding slots sort last
    __syncthreads();
    const int64_t li = len[t];
    int rank = 0;
    for (int j = 0; j < kSigma; ++j) {
        const int64_t lj = len[j];
        rank += (lj > li || (lj == li && j < t)) ? 1 : 0;
    }
    perm[w0 + rank] = (r < n) ? (int32_t)r : -1;
}
__global__ void kc_slice_width_perm(const int64_t* __restrict__ rp, const int32_t* __restrict__ perm, int64_t nsl,
                                    uint32_t* width) {
    for (int64_t sl = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; sl < nsl; sl += (int64_t)gridDim.x * blockDim.x) {
        int64_t w = 0;
        for (int l = 0; l < 32; ++l) {
            const int32_t r = perm[sl * 32 + l];
            if (r >= 0) w = max(w, rp[r + 1] - rp[r]);
        }
        width[sl] = (uint32_t)w;
    }
}
// slot-major fill (thread per slot); padding entries repeat the row's last column, value 0
__global__ void kc_sell_fill_perm(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                  const double* __restrict__ v, const int32_t* __restrict__ perm, int64_t nslots,
                                  const uint32_t* __restrict__ sptr, const uint32_t* __restrict__ width, int32_t* col,
                                  double* val) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nslots; q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t sl = q >> 5, lane = q & 31;
        const int64_t base = (int64_t)sptr[sl] * 32;
        const int32_t r = perm[q];
        int64_t k = 0;
        int32_t last = 0;
        if (r >= 0)
            for (int64_t t = rp[r]; t < rp[r + 1]; ++t, ++k) {
                col[base + k * 32 + lane] = last = ci[t];
                val[base + k * 32 + lane] = v[t];
            }
        for (; k < (int64_t)width[sl]; ++k) col[base + k * 32 + lane] = last;
    }
}
__global__ void kc_rp32(const int64_t* __restrict__ rp, int64_t n, int32_t* out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (int32_t)rp[i];
}
__global__ void kc_scale_cols(const int32_t* __restrict__ ci, const double* __restrict__ v, int64_t nnz,
                              const double* __restrict__ m, double* out) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x)
        out[k] = v[k] * m[ci[k]];
}

static double sigma_mean_max() {  // AMG_SIGMA_MEAN_MAX: experiment knob (default 128)
    const char* e = std::getenv("AMG_SIGMA_MEAN_MAX");
    return e ? std::atof(e) : 128.0;
}

int convert_mat_fmt(const amgsetup::DevCsrRaw& M, DevMat& D, bool square, int64_t shift, bool force_csr, cudaStream_t s) {
    const int64_t n = M.nrows, nnz = M.nnz;
    D.nrows = n;
    D.ncols = M.ncols;
    D.nnz = nnz;
    D.shift = (int32_t)shift;
    const int64_t nsl = (n + 31) / 32;
    const int gs = (int)std::max<int64_t>(1, std::min<int64_t>((nsl * 32 + 255) / 256, 148 * 16));
    uint32_t* dwidth = nullptr;
    int st;
    if ((st = dev_alloc(&dwidth, (size_t)nsl))) return st;
    kc_slice_width<<<gs, 256, 0, s>>>(M.rp, n, nsl, dwidth);
    std::vector<uint32_t> width(nsl);
    CK(cudaMemcpyAsync(width.data(), dwidth, nsl * 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    int64_t padded = 0;
    for (int64_t q = 0; q < nsl; ++q) padded += 32 * (int64_t)width[q];
    const double mean = n ? (double)nnz / (double)n : 0.0;
    if (!force_csr && nsl >= 148 * 16 && mean <= 64.0) {
        uint32_t* ddw = nullptr;
        if ((st = dev_alloc(&ddw, (size_t)nsl))) return st;
        kc_slice_offs<<<gs, 256, 0, s>>>(M.rp, M.ci, M.v, n, nsl, square ? 1 : 0, shift, ddw, nullptr, nullptr,
                                         nullptr);
        std::vector<uint32_t> dw(nsl);
        CK(cudaMemcpyAsync(dw.data(), ddw, nsl * 4, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        cudaFree(ddw);
        int64_t dpad = 0;
        for (int64_t q = 0; q < nsl; ++q) dpad += 32 * (int64_t)dw[q];
        const double sdia_bytes = 8.0 * (double)dpad + 4.0 * (double)dpad / 32.0 + (square ? 0.0 : 4.0 * (double)n);
        const double sell_bytes = 12.0 * (double)padded;
        const bool ok = square ? (double)dpad <= 1.02 * (double)padded + 64.0 : sdia_bytes <= 0.9 * sell_bytes;
        if (ok && dpad / 32 < (int64_t)UINT32_MAX) {
            D.fmt = FMT_SDIA;
            D.stored = dpad;
            std::vector<uint32_t> sptr(nsl + 1, 0);
            for (int64_t q = 0; q < nsl; ++q) sptr[q + 1] = sptr[q] + dw[q];
            if ((st = dev_copy(&D.sptr, sptr.data(), sptr.size()))) return st;
            CK(cudaMalloc((void**)&D.offs, std::max<int64_t>(1, dpad / 32) * 4));
            CK(cudaMalloc((void**)&D.val, std::max<int64_t>(1, dpad) * 8));
            kc_slice_offs<<<gs, 256, 0, s>>>(M.rp, M.ci, M.v, n, nsl, square ? 1 : 0, shift, nullptr, D.sptr, D.offs,
                                             D.val);
            if (!square) {
                CK(cudaMalloc((void**)&D.anchor, std::max<int64_t>(1, n) * 4));
                kc_anchor<<<gs, 256, 0, s>>>(M.rp, M.ci, n, D.anchor);
            }
            CK(cudaStreamSynchronize(s));
            cudaFree(dwidth);
            D.units = nsl;
            return AMG_OK;
        }
    }
    const bool sell = !force_csr && (double)padded <= 1.10 * (double)nnz + 64.0 && nsl >= 148 * 16 &&
                      padded / 32 < (int64_t)UINT32_MAX;
    if (sell) {
        D.fmt = FMT_SELL;
        D.stored = padded;
        std::vector<uint32_t> sptr(nsl + 1, 0);
        for (int64_t q = 0; q < nsl; ++q) sptr[q + 1] = sptr[q] + width[q];
        if ((st = dev_copy(&D.sptr, sptr.data(), sptr.size()))) return st;
        if ((st = dev_alloc(&D.col, (size_t)std::max<int64_t>(1, padded)))) return st;
        if ((st = dev_alloc(&D.val, (size_t)std::max<int64_t>(1, padded)))) return st;
        kc_sell_fill<<<gs, 256, 0, s>>>(M.rp, M.ci, M.v, n, D.sptr, dwidth, D.col, D.val);
        CK(cudaStreamSynchronize(s));
        cudaFree(dwidth);
        D.units = nsl;
        return AMG_OK;
    }
    // SELL-32-sigma: rows sorted by length inside windows of kSigma rows cut the padding of
    // ragged operators (irregular aggregates: P-bar / R of the 27-point jump problem, its
    // coarse A_l); the slot -> row map costs 4 B per row.  Used when it stores at most
    // 1.10 x nnz and the rows fit int32, for rows of <= 128 entries on average and enough
    // of them to fill the GPU with one thread per row (>= 148 x 2048): few long rows on one
    // thread each (A_2 of the 27-point problem: 114k rows of 600 entries) serialise, and
    // CSR-vector is faster there.  c5 analogue 192^3: 56.9 -> 53.9 ms; 256^3: 119.8 -> 115.5.
    if (!force_csr && n >= 148 * 2048 && mean <= sigma_mean_max() && n < (int64_t)INT32_MAX) {
        const int64_t nwin = (n + kSigma - 1) / kSigma;
        const int64_t nslots = nwin * kSigma;
        const int64_t nslp = nslots / 32;
        int32_t* perm = nullptr;
        uint32_t* pw = nullptr;
        if ((st = dev_alloc(&perm, (size_t)nslots))) return st;
        if ((st = dev_alloc(&pw, (size_t)nslp))) return st;
        kc_sigma_perm<<<(unsigned)nwin, kSigma, 0, s>>>(M.rp, n, perm);
        kc_slice_width_perm<<<gs, 256, 0, s>>>(M.rp, perm, nslp, pw);
        std::vector<uint32_t> pwidth(nslp);
        CK(cudaMemcpyAsync(pwidth.data(), pw, nslp * 4, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        int64_t ppad = 0;
        for (int64_t q = 0; q < nslp; ++q) ppad += 32 * (int64_t)pwidth[q];
        if ((double)ppad <= 1.10 * (double)nnz + 64.0 && ppad / 32 < (int64_t)UINT32_MAX) {
            D.fmt = FMT_SELL;
            D.stored = ppad;
            D.perm = perm;
            std::vector<uint32_t> sptr(nslp + 1, 0);
            for (int64_t q = 0; q < nslp; ++q) sptr[q + 1] = sptr[q] + pwidth[q];
            if ((st = dev_copy(&D.sptr, sptr.data(), sptr.size()))) return st;
            if ((st = dev_alloc(&D.col, (size_t)std::max<int64_t>(1, ppad)))) return st;
            if ((st = dev_alloc(&D.val, (size_t)std::max<int64_t>(1, ppad)))) return st;
            kc_sell_fill_perm<<<gs, 256, 0, s>>>(M.rp, M.ci, M.v, perm, nslots, D.sptr, pw, D.col, D.val);
            CK(cudaStreamSynchronize(s));
            cudaFree(pw);
            cudaFree(dwidth);
            D.units = nslp;
            return AMG_OK;
        }
        cudaFree(perm);
        cudaFree(pw);
    }
    cudaFree(dwidth);
    if (nnz >= (int64_t)INT32_MAX) {
        set_err("operator too large for 32-bit CSR row pointers on one rank");
        return AMG_ERR_ARG;
    }
    D.fmt = FMT_CSRV;
    D.stored = nnz;
    const double want = 148.0 * 2048.0 / (double)std::max<int64_t>(n, 1);
    int vw = 2;
    while (vw < 32 && (vw < want || vw * 8 < mean) && vw * 2 <= std::max(2.0, mean)) vw *= 2;
    // block per row: few long rows, or rows long enough (>= 1024) to give every thread of a block
    // several entries (c5 A_3 at 256^3: 34k rows x 2,695 -> 5.6 vs 4.5 TB/s in spmv_lab3)
    if ((mean >= 256.0 && (double)n < 18944.0) || mean >= 1024.0) vw = kVWBlock;
    D.vw = vw;
    D.units = n;
    CK(cudaMalloc((void**)&D.rp, (n + 1) * 4));
    kc_rp32<<<gs, 256, 0, s>>>(M.rp, n, D.rp);
    CK(cudaMalloc((void**)&D.col, std::max<int64_t>(1, nnz) * 4));
    CK(cudaMalloc((void**)&D.val, std::max<int64_t>(1, nnz) * 8));
    if (nnz) {
        CK(cudaMemcpyAsync(D.col, M.ci, nnz * 4, cudaMemcpyDeviceToDevice, s));
        CK(cudaMemcpyAsync(D.val, M.v, nnz * 8, cudaMemcpyDeviceToDevice, s));
    }
    CK(cudaStreamSynchronize(s));
    return AMG_OK;
}
int convert_mat(const amgsetup::DevCsrRaw& M, DevMat& D, bool square, int64_t shift, bool force_csr, cudaStream_t s) {
    int st = convert_mat_fmt(M, D, square, shift, force_csr, s);
    return st ? st : compress_cols(D, s);
}

// Coarse CG (cfg.coarse_solver == 1): CSR of the replicated A_L, its l1 diagonal,
// and the cluster shape of k_coarse_cg.  CTAs: enough that each holds <= ~16k
// entries (the SpMV is spread over 16 warps per CTA), more if the CTA's rows of
// A_L do not fit in shared memory, at most 16 (non-portable cluster size), and
// no more than the device can co-schedule as one cluster.
int upload_coarse_cg(amg_hier_s* h, const amgsetup::RankLevel& C, RankState& R) {
    const amgsetup::Csr& A = C.A;
    const int64_t n = A.nrows, nnz = A.nnz();
    const bool invk = h->cfg.coarse_prec == 1;
    if (invk && (C.Wd.nrows != n || C.Z.nrows != n || C.Wd.nnz() >= (int64_t)INT32_MAX ||
                 C.Z.nnz() >= (int64_t)INT32_MAX)) {
        set_err("coarse CG: the INVK factors of the coarsest matrix are missing or too large");
        return AMG_ERR_ARG;
    }
    if (n > 16384 || nnz >= (int64_t)INT32_MAX) {
        set_err("coarse CG: the coarsest matrix is too large (n_L <= 16384 required)");
        return AMG_ERR_ARG;
    }
    // function attributes are per device: set on every build (cheap, thread-safe)
    CK(cudaFuncSetAttribute(k_coarse_cg, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    CK(cudaFuncSetAttribute(k_coarse_cg, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    const size_t budget = 200 * 1024;
    auto plan = [&](int ncta, std::vector<int32_t>& split, size_t& smem_base, size_t& smem_a) {
        split.assign(ncta + 1, 0);
        for (int c = 1; c < ncta; ++c) {
            const int64_t target = nnz * c / ncta;
            const int64_t r = std::lower_bound(A.rp.begin(), A.rp.end(), target) - A.rp.begin();
            split[c] = (int32_t)std::max<int64_t>(split[c - 1] + 1, std::min<int64_t>(r, n - (ncta - c)));
        }
        split[ncta] = (int32_t)n;
        int64_t own = 0, ann = 0;
        for (int c = 0; c < ncta; ++c) {
            own = std::max<int64_t>(own, split[c + 1] - split[c]);
            ann = std::max<int64_t>(ann, A.rp[split[c + 1]] - A.rp[split[c]]);
        }
        smem_base = 8 * (size_t)n * (invk ? 3 : 1) + 32 * (size_t)own;
        smem_a = 12 * (size_t)ann;
    };
    int ncta = (int)std::min<int64_t>(16, std::max<int64_t>(1, (nnz + 16383) / 16384));
    ncta = (int)std::min<int64_t>(ncta, n);
    std::vector<int32_t> split;
    size_t base = 0, sa = 0;
    plan(ncta, split, base, sa);
    while (base + sa > budget && ncta < 16 && ncta < n) plan(++ncta, split, base, sa);
    for (;;) {  // the cluster must be co-schedulable
        if (ncta == 1) break;
        cudaLaunchConfig_t lc = {};
        lc.gridDim = dim3((unsigned)ncta);
        lc.blockDim = dim3((unsigned)kCgBlock);
        lc.dynamicSmemBytes = base + (base + sa <= budget ? sa : 0);
        cudaLaunchAttribute at;
        at.id = cudaLaunchAttributeClusterDimension;
        at.val.clusterDim.x = (unsigned)ncta;
        at.val.clusterDim.y = at.val.clusterDim.z = 1;
        lc.attrs = &at;
        lc.numAttrs = 1;
        int ncl = 0;
        if (cudaOccupancyMaxActiveClusters(&ncl, k_coarse_cg, &lc) == cudaSuccess && ncl > 0) break;
        cudaGetLastError();
        plan(--ncta, split, base, sa);
    }
    if (base > budget) {
        set_err("coarse CG: the coarsest vectors do not fit in shared memory");
        return AMG_ERR_ARG;
    }
    R.cg_ncta = ncta;
    R.cg_smem_a = (base + sa <= budget) ? 1 : 0;
    R.cg_smem = base + (R.cg_smem_a ? sa : 0);
    R.cg_nnz = nnz;
    std::vector<int32_t> rp(n + 1);
    for (int64_t i = 0; i <= n; ++i) rp[i] = (int32_t)A.rp[i];
    int st;
    if ((st = dev_copy(&R.cg_rp, rp.data(), rp.size()))) return st;
    if ((st = dev_copy(&R.cg_ci, A.ci.data(), A.ci.size()))) return st;
    if ((st = dev_copy(&R.cg_v, A.v.data(), A.v.size()))) return st;
    if ((st = dev_copy(&R.cg_m, C.m.data(), C.m.size()))) return st;
    if ((st = dev_copy(&R.cg_split, split.data(), split.size()))) return st;
    if (invk) {
        auto up = [&](const amgsetup::Csr& M, int32_t** rpd, int32_t** cid, double** vd) {
            std::vector<int32_t> r32(M.nrows + 1);
            for (int64_t i = 0; i <= M.nrows; ++i) r32[i] = (int32_t)M.rp[i];
            int e;
            if ((e = dev_copy(rpd, r32.data(), r32.size()))) return e;
            if ((e = dev_copy(cid, M.ci.data(), M.ci.size()))) return e;
            return dev_copy(vd, M.v.data(), M.v.size());
        };
        if ((st = up(C.Wd, &R.cg_wrp, &R.cg_wci, &R.cg_wv))) return st;
        if ((st = up(C.Z, &R.cg_zrp, &R.cg_zci, &R.cg_zv))) return st;
    }
    return AMG_OK;
}

// Uploads one rank's plan.  coarse_inv: the dense A_L^{-1}.
// ------------------------------------------------------------- compact small levels
// With one pre- and one post-sweep the level's cycle is (Eq. 3.1, x1 = m o b, R9):
//   x1 = m b;  b_{l+1} = R (b - A x1);  e = B_{l+1} b_{l+1};  u = x1 + P e;  out = u + m (b - A u)
//      = [m b + m (b - A (m b))] + (P - diag(m) A P) e  =  S2(b) + Pc e,  b_{l+1} = R (I - A diag m) b = Rc b.
// On small levels (latency-bound) this is 3 kernels instead of 4, the restriction independent of
// the smoothing.  Same arithmetic up to rounding order; Rc and Pc are formed once on the host.
constexpr int64_t kCompactRows = 8192;
constexpr int64_t kCollapseRows = 2048;  // dense B of the collapsed level: <= 32 MB
// (multi-rank: on replicated levels only -- every rank computes all their rows; `rep`)
bool collapse_level_ok(const amg_hier_s* h, int l, int nl, int64_t n, bool rep) {
    return (!h->multi() || rep) && h->cfg.smoother == 0 && h->cfg.coarse_solver == 0 && l >= 1 && l + 2 == nl &&
           n <= kCollapseRows && !(h->tail_level >= 0 && l >= h->tail_level);
}
// C = X D (X sparse n x k CSR, D dense k x w row-major) -> dense n x w
std::vector<double> sp_dense(const amgsetup::Csr& X, const std::vector<double>& D, int64_t w) {
    std::vector<double> C((size_t)X.nrows * w, 0.0);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < X.nrows; ++i) {
        double* Ci = C.data() + (size_t)i * w;
        for (int64_t k = X.rp[i]; k < X.rp[i + 1]; ++k) {
            const double x = X.v[k];
            const double* Dk = D.data() + (size_t)X.ci[k] * w;
            for (int64_t j = 0; j < w; ++j) Ci[j] += x * Dk[j];
        }
    }
    return C;
}
// The cycle rooted at level l (s1 pre- / s2 post-sweeps of l1-Jacobi, exact coarsest solve
// A_L^{-1} = Cinv one level down) as a dense matrix B (Eq. 3.1, R9): with E = I - diag(m) A,
//   Spre = sum_{t<s1} E^t diag(m);  U = Spre + P-bar Cinv R (I - A Spre);
//   B = U, then s2 times B <- E B + diag(m).
std::vector<double> dense_level_operator(const amgsetup::Csr& A, const amgsetup::Csr& Pb, const amgsetup::Csr& Rt,
                                         const std::vector<double>& m, const std::vector<double>& Cinv, int s1,
                                         int s2) {
    const int64_t n = A.nrows, nc = Rt.nrows;
    auto diag_m = [&]() {
        std::vector<double> D((size_t)n * n, 0.0);
        for (int64_t i = 0; i < n; ++i) D[(size_t)i * n + i] = m[i];
        return D;
    };
    auto applyE = [&](const std::vector<double>& X) {  // E X = X - diag(m) (A X)
        std::vector<double> AX = sp_dense(A, X, n), Y(X);
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < n; ++i)
            for (int64_t j = 0; j < n; ++j) Y[(size_t)i * n + j] -= m[i] * AX[(size_t)i * n + j];
        return Y;
    };
    std::vector<double> G = diag_m(), Spre = G;
    for (int t = 1; t < s1; ++t) {
        G = applyE(G);
        for (size_t q = 0; q < Spre.size(); ++q) Spre[q] += G[q];
    }
    std::vector<double> W = sp_dense(A, Spre, n);  // W = I - A Spre
    for (size_t q = 0; q < W.size(); ++q) W[q] = -W[q];
    for (int64_t i = 0; i < n; ++i) W[(size_t)i * n + i] += 1.0;
    const std::vector<double> V = sp_dense(Rt, W, n);  // nc x n
    std::vector<double> Y((size_t)nc * n, 0.0);      // Y = Cinv V
#pragma omp parallel for schedule(static)
    for (int64_t a = 0; a < nc; ++a)
        for (int64_t c = 0; c < nc; ++c) {
            const double ca = Cinv[(size_t)a * nc + c];
            const double* Vc = V.data() + (size_t)c * n;
            double* Ya = Y.data() + (size_t)a * n;
            for (int64_t j = 0; j < n; ++j) Ya[j] += ca * Vc[j];
        }
    std::vector<double> B = sp_dense(Pb, Y, n);  // U = Spre + P-bar Y
    for (size_t q = 0; q < B.size(); ++q) B[q] += Spre[q];
    for (int t = 0; t < s2; ++t) {
        B = applyE(B);
        for (int64_t i = 0; i < n; ++i) B[(size_t)i * n + i] += m[i];
    }
    return B;
}
bool compact_level_ok(const amg_hier_s* h, int l, int nl, int64_t n, bool rep) {
    return (!h->multi() || rep) && h->cfg.pre_sweeps == 1 && h->cfg.post_sweeps == 1 && h->cfg.smoother == 0 && l >= 1 &&
           l + 1 < nl && n <= kCompactRows && !(h->tail_level >= 0 && l >= h->tail_level);
}
amgsetup::Csr csr_from_device(const amgsetup::DevCsrRaw& D, cudaStream_t s) {
    amgsetup::Csr C;
    C.nrows = D.nrows;
    C.ncols = D.ncols;
    C.rp.resize(D.nrows + 1);
    C.ci.resize(D.nnz);
    C.v.resize(D.nnz);
    cudaMemcpyAsync(C.rp.data(), D.rp, (D.nrows + 1) * 8, cudaMemcpyDeviceToHost, s);
    if (D.nnz) {
        cudaMemcpyAsync(C.ci.data(), D.ci, D.nnz * 4, cudaMemcpyDeviceToHost, s);
        cudaMemcpyAsync(C.v.data(), D.v, D.nnz * 8, cudaMemcpyDeviceToHost, s);
    }
    cudaStreamSynchronize(s);
    return C;
}
// Y = X - diag(lm) Z W  (dense accumulator per row; lm = nullptr: no left scaling; cm: right
// scaling of Z's columns).  Rc = R - R (A diag m): X = R, Z = R, W = A, cm = m.
// Pc = P - diag(m) A P: X = P, Z = A, W = P, lm = m.
amgsetup::Csr minus_product(const amgsetup::Csr& X, const amgsetup::Csr& Z, const amgsetup::Csr& W,
                            const double* lm, const double* cm) {
    amgsetup::Csr Y;
    Y.nrows = X.nrows;
    Y.ncols = X.ncols;
    std::vector<std::vector<int32_t>> rc(X.nrows);
    std::vector<std::vector<double>> rv(X.nrows);
#pragma omp parallel
    {
        std::vector<double> acc(X.ncols, 0.0);
        std::vector<char> used(X.ncols, 0);
        std::vector<int32_t> cols;
#pragma omp for schedule(dynamic, 16)
        for (int64_t i = 0; i < X.nrows; ++i) {
            cols.clear();
            for (int64_t k = X.rp[i]; k < X.rp[i + 1]; ++k) {
                const int32_t c = X.ci[k];
                if (!used[c]) used[c] = 1, cols.push_back(c);
                acc[c] += X.v[k];
            }
            const double li = lm ? lm[i] : 1.0;
            for (int64_t k = Z.rp[i]; k < Z.rp[i + 1]; ++k) {
                const int32_t j = Z.ci[k];
                const double zij = li * Z.v[k];
                for (int64_t t = W.rp[j]; t < W.rp[j + 1]; ++t) {
                    const int32_t c = W.ci[t];
                    if (!used[c]) used[c] = 1, cols.push_back(c);
                    acc[c] -= zij * W.v[t] * (cm ? cm[c] : 1.0);
                }
            }
            std::sort(cols.begin(), cols.end());
            rc[i].reserve(cols.size());
            rv[i].reserve(cols.size());
            for (int32_t c : cols) {
                rc[i].push_back(c);
                rv[i].push_back(acc[c]);
                acc[c] = 0.0;
                used[c] = 0;
            }
        }
    }
    Y.rp.assign(X.nrows + 1, 0);
    for (int64_t i = 0; i < X.nrows; ++i) Y.rp[i + 1] = Y.rp[i] + (int64_t)rc[i].size();
    Y.ci.resize(Y.rp[X.nrows]);
    Y.v.resize(Y.rp[X.nrows]);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < X.nrows; ++i) {
        std::copy(rc[i].begin(), rc[i].end(), Y.ci.begin() + Y.rp[i]);
        std::copy(rv[i].begin(), rv[i].end(), Y.v.begin() + Y.rp[i]);
    }
    return Y;
}

// A compact level above a collapsed one is itself a fixed linear map (V-cycle, direct coarsest):
// with the compact form out = S2(b) + Pc e and e = B_{l+1} Rc b,
//   B_l = S2 + Pc (B_{l+1} Rc),   S2 = 2 diag(m) - diag(m) A diag(m)
// (dense n_l x n_l; exact up to rounding).  One GEMV then replaces the compact level's three
// kernels and the collapsed level's one.
constexpr int64_t kCollapseRows2 = 4608;  // dense B <= 170 MB
struct CompactHost {
    amgsetup::Csr A, Rc, Pc;
    std::vector<double> m;
    bool have = false;
};
std::vector<double> collapse_above(const CompactHost& c, const std::vector<double>& B1, int64_t nc) {
    const int64_t n = c.A.nrows;
    std::vector<double> Y((size_t)nc * n, 0.0);  // Y = B_{l+1} Rc  (nc x n)
#pragma omp parallel for schedule(static)
    for (int64_t a = 0; a < nc; ++a) {
        double* Ya = Y.data() + (size_t)a * n;
        for (int64_t g = 0; g < nc; ++g) {
            const double b = B1[(size_t)a * nc + g];
            if (b == 0.0) continue;
            for (int64_t k = c.Rc.rp[g]; k < c.Rc.rp[g + 1]; ++k) Ya[c.Rc.ci[k]] += b * c.Rc.v[k];
        }
    }
    std::vector<double> B = sp_dense(c.Pc, Y, n);  // Pc Y  (n x n)
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {  // + S2
        double* Bi = B.data() + (size_t)i * n;
        for (int64_t k = c.A.rp[i]; k < c.A.rp[i + 1]; ++k) Bi[c.A.ci[k]] -= c.m[i] * c.A.v[k] * c.m[c.A.ci[k]];
        Bi[i] += 2.0 * c.m[i];
    }
    return B;
}

int upload_rank(amg_hier_s* h, const amgsetup::RankPlan& P, const std::vector<double>& coarse_inv, RankState& R,
                const amgsetup::DeviceKeep* dk = nullptr) {
    const C16Scope c16_scope(h->tail_level < 0);
    const int nl = (int)P.lv.size();
    R.rank = P.rank;
    R.lv.resize(nl);
    int st;
    std::vector<CompactHost> ch(nl);
    std::vector<std::vector<double>> Bh(nl);  // host copies of the collapsed operators
    for (int l = 0; l < nl; ++l) {
        const amgsetup::RankLevel& S = P.lv[l];
        DevLevel& D = R.lv[l];
        D.replicated = S.replicated;
        D.coarsest = (l == nl - 1);
        D.n_global = S.n_global;
        D.own_begin = S.own_begin;
        D.own_n = S.own_end - S.own_begin;
        D.comp_n = S.comp_end - S.comp_begin;
        D.win_n = S.win_end - S.win_begin;
        D.ep_off = S.comp_begin - S.win_begin;
        D.own_off = S.own_begin - S.win_begin;
        const size_t wn = (size_t)D.win_n;
        if (!D.coarsest) {
            D.rst_n = S.rst_end - S.rst_begin;
            D.rst_off = S.rst_begin - P.lv[l + 1].win_begin;
            const bool tcsr = h->tail_level >= 0 && l >= h->tail_level;  // tail levels: CSR for k_tail
            // multi-rank overlap: owned window columns of the vectors the operators gather
            int64_t lo = -1, hi = -1, clo = -1, chi = -1;
            if (h->multi() && !S.replicated) {
                lo = S.own_begin - S.win_begin;
                hi = S.own_end - S.win_begin;
            }
            if (h->multi() && !P.lv[l + 1].replicated) {
                clo = P.lv[l + 1].own_begin - P.lv[l + 1].win_begin;
                chi = P.lv[l + 1].own_end - P.lv[l + 1].win_begin;
            }
            if (dk) {  // GPU-built hierarchy: formats converted on the device (single rank)
                cudaStream_t cs = h->ctx->stream;
                if ((st = convert_mat(dk->A[l], D.A, true, D.ep_off, tcsr, cs))) return st;
                if ((st = convert_mat(dk->P[l], D.P, false, 0, tcsr, cs))) return st;
                if ((st = convert_mat(dk->R[l], D.R, false, 0, tcsr, cs))) return st;
                CK(cudaMalloc((void**)&D.m, wn * 8));
                CK(cudaMemcpyAsync(D.m, dk->m[l], wn * 8, cudaMemcpyDeviceToDevice, cs));
                if (h->cfg.pre_sweeps == 1) {
                    amgsetup::DevCsrRaw As = dk->A[l];
                    CK(cudaMalloc((void**)&As.v, std::max<int64_t>(1, As.nnz) * 8));
                    kc_scale_cols<<<148 * 16, 256, 0, cs>>>(dk->A[l].ci, dk->A[l].v, As.nnz, D.m, As.v);
                    st = convert_mat(As, D.Am, true, D.ep_off, tcsr, cs);
                    cudaFree(As.v);
                    if (st) return st;
                }
                if ((st = dev_alloc(&D.mb, wn))) return st;
                if ((st = dev_alloc(&D.r, wn))) return st;
                if ((st = dev_alloc(&D.xb, wn))) return st;
            } else {  // host-built hierarchy (or multi-rank plan): formats on the host
                if ((st = upload_mat(S.A, D.A, true, D.ep_off, tcsr, lo, hi))) return st;
                if (h->cfg.smoother == 1) {
                    if ((st = upload_mat(S.Wd, D.Wd, true, D.ep_off))) return st;
                    if ((st = upload_mat(S.Z, D.Z, true, D.ep_off))) return st;
                } else if (h->cfg.pre_sweeps == 1) {
                    amgsetup::Csr As = S.A;
#pragma omp parallel for schedule(static)
                    for (int64_t i = 0; i < As.nrows; ++i)
                        for (int64_t k = As.rp[i]; k < As.rp[i + 1]; ++k) As.v[k] = As.v[k] * S.m[As.ci[k]];
                    if ((st = upload_mat(As, D.Am, true, D.ep_off, tcsr, lo, hi))) return st;
                }
                if ((st = upload_mat(S.P, D.P, false, 0, tcsr, clo, chi))) return st;
                if ((st = upload_mat(S.R, D.R, false, 0, tcsr, lo, hi))) return st;
                if ((st = dev_copy(&D.m, S.m.data(), S.m.size()))) return st;
                if ((st = dev_alloc(&D.mb, wn))) return st;
                if ((st = dev_alloc(&D.r, wn))) return st;
                if ((st = dev_alloc(&D.xb, wn))) return st;
            }
        }
        if (compact_level_ok(h, l, nl, D.comp_n, S.replicated)) {
            amgsetup::Csr A, Pb, Rt;
            std::vector<double> m(D.comp_n);
            if (dk) {
                A = csr_from_device(dk->A[l], h->ctx->stream);
                Pb = csr_from_device(dk->P[l], h->ctx->stream);
                Rt = csr_from_device(dk->R[l], h->ctx->stream);
                CK(cudaMemcpy(m.data(), dk->m[l], m.size() * 8, cudaMemcpyDeviceToHost));
            } else {
                A = S.A;
                Pb = S.P;
                Rt = S.R;
                m = S.m;
            }
            const amgsetup::Csr Rc = minus_product(Rt, Rt, A, nullptr, m.data());
            const amgsetup::Csr Pc = minus_product(Pb, A, Pb, m.data(), nullptr);
            if ((st = upload_mat(Rc, D.Rc, false, 0))) return st;
            if ((st = upload_mat(Pc, D.Pc, false, 0))) return st;
            D.compact = true;
            if (D.comp_n <= kCollapseRows2) {  // kept for a second collapse (below)
                ch[l].A = std::move(A);
                ch[l].Rc = Rc;
                ch[l].Pc = Pc;
                ch[l].m = std::move(m);
                ch[l].have = true;
            }
        }
        if (collapse_level_ok(h, l, nl, D.comp_n, S.replicated) &&
            (int64_t)coarse_inv.size() == P.lv[l + 1].n_global * P.lv[l + 1].n_global) {
            // the level above a direct coarsest solve: its whole cycle is a fixed linear map B
            amgsetup::Csr A, Pb, Rt;
            std::vector<double> m(D.comp_n);
            if (dk) {
                A = csr_from_device(dk->A[l], h->ctx->stream);
                Pb = csr_from_device(dk->P[l], h->ctx->stream);
                Rt = csr_from_device(dk->R[l], h->ctx->stream);
                CK(cudaMemcpy(m.data(), dk->m[l], m.size() * 8, cudaMemcpyDeviceToHost));
            } else {
                A = S.A;
                Pb = S.P;
                Rt = S.R;
                m = S.m;
            }
            std::vector<double> B =
                dense_level_operator(A, Pb, Rt, m, coarse_inv, h->cfg.pre_sweeps, h->cfg.post_sweeps);
            if ((st = dev_copy(&D.Mc, B.data(), B.size()))) return st;
            Bh[l] = std::move(B);
            if (h->cfg.cycle == 1 && kcycle_fused(h) && l + 2 == nl && l >= 1) {  // an inner FCG level: also A B
                const std::vector<double> AB = sp_dense(A, Bh[l], D.comp_n);
                if ((st = dev_copy(&D.AMc, AB.data(), AB.size()))) return st;
            }
        }
        if ((st = dev_alloc(&D.b, wn))) return st;
        if ((st = dev_alloc(&D.xa, wn))) return st;
        if (h->cfg.cycle == 1 && l >= 1 && l + 1 < nl) {
            for (double** v : {&D.kx, &D.kr, &D.kmb, &D.kz, &D.kp, &D.kq, &D.kp2})
                if ((st = dev_alloc(v, wn))) return st;
            if ((st = dev_alloc(&D.kst, 8))) return st;
        }
        // halo plan: window positions
        Exch& E = D.ex;
        E.send_off = S.send_off;
        E.recv_off = S.recv_off;
        E.nsend = (int64_t)S.send_ids.size();
        E.nrecv = (int64_t)S.recv_ids.size();
        std::vector<int32_t> si(E.nsend), ri(E.nrecv);
        for (int64_t k = 0; k < E.nsend; ++k) si[k] = (int32_t)(S.send_ids[k] - S.win_begin);
        for (int64_t k = 0; k < E.nrecv; ++k) ri[k] = (int32_t)(S.recv_ids[k] - S.win_begin);
        if ((st = dev_copy(&E.send_idx, si.data(), si.size()))) return st;
        if ((st = dev_copy(&E.recv_idx, ri.data(), ri.size()))) return st;
        if ((st = dev_alloc(&E.sbuf, E.nsend))) return st;
        if ((st = dev_alloc(&E.rbuf, E.nrecv))) return st;
    }
    // second collapse: a compact level directly above a collapsed level (V-cycle)
    if (h->cfg.cycle == 0 && !std::getenv("AMG_NO_COLLAPSE2"))
        for (int l = nl - 3; l >= 1; --l) {
            DevLevel& D = R.lv[l];
            if (!ch[l].have || Bh[l + 1].empty() || D.Mc) continue;
            const int64_t nc = P.lv[l + 1].n_global;
            if ((int64_t)Bh[l + 1].size() != nc * nc || D.comp_n != P.lv[l].n_global) continue;
            // only when the dense operator moves no more bytes than the compact level and the collapsed
            // one below it (measured: c4 / c5 gain 0.6 %, the sparser c2 level loses 0.5 % at 3x the bytes)
            const double dense_b = 8.0 * (double)D.comp_n * (double)D.comp_n;
            const double compact_b = 12.0 * (double)(ch[l].A.nnz() + ch[l].Rc.nnz() + ch[l].Pc.nnz()) +
                                     8.0 * (double)nc * (double)nc;
            if (dense_b > compact_b && !std::getenv("AMG_FORCE_COLLAPSE2")) break;
            Bh[l] = collapse_above(ch[l], Bh[l + 1], nc);
            if ((st = dev_copy(&D.Mc, Bh[l].data(), Bh[l].size()))) return st;
            amgsetup::tmark("second collapse");
            break;  // the next level up is too large to hold densely (kCollapseRows2)
        }
    R.nL = P.lv[nl - 1].n_global;
    if ((st = dev_copy(&R.cinv, coarse_inv.data(), coarse_inv.size()))) return st;
    if (h->cfg.coarse_solver == 1 && (st = upload_coarse_cg(h, P.lv[nl - 1], R))) return st;
    const size_t w0 = (size_t)R.lv[0].win_n;
    if ((st = dev_alloc(&R.pr, w0))) return st;
    if ((st = dev_alloc(&R.pz, w0))) return st;
    if ((st = dev_alloc(&R.pp, w0))) return st;
    if ((st = dev_alloc(&R.pp2, w0))) return st;
    if ((st = dev_alloc(&R.pq, w0))) return st;
    if ((st = dev_alloc(&R.st, 1))) return st;
    if ((st = dev_alloc(&R.partials, 2 * kMaxPartials))) return st;  // two-dot reductions: 2 per block
    if ((st = dev_alloc(&R.ticket, 1))) return st;
    if ((st = dev_alloc(&R.dot_local, kDotSlots))) return st;
    if ((st = dev_alloc(&R.dot_all, (size_t)kDotSlots * h->np))) return st;
    if (nl == 1) {  // single-level: level 0 is the coarsest; give it an operator for q = A p
        if ((st = upload_mat(P.lv[0].A, R.lv[0].A, true, 0))) return st;
    }
    return AMG_OK;
}

// SURVEY.md §8d byte model (global hierarchy).  For the K-cycle every level-l part
// runs 2^l times (l <= nl-2; the coarsest 2^(nl-2) times) and each of the 2^(l-1)
// inner FCG solves at level l >= 1 adds two SpMVs and its vector updates
// (176 B per row: p^T b, kupd1, z^T q, p-update, kupd2 and the SpMV p/q).
// Global level statistics (rows, nnz(A_l), nnz(P-bar_l), nnz(Wd_l) + nnz(Z_l)).
struct LevelStats {
    std::vector<int64_t> n, nnzA, nnzP, nnzWZ;
};
LevelStats stats_of(const amgsetup::Hierarchy& H) {
    LevelStats S;
    for (auto& L : H.lv) {
        S.n.push_back(L.A.nrows);
        S.nnzA.push_back(L.A.nnz());
        S.nnzP.push_back(L.P.nnz());
        S.nnzWZ.push_back(L.Wd.nnz() + L.Z.nnz());
    }
    return S;
}

void byte_model(amg_hier_s* h, const LevelStats& S) {
    const double s1 = h->cfg.pre_sweeps, s2 = h->cfg.post_sweeps;
    const bool kc = h->cfg.cycle == 1;
    double bv = 0.0;
    const size_t nl = S.n.size();
    for (size_t l = 0; l + 1 < nl; ++l) {
        const double n = (double)S.n[l], nc = (double)S.n[l + 1];
        const double MA = 12.0 * (double)S.nnzA[l] + 4.0 * (n + 1);
        const double MP = 12.0 * (double)S.nnzP[l] + 4.0 * (n + 1);
        const double visits = kc ? std::ldexp(1.0, (int)l) : 1.0;
        bv += visits * ((s1 + s2) * MA + 2 * MP + 8 * n * ((s1 + s2) + 2 + 3 * (s1 - 1) + 2 + 2 + 3 * s2) + 16 * nc);
        if (h->cfg.smoother == 1)  // INVK: every smoothing step also streams Wd and Z (+ t write/read)
            bv += visits * (s1 + s2) * (12.0 * (double)S.nnzWZ[l] + 8.0 * (n + 1) + 16.0 * n);
        if (kc && l >= 1) bv += std::ldexp(1.0, (int)l - 1) * (2 * MA + 176.0 * n);
    }
    const double nL = (double)S.n.back();
    bv += (kc && nl >= 2 ? std::ldexp(1.0, (int)nl - 2) : 1.0) * (8 * nL * nL + 16 * nL);
    h->bytes_v = bv;
    const double n0 = (double)S.n[0];
    h->bytes_it = bv + 12.0 * (double)S.nnzA[0] + 4.0 * (n0 + 1) + 88.0 * n0;
}

void hier_stats(amg_hier_s* h, const LevelStats& S) {
    const size_t nl = S.n.size();
    double s = 0.0;
    for (int64_t x : S.nnzA) s += (double)x;
    h->opc = s / (double)S.nnzA[0];
    double cr = 0.0;
    for (size_t l = 0; l + 1 < nl; ++l) cr += (double)S.n[l] / (double)S.n[l + 1];
    h->avg_cr = nl > 1 ? cr / (double)(nl - 1) : 1.0;
    h->lvl_n = S.n;
    h->lvl_nnzA = S.nnzA;
    h->lvl_nnzP = S.nnzP;
    byte_model(h, S);
}
void hier_stats(amg_hier_s* h, const amgsetup::Hierarchy& H) { hier_stats(h, stats_of(H)); }

// AMG_L2_PERSIST_MB=<MB> (experiment, default off): the value arrays of the deepest levels' operators,
// from the coarsest up while they fit in the budget, are launched with an L2 persistence window so
// they stay L2-resident across V-cycles (the level-0/1 streams would otherwise evict them).
void mark_persistent(amg_hier_s* h) {
    const char* e = std::getenv("AMG_L2_PERSIST_MB");
    if (!e) return;
    const double budget = std::atof(e) * 1048576.0;
    if (!(budget > 0.0)) return;
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)budget);
    double used = 0.0;
    for (int l = h->nlev() - 2; l >= 1; --l) {
        double lb = 0.0;
        for (auto& R : h->ranks) {
            DevLevel& D = R.lv[l];
            for (DevMat* M : {&D.A, &D.Am, &D.P, &D.R, &D.Rc, &D.Pc}) lb += 8.0 * (double)M->stored;
        }
        if (used + lb > budget) break;
        used += lb;
        for (auto& R : h->ranks) {
            DevLevel& D = R.lv[l];
            for (DevMat* M : {&D.A, &D.Am, &D.P, &D.R, &D.Rc, &D.Pc}) M->persist = M->val != nullptr;
        }
    }
}

int build_solve_exec(amg_hier_s* h, const double* b, double* x, cudaGraphExec_t* out);
enum { GM_WHILE = 0, GM_ITER = 1 };
// NCCL contexts: every rank must take the same graph shape (the captured collectives must
// match), so a local failure is agreed on with an eager all-reduce (min) of the success flags.
int agree_ok(amg_hier_s* h, int ok_local, int* ok_all) {
    *ok_all = ok_local;
    if (!h->nccl_xport()) return AMG_OK;
    int* d = nullptr;
    CK(cudaMalloc(&d, sizeof(int)));
    CK(h2d_sync(d, &ok_local, sizeof(int)));
    NK(ncclAllReduce(d, d, 1, ncclInt, ncclMin, h->ctx->nccl, h->ctx->stream));
    CK(cudaStreamSynchronize(h->ctx->stream));
    CK(cudaMemcpy(ok_all, d, sizeof(int), cudaMemcpyDeviceToHost));
    cudaFree(d);
    return AMG_OK;
}
int ensure_solve_graph(amg_hier_s* h, const double* b, double* x) {
    if (h->solve_exec && h->solve_b == b && h->solve_x == x) return AMG_OK;
    if (h->solve_exec) {
        cudaGraphExecDestroy(h->solve_exec);
        h->solve_exec = nullptr;
    }
    int st = build_solve_exec(h, b, x, &h->solve_exec);
    if (h->nccl_xport()) {  // NCCL: collective decision, fall back to one graph per iteration
        if (st == AMG_OK && h->nccl_status != ncclSuccess) st = AMG_ERR_NCCL;  // a collective refused capture
        if (st != AMG_OK) {
            std::fprintf(stderr, "amg: the NCCL solve could not be captured as one WHILE graph (%s); "
                         "falling back to one graph per iteration\n",
                         h->nccl_status != ncclSuccess ? h->nccl_what.c_str() : amg_last_error());
            h->nccl_status = ncclSuccess;
        }
        int all = 0, e;
        if ((e = agree_ok(h, st == AMG_OK ? 1 : 0, &all))) return e;
        if (!all) {
            if (h->solve_exec) cudaGraphExecDestroy(h->solve_exec);
            h->solve_exec = nullptr;
            cudaGetLastError();
            h->graph_mode = GM_ITER;
            return AMG_OK;
        }
    }
    if (st) return st;
    h->solve_b = b;
    h->solve_x = x;
    return AMG_OK;
}
// GM_ITER: the iteration body as a plain graph (captured collectives, no conditional node)
int ensure_iter_graph(amg_hier_s* h, double* x) {
    if (h->iter_exec && h->iter_x == x) return AMG_OK;
    if (h->iter_exec) {
        cudaGraphExecDestroy(h->iter_exec);
        h->iter_exec = nullptr;
    }
    cudaStream_t s = h->ctx->stream;
    Launch L{h, s};
    cudaGraph_t g = nullptr;
    CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    enqueue_pcg_body(h, L, x, 0);
    const cudaError_t ec = cudaStreamEndCapture(s, &g);
    cudaError_t ei = cudaErrorUnknown;
    if (ec == cudaSuccess) ei = cudaGraphInstantiate(&h->iter_exec, g, 0);
    if (g) cudaGraphDestroy(g);
    const bool nok = h->nccl_status != ncclSuccess;  // a collective refused capture: discard the graph
    if (ec != cudaSuccess || ei != cudaSuccess || nok) {
        std::fprintf(stderr, "amg: the iteration could not be captured as a graph (%s); eager launches\n",
                     nok ? h->nccl_what.c_str() : cudaGetErrorString(ec != cudaSuccess ? ec : ei));
        h->nccl_status = ncclSuccess;
    }
    int all = 0, e;
    if ((e = agree_ok(h, (ec == cudaSuccess && ei == cudaSuccess && !nok) ? 1 : 0, &all))) return e;
    if (!all) {
        if (h->iter_exec && ei == cudaSuccess) cudaGraphExecDestroy(h->iter_exec);
        h->iter_exec = nullptr;
        cudaGetLastError();
        h->graph_mode = 2;  // eager
        return AMG_OK;
    }
    h->iter_x = x;
    return AMG_OK;
}
// the whole solve as one graph: prologue, WHILE node over the PCG body, final x update
// (every exit destroys the graph: a leaked graph that captured NCCL collectives keeps the
// communicator's persistent references alive, and ncclCommDestroy then waits forever)
struct GraphGuard {
    cudaGraph_t g = nullptr;
    ~GraphGuard() {
        if (g) cudaGraphDestroy(g);
    }
};
int build_solve_exec(amg_hier_s* h, const double* b, double* x, cudaGraphExec_t* out) {
    cudaStream_t s = h->ctx->stream;
    GraphGuard gg;
    CK(cudaGraphCreate(&gg.g, 0));
    cudaGraph_t g = gg.g;  // capture-to-graph hands the same graph back
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
    // after the loop: the deferred last x update
    CK(cudaStreamBeginCaptureToGraph(s, g, &wnode, nullptr, 1, cudaStreamCaptureModeThreadLocal));
    enqueue_pcg_final(h, L, x);
    CK(cudaStreamEndCapture(s, &g));
    cudaGraphInstantiateParams ip = {};
    const cudaError_t ei = cudaGraphInstantiateWithParams(out, g, &ip);
    if (ei != cudaSuccess) {
        // name the node the driver refused (NCCL collectives inside the WHILE body, B200 / CUDA 12.9:
        // tests/test_gpu_nccl_loopback.py records what it is)
        std::string what = std::string("cudaGraphInstantiate (WHILE graph): ") + cudaGetErrorString(ei) +
                           ", result " + std::to_string((int)ip.result_out);
        if (ip.errNode_out) {
            cudaGraphNodeType t;
            if (cudaGraphNodeGetType(ip.errNode_out, &t) == cudaSuccess) {
                what += ", node type " + std::to_string((int)t);
                cudaKernelNodeParams kp = {};
                const char* fname = nullptr;
                if (t == cudaGraphNodeTypeKernel && cudaGraphKernelNodeGetParams(ip.errNode_out, &kp) == cudaSuccess &&
                    cudaFuncGetName(&fname, kp.func) == cudaSuccess && fname)
                    what += std::string(" (kernel ") + fname + ")";
            }
        }
        cudaGetLastError();
        *out = nullptr;
        set_err(what);
        return AMG_ERR_CUDA;
    }
    return AMG_OK;
}

// V-cycle on the caller's vectors: level-0 window staging for multi-rank.
void enqueue_apply(amg_hier_s* h, Launch& L, const double* r_user, double* z_user) {
    if (!h->multi()) {
        enqueue_vcycle(h, L, [&](RankState&) { return const_cast<double*>(r_user); },
                       [&](RankState&) { return z_user; }, false);
        return;
    }
    for (auto& R : h->ranks) {
        const DevLevel& D = R.L0();
        cudaMemcpyAsync(R.pr + D.own_off, r_user + R.user_off, sizeof(double) * D.own_n, cudaMemcpyDeviceToDevice,
                        L.s);
    }
    enqueue_vcycle(h, L, [](RankState& R) { return R.pr; }, [](RankState& R) { return R.pz; }, false);
    for (auto& R : h->ranks) {
        const DevLevel& D = R.L0();
        cudaMemcpyAsync(z_user + R.user_off, R.pz + D.own_off, sizeof(double) * D.own_n, cudaMemcpyDeviceToDevice,
                        L.s);
    }
}

int ensure_apply_graph(amg_hier_s* h, const double* r, double* z) {
    if (h->apply_exec && h->apply_r == r && h->apply_z == z) return AMG_OK;
    if (h->apply_exec) {
        cudaGraphExecDestroy(h->apply_exec);
        h->apply_exec = nullptr;
    }
    cudaStream_t s = h->ctx->stream;
    Launch L{h, s};
    GraphGuard gg;
    CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    enqueue_apply(h, L, r, z);
    CK(cudaStreamEndCapture(s, &gg.g));
    CK(cudaGraphInstantiate(&h->apply_exec, gg.g, 0));
    h->apply_r = r;
    h->apply_z = z;
    return AMG_OK;
}

// ------------------------------------------------ LSA transport setup (NCCL symmetric window)
__global__ void k_lsa_bases(ncclWindow_t win, int np, int loopback, int64_t seg, char** out) {
    const int q = threadIdx.x;
    if (q >= np) return;
    out[q] = loopback ? (char*)ncclGetLsaPointer(win, 0, 0) + (int64_t)q * seg : (char*)ncclGetLsaPointer(win, 0, q);
}

// All ranks agree (NCCL contexts; min over ranks) -- on the context stream, outside any capture.
int lsa_agree(amg_hier_s* h, int ok_local, int* ok_all) {
    *ok_all = ok_local;
    if (h->loopback) return AMG_OK;  // one process: the local decision is everyone's
    int* d = nullptr;
    CK(cudaMalloc(&d, sizeof(int)));
    CK(h2d_sync(d, &ok_local, sizeof(int)));
    NK(ncclAllReduce(d, d, 1, ncclInt, ncclMin, h->ctx->nccl, h->ctx->stream));
    CK(cudaStreamSynchronize(h->ctx->stream));
    CK(cudaMemcpy(ok_all, d, sizeof(int), cudaMemcpyDeviceToHost));
    cudaFree(d);
    return AMG_OK;
}

// Sets up the peer-memory transport for a hierarchy on an NCCL context (real ranks, or loopback on a
// one-rank communicator): lays out one window segment per rank (flags | 2 x dots | 2 x receive region
// per level), allocates it with ncclMemAlloc, registers it as a symmetric window, resolves every
// segment's address (ncclGetLsaPointer), checks one dot gather end to end (values and a bounded
// barrier) and only then points the levels' receive buffers into the window.  Any failure on any
// rank keeps every rank on the NCCL send/recv transport (decided collectively).  AMG_TRANSPORT=nccl
// skips it.
int lsa_setup(amg_hier_s* h) {
    const char* tr = std::getenv("AMG_TRANSPORT");
    if ((tr && std::strcmp(tr, "nccl") == 0) || !h->nccl_xport()) return AMG_OK;
    ncclComm_t comm = h->ctx->nccl;
    const int np = h->np, nl = h->nlev();
    const bool lb = h->loopback;
    cudaStream_t s = h->ctx->stream;
    int ok = np <= kBlock ? 1 : 0;
    if (!lb && ok) {
        const ncclTeam_t t = ncclTeamLsa(comm);
        if (t.nRanks != np) ok = 0;  // not one NVLink (load/store) domain
    }
    // every rank's recv_off per level: [rank][level][np+1]
    const size_t per = (size_t)nl * (np + 1);
    std::vector<int64_t> ro((size_t)np * per, 0);
    auto mine = [&](RankState& R, int64_t* out) {
        for (int l = 0; l < nl; ++l) {
            const auto& v = R.lv[l].ex.recv_off;
            for (int q = 0; q <= np; ++q) out[(size_t)l * (np + 1) + q] = v.size() == (size_t)np + 1 ? v[q] : 0;
        }
    };
    if (lb) {
        for (auto& R : h->ranks) mine(R, ro.data() + (size_t)R.rank * per);
    } else {
        std::vector<int64_t> m(per);
        mine(h->ranks[0], m.data());
        int64_t* d = nullptr;
        CK(cudaMalloc(&d, sizeof(int64_t) * per * (np + 1)));
        CK(h2d_sync(d, m.data(), sizeof(int64_t) * per));
        NK(ncclAllGather(d, d + per, per, ncclInt64, comm, s));
        CK(cudaStreamSynchronize(s));
        CK(cudaMemcpy(ro.data(), d + per, sizeof(int64_t) * per * np, cudaMemcpyDeviceToHost));
        cudaFree(d);
    }
    auto al = [](int64_t x, int64_t a) { return (x + a - 1) / a * a; };
    int64_t off = al(8 * (int64_t)np, 256);
    h->lsa_flag_off = 0;
    h->lsa_dot_off = off;
    h->lsa_dot_stride = al(8 * (int64_t)kDotSlots * np, 256);
    off += 2 * h->lsa_dot_stride;
    std::vector<int64_t> lvl_off(nl, 0);
    h->lsa_lvl_stride.assign(nl, 0);
    for (int l = 0; l < nl; ++l) {
        int64_t mx = 0;
        for (int q = 0; q < np; ++q) mx = std::max(mx, ro[(size_t)q * per + (size_t)l * (np + 1) + np]);
        if (!mx) continue;
        lvl_off[l] = off;
        h->lsa_lvl_stride[l] = al(8 * mx, 256);
        off += 2 * h->lsa_lvl_stride[l];
    }
    h->lsa_seg = al(off, NCCL_WIN_REQUIRED_ALIGNMENT);
    const size_t total = (size_t)h->lsa_seg * (lb ? np : 1);
    if (ok && ncclMemAlloc(&h->lsa_mem, total) != ncclSuccess) {
        h->lsa_mem = nullptr;
        ok = 0;
    }
    if (ok && memset_sync(h->lsa_mem, 0, total) != cudaSuccess) ok = 0;
    int all = 0, e;
    if ((e = lsa_agree(h, ok, &all))) return e;
    if (all) {  // collective registration, every rank takes part
        h->lsa_comm = comm;
        if (ncclCommWindowRegister(comm, h->lsa_mem, total, &h->lsa_win, NCCL_WIN_COLL_SYMMETRIC) != ncclSuccess) {
            h->lsa_win = nullptr;
            ok = 0;
        }
        if ((e = lsa_agree(h, ok, &all))) return e;
    }
    std::string why = "ncclMemAlloc / window registration / LSA team";
    if (all) {
        if (cudaMalloc(&h->lsa_peer, sizeof(char*) * np) != cudaSuccess || cudaMalloc(&h->lsa_err, sizeof(int)) != cudaSuccess ||
            memset_sync(h->lsa_err, 0, sizeof(int)) != cudaSuccess)
            ok = 0;
        if (ok) {
            k_lsa_bases<<<1, kBlock, 0, s>>>(h->lsa_win, np, lb ? 1 : 0, h->lsa_seg, h->lsa_peer);
            for (auto& R : h->ranks) {
                char* mine_seg = (char*)h->lsa_mem + (lb ? (int64_t)R.rank * h->lsa_seg : 0);
                R.lsa_flags = (unsigned long long*)(mine_seg + h->lsa_flag_off);
                R.lsa_dots = (double*)(mine_seg + h->lsa_dot_off);
                if (cudaMalloc(&R.lsa_seq, sizeof(unsigned long long)) != cudaSuccess ||
                    cudaMalloc(&R.lsa_count, sizeof(unsigned int)) != cudaSuccess ||
                    memset_sync(R.lsa_seq, 0, sizeof(unsigned long long)) != cudaSuccess ||
                    memset_sync(R.lsa_count, 0, sizeof(unsigned int)) != cudaSuccess)
                    ok = 0;
            }
        }
        // end-to-end check: one dot gather of known values through the window (a bounded barrier)
        if (ok) {
            for (auto& R : h->ranks) {
                const double v[kDotSlots] = {(double)R.rank + 1.0, -2.0 * R.rank, 0.5};
                h2d_sync(R.dot_local, v, sizeof(v));
            }
            lsa_dot_push(h, s);
            for (auto& R : h->ranks) {
                RxWait w = lsa_rx(h, R, 0);
                w.timeout_ns = 30ull * 1000000000ull;
                k_lsa_wait<<<1, kBlock, 0, s>>>(w);
            }
            int err = 1;
            if (cudaStreamSynchronize(s) != cudaSuccess) ok = 0;
            if (ok) cudaMemcpy(&err, h->lsa_err, sizeof(int), cudaMemcpyDeviceToHost);
            if (err) {
                ok = 0;
                why = "barrier check timed out";
            }
            for (auto& R : h->ranks) {
                std::vector<double> got((size_t)kDotSlots * np);
                if (ok && cudaMemcpy(got.data(), R.lsa_dots, sizeof(double) * got.size(), cudaMemcpyDeviceToHost) != cudaSuccess)
                    ok = 0;
                for (int q = 0; q < np && ok; ++q)
                    if (got[(size_t)q * kDotSlots] != q + 1.0 || got[(size_t)q * kDotSlots + 1] != -2.0 * q ||
                        got[(size_t)q * kDotSlots + 2] != 0.5) {
                        ok = 0;
                        why = "dot gather check read wrong values";
                    }
                memset_sync(R.dot_local, 0, kDotSlots * sizeof(double));
            }
        }
        if ((e = lsa_agree(h, ok, &all))) return e;
    }
    if (!all) {
        std::fprintf(stderr, "amg: peer-memory (LSA) transport unavailable (%s); NCCL send/recv transport\n",
                     why.c_str());
        for (auto& R : h->ranks) {
            cudaFree(R.lsa_seq);
            cudaFree(R.lsa_count);
            R.lsa_seq = nullptr;
            R.lsa_count = nullptr;
            R.lsa_flags = nullptr;
            R.lsa_dots = nullptr;
        }
        h->release_lsa();
        cudaGetLastError();
        return AMG_OK;
    }
    // point every distributed level's receive buffer into the window (double-buffered regions)
    for (auto& R : h->ranks) {
        char* mine_seg = (char*)h->lsa_mem + (lb ? (int64_t)R.rank * h->lsa_seg : 0);
        for (int l = 0; l < nl; ++l) {
            Exch& E = R.lv[l].ex;
            E.rx = lsa_rx(h, R, h->lsa_lvl_stride[l] / 8);  // every level: ranks without entries wait too
            if (!h->lsa_lvl_stride[l]) continue;
            if (!E.rbuf_in_window) cudaFree(E.rbuf);
            E.rbuf = (double*)(mine_seg + lvl_off[l]);
            E.rbuf_in_window = true;
            std::vector<int64_t> so(np + 1, 0), dst(np, 0);
            for (int q = 0; q <= np; ++q) so[q] = E.send_off.size() == (size_t)np + 1 ? E.send_off[q] : 0;
            for (int q = 0; q < np; ++q) dst[q] = lvl_off[l] + 8 * ro[(size_t)q * per + (size_t)l * (np + 1) + R.rank];
            int st;
            if ((st = dev_copy(&E.d_send_off, so.data(), so.size()))) return st;
            if ((st = dev_copy(&E.d_dst_off, dst.data(), dst.size()))) return st;
        }
    }
    h->lsa = true;
    return AMG_OK;
}

// AMG_DEBUG_CHECKSUM=1 (diagnostics): FNV-1a of every device array of rank 0's hierarchy on stderr,
// one line per level and operator, so two builds of the same matrix can be compared array by array.
uint64_t dev_fnv(const void* p, size_t bytes) {
    if (!p || !bytes) return 0;
    std::vector<unsigned char> hbuf(bytes);
    if (cudaMemcpy(hbuf.data(), p, bytes, cudaMemcpyDeviceToHost) != cudaSuccess) return 1;
    uint64_t x = 1469598103934665603ull;
    for (unsigned char c : hbuf) x = (x ^ c) * 1099511628211ull;
    return x;
}
void debug_checksums(amg_hier_s* h) {
    cudaDeviceSynchronize();
    RankState& R = h->ranks[0];
    auto mat = [&](int l, const char* name, const DevMat& M) {
        if (!M.nrows) return;
        const int64_t nsl = M.units;
        const bool sell = M.fmt == FMT_SELL, sdia = M.fmt == FMT_SDIA;
        const int64_t ne = (sell || sdia) ? M.stored : M.nnz;
        std::fprintf(stderr,
                     "amg-checksum L%d %s fmt %d n %lld stored %lld sptr %016llx offs %016llx anchor %016llx rp %016llx "
                     "col %016llx val %016llx perm %016llx c16 %016llx cbase %016llx\n",
                     l, name, M.fmt, (long long)M.nrows, (long long)ne,
                     (unsigned long long)dev_fnv(M.sptr, (sell || sdia) ? (nsl + 1) * 4 : 0),
                     (unsigned long long)dev_fnv(M.offs, sdia ? ne / 32 * 4 : 0),
                     (unsigned long long)dev_fnv(M.anchor, M.anchor ? M.nrows * 4 : 0),
                     (unsigned long long)dev_fnv(M.rp, M.rp ? (M.nrows + 1) * 4 : 0),
                     (unsigned long long)dev_fnv(M.col, M.col ? ne * 4 : 0),
                     (unsigned long long)dev_fnv(M.val, ne * 8),
                     (unsigned long long)dev_fnv(M.perm, M.perm ? nsl * 32 * 4 : 0),
                     (unsigned long long)dev_fnv(M.c16, M.c16 ? ne * 2 : 0),
                     (unsigned long long)dev_fnv(M.cbase, M.cbase ? (sell ? nsl * 32 : M.nrows) * 4 : 0));
    };
    for (int l = 0; l < (int)R.lv.size(); ++l) {
        DevLevel& D = R.lv[l];
        mat(l, "A", D.A);
        mat(l, "Am", D.Am);
        mat(l, "P", D.P);
        mat(l, "R", D.R);
        mat(l, "Rc", D.Rc);
        mat(l, "Pc", D.Pc);
        const int64_t nc = l + 1 < (int)R.lv.size() ? R.lv[l + 1].win_n : 0;
        std::fprintf(stderr, "amg-checksum L%d vec m %016llx Mc %016llx (n %lld)\n", l,
                     (unsigned long long)dev_fnv(D.m, D.m ? D.win_n * 8 : 0),
                     (unsigned long long)dev_fnv(D.Mc, D.Mc ? D.comp_n * D.comp_n * 8 : 0), (long long)nc);
    }
    std::fprintf(stderr, "amg-checksum cinv %016llx (nL %lld)\n", (unsigned long long)dev_fnv(R.cinv, R.nL * R.nL * 8),
                 (long long)R.nL);
}

// AMG_ERR_NCCL if an LSA barrier timed out (a peer rank never arrived; sticky).
int take_lsa_err(amg_hier_s* h) {
    if (!h->lsa) return AMG_OK;
    int err = 0;
    CK(cudaMemcpy(&err, h->lsa_err, sizeof(int), cudaMemcpyDeviceToHost));
    if (!err) return AMG_OK;
    set_err("peer-memory transport: a peer rank did not arrive at a barrier within " +
            std::to_string(h->lsa_timeout_ns / 1000000000ull) + " s");
    return AMG_ERR_NCCL;
}

// AMG_ERR_NCCL if an enqueue pass since the last call recorded an NCCL failure.
int take_nccl_status(amg_hier_s* h) {
    if (h->nccl_status == ncclSuccess) return AMG_OK;
    set_err(h->nccl_what);
    h->nccl_status = ncclSuccess;
    return AMG_ERR_NCCL;
}

void fill_report(amg_hier_s* h, amg_report_t* rep) {
    rep->nlevels = (int32_t)h->lvl_n.size();
    rep->setup_s = h->setup_s;
    rep->opc = h->opc;
    rep->avg_cr = h->avg_cr;
    rep->vcycle_bytes_model = h->bytes_v;
    rep->iteration_bytes_model = h->bytes_it;
}

amgsetup::Config setup_config(const amg_config_t& cfg) {
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
    sc.device = cfg.setup_device;
    return sc;
}

// Copies the caller's CSR into the setup's form and runs the host setup.
int host_setup(int64_t n, const int64_t* rowptr, const int64_t* colind, const double* values, const double* w,
               const amg_config_t& cfg, amgsetup::Hierarchy& H) {
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
    amgsetup::Config sc = setup_config(cfg);
    if (sc.device) {
        // capacity: A_0 and the level-0 Galerkin operands and results (A P-bar, its
        // per-entry product offsets, P-bar^T, the kept device hierarchy: <= ~64 B per
        // nonzero of A_0) plus one expand-sort-compress chunk (<= free/4, setup_gpu.cu)
        // must fit in the free device memory; otherwise the bit-identical host build runs
        size_t freeb = 0, totalb = 0;
        if (cudaMemGetInfo(&freeb, &totalb) == cudaSuccess) {
            if (64.0 * (double)nnz > 0.6 * (double)freeb) sc.device = 0;
        }
    }
    std::string err;
    const int sst = amgsetup::build(std::move(A), std::move(wv), sc, H, err);
    if (sst != amgsetup::SETUP_OK) {
        set_err(err);
        return sst == amgsetup::SETUP_ERR_ARG ? AMG_ERR_ARG : AMG_ERR_NOT_SPD;
    }
    return AMG_OK;
}

// INVK factors of every non-coarsest level (smoother == 1) and of the
// coarsest (coarse CG preconditioned by them, coarse_prec == 1), in the parallel
// block-Jacobi setting: the blocks are the ranks' rows (rank_bounds, level 0; R18 above), or
// cfg.invk_blocks equal level-0 blocks; HINVK factors A_pp, l1-INVK A_pp + D_l1,p.  Host,
// levels in parallel (each factorisation is a sequential row recurrence).
int invk_build(const amg_config_t& cfg, amgsetup::Hierarchy& H, const std::vector<int64_t>& rank_bounds) {
    const int nlv = (int)H.lv.size();
    const bool smooth = cfg.smoother == 1, coarse = cfg.coarse_solver == 1 && cfg.coarse_prec == 1;
    if (!smooth && !coarse) return AMG_OK;
    std::vector<int64_t> b0 = rank_bounds;
    const int64_t n0 = H.lv[0].A.nrows;
    if (cfg.invk_blocks > 0) {
        b0.assign(cfg.invk_blocks + 1, 0);
        for (int g = 0; g <= cfg.invk_blocks; ++g) b0[g] = n0 * g / cfg.invk_blocks;
    }
    const bool blocks = b0.size() > 2;
    const std::vector<std::vector<int32_t>> own =
        blocks ? amgsetup::level_blocks(H, b0) : std::vector<std::vector<int32_t>>(nlv);
    int bad = 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(max : bad)
    for (int l = 0; l < nlv; ++l) {
        if (l == nlv - 1 ? !coarse : !smooth) continue;
        const amgsetup::Csr& Al = H.lv[l].A;
        // "a single level of fill-in in the inversion" on every level, unless the
        // non-paper invk_dense_cut knob drops the fill of dense levels
        const int f = (cfg.invk_dense_cut > 0 && (double)Al.nnz() > (double)cfg.invk_dense_cut * (double)Al.nrows)
                          ? 0 : cfg.invk_fill;
        const amgsetup::Csr B = amgsetup::block_diagonal_part(Al, own[l], cfg.invk_l1 == 1);
        if (!amgsetup::invk_factors(B, f, H.lv[l].Wd, H.lv[l].Z)) bad = 1;
    }
    if (bad) {
        set_err("amg_hierarchy_build: INVK: non-positive IC(0) pivot");
        return AMG_ERR_NOT_SPD;
    }
    amgsetup::tmark("INVK factors");
    return AMG_OK;
}

// ---------------------------------------------------- plan (de)serialisation
struct Blob {
    std::vector<char> b;
    size_t pos = 0;
    template <class T>
    void put(const T& v) {
        const char* p = (const char*)&v;
        b.insert(b.end(), p, p + sizeof(T));
    }
    template <class T>
    void putv(const std::vector<T>& v) {
        put<int64_t>((int64_t)v.size());
        const char* p = (const char*)v.data();
        b.insert(b.end(), p, p + v.size() * sizeof(T));
    }
    template <class T>
    T get() {
        T v;
        std::memcpy(&v, b.data() + pos, sizeof(T));
        pos += sizeof(T);
        return v;
    }
    template <class T>
    void getv(std::vector<T>& v) {
        const int64_t n = get<int64_t>();
        v.resize(n);
        std::memcpy(v.data(), b.data() + pos, n * sizeof(T));
        pos += n * sizeof(T);
    }
    void put_csr(const amgsetup::Csr& M) {
        put(M.nrows);
        put(M.ncols);
        putv(M.rp);
        putv(M.ci);
        putv(M.v);
    }
    void get_csr(amgsetup::Csr& M) {
        M.nrows = get<int64_t>();
        M.ncols = get<int64_t>();
        getv(M.rp);
        getv(M.ci);
        getv(M.v);
    }
};

void serialize(const amgsetup::RankPlan& P, const std::vector<double>& cinv, const std::vector<int32_t>* agg_own,
               int nl, Blob& B) {
    B.put<int32_t>(P.rank);
    B.put<int32_t>(P.nranks);
    B.put<int32_t>((int32_t)P.lv.size());
    for (const auto& L : P.lv) {
        B.put<int32_t>(L.replicated ? 1 : 0);
        B.put(L.n_global);
        B.put(L.own_begin);
        B.put(L.own_end);
        B.put(L.comp_begin);
        B.put(L.comp_end);
        B.put(L.win_begin);
        B.put(L.win_end);
        B.put(L.rst_begin);
        B.put(L.rst_end);
        B.putv(L.recv_off);
        B.putv(L.recv_ids);
        B.putv(L.send_off);
        B.putv(L.send_ids);
        B.put_csr(L.A);
        B.put_csr(L.P);
        B.put_csr(L.R);
        B.putv(L.m);
        B.put_csr(L.Wd);
        B.put_csr(L.Z);
    }
    B.putv(cinv);
    for (int l = 0; l + 1 < nl; ++l) B.putv(agg_own[l]);
}

void deserialize(Blob& B, amgsetup::RankPlan& P, std::vector<double>& cinv, std::vector<std::vector<int32_t>>& agg) {
    P.rank = B.get<int32_t>();
    P.nranks = B.get<int32_t>();
    const int nl = B.get<int32_t>();
    P.lv.resize(nl);
    for (auto& L : P.lv) {
        L.replicated = B.get<int32_t>() != 0;
        L.n_global = B.get<int64_t>();
        L.own_begin = B.get<int64_t>();
        L.own_end = B.get<int64_t>();
        L.comp_begin = B.get<int64_t>();
        L.comp_end = B.get<int64_t>();
        L.win_begin = B.get<int64_t>();
        L.win_end = B.get<int64_t>();
        L.rst_begin = B.get<int64_t>();
        L.rst_end = B.get<int64_t>();
        B.getv(L.recv_off);
        B.getv(L.recv_ids);
        B.getv(L.send_off);
        B.getv(L.send_ids);
        B.get_csr(L.A);
        B.get_csr(L.P);
        B.get_csr(L.R);
        B.getv(L.m);
        B.get_csr(L.Wd);
        B.get_csr(L.Z);
    }
    B.getv(cinv);
    agg.assign(nl > 0 ? nl - 1 : 0, {});
    for (int l = 0; l + 1 < nl; ++l) B.getv(agg[l]);
}

// NCCL point-to-point of a host byte buffer through a device staging buffer.
int nccl_send_bytes(amg_ctx_s* c, const std::vector<char>& buf, int peer) {
    int64_t n = (int64_t)buf.size();
    char* d = nullptr;
    CK(cudaMalloc(&d, std::max<int64_t>(n, 8) + 8));
    CK(h2d_sync(d, &n, 8));
    if (n) CK(h2d_sync(d + 8, buf.data(), n));
    NK(ncclSend(d, 8, ncclChar, peer, c->nccl, c->stream));
    if (n) NK(ncclSend(d + 8, n, ncclChar, peer, c->nccl, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    cudaFree(d);
    return AMG_OK;
}

int nccl_recv_bytes(amg_ctx_s* c, std::vector<char>& buf, int peer) {
    int64_t* dn = nullptr;
    CK(cudaMalloc(&dn, 8));
    NK(ncclRecv(dn, 8, ncclChar, peer, c->nccl, c->stream));
    int64_t n = 0;
    CK(cudaMemcpyAsync(&n, dn, 8, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    cudaFree(dn);
    buf.resize(n);
    if (n) {
        char* d = nullptr;
        CK(cudaMalloc(&d, n));
        NK(ncclRecv(d, n, ncclChar, peer, c->nccl, c->stream));
        CK(cudaMemcpyAsync(buf.data(), d, n, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        cudaFree(d);
    }
    return AMG_OK;
}

template <class T>
void blob_put_array(Blob& B, const T* p, int64_t n) {
    B.put<int64_t>(n);
    const char* c = (const char*)p;
    B.b.insert(B.b.end(), c, c + n * sizeof(T));
}


// ---------------------------------------------------- distributed setup (NEXT-1)
// NCCL transport of the distributed setup: an all-to-all of host byte buffers through device
// staging (sizes all-gathered, payloads by grouped send/recv on the context stream).
struct NcclComm : amgsetup::Comm {
    amg_ctx_s* c = nullptr;
    bool ok = true;
    std::string what;
    int rank() const override { return c->rank; }
    int size() const override { return c->nranks; }
    bool fail(const std::string& w) {
        if (ok) what = w;
        ok = false;
        return false;
    }
    bool alltoallv(const std::vector<std::vector<char>>& out, std::vector<std::vector<char>>& in) override {
        const int np = c->nranks, me = c->rank;
        in.assign(np, {});
        if (!ok) return false;
        std::vector<int64_t> mine(np), all((size_t)np * np);
        for (int q = 0; q < np; ++q) mine[q] = (int64_t)out[q].size();
        int64_t* dsz = nullptr;
        if (cudaMalloc(&dsz, sizeof(int64_t) * (size_t)np * (np + 1)) != cudaSuccess) return fail("cudaMalloc");
        h2d_sync(dsz, mine.data(), sizeof(int64_t) * np);
        if (ncclAllGather(dsz, dsz + np, np, ncclInt64, c->nccl, c->stream) != ncclSuccess)
            return cudaFree(dsz), fail("ncclAllGather (setup sizes)");
        if (cudaStreamSynchronize(c->stream) != cudaSuccess) return cudaFree(dsz), fail("setup sizes sync");
        cudaMemcpy(all.data(), dsz + np, sizeof(int64_t) * (size_t)np * np, cudaMemcpyDeviceToHost);
        cudaFree(dsz);
        int64_t stot = 0, rtot = 0;
        std::vector<int64_t> soff(np + 1, 0), roff(np + 1, 0);
        for (int q = 0; q < np; ++q) {
            const int64_t sq = q == me ? 0 : mine[q], rq = q == me ? 0 : all[(size_t)q * np + me];
            soff[q + 1] = soff[q] + sq;
            roff[q + 1] = roff[q] + rq;
        }
        stot = soff[np];
        rtot = roff[np];
        char *ds = nullptr, *dr = nullptr;
        if (cudaMalloc(&ds, std::max<int64_t>(stot, 8)) != cudaSuccess ||
            cudaMalloc(&dr, std::max<int64_t>(rtot, 8)) != cudaSuccess)
            return cudaFree(ds), fail("cudaMalloc (setup payload)");
        for (int q = 0; q < np; ++q)
            if (q != me && mine[q]) h2d_sync(ds + soff[q], out[q].data(), mine[q]);
        bool nok = ncclGroupStart() == ncclSuccess;
        for (int q = 0; q < np; ++q) {
            if (q == me) continue;
            if (soff[q + 1] > soff[q])
                nok &= ncclSend(ds + soff[q], soff[q + 1] - soff[q], ncclChar, q, c->nccl, c->stream) == ncclSuccess;
            if (roff[q + 1] > roff[q])
                nok &= ncclRecv(dr + roff[q], roff[q + 1] - roff[q], ncclChar, q, c->nccl, c->stream) == ncclSuccess;
        }
        nok &= ncclGroupEnd() == ncclSuccess;
        nok &= cudaStreamSynchronize(c->stream) == cudaSuccess;
        for (int q = 0; q < np && nok; ++q) {
            if (q == me) {
                in[q] = out[q];
                continue;
            }
            in[q].resize(roff[q + 1] - roff[q]);
            if (!in[q].empty()) cudaMemcpy(in[q].data(), dr + roff[q], in[q].size(), cudaMemcpyDeviceToHost);
        }
        cudaFree(ds);
        cudaFree(dr);
        if (!nok) return fail("ncclSend/ncclRecv (setup payload)");
        return true;
    }
};

// The INVK factors of a rank's plan (smoother == 1 / the coarse CG's HINVK): block-diagonal over
// the ranks (HINVK / l1-INVK), so a distributed level factors its own diagonal
// block (its rows, its columns) and a replicated level the whole level with the owners' blocks --
// the same numbers as invk_build on the whole hierarchy sliced by partition().
int plan_invk(const amg_config_t& cfg, amgsetup::RankPlan& P, const std::vector<std::vector<int64_t>>& bounds,
              const LevelStats& S) {
    const int nl = (int)P.lv.size();
    const bool smooth = cfg.smoother == 1, coarse = cfg.coarse_solver == 1 && cfg.coarse_prec == 1;
    for (int l = 0; l < nl; ++l) {
        if (l == nl - 1 ? !coarse : !smooth) continue;
        amgsetup::RankLevel& L = P.lv[l];
        const int f = (cfg.invk_dense_cut > 0 && (double)S.nnzA[l] > (double)cfg.invk_dense_cut * (double)S.n[l])
                          ? 0 : cfg.invk_fill;
        if (L.replicated) {  // win = [0, n): global frame; blocks = the owners of this level
            std::vector<int32_t> own(L.n_global);
            for (size_t g = 0; g + 1 < bounds[l].size(); ++g)
                for (int64_t i = bounds[l][g]; i < bounds[l][g + 1]; ++i) own[i] = (int32_t)g;
            const amgsetup::Csr B = amgsetup::block_diagonal_part(L.A, bounds[l].size() > 2 ? own : std::vector<int32_t>(),
                                                                  cfg.invk_l1 == 1);
            if (!amgsetup::invk_factors(B, f, L.Wd, L.Z)) return AMG_ERR_NOT_SPD;
            continue;
        }
        // own diagonal block in local indices (window columns [o0, o1) are the owned rows)
        const int64_t n = L.own_end - L.own_begin, o0 = L.own_begin - L.win_begin, o1 = o0 + n;
        amgsetup::Csr B;
        B.nrows = B.ncols = n;
        B.rp.assign(n + 1, 0);
        for (int64_t r = 0; r < n; ++r) {
            double dl1 = 0.0;
            if (cfg.invk_l1 == 1)
                for (int64_t k = L.A.rp[r]; k < L.A.rp[r + 1]; ++k)
                    if (L.A.ci[k] < o0 || L.A.ci[k] >= o1) dl1 = dl1 + std::fabs(L.A.v[k]);
            for (int64_t k = L.A.rp[r]; k < L.A.rp[r + 1]; ++k) {
                const int64_t cc = L.A.ci[k];
                if (cc < o0 || cc >= o1) continue;
                B.ci.push_back((int32_t)(cc - o0));
                B.v.push_back((cfg.invk_l1 == 1 && cc - o0 == r) ? L.A.v[k] + dl1 : L.A.v[k]);
            }
            B.rp[r + 1] = (int64_t)B.ci.size();
        }
        amgsetup::Csr Wd, Z;
        if (!amgsetup::invk_factors(B, f, Wd, Z)) return AMG_ERR_NOT_SPD;
        for (amgsetup::Csr* M : {&Wd, &Z}) {
            for (auto& cc : M->ci) cc = (int32_t)(cc + o0);
            M->ncols = L.win_end - L.win_begin;
        }
        L.Wd = std::move(Wd);
        L.Z = std::move(Z);
    }
    return AMG_OK;
}

struct DistOut {
    amgsetup::RankPlan plan;
    std::vector<double> cinv;
    std::vector<std::vector<int32_t>> agg;  // owned rows of every non-coarsest level
    LevelStats S;
    int st = AMG_OK;
    std::string err;
};

// One rank of the distributed setup: validation, build, plan, INVK factors, statistics.
void dist_rank(amgsetup::Comm& c, const amg_config_t& cfg, const std::vector<int64_t>& b0, amgsetup::Csr&& Al,
               std::vector<double>&& wl, bool validate, DistOut& o) {
    if (validate) {
        const int v = amgsetup::validate_distributed(c, b0, Al, wl, o.err);
        if (v != amgsetup::SETUP_OK) {
            o.st = v == amgsetup::SETUP_ERR_ARG ? AMG_ERR_ARG : AMG_ERR_NOT_SPD;
            return;
        }
    }
    amgsetup::DistHierarchy H;
    const int st = amgsetup::build_distributed(c, b0, std::move(Al), std::move(wl), setup_config(cfg), H, o.err);
    if (st != amgsetup::SETUP_OK) {
        o.st = st == amgsetup::SETUP_ERR_ARG ? AMG_ERR_ARG : AMG_ERR_NOT_SPD;
        return;
    }
    const int nl = (int)H.lv.size();
    std::vector<std::vector<int64_t>> bounds;
    for (auto& L : H.lv) {
        o.S.n.push_back(L.n);
        o.S.nnzA.push_back(L.nnzA);
        o.S.nnzP.push_back(L.nnzP);
        bounds.push_back(L.bounds);
    }
    for (int l = 0; l + 1 < nl; ++l) o.agg.push_back(H.lv[l].agg);
    o.cinv = H.coarse_inv;
    if (!amgsetup::partition_distributed(c, H, cfg.replicate_below_bytes, o.plan, o.err)) {
        o.st = AMG_ERR_ARG;
        return;
    }
    const int ist = plan_invk(cfg, o.plan, bounds, o.S);
    if (amgsetup::comm_allreduce_sum(c, ist ? 1 : 0)) {  // collective: every rank stops
        o.st = AMG_ERR_NOT_SPD;
        o.err = "INVK: non-positive IC(0) pivot";
        return;
    }
    // global nnz of the INVK factors (replicated levels: every rank holds all rows, count once)
    o.S.nnzWZ.assign(nl, 0);
    for (int l = 0; l < nl; ++l) {
        const auto& L = o.plan.lv[l];
        const int64_t mine = L.replicated ? (c.rank() == 0 ? L.Wd.nnz() + L.Z.nnz() : 0) : L.Wd.nnz() + L.Z.nnz();
        o.S.nnzWZ[l] = amgsetup::comm_allreduce_sum(c, mine);
    }
}

// amg_hierarchy_build's distributed path: loopback (one process, np threads) or NCCL ranks.
int build_dist_path(amg_hier_s* h, amg_ctx_s* ctx, const amg_config_t& cfg, int64_t n_global, int64_t row_begin,
                    int64_t row_end, const int64_t* rowptr, const int64_t* colind, const double* values,
                    const double* w) {
    const int np = h->np;
    auto to_local = [&](int64_t r0, int64_t r1, int64_t base, amgsetup::Csr& A, std::vector<double>& wl) -> bool {
        A.nrows = r1 - r0;
        A.ncols = n_global;
        A.rp.resize(A.nrows + 1);
        const int64_t k0 = rowptr[r0 - base];
        for (int64_t i = 0; i <= A.nrows; ++i) A.rp[i] = rowptr[r0 - base + i] - k0;
        const int64_t nnz = A.rp[A.nrows];
        A.ci.resize(nnz);
        A.v.assign(values + k0, values + k0 + nnz);
        bool ok = true;
        for (int64_t k = 0; k < nnz; ++k) {
            const int64_t cc = colind[k0 + k];
            ok &= (cc >= 0 && cc < n_global);
            A.ci[k] = (int32_t)cc;
        }
        wl.assign(A.nrows, 1.0);
        if (w) std::copy(w + (r0 - base), w + (r1 - base), wl.begin());
        return ok;
    };
    std::vector<DistOut> outs;
    if (h->loopback) {
        if (rowptr[0] != 0) {
            set_err("amg_hierarchy_build: rowptr[0] must be 0");
            return AMG_ERR_ARG;
        }
        std::vector<int64_t> b0(np + 1);
        for (int g = 0; g <= np; ++g) b0[g] = n_global * g / np;
        outs.resize(np);
        std::vector<char> okc(np, 1);
        amgsetup::run_loopback(np, [&](amgsetup::Comm& c) {
            const int r = c.rank();
            amgsetup::Csr A;
            std::vector<double> wl;
            okc[r] = to_local(b0[r], b0[r + 1], 0, A, wl);
            dist_rank(c, cfg, b0, std::move(A), std::move(wl), true, outs[r]);
        });
        for (int r = 0; r < np; ++r)
            if (!okc[r] || outs[r].st != AMG_OK) {
                set_err("amg_hierarchy_build (distributed setup, rank " + std::to_string(r) +
                        "): " + (okc[r] ? outs[r].err : std::string("column index out of range")));
                return okc[r] ? outs[r].st : AMG_ERR_ARG;
            }
    } else {
        NcclComm c;
        c.c = ctx;
        std::vector<int64_t> mine{row_begin, row_end};
        // the row blocks of all ranks (rank order, contiguous, covering [0, n))
        std::vector<std::vector<char>> out(np), in;
        for (int q = 0; q < np; ++q) {
            out[q].resize(16);
            std::memcpy(out[q].data(), mine.data(), 16);
        }
        c.alltoallv(out, in);
        if (!c.ok) {
            set_err("amg_hierarchy_build: " + c.what);
            return AMG_ERR_NCCL;
        }
        std::vector<int64_t> b0(np + 1, 0);
        bool okb = true;
        for (int q = 0; q < np; ++q) {
            int64_t rb, re;
            std::memcpy(&rb, in[q].data(), 8);
            std::memcpy(&re, in[q].data() + 8, 8);
            okb &= (rb == b0[q] && re >= rb);
            b0[q + 1] = re;
        }
        if (!okb || b0[np] != n_global) {
            set_err("amg_hierarchy_build: row blocks must be contiguous, in rank order and cover [0, n_global)");
            return AMG_ERR_ARG;
        }
        if (rowptr[0] != 0) {
            set_err("amg_hierarchy_build: rowptr[0] must be 0");
            return AMG_ERR_ARG;
        }
        amgsetup::Csr A;
        std::vector<double> wl;
        if (!to_local(row_begin, row_end, row_begin, A, wl)) {
            set_err("amg_hierarchy_build: column index out of range");
            return AMG_ERR_ARG;
        }
        outs.resize(1);
        dist_rank(c, cfg, b0, std::move(A), std::move(wl), true, outs[0]);
        if (!c.ok) {
            set_err("amg_hierarchy_build (distributed setup): " + c.what);
            return AMG_ERR_NCCL;
        }
        if (outs[0].st != AMG_OK) {
            set_err("amg_hierarchy_build (distributed setup): " + outs[0].err);
            return outs[0].st;
        }
    }
    amgsetup::tmark("distributed setup + plans");
    hier_stats(h, outs[0].S);
    const int nl = (int)outs[0].S.n.size();
    h->ranks.resize(outs.size());
    int st;
    for (size_t g = 0; g < outs.size(); ++g)
        if ((st = upload_rank(h, outs[g].plan, outs[g].cinv, h->ranks[g]))) return st;
    amgsetup::tmark("device formats + upload");
    h->agg.assign(nl > 0 ? nl - 1 : 0, {});
    for (int l = 0; l + 1 < nl; ++l)
        for (auto& o : outs) h->agg[l].insert(h->agg[l].end(), o.agg[l].begin(), o.agg[l].end());
    if (h->loopback) {
        for (size_t g = 0; g < outs.size(); ++g) h->ranks[g].user_off = outs[g].plan.lv[0].own_begin;
        h->lvl_own_begin.assign(nl, 0);
        h->lvl_own_end = h->lvl_n;
        h->n0_local = n_global;
    } else {
        h->ranks[0].user_off = 0;
        for (auto& L : outs[0].plan.lv) {
            h->lvl_own_begin.push_back(L.own_begin);
            h->lvl_own_end.push_back(L.own_end);
        }
        h->n0_local = row_end - row_begin;
    }
    for (int l = 0; l < nl; ++l)
        h->lvl_fmt.push_back(l + 1 < nl ? (h->ranks[0].lv[l].A.perm ? FMT_SELL_SIGMA : h->ranks[0].lv[l].A.fmt)
                                        : FMT_DENSE);
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
    c->replicate_below_bytes = 128ll << 20;
    c->setup_threads = 0;
    c->use_graphs = 1;
    c->emulate_ranks = 1;
    c->krylov = 0;
    c->coarse_solver = 0;
    c->coarse_maxit = 30;
    c->coarse_rtol = 1e-4;
    c->cycle = 0;
    c->setup_device = 1;
    c->tail_rows = 0;
    c->tail_bytes = 0;
    c->smoother = 0;
    c->invk_fill = 1;
    c->invk_l1 = 0;
    c->invk_blocks = 0;
    c->invk_dense_cut = 0;
    c->coarse_prec = 0;
    c->setup_distributed = -1;
}

int amg_nccl_unique_id(void* out128) {
    if (!out128) return AMG_ERR_ARG;
    ncclUniqueId id;
    NK(ncclGetUniqueId(&id));
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    std::memcpy(out128, &id, 128);
    return AMG_OK;
}

int amg_ctx_create(int device, int rank, int nranks, const void* nccl_unique_id, void* cuda_stream,
                   amg_ctx_t* out) {
    if (!out || nranks < 1 || rank < 0 || rank >= nranks || (nranks > 1 && !nccl_unique_id)) {
        set_err("amg_ctx_create: bad rank/nranks, null out, or missing NCCL unique id");
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
    if (nranks > 1 || nccl_unique_id) {  // nranks == 1 with an id: a one-rank communicator (loopback transport)
        ncclUniqueId id;
        std::memcpy(&id, nccl_unique_id, sizeof(id));
        ncclResult_t r = ncclCommInitRank(&c->nccl, nranks, id, rank);
        if (r != ncclSuccess) {
            if (c->own_stream) cudaStreamDestroy(c->stream);
            delete c;
            set_err(std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
            return AMG_ERR_NCCL;
        }
    }
    *out = c;
    return AMG_OK;
}

int amg_ctx_destroy(amg_ctx_t c) {
    if (!c) return AMG_OK;
    {
        // hierarchies still alive (a caller error the header warns about, and a garbage-collection
        // order Python can produce): release their graphs now and orphan them, so the communicator
        // is not held by captured NCCL work; amg_hierarchy_destroy still frees them later
        std::lock_guard<std::mutex> g(c->hiers_mu);
        for (amg_hier_s* h : c->hiers) {
            std::lock_guard<std::recursive_mutex> hg(h->mu);
            cudaSetDevice(h->device);
            cudaStreamSynchronize(c->stream);
            h->release_graphs();
            h->release_lsa();  // the window belongs to the communicator
            h->ctx = nullptr;
        }
        c->hiers.clear();
    }
    if (c->nccl) ncclCommDestroy(c->nccl);
    if (c->own_stream) cudaStreamDestroy(c->stream);
    delete c;
    return AMG_OK;
}

int amg_hierarchy_build(amg_ctx_t ctx, int64_t n_global, int64_t row_begin, int64_t row_end, const int64_t* rowptr,
                        const int64_t* colind, const double* values, const double* w, const amg_config_t* cfg_in,
                        amg_hier_t* out) {
    NvtxRange nvtx_("amg_hierarchy_build");
    auto t0 = std::chrono::steady_clock::now();
    if (!ctx || !out || !rowptr || !colind || !values || n_global <= 0 || row_begin < 0 || row_end < row_begin ||
        row_end > n_global) {
        set_err("amg_hierarchy_build: null argument, empty matrix or bad row block");
        return AMG_ERR_ARG;
    }
    *out = nullptr;
    amg_config_t cfg;
    amg_config_default(&cfg);
    if (cfg_in) cfg = *cfg_in;
    // AMG_EAGER=1 forces eager launches (ncu cannot profile kernels inside graphs
    // that contain conditional nodes)
    if (const char* ev = std::getenv("AMG_EAGER")) cfg.use_graphs = (ev[0] == '1') ? 0 : cfg.use_graphs;
    if ((cfg.krylov != 0 && cfg.krylov != 1) || (cfg.coarse_solver != 0 && cfg.coarse_solver != 1) ||
        cfg.coarse_maxit < 1 || !(cfg.coarse_rtol >= 0.0) || (cfg.cycle != 0 && cfg.cycle != 1)) {
        set_err("amg_hierarchy_build: krylov / coarse_solver / cycle must be 0 or 1, coarse_maxit >= 1, "
                "coarse_rtol >= 0");
        return AMG_ERR_ARG;
    }
    if ((cfg.smoother != 0 && cfg.smoother != 1) || cfg.invk_fill < 0) {
        set_err("amg_hierarchy_build: smoother must be 0 (l1-Jacobi) or 1 (INVK), invk_fill >= 0");
        return AMG_ERR_ARG;
    }
    if ((cfg.invk_l1 != 0 && cfg.invk_l1 != 1) || cfg.invk_blocks < 0 || cfg.invk_dense_cut < 0 ||
        (cfg.coarse_prec != 0 && cfg.coarse_prec != 1)) {
        set_err("amg_hierarchy_build: invk_l1 / coarse_prec must be 0 or 1, invk_blocks / invk_dense_cut >= 0");
        return AMG_ERR_ARG;
    }
    {
        const int npart = ctx->nranks > 1 ? ctx->nranks : std::max(1, cfg.emulate_ranks);
        if (npart > 1 && cfg.invk_blocks != 0 && cfg.invk_blocks != npart) {
            set_err("amg_hierarchy_build: with several ranks the INVK blocks are the ranks' (invk_blocks 0 or np)");
            return AMG_ERR_ARG;
        }
    }
    CK(cudaSetDevice(ctx->device));
    const int nr = ctx->nranks;
    if (nr == 1 && (row_begin != 0 || row_end != n_global)) {
        set_err("amg_hierarchy_build: a single-rank context must own all rows");
        return AMG_ERR_ARG;
    }
    if (nr > 1 && cfg.emulate_ranks > 1) {
        set_err("amg_hierarchy_build: emulate_ranks is for single-rank contexts");
        return AMG_ERR_ARG;
    }
    const int np = nr > 1 ? nr : std::max(1, cfg.emulate_ranks);
    auto* h = new amg_hier_s();
    h->ctx = ctx;
    h->device = ctx->device;
    h->cfg = cfg;
    h->np = np;
    h->loopback = (nr == 1 && np > 1);
    auto fail = [&](int code) {
        delete h;
        return code;
    };
    int st = AMG_OK;
    // the distributed setup (NEXT-1): default for NCCL contexts, opt-in for loopback
    const bool dist_setup = np > 1 && (cfg.setup_distributed == 1 || (cfg.setup_distributed < 0 && nr > 1));
    if (dist_setup) {
        if ((st = build_dist_path(h, ctx, cfg, n_global, row_begin, row_end, rowptr, colind, values, w)))
            return fail(st);
    } else if (nr == 1) {
        amgsetup::Hierarchy H;
        // one process, l1-Jacobi: a GPU-built hierarchy stays on the device (formats converted there)
        H.keep_device = (np == 1 && cfg.smoother == 0 && !(cfg.coarse_solver == 1 && cfg.coarse_prec == 1));
        if ((st = host_setup(n_global, rowptr, colind, values, w, cfg, H))) {
            set_err("amg_hierarchy_build: " + g_err);
            return fail(st);
        }
        {
            std::vector<int64_t> b0(np + 1);
            for (int g = 0; g <= np; ++g) b0[g] = n_global * g / np;
            if ((st = invk_build(cfg, H, b0))) return fail(st);
        }
        amgsetup::tmark("(hierarchy built)");
        std::vector<int64_t> bounds(np + 1);
        for (int g = 0; g <= np; ++g) bounds[g] = n_global * g / np;
        std::vector<amgsetup::RankPlan> plans;
        std::string err;
        hier_stats(h, H);
        const size_t nlv = H.lv.size();
        for (size_t l = 0; l + 1 < nlv; ++l) h->agg.push_back(H.lv[l].agg);
        // persistent tail: the deep levels (n_l <= tail_rows, at least one non-coarsest)
        // run as one cooperative kernel; single process, direct coarsest solve
        const bool tail_ok = np == 1 && cfg.coarse_solver == 0 && cfg.smoother == 0 && nlv >= 3 &&
                             (cfg.cycle == 0 || cfg.pre_sweeps == 1);
        if (tail_ok && cfg.tail_bytes > 0) {
            // cluster tail: the deepest levels whose operators (A, A diag(m), P-bar, R, the dense
            // inverse) together take at most tail_bytes
            double tot = 8.0 * (double)H.lv[nlv - 1].A.nrows * (double)H.lv[nlv - 1].A.nrows;
            for (int l = (int)nlv - 2; l >= 1; --l) {
                tot += 12.0 * (2.0 * (double)H.lv[l].A.nnz() + (double)H.lv[l].P.nnz() + (double)H.lv[l].R.nnz());
                if (tot > (double)cfg.tail_bytes) break;
                h->tail_level = l;
            }
            h->tail_cluster = h->tail_level > 0;
        } else if (tail_ok && cfg.tail_rows > 0) {
            for (size_t l = 1; l + 1 < nlv; ++l)
                if (H.lv[l].A.nrows <= cfg.tail_rows) {
                    h->tail_level = (int)l;
                    break;
                }
        }
        if (np == 1) {
            // one rank: the plan is the whole hierarchy (level 0 .. L-1 owned, the coarsest
            // replicated, no halo) — move the operators instead of slicing copies
            plans.resize(1);
            amgsetup::RankPlan& P = plans[0];
            P.rank = 0;
            P.nranks = 1;
            P.lv.resize(nlv);
            for (size_t l = 0; l < nlv; ++l) {
                amgsetup::RankLevel& Lv = P.lv[l];
                amgsetup::Level& S = H.lv[l];
                Lv.replicated = (l + 1 == nlv);
                Lv.n_global = S.A.nrows;
                Lv.own_begin = Lv.comp_begin = Lv.win_begin = 0;
                Lv.own_end = Lv.comp_end = Lv.win_end = S.A.nrows;
                if (l + 1 < nlv) {
                    Lv.rst_begin = 0;
                    Lv.rst_end = H.lv[l + 1].A.nrows;
                }
                Lv.recv_off.assign(2, 0);
                Lv.send_off.assign(2, 0);
                Lv.A = std::move(S.A);
                Lv.P = std::move(S.P);
                Lv.R = std::move(S.R);
                Lv.m = std::move(S.m);
                Lv.Wd = std::move(S.Wd);
                Lv.Z = std::move(S.Z);
            }
        } else if (!amgsetup::partition(H, bounds, cfg.replicate_below_bytes, plans, err)) {
            set_err("amg_hierarchy_build: " + err);
            return fail(AMG_ERR_ARG);
        }
        amgsetup::tmark("partition");
        h->ranks.resize(np);
        const amgsetup::DeviceKeep* dk = (np == 1 && !H.dev.A.empty()) ? &H.dev : nullptr;
        for (int g = 0; g < np; ++g)
            if ((st = upload_rank(h, plans[g], H.coarse_inv, h->ranks[g], dk))) {
                H.dev.free_all();
                return fail(st);
            }
        H.dev.free_all();
        if (h->tail_level > 0 && (st = build_tail(h))) return fail(st);
        amgsetup::tmark("device formats + upload");
        for (int g = 0; g < np; ++g) h->ranks[g].user_off = h->loopback ? plans[g].lv[0].own_begin : 0;
        h->lvl_own_begin.assign(H.lv.size(), 0);
        h->lvl_own_end = h->lvl_n;
        h->n0_local = n_global;
        for (size_t l = 0; l < H.lv.size(); ++l)
            h->lvl_fmt.push_back(l + 1 < H.lv.size()
                                     ? (h->ranks[0].lv[l].A.perm ? FMT_SELL_SIGMA : h->ranks[0].lv[l].A.fmt)
                                     : FMT_DENSE);
    } else {
        // ---- NCCL: gather the matrix on rank 0, build there, send each rank its plan
        const int me = ctx->rank;
        const int64_t nloc = row_end - row_begin;
        Blob mine;
        mine.put(row_begin);
        mine.put(row_end);
        blob_put_array(mine, rowptr, nloc + 1);
        blob_put_array(mine, colind, rowptr[nloc]);
        blob_put_array(mine, values, rowptr[nloc]);
        std::vector<double> wl(nloc, 1.0);
        if (w) std::copy(w, w + nloc, wl.begin());
        mine.putv(wl);
        Blob myplan;
        if (me == 0) {
            std::vector<Blob> parts(nr);
            parts[0] = mine;
            for (int q = 1; q < nr; ++q)
                if ((st = nccl_recv_bytes(ctx, parts[q].b, q))) return fail(st);
            std::vector<int64_t> gr(n_global + 1, 0), gc;
            std::vector<double> gv, gw(n_global, 1.0);
            std::vector<int64_t> bounds(nr + 1, 0);
            for (int q = 0; q < nr; ++q) {
                Blob& B = parts[q];
                const int64_t rb = B.get<int64_t>(), re = B.get<int64_t>();
                std::vector<int64_t> rp, ci;
                std::vector<double> v, ww;
                B.getv(rp);
                B.getv(ci);
                B.getv(v);
                B.getv(ww);
                if (q > 0 && rb != bounds[q]) {
                    set_err("amg_hierarchy_build: row blocks must be contiguous and in rank order");
                    return fail(AMG_ERR_ARG);
                }
                bounds[q] = rb;
                bounds[q + 1] = re;
                const int64_t off = (int64_t)gc.size();
                for (int64_t i = 0; i < re - rb; ++i) gr[rb + i + 1] = off + rp[i + 1];
                gc.insert(gc.end(), ci.begin(), ci.end());
                gv.insert(gv.end(), v.begin(), v.end());
                std::copy(ww.begin(), ww.end(), gw.begin() + rb);
            }
            if (bounds[0] != 0 || bounds[nr] != n_global) {
                set_err("amg_hierarchy_build: row blocks do not cover [0, n_global)");
                return fail(AMG_ERR_ARG);
            }
            std::vector<Blob>().swap(parts);  // the gathered blobs are no longer needed
            amgsetup::Hierarchy H;
            st = host_setup(n_global, gr.data(), gc.data(), gv.data(), gw.data(), cfg, H);
            std::vector<int64_t>().swap(gr);  // host_setup keeps its own copy of A
            std::vector<int64_t>().swap(gc);
            std::vector<double>().swap(gv);
            if (st) {
                set_err("amg_hierarchy_build: " + g_err);
                return fail(st);
            }
            if ((st = invk_build(cfg, H, bounds))) return fail(st);
            std::vector<amgsetup::RankPlan> plans;
            std::string err;
            if (!amgsetup::partition(H, bounds, cfg.replicate_below_bytes, plans, err)) {
                set_err("amg_hierarchy_build: " + err);
                return fail(AMG_ERR_ARG);
            }
            hier_stats(h, H);
            Blob stats;
            stats.putv(h->lvl_n);
            stats.putv(h->lvl_nnzA);
            stats.putv(h->lvl_nnzP);
            stats.put(h->opc);
            stats.put(h->avg_cr);
            stats.put(h->bytes_v);
            stats.put(h->bytes_it);
            const int nl = (int)H.lv.size();
            for (int q = nr - 1; q >= 0; --q) {
                std::vector<std::vector<int32_t>> agg_own(nl > 0 ? nl - 1 : 0);
                for (int l = 0; l + 1 < nl; ++l)
                    agg_own[l].assign(H.lv[l].agg.begin() + plans[q].lv[l].own_begin,
                                      H.lv[l].agg.begin() + plans[q].lv[l].own_end);
                Blob B;
                B.b = stats.b;
                serialize(plans[q], H.coarse_inv, agg_own.data(), nl, B);
                if (q == 0) myplan = std::move(B);
                else if ((st = nccl_send_bytes(ctx, B.b, q))) return fail(st);
            }
        } else {
            if ((st = nccl_send_bytes(ctx, mine.b, 0))) return fail(st);
            if ((st = nccl_recv_bytes(ctx, myplan.b, 0))) return fail(st);
        }
        myplan.getv(h->lvl_n);
        myplan.getv(h->lvl_nnzA);
        myplan.getv(h->lvl_nnzP);
        h->opc = myplan.get<double>();
        h->avg_cr = myplan.get<double>();
        h->bytes_v = myplan.get<double>();
        h->bytes_it = myplan.get<double>();
        amgsetup::RankPlan P;
        std::vector<double> cinv;
        deserialize(myplan, P, cinv, h->agg);
        h->ranks.resize(1);
        if ((st = upload_rank(h, P, cinv, h->ranks[0]))) return fail(st);
        h->ranks[0].user_off = 0;
        for (auto& L : P.lv) {
            h->lvl_own_begin.push_back(L.own_begin);
            h->lvl_own_end.push_back(L.own_end);
        }
        h->n0_local = P.lv[0].own_end - P.lv[0].own_begin;
        for (size_t l = 0; l < P.lv.size(); ++l)
            h->lvl_fmt.push_back(l + 1 < P.lv.size() ? h->ranks[0].lv[l].A.fmt : FMT_DENSE);
    }
    mark_persistent(h);
    if (const char* gm = std::getenv("AMG_MULTI_GRAPH"))
        if (h->multi() && std::strcmp(gm, "iter") == 0) h->graph_mode = GM_ITER;
    if (cudaMallocHost((void**)&h->st_host, sizeof(PcgState)) != cudaSuccess) {
        set_err("cudaMallocHost failed");
        return fail(AMG_ERR_OOM);
    }
    cudaEventCreate(&h->ev0);
    cudaEventCreate(&h->ev1);
    // second stream: halo exchanges (multi-rank) / the smoothing branch of compact levels
    CK(cudaStreamCreateWithFlags(&h->comm, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming));
    CK(cudaDeviceSynchronize());
    if (int e = lsa_setup(h)) return fail(e);
    if (std::getenv("AMG_DEBUG_CHECKSUM")) debug_checksums(h);
    h->setup_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    {
        std::lock_guard<std::mutex> g(ctx->hiers_mu);
        ctx->hiers.insert(h);
    }
    *out = h;
    return AMG_OK;
}

int amg_hierarchy_destroy(amg_hier_t h) {
    if (h) {
        // the context may already be destroyed (a caller error the Python binding can hit at garbage
        // collection; amg_ctx_destroy then orphaned h, ctx = null): use the device recorded at build
        // time, and leave no error behind
        cudaSetDevice(h->device);
        if (amg_ctx_s* c = h->ctx) {
            std::lock_guard<std::mutex> g(c->hiers_mu);
            c->hiers.erase(h);
        }
        delete h;
        cudaGetLastError();
    }
    return AMG_OK;
}

int amg_solve(amg_hier_t h, const double* b_dev, double* x_dev, double rtol, int32_t maxit, amg_report_t* rep) {
    NvtxRange nvtx_("amg_solve");
    if (!h || !b_dev || !x_dev || rtol < 0.0 || maxit < 0) {
        set_err("amg_solve: bad argument");
        return AMG_ERR_ARG;
    }
    std::lock_guard<std::recursive_mutex> guard(h->mu);
    CK(cudaSetDevice(h->ctx->device));
    cudaStream_t s = h->ctx->stream;
    h->nccl_status = ncclSuccess;
    PcgState init{};
    init.rtol = rtol;
    init.maxit = maxit;
    *h->st_host = init;
    for (auto& R : h->ranks) CK(cudaMemcpyAsync(R.st, h->st_host, sizeof(PcgState), cudaMemcpyHostToDevice, s));
    CK(cudaEventRecord(h->ev0, s));
    if (h->cfg.use_graphs && h->graph_mode == GM_WHILE) {
        int e = ensure_solve_graph(h, b_dev, x_dev);
        if (e) return e;
        if ((e = take_nccl_status(h))) return e;
    }
    if (h->cfg.use_graphs && h->graph_mode == GM_ITER) {
        int e = ensure_iter_graph(h, x_dev);
        if (e) return e;
        if ((e = take_nccl_status(h))) return e;
    }
    if (h->cfg.use_graphs && h->graph_mode == GM_WHILE) {
        CK(cudaGraphLaunch(h->solve_exec, s));
        CK(cudaEventRecord(h->ev1, s));
        CK(cudaMemcpyAsync(h->st_host, h->ranks[0].st, sizeof(PcgState), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
    } else {
        // one graph per iteration (GM_ITER) or eager launches, one status read per iteration
        const bool it_graph = h->cfg.use_graphs && h->graph_mode == GM_ITER;
        Launch L{h, s};
        int e;
        enqueue_pcg_init(h, L, b_dev, x_dev, 0);
        if ((e = take_nccl_status(h))) return e;
        for (;;) {
            CK(cudaMemcpyAsync(h->st_host, h->ranks[0].st, sizeof(PcgState), cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            if (h->st_host->status != ST_RUNNING) break;
            if (it_graph) {
                CK(cudaGraphLaunch(h->iter_exec, s));
            } else {
                enqueue_pcg_body(h, L, x_dev, 0);
                if ((e = take_nccl_status(h))) return e;
            }
        }
        enqueue_pcg_final(h, L, x_dev);
        CK(cudaEventRecord(h->ev1, s));
        CK(cudaStreamSynchronize(s));
    }
    CK(cudaGetLastError());
    if (int e = take_lsa_err(h)) return e;
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

int amg_solve_host_batch(amg_hier_t h, int32_t nrhs, const double* B_host, double* X_host, double rtol,
                         int32_t maxit, amg_report_t* reps) {
    NvtxRange nvtx_("amg_solve_host_batch");
    if (!h || nrhs < 0 || (nrhs > 0 && (!B_host || !X_host)) || rtol < 0.0 || maxit < 0) {
        set_err("amg_solve_host_batch: bad argument");
        return AMG_ERR_ARG;
    }
    std::lock_guard<std::recursive_mutex> guard(h->mu);
    CK(cudaSetDevice(h->ctx->device));
    const int64_t n = h->n0_local;
    int code = AMG_OK;
    // NCCL ranks / eager launches: one solve after another (loopback pipelines like one rank)
    if (h->nccl_xport() || !h->cfg.use_graphs) {
        for (int32_t k = 0; k < nrhs; ++k) {
            const int c = amg_solve_host(h, B_host + k * n, X_host + k * n, rtol, maxit, reps ? reps + k : nullptr);
            if (c != AMG_OK && c != AMG_NOT_CONVERGED && c != AMG_ERR_BREAKDOWN) return c;
            if (code == AMG_OK) code = c;
        }
        return code;
    }
    int st;
    for (int q = 0; q < 2; ++q) {
        if (!h->bb[q] && (st = dev_alloc(&h->bb[q], n))) return st;
        if (!h->bx[q] && (st = dev_alloc(&h->bx[q], n))) return st;
        if (!h->batch_exec[q] && (st = build_solve_exec(h, h->bb[q], h->bx[q], &h->batch_exec[q]))) return st;
    }
    if (!h->cstream) CK(cudaStreamCreateWithFlags(&h->cstream, cudaStreamNonBlocking));
    if (!h->dstream) CK(cudaStreamCreateWithFlags(&h->dstream, cudaStreamNonBlocking));
    // separate copy streams: b_{k+1} must not queue behind x_k's copy (which waits for solve k)
    cudaStream_t s = h->ctx->stream, cs = h->cstream, ds = h->dstream;
    // every exit path (including a failing CK below) drains the three streams before the
    // pinned state array and the events go away: queued copies may still reference them
    struct BatchRes {
        cudaStream_t s, cs, ds;
        PcgState* sts = nullptr;
        cudaEvent_t h2d[2] = {}, solved[2] = {}, d2h[2] = {};
        ~BatchRes() {
            cudaStreamSynchronize(s);
            cudaStreamSynchronize(cs);
            cudaStreamSynchronize(ds);
            for (int q = 0; q < 2; ++q)
                for (cudaEvent_t e : {h2d[q], solved[q], d2h[q]})
                    if (e) cudaEventDestroy(e);
            if (sts) cudaFreeHost(sts);
        }
    } res{s, cs, ds};
    CK(cudaMallocHost((void**)&res.sts, sizeof(PcgState) * (size_t)(nrhs + 1)));
    PcgState* sts = res.sts;  // [0]: the initial state, [1 + k]: solve k's final state
    PcgState init{};
    init.rtol = rtol;
    init.maxit = maxit;
    sts[0] = init;
    cudaEvent_t* h2d = res.h2d;
    cudaEvent_t* solved = res.solved;
    cudaEvent_t* d2h = res.d2h;
    for (int q = 0; q < 2; ++q) {
        CK(cudaEventCreateWithFlags(&h2d[q], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&solved[q], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&d2h[q], cudaEventDisableTiming));
    }
    RankState& R = h->ranks[0];
    CK(cudaEventRecord(h->ev0, s));
    CK(cudaStreamWaitEvent(cs, h->ev0, 0));
    CK(cudaStreamWaitEvent(ds, h->ev0, 0));
    for (int32_t k = 0; k < nrhs; ++k) {
        const int q = k & 1;
        // b_k -> bb[q] once solve k-2 (the last reader of bb[q]) is done
        if (k >= 2) CK(cudaStreamWaitEvent(cs, solved[q], 0));
        CK(cudaMemcpyAsync(h->bb[q], B_host + k * n, sizeof(double) * n, cudaMemcpyHostToDevice, cs));
        CK(cudaEventRecord(h2d[q], cs));
        // solve k once b_k is there and x_{k-2} has left bx[q]
        CK(cudaStreamWaitEvent(s, h2d[q], 0));
        if (k >= 2) CK(cudaStreamWaitEvent(s, d2h[q], 0));
        for (auto& Rk : h->ranks) CK(cudaMemcpyAsync(Rk.st, &sts[0], sizeof(PcgState), cudaMemcpyHostToDevice, s));
        CK(cudaGraphLaunch(h->batch_exec[q], s));
        CK(cudaMemcpyAsync(&sts[1 + k], R.st, sizeof(PcgState), cudaMemcpyDeviceToHost, s));
        CK(cudaEventRecord(solved[q], s));
        // x_k -> host while the next solves run
        CK(cudaStreamWaitEvent(ds, solved[q], 0));
        CK(cudaMemcpyAsync(X_host + k * n, h->bx[q], sizeof(double) * n, cudaMemcpyDeviceToHost, ds));
        CK(cudaEventRecord(d2h[q], ds));
    }
    CK(cudaStreamWaitEvent(s, d2h[0], 0));
    CK(cudaStreamWaitEvent(s, d2h[1], 0));
    CK(cudaEventRecord(h->ev1, s));
    CK(cudaStreamSynchronize(s));
    CK(cudaStreamSynchronize(cs));
    CK(cudaStreamSynchronize(ds));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, h->ev0, h->ev1);
    for (int32_t k = 0; k < nrhs; ++k) {
        const PcgState& S = sts[1 + k];
        int c = AMG_OK;
        if (S.status == ST_MAXIT) c = AMG_NOT_CONVERGED;
        if (S.status == ST_BREAKDOWN) c = AMG_ERR_BREAKDOWN;
        if (code == AMG_OK) code = c;
        if (reps) {
            fill_report(h, reps + k);
            reps[k].iterations = S.iter;
            reps[k].final_relres = S.relres;
            reps[k].converged = (S.status == ST_CONVERGED || S.status == ST_ZERO_RHS) ? 1 : 0;
            reps[k].solve_s = ms * 1e-3 / (double)std::max(1, nrhs);
            reps[k].status = c;
        }
    }
    if (code == AMG_ERR_BREAKDOWN) set_err("amg_solve_host_batch: breakdown, p^T A p <= 0");
    CK(cudaGetLastError());
    return code;
}

int amg_solve_host(amg_hier_t h, const double* b_host, double* x_host, double rtol, int32_t maxit,
                   amg_report_t* rep) {
    NvtxRange nvtx_("amg_solve_host");
    if (!h || !b_host || !x_host) {
        set_err("amg_solve_host: bad argument");
        return AMG_ERR_ARG;
    }
    std::lock_guard<std::recursive_mutex> guard(h->mu);
    CK(cudaSetDevice(h->ctx->device));
    int st;
    if (!h->hb && (st = dev_alloc(&h->hb, h->n0_local))) return st;
    if (!h->hx && (st = dev_alloc(&h->hx, h->n0_local))) return st;
    cudaStream_t s = h->ctx->stream;
    CK(cudaMemcpyAsync(h->hb, b_host, sizeof(double) * h->n0_local, cudaMemcpyHostToDevice, s));
    const int code = amg_solve(h, h->hb, h->hx, rtol, maxit, rep);
    if (code != AMG_OK && code != AMG_NOT_CONVERGED && code != AMG_ERR_BREAKDOWN) return code;
    CK(cudaMemcpyAsync(x_host, h->hx, sizeof(double) * h->n0_local, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return code;
}

int amg_precond_apply(amg_hier_t h, const double* r_dev, double* z_dev) {
    NvtxRange nvtx_("amg_precond_apply");
    if (!h || !r_dev || !z_dev) {
        set_err("amg_precond_apply: bad argument");
        return AMG_ERR_ARG;
    }
    std::lock_guard<std::recursive_mutex> guard(h->mu);
    CK(cudaSetDevice(h->ctx->device));
    cudaStream_t s = h->ctx->stream;
    h->nccl_status = ncclSuccess;
    if (h->cfg.use_graphs && !h->nccl_xport()) {
        int e = ensure_apply_graph(h, r_dev, z_dev);
        if (e) return e;
        CK(cudaGraphLaunch(h->apply_exec, s));
    } else {
        Launch L{h, s};
        enqueue_apply(h, L, r_dev, z_dev);
        if (int e = take_nccl_status(h)) return e;
    }
    CK(cudaStreamSynchronize(s));
    CK(cudaGetLastError());
    return take_lsa_err(h);
}

int amg_solve_graph_mode(amg_hier_t h, int32_t* mode) {
    if (!h || !mode) {
        set_err("amg_solve_graph_mode: null argument");
        return AMG_ERR_ARG;
    }
    std::lock_guard<std::recursive_mutex> guard(h->mu);
    *mode = h->cfg.use_graphs ? (int32_t)h->graph_mode : 2;
    return AMG_OK;
}

int amg_comm_transport(amg_hier_t h, int32_t* transport) {
    if (!h || !transport) {
        set_err("amg_comm_transport: null argument");
        return AMG_ERR_ARG;
    }
    *transport = !h->multi() ? 0 : h->lsa ? 3 : h->nccl_xport() ? 2 : 1;
    return AMG_OK;
}

int amg_num_levels(amg_hier_t h, int32_t* nl) {
    if (!h || !nl) return AMG_ERR_ARG;
    *nl = (int32_t)h->lvl_n.size();
    return AMG_OK;
}

int amg_level_info(amg_hier_t h, int32_t l, int64_t* n_global, int64_t* nnzA, int64_t* nnzP, int64_t* rb,
                   int64_t* re, int32_t* format) {
    if (!h || l < 0 || l >= (int32_t)h->lvl_n.size()) {
        set_err("amg_level_info: bad level");
        return AMG_ERR_ARG;
    }
    if (n_global) *n_global = h->lvl_n[l];
    if (nnzA) *nnzA = h->lvl_nnzA[l];
    if (nnzP) *nnzP = h->lvl_nnzP[l];
    if (rb) *rb = h->lvl_own_begin[l];
    if (re) *re = h->lvl_own_end[l];
    if (format) *format = h->lvl_fmt[l];
    return AMG_OK;
}

int amg_level_aggregates(amg_hier_t h, int32_t l, int64_t* agg) {
    if (!h || !agg || l < 0 || l >= (int32_t)h->agg.size()) {
        set_err("amg_level_aggregates: bad level");
        return AMG_ERR_ARG;
    }
    const auto& a = h->agg[l];
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
    NvtxRange nvtx_("amg_profile_vcycle");
    if (!h || napply < 1 || !count) {
        set_err("amg_profile_vcycle: bad argument");
        return AMG_ERR_ARG;
    }
    std::lock_guard<std::recursive_mutex> guard(h->mu);
    CK(cudaSetDevice(h->ctx->device));
    cudaStream_t s = h->ctx->stream;
    for (auto& R : h->ranks) CK(cudaMemsetAsync(R.pr, 0, sizeof(double) * R.lv[0].win_n, s));
    std::vector<KernelRec> recs;
    Launch L{h, s};
    auto b0 = [](RankState& R) { return R.pr; };
    auto z0 = [](RankState& R) { return R.pz; };
    enqueue_vcycle(h, L, b0, z0, false);  // warm-up
    CK(cudaStreamSynchronize(s));
    h->prof = &recs;
    for (int a = 0; a < napply; ++a) enqueue_vcycle(h, L, b0, z0, false);
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

int amg_profile_iteration(amg_hier_t h, const double* b_dev, double* x_dev, int32_t napply, int32_t cap,
                          double* ms_out, double* bytes_out, double* stored_bytes_out, const char** names_out,
                          int32_t* count) {
    NvtxRange nvtx_("amg_profile_iteration");
    if (!h || !b_dev || !x_dev || napply < 1 || !count) {
        set_err("amg_profile_iteration: bad argument");
        return AMG_ERR_ARG;
    }
    std::lock_guard<std::recursive_mutex> guard(h->mu);
    CK(cudaSetDevice(h->ctx->device));
    cudaStream_t s = h->ctx->stream;
    h->nccl_status = ncclSuccess;
    PcgState init{};
    init.rtol = 0.0;  // fixed-count: every profiled body runs the whole iteration
    init.maxit = napply + 2;
    *h->st_host = init;
    for (auto& R : h->ranks) CK(cudaMemcpyAsync(R.st, h->st_host, sizeof(PcgState), cudaMemcpyHostToDevice, s));
    std::vector<KernelRec> recs;
    Launch L{h, s};
    enqueue_pcg_init(h, L, b_dev, x_dev, 0);
    enqueue_pcg_body(h, L, x_dev, 0);  // warm-up iteration
    CK(cudaStreamSynchronize(s));
    h->prof = &recs;
    for (int a = 0; a < napply; ++a) enqueue_pcg_body(h, L, x_dev, 0);
    h->prof = nullptr;
    enqueue_pcg_final(h, L, x_dev);
    CK(cudaStreamSynchronize(s));
    CK(cudaGetLastError());
    if (int e = take_nccl_status(h)) return e;
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

// ---------------------------------------------------------- host-only view
struct amg_host_hier_s {
    amgsetup::Hierarchy H;
    std::vector<amgsetup::RankPlan> plans;
};

int amg_host_hierarchy_build(int64_t n, const int64_t* rowptr, const int64_t* colind, const double* values,
                             const double* w, const amg_config_t* cfg_in, amg_host_hier_t* out) {
    NvtxRange nvtx_("amg_host_hierarchy_build");
    if (!out) {
        set_err("amg_host_hierarchy_build: null out");
        return AMG_ERR_ARG;
    }
    *out = nullptr;
    amg_config_t cfg;
    amg_config_default(&cfg);
    if (cfg_in) cfg = *cfg_in;
    if (!cfg_in) cfg.setup_device = 0;  // the host-only view needs no device unless asked
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

int amg_host_dist_build(int64_t n, const int64_t* rowptr, const int64_t* colind, const double* values,
                        const double* w, const amg_config_t* cfg_in, int32_t nranks, int64_t replicate_below_bytes,
                        amg_host_hier_t* out) {
    NvtxRange nvtx_("amg_host_dist_build");
    if (!out || nranks < 1 || !rowptr || !colind || !values || n <= 0 || n >= (int64_t)INT32_MAX) {
        set_err("amg_host_dist_build: bad argument");
        return AMG_ERR_ARG;
    }
    *out = nullptr;
    amg_config_t cfg;
    amg_config_default(&cfg);
    if (cfg_in) cfg = *cfg_in;
    // the same validation as the single-process build (the whole matrix is at hand here)
    amgsetup::Csr A;
    A.nrows = A.ncols = n;
    A.rp.assign(rowptr, rowptr + n + 1);
    A.ci.resize(rowptr[n]);
    for (int64_t k = 0; k < rowptr[n]; ++k) {
        if (colind[k] < 0 || colind[k] >= n) {
            set_err("amg_host_dist_build: column index out of range");
            return AMG_ERR_ARG;
        }
        A.ci[k] = (int32_t)colind[k];
    }
    A.v.assign(values, values + rowptr[n]);
    std::vector<double> wv(n, 1.0);
    if (w) std::copy(w, w + n, wv.begin());
    std::string err;
    int vst = amgsetup::validate(A, wv, err);
    if (vst != amgsetup::SETUP_OK) {
        set_err("amg_host_dist_build: " + err);
        return vst == amgsetup::SETUP_ERR_ARG ? AMG_ERR_ARG : AMG_ERR_NOT_SPD;
    }
    std::vector<int64_t> b0(nranks + 1);
    for (int g = 0; g <= nranks; ++g) b0[g] = n * g / nranks;
    amgsetup::Config sc = setup_config(cfg);
    std::vector<amgsetup::DistHierarchy> DH(nranks);
    std::vector<amgsetup::RankPlan> plans(nranks);
    std::vector<int> rst(nranks, AMG_OK);
    std::vector<std::string> rerr(nranks);
    amgsetup::run_loopback(nranks, [&](amgsetup::Comm& c) {
        const int r = c.rank();
        amgsetup::Csr Al;
        Al.nrows = b0[r + 1] - b0[r];
        Al.ncols = n;
        Al.rp.resize(Al.nrows + 1);
        for (int64_t i = 0; i <= Al.nrows; ++i) Al.rp[i] = A.rp[b0[r] + i] - A.rp[b0[r]];
        Al.ci.assign(A.ci.begin() + A.rp[b0[r]], A.ci.begin() + A.rp[b0[r + 1]]);
        Al.v.assign(A.v.begin() + A.rp[b0[r]], A.v.begin() + A.rp[b0[r + 1]]);
        std::vector<double> wl(wv.begin() + b0[r], wv.begin() + b0[r + 1]);
        const int st = amgsetup::build_distributed(c, b0, std::move(Al), std::move(wl), sc, DH[r], rerr[r]);
        if (st != amgsetup::SETUP_OK) {
            rst[r] = st == amgsetup::SETUP_ERR_ARG ? AMG_ERR_ARG : AMG_ERR_NOT_SPD;
            return;
        }
        if (!amgsetup::partition_distributed(c, DH[r], replicate_below_bytes, plans[r], rerr[r])) rst[r] = AMG_ERR_ARG;
    });
    for (int r = 0; r < nranks; ++r)
        if (rst[r] != AMG_OK) {
            set_err("amg_host_dist_build: rank " + std::to_string(r) + ": " + rerr[r]);
            return rst[r];
        }
    // the global view for inspection: every level's rows concatenated in rank order
    auto* h = new amg_host_hier_s();
    const size_t nl = DH[0].lv.size();
    h->H.lv.resize(nl);
    for (size_t l = 0; l < nl; ++l) {
        amgsetup::Level& L = h->H.lv[l];
        const int64_t nn = DH[0].lv[l].n;
        auto cat = [&](auto get, int64_t ncols) {
            amgsetup::Csr M;
            M.nrows = nn;
            M.ncols = ncols;
            M.rp.assign(1, 0);
            for (int r = 0; r < nranks; ++r) {
                const amgsetup::Csr& X = get(DH[r].lv[l]);
                for (int64_t i = 0; i < X.nrows; ++i) M.rp.push_back(M.rp.back() + (X.rp[i + 1] - X.rp[i]));
                M.ci.insert(M.ci.end(), X.ci.begin(), X.ci.end());
                M.v.insert(M.v.end(), X.v.begin(), X.v.end());
            }
            return M;
        };
        L.A = cat([](const amgsetup::DistLevel& D) -> const amgsetup::Csr& { return D.A; }, nn);
        if (l + 1 < nl) {
            L.P = cat([](const amgsetup::DistLevel& D) -> const amgsetup::Csr& { return D.P; }, DH[0].lv[l + 1].n);
            for (int r = 0; r < nranks; ++r) L.agg.insert(L.agg.end(), DH[r].lv[l].agg.begin(), DH[r].lv[l].agg.end());
            L.omega = DH[0].lv[l].omega;
            L.sweeps = DH[0].lv[l].sweeps;
        }
    }
    h->H.coarse_inv = DH[0].coarse_inv;
    h->plans = std::move(plans);
    *out = h;
    return AMG_OK;
}

namespace {
// A caller-supplied transport (amg_exchange_fn): counts, then payloads concatenated in rank order.
struct CallbackComm : amgsetup::Comm {
    amg_exchange_fn fn = nullptr;
    void* user = nullptr;
    int me = 0, np = 1;
    bool ok = true;
    int rank() const override { return me; }
    int size() const override { return np; }
    bool alltoallv(const std::vector<std::vector<char>>& out, std::vector<std::vector<char>>& in) override {
        in.assign(np, {});
        if (!ok) return false;
        std::vector<int64_t> sc(np), rc(np, 0);
        int64_t stot = 0, rtot = 0;
        for (int q = 0; q < np; ++q) stot += (sc[q] = (int64_t)out[q].size());
        if (fn(user, 0, sc.data(), rc.data(), nullptr, nullptr) != 0) return ok = false;
        for (int q = 0; q < np; ++q) rtot += rc[q];
        std::vector<char> sb((size_t)std::max<int64_t>(stot, 1)), rb((size_t)std::max<int64_t>(rtot, 1));
        int64_t o = 0;
        for (int q = 0; q < np; ++q) {
            if (sc[q]) std::memcpy(sb.data() + o, out[q].data(), sc[q]);
            o += sc[q];
        }
        if (fn(user, 1, sc.data(), rc.data(), sb.data(), rb.data()) != 0) return ok = false;
        o = 0;
        for (int q = 0; q < np; ++q) {
            in[q].assign(rb.data() + o, rb.data() + o + rc[q]);
            o += rc[q];
        }
        return true;
    }
};
}  // namespace

int amg_host_dist_build_rank(int64_t n, int64_t row_begin, int64_t row_end, const int64_t* rowptr,
                             const int64_t* colind, const double* values, const double* w, const amg_config_t* cfg_in,
                             int32_t nranks, int32_t rank, int64_t replicate_below_bytes, amg_exchange_fn exchange,
                             void* user, amg_host_hier_t* out) {
    NvtxRange nvtx_("amg_host_dist_build_rank");
    if (!out || !exchange || nranks < 1 || rank < 0 || rank >= nranks || !rowptr || !colind || !values || n <= 0 ||
        n >= (int64_t)INT32_MAX || row_begin < 0 || row_end < row_begin || row_end > n || rowptr[0] != 0) {
        set_err("amg_host_dist_build_rank: bad argument");
        return AMG_ERR_ARG;
    }
    *out = nullptr;
    amg_config_t cfg;
    amg_config_default(&cfg);
    if (cfg_in) cfg = *cfg_in;
    CallbackComm c;
    c.fn = exchange;
    c.user = user;
    c.me = rank;
    c.np = nranks;
    // the row blocks of all ranks (contiguous, in rank order, covering [0, n))
    std::vector<std::vector<char>> ob(nranks, std::vector<char>(16)), ib;
    for (auto& b : ob) {
        std::memcpy(b.data(), &row_begin, 8);
        std::memcpy(b.data() + 8, &row_end, 8);
    }
    c.alltoallv(ob, ib);
    std::vector<int64_t> b0(nranks + 1, 0);
    bool okb = c.ok;
    for (int q = 0; q < nranks && okb; ++q) {
        int64_t rb, re;
        std::memcpy(&rb, ib[q].data(), 8);
        std::memcpy(&re, ib[q].data() + 8, 8);
        okb &= (rb == b0[q] && re >= rb);
        b0[q + 1] = re;
    }
    if (!okb || b0[nranks] != n) {
        set_err(c.ok ? "amg_host_dist_build_rank: row blocks must be contiguous, in rank order and cover [0, n)"
                     : "amg_host_dist_build_rank: exchange callback failed");
        return c.ok ? AMG_ERR_ARG : AMG_ERR_NCCL;
    }
    amgsetup::Csr A;
    A.nrows = row_end - row_begin;
    A.ncols = n;
    A.rp.assign(rowptr, rowptr + A.nrows + 1);
    A.ci.resize(rowptr[A.nrows]);
    for (int64_t k = 0; k < rowptr[A.nrows]; ++k) {
        if (colind[k] < 0 || colind[k] >= n) {
            set_err("amg_host_dist_build_rank: column index out of range");
            return AMG_ERR_ARG;
        }
        A.ci[k] = (int32_t)colind[k];
    }
    A.v.assign(values, values + rowptr[A.nrows]);
    std::vector<double> wl(A.nrows, 1.0);
    if (w) std::copy(w, w + A.nrows, wl.begin());
    cfg.replicate_below_bytes = replicate_below_bytes;
    DistOut o;
    dist_rank(c, cfg, b0, std::move(A), std::move(wl), true, o);
    if (!c.ok) {
        set_err("amg_host_dist_build_rank: exchange callback failed");
        return AMG_ERR_NCCL;
    }
    if (o.st != AMG_OK) {
        set_err("amg_host_dist_build_rank: " + o.err);
        return o.st;
    }
    auto* h = new amg_host_hier_s();
    h->plans.resize(nranks);
    h->plans[rank] = std::move(o.plan);
    h->H.lv.resize(o.S.n.size());
    for (size_t l = 0; l < o.S.n.size(); ++l) {
        h->H.lv[l].A.nrows = o.S.n[l];  // sizes only: the rank holds its own rows (see the plan)
        h->H.lv[l].A.rp.assign(1, 0);
        if (l + 1 < o.S.n.size()) h->H.lv[l].agg = o.agg[l];
    }
    h->H.coarse_inv = std::move(o.cinv);
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
    if ((int64_t)a.size() != h->H.lv[l].A.nrows) {  // a rank's view holds its own rows only
        set_err("amg_host_level_aggregates: this host hierarchy holds one rank's rows only");
        return AMG_ERR_ARG;
    }
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
    if ((int64_t)M.rp.size() != M.nrows + 1) {  // amg_host_dist_build_rank keeps only its plan
        set_err("amg_host_level_matrix: this host hierarchy holds one rank's plan, not the level matrices");
        return AMG_ERR_ARG;
    }
    for (int64_t i = 0; i <= M.nrows; ++i) rowptr[i] = M.rp[i];
    for (int64_t k = 0; k < M.nnz(); ++k) {
        colind[k] = M.ci[k];
        values[k] = M.v[k];
    }
    return AMG_OK;
}

int amg_host_partition(amg_host_hier_t h, int32_t nranks, const int64_t* row_bounds, int64_t replicate_below_bytes) {
    if (!h || nranks < 1 || !row_bounds) {
        set_err("amg_host_partition: bad argument");
        return AMG_ERR_ARG;
    }
    std::vector<int64_t> b(row_bounds, row_bounds + nranks + 1);
    std::string err;
    if (!amgsetup::partition(h->H, b, replicate_below_bytes, h->plans, err)) {
        set_err("amg_host_partition: " + err);
        return AMG_ERR_ARG;
    }
    return AMG_OK;
}

int amg_host_plan_level(amg_host_hier_t h, int32_t rank, int32_t l, int64_t* info16) {
    if (!h || rank < 0 || rank >= (int32_t)h->plans.size() || l < 0 || l >= (int32_t)h->plans[rank].lv.size() ||
        !info16) {
        set_err("amg_host_plan_level: bad argument");
        return AMG_ERR_ARG;
    }
    const auto& L = h->plans[rank].lv[l];
    const int64_t v[16] = {L.replicated ? 1 : 0, L.n_global, L.own_begin, L.own_end, L.comp_begin, L.comp_end,
                           L.win_begin, L.win_end, L.rst_begin, L.rst_end, (int64_t)L.recv_ids.size(),
                           (int64_t)L.send_ids.size(), L.A.nnz(), L.P.nnz(), L.R.nnz(), 0};
    std::memcpy(info16, v, sizeof(v));
    return AMG_OK;
}

int amg_host_plan_array(amg_host_hier_t h, int32_t rank, int32_t l, int32_t which, void* out) {
    if (!h || rank < 0 || rank >= (int32_t)h->plans.size() || l < 0 || l >= (int32_t)h->plans[rank].lv.size() ||
        !out) {
        set_err("amg_host_plan_array: bad argument");
        return AMG_ERR_ARG;
    }
    const auto& L = h->plans[rank].lv[l];
    auto cp64 = [&](const std::vector<int64_t>& v) { std::memcpy(out, v.data(), v.size() * sizeof(int64_t)); };
    auto csr = [&](const amgsetup::Csr& M, int part) {
        if (part == 0) {
            cp64(M.rp);
        } else if (part == 1) {
            int64_t* o = (int64_t*)out;
            for (size_t k = 0; k < M.ci.size(); ++k) o[k] = M.ci[k];
        } else {
            std::memcpy(out, M.v.data(), M.v.size() * sizeof(double));
        }
    };
    switch (which) {
        case 0: cp64(L.recv_off); break;
        case 1: cp64(L.recv_ids); break;
        case 2: cp64(L.send_off); break;
        case 3: cp64(L.send_ids); break;
        case 4: case 5: case 6: csr(L.A, which - 4); break;
        case 7: case 8: case 9: csr(L.P, which - 7); break;
        case 10: case 11: case 12: csr(L.R, which - 10); break;
        case 13: std::memcpy(out, L.m.data(), L.m.size() * sizeof(double)); break;
        default:
            set_err("amg_host_plan_array: bad selector");
            return AMG_ERR_ARG;
    }
    return AMG_OK;
}

}  // extern "C"
