// wave_lab.cu — L2 temporal blocking of consecutive l1-Jacobi sweeps on B200.
// Operator: 7-point 256^3 Laplacian in SDIA-32 (per-slice offsets, values
// column-major per slice, no column indices), as the library stores A_0.
// Stages: S-1 out-of-place sweeps x' = x + (b - A x) / sum_j |a_ij|, then the
// residual r = b - A x (the pre-smoothing + residual of a V-cycle level).
//   SEP   one launch per stage (the library's current schedule)
//   WAVE  one persistent launch: items (stage s, block p of BR rows) are taken
//         from an atomic ticket counter in diagonal order t = p + s (d+1), ties
//         by s; an item waits for stage s-1 on blocks p-d..p+d (d = bandwidth /
//         BR) through per-item flags, so stage s+1 re-reads A's block from L2.
// Results must be bit-identical (same per-row arithmetic).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o wave_lab tools/wave_lab.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ double ld_stream(const double* p) {
    double r;
    asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(r) : "l"(p));
    return r;
}
__device__ __forceinline__ double ld_l2(const double* p) {  // may be re-read from L2 by a later stage
    double r;
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(r) : "l"(p), "l"(pol));
    return r;
}

// x is written by an earlier stage of the same launch: coherent (L1-invalidated on
// acquire) loads, never the non-coherent read-only path
__device__ __forceinline__ double ld_coh(const double* p) {
    double r;
    asm volatile("ld.global.f64 %0, [%1];" : "=d"(r) : "l"(p));
    return r;
}

struct Sdia {
    const uint32_t* sptr;
    const int32_t* offs;
    const double* val;
    int64_t n;
};

struct Stages {
    const double* xin[8];
    double* xout[8];
    const double* b;
    int S;  // number of stages; the last one is the residual
};

template <bool L2KEEP, bool COH = L2KEEP>
__device__ __forceinline__ void slice_apply(const Sdia& A, int64_t s, int lane, const double* __restrict__ x,
                                            const double* __restrict__ b, double* __restrict__ y, bool resid) {
    const uint32_t b0 = __ldg(A.sptr + s);
    const uint32_t w = __ldg(A.sptr + s + 1) - b0;
    const int64_t row = (s << 5) + lane;
    const int32_t* o = A.offs + b0;
    const double* v = A.val + (int64_t)b0 * 32 + lane;
    const int32_t rmax = (int32_t)A.n - 1;
    double acc = 0.0, asum = 0.0;
    auto gx = [](const double* q) { return COH ? ld_coh(q) : __ldg(q); };
    uint32_t k = 0;
    for (; k + 8 <= w; k += 8) {
        double a[8], xx[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) a[j] = L2KEEP ? ld_l2(v + 32 * (k + j)) : ld_stream(v + 32 * (k + j));
#pragma unroll
        for (int j = 0; j < 8; ++j) xx[j] = gx(x + min(max((int32_t)row + __ldg(o + k + j), 0), rmax));
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            acc += a[j] * xx[j];
            asum += fabs(a[j]);
        }
    }
    if (k < w) {
        double a[8], xx[8];
#pragma unroll
        for (int j = 0; j < 8; ++j)
            a[j] = (k + j < w) ? (L2KEEP ? ld_l2(v + 32 * (k + j)) : ld_stream(v + 32 * (k + j))) : 0.0;
#pragma unroll
        for (int j = 0; j < 8; ++j)
            xx[j] = (k + j < w) ? gx(x + min(max((int32_t)row + __ldg(o + k + j), 0), rmax)) : 0.0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            acc += a[j] * xx[j];
            asum += fabs(a[j]);
        }
    }
    if (row < A.n) {
        const double bi = b[row];
        y[row] = resid ? bi - acc : gx(x + row) + (bi - acc) / asum;
    }
}

__global__ void __launch_bounds__(256) k_sep(Sdia A, const double* x, const double* b, double* y, bool resid) {
    const int lane = threadIdx.x & 31;
    const int64_t nsl = (A.n + 31) / 32;
    for (int64_t s = ((int64_t)blockIdx.x * 256 + threadIdx.x) >> 5; s < nsl; s += ((int64_t)gridDim.x * 256) >> 5)
        slice_apply<false>(A, s, lane, x, b, y, resid);
}

// items: block p covers slices [p*spb, (p+1)*spb).  cnt[s*ng + g] counts the
// finished blocks of stage s in group g (G consecutive blocks).  Ticket order:
// diagonal t = p + s*L (L >= d: stage s+1 lags stage s by L blocks), ties by s;
// an item of stage s waits until stage s-1 has finished every group that
// intersects blocks [p-d, p+d] (all those blocks have smaller tickets).
template <bool L2KEEP>
__global__ void __launch_bounds__(256) k_wave(Sdia A, const Stages st, int spb, int64_t nb, int d, int G, int L,
                                              unsigned long long* ticket, int* cnt) {
    __shared__ long long item;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t nsl = (A.n + 31) / 32;
    const int S = st.S;
    const int64_t ng = (nb + G - 1) / G;
    const int64_t ndiag = nb + (int64_t)(S - 1) * L;
    for (;;) {
        if (threadIdx.x == 0) {
            long long it = -1;
            for (;;) {
                const unsigned long long tk = atomicAdd(ticket, 1ull);
                const long long t = (long long)(tk / S), s = (long long)(tk % S);
                if (t >= ndiag) break;
                const long long p = t - s * L;
                if (p >= 0 && p < nb) {
                    it = s * nb + p;
                    break;
                }
            }
            if (it >= nb) {
                const long long s = it / nb, p = it % nb;
                const long long g0 = max(0ll, p - d) / G, g1 = min((long long)nb - 1, p + d) / G;
                for (long long g = g1; g >= g0; --g) {
                    const int need = (int)min((long long)G, (long long)nb - g * G);
                    const int* f = cnt + (s - 1) * ng + g;
                    int v;
                    do {
                        asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(f));
                    } while (v < need);
                }
                asm volatile("fence.acq_rel.gpu;" ::: "memory");
            }
            item = it;
        }
        __syncthreads();
        const long long it = item;
        if (it < 0) break;
        const int s = (int)(it / nb);
        const int64_t p = it % nb;
        const int64_t sl0 = p * spb, sl1 = min(nsl, sl0 + spb);
        for (int64_t sl = sl0 + wid; sl < sl1; sl += 8)
            slice_apply<L2KEEP, true>(A, sl, lane, st.xin[s], st.b, st.xout[s], s == S - 1);
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            atomicAdd(cnt + (int64_t)s * ng + p / G, 1);
        }
    }
}

// Static schedule (cooperative launch: all CTAs co-resident): CTA c takes the
// valid items of tickets c, c + grid, c + 2 grid, ... in order — no ticket atomic.
// Deadlock-free: the smallest unfinished ticket's dependencies are all smaller.
template <bool L2KEEP>
__global__ void __launch_bounds__(256, 8) k_wave_static(Sdia A, const Stages st, int spb, int64_t nb, int d, int G,
                                                     int L, int* cnt) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t nsl = (A.n + 31) / 32;
    const int S = st.S;
    const int64_t ng = (nb + G - 1) / G;
    const int64_t ntk = (nb + (int64_t)(S - 1) * L) * S;
    for (int64_t tk = blockIdx.x; tk < ntk; tk += gridDim.x) {
        const int64_t t = tk / S;
        const int s = (int)(tk % S);
        const int64_t p = t - (int64_t)s * L;
        if (p < 0 || p >= nb) continue;
        if (s > 0) {
            if (threadIdx.x == 0) {
                const long long g0 = max(0ll, (long long)p - d) / G, g1 = min((long long)nb - 1, (long long)p + d) / G;
                for (long long g = g1; g >= g0; --g) {
                    const int need = (int)min((long long)G, (long long)nb - g * G);
                    const int* f = cnt + (int64_t)(s - 1) * ng + g;
                    int v;
                    do {
                        asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(f));
                    } while (v < need);
                }
            }
            __syncthreads();
        }
        const int64_t sl0 = p * spb, sl1 = min(nsl, sl0 + spb);
        for (int64_t sl = sl0 + wid; sl < sl1; sl += 8)
            slice_apply<L2KEEP, true>(A, sl, lane, st.xin[s], st.b, st.xout[s], s == S - 1);
        __syncthreads();
        if (threadIdx.x == 0) {
            int* c = cnt + (int64_t)s * ng + p / G;
            asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(c), "r"(1) : "memory");
        }
    }
}

int main(int argc, char** argv) {
    const int N = 256;
    const int64_t n = (int64_t)N * N * N, plane = (int64_t)N * N;
    const int64_t nsl = n / 32;
    // SDIA: per slice the union of the 7 offsets present (interior: all 7)
    std::vector<uint32_t> sptr(nsl + 1, 0);
    std::vector<int32_t> offs;
    std::vector<double> val;
    const int64_t O[7] = {-plane, -N, -1, 0, 1, N, plane};
    for (int64_t s = 0; s < nsl; ++s) {
        int w = 0;
        for (int k = 0; k < 7; ++k) {
            bool any = false;
            for (int l = 0; l < 32; ++l) {
                const int64_t i = s * 32 + l, x = i % N, y = (i / N) % N, z = i / plane;
                const bool in = (k == 0 ? z > 0 : k == 1 ? y > 0 : k == 2 ? x > 0 : k == 3 ? true
                                 : k == 4 ? x < N - 1 : k == 5 ? y < N - 1 : z < N - 1);
                any |= in;
            }
            if (!any) continue;
            offs.push_back((int32_t)O[k]);
            for (int l = 0; l < 32; ++l) {
                const int64_t i = s * 32 + l, x = i % N, y = (i / N) % N, z = i / plane;
                const bool in = (k == 0 ? z > 0 : k == 1 ? y > 0 : k == 2 ? x > 0 : k == 3 ? true
                                 : k == 4 ? x < N - 1 : k == 5 ? y < N - 1 : z < N - 1);
                val.push_back(!in ? 0.0 : (k == 3 ? 6.0 : -1.0));
            }
            ++w;
        }
        sptr[s + 1] = sptr[s] + w;
    }
    uint32_t* dsptr;
    int32_t* doffs;
    double *dval, *db, *dx0, *bufs[8];
    CK(cudaMalloc(&dsptr, sptr.size() * 4));
    CK(cudaMalloc(&doffs, offs.size() * 4));
    CK(cudaMalloc(&dval, val.size() * 8));
    CK(cudaMemcpy(dsptr, sptr.data(), sptr.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(doffs, offs.data(), offs.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dval, val.data(), val.size() * 8, cudaMemcpyHostToDevice));
    std::vector<double> hb(n);
    uint64_t z = 88172645463325252ull;
    for (auto& t : hb) {
        z ^= z << 13; z ^= z >> 7; z ^= z << 17;
        t = (double)(z >> 11) * (1.0 / 9007199254740992.0);
    }
    CK(cudaMalloc(&db, n * 8));
    CK(cudaMalloc(&dx0, n * 8));
    CK(cudaMemcpy(db, hb.data(), n * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dx0, hb.data(), n * 8, cudaMemcpyHostToDevice));  // x0 = b (any start)
    for (int i = 0; i < 3; ++i) CK(cudaMalloc(&bufs[i], n * 8));
    Sdia A{dsptr, doffs, dval, n};
    const double abytes = 8.0 * val.size() + 4.0 * offs.size();
    printf("A: %lld rows, stored %zu entries, %.1f MB; L2-flush between reps\n", (long long)n, val.size(), abytes / 1e6);
    double* flush;
    const int64_t nf = 40 << 20;
    CK(cudaMalloc(&flush, nf * 8));
    unsigned long long* ticket;
    int* flags;
    CK(cudaMalloc(&ticket, 8));
    const int maxS = 6;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    int dev_sm = 0;
    cudaDeviceGetAttribute(&dev_sm, cudaDevAttrMultiProcessorCount, 0);
    auto flush_l2 = [&] { CK(cudaMemsetAsync(flush, 0, nf * 8)); };
    for (int S : {2, 3, 5}) {
        // stage pointers: x0 -> buf0 -> buf1 -> buf0 ... ; last stage -> buf2 (residual)
        Stages st;
        st.S = S;
        st.b = db;
        const double* cur = dx0;
        for (int s = 0; s < S; ++s) {
            st.xin[s] = cur;
            st.xout[s] = (s == S - 1) ? bufs[2] : bufs[s % 2];
            cur = st.xout[s];
        }
        // reference: separate launches
        const int gsep = dev_sm * 8;
        float tsep = 0.f;
        const int reps = 10;
        for (int r = 0; r < reps + 2; ++r) {
            flush_l2();
            cudaEventRecord(e0);
            for (int s = 0; s < S; ++s) k_sep<<<gsep, 256>>>(A, st.xin[s], db, st.xout[s], s == S - 1);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (r >= 2) tsep += ms;
        }
        CK(cudaGetLastError());
        std::vector<double> ref(n), got(n);
        CK(cudaMemcpy(ref.data(), bufs[2], n * 8, cudaMemcpyDeviceToHost));
        printf("S=%d  SEP  %.3f ms  (%.0f GB/s of A+vectors per stage-pass model)\n", S, tsep / reps,
               S * (abytes + 24.0 * n) / (tsep / reps * 1e-3) / 1e9);
        struct Cfg { int spb, G, L; };
        for (Cfg c : {Cfg{16, 64, 320}, Cfg{32, 32, 320}, Cfg{32, 32, 640}, Cfg{64, 16, 160}, Cfg{64, 16, 320},
                      Cfg{128, 8, 160}}) {
            const int spb = c.spb;
            const int64_t nb = (nsl + spb - 1) / spb;
            const int d = (int)((plane + 32 * spb - 1) / (32 * spb)) + 1;  // bandwidth in blocks (+1: slice misalignment)
            const int L = std::max(c.L, d + c.G);  // every dependency has a smaller ticket (no deadlock)
            const int64_t ng = (nb + c.G - 1) / c.G;
            CK(cudaMalloc(&flags, (size_t)S * ng * 4));
            for (int keep = 0; keep < 1; ++keep) {
                for (int occ : {4}) {
                    float tw = 0.f;
                    for (int r = 0; r < reps + 2; ++r) {
                        flush_l2();
                        CK(cudaMemsetAsync(ticket, 0, 8));
                        CK(cudaMemsetAsync(flags, 0, (size_t)S * ng * 4));
                        cudaEventRecord(e0);
                        if (keep) k_wave<true><<<dev_sm * occ, 256>>>(A, st, spb, nb, d, c.G, L, ticket, flags);
                        else k_wave<false><<<dev_sm * occ, 256>>>(A, st, spb, nb, d, c.G, L, ticket, flags);
                        cudaEventRecord(e1);
                        CK(cudaEventSynchronize(e1));
                        float ms;
                        cudaEventElapsedTime(&ms, e0, e1);
                        if (r >= 2) tw += ms;
                    }
                    CK(cudaGetLastError());
                    CK(cudaMemcpy(got.data(), bufs[2], n * 8, cudaMemcpyDeviceToHost));
                    const bool same = std::memcmp(ref.data(), got.data(), n * 8) == 0;
                    printf("S=%d  WAVE spb %3d G %3d L %4d d %3d keep %d occ %d  %.3f ms  speedup %.2fx  %s\n", S, spb,
                           c.G, L, d, keep, occ, tw / reps, tsep / tw, same ? "bit-identical" : "MISMATCH");
                }
            }
            {
                int nbk = 0;
                CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nbk, k_wave_static<false>, 256, 0));
                for (int occ : {4, nbk}) {
                    if (occ > nbk) continue;
                    const int grid = occ * dev_sm;
                    float tw = 0.f;
                    for (int r = 0; r < reps + 2; ++r) {
                        flush_l2();
                        CK(cudaMemsetAsync(flags, 0, (size_t)S * ng * 4));
                        cudaEventRecord(e0);
                        int spb_ = spb, d_ = d, G_ = c.G, L_ = L;
                        int64_t nb_ = nb;
                        Sdia A_ = A;
                        Stages st_ = st;
                        int* fl_ = flags;
                        void* args[] = {&A_, &st_, &spb_, &nb_, &d_, &G_, &L_, &fl_};
                        CK(cudaLaunchCooperativeKernel((void*)k_wave_static<false>, grid, 256, args, 0, 0));
                        cudaEventRecord(e1);
                        CK(cudaEventSynchronize(e1));
                        float ms;
                        cudaEventElapsedTime(&ms, e0, e1);
                        if (r >= 2) tw += ms;
                    }
                    CK(cudaMemcpy(got.data(), bufs[2], n * 8, cudaMemcpyDeviceToHost));
                    const bool same = std::memcmp(ref.data(), got.data(), n * 8) == 0;
                    printf("S=%d  STAT spb %3d G %3d L %4d d %3d occ %d/%d  %.3f ms  speedup %.2fx  %s\n", S, spb, c.G, L,
                           d, occ, nbk, tw / reps, tsep / tw, same ? "bit-identical" : "MISMATCH");
                }
            }
            cudaFree(flags);
        }
    }
    (void)maxS;
    return 0;
}
