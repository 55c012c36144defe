// tma_lab.cu -- SDIA-32 first post-sweep (x' = m b + u + m (r - A u)) with the matrix VALUE stream
// staged into shared memory by bulk async copies (cp.async.bulk, mbarrier complete_tx; SASS UBLKCP):
// one producer warp streams each block's contiguous slice range through an S-stage ring while NC
// consumer warps gather u and reduce the rows, vs the library's register-chunk kernel (ks).
// Derived from spmv_lab2.cu (same operators, same epilogue, bitwise-equal results).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tma_lab tools/tma_lab.cu
// (old header follows)
// spmv_lab2.cu — ILP variants of the SDIA-32 sweep kernel on two operators:
//   P7   256^3 7-point  (A_0 of c4: widths 4..7 per slice)
//   P27  128^3 27-point (stands in for A_1 of c4: ~27-33 entries per row)
// Kernel: first post-sweep x' = m b + u + m (r - A u), m = 1/sum|a| (EPost1).
//   K0   the library's current loop (#pragma unroll 8 over a runtime width)
//   C<U> chunks of U entries: U value loads, then U column offsets, then U
//        gathers, then the U FMAs (predicated on k < w); registers <= 32 or 40
//   S7   fully unrolled switch on the slice width (<= 8), chunks of 8 above
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o spmv_lab2 tools/spmv_lab2.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ double ld_stream(const double* p) {
    double r;
    asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(r) : "l"(p));
    return r;
}

struct View {
    const uint32_t* __restrict__ sptr;
    const int32_t* __restrict__ offs;
    const double* __restrict__ val;
    int64_t n;
};
struct Vecs {
    const double* __restrict__ u;
    const double* __restrict__ b;
    const double* __restrict__ r;
    double* __restrict__ xo;
};

__device__ __forceinline__ void epi(const Vecs& V, int64_t row, double acc, double asum) {
    const double mi = 1.0 / asum, bi = V.b[row];
    V.xo[row] = mi * bi + V.u[row] + mi * (V.r[row] - acc);
}

// exact-width specialisation
template <int W>
__device__ __forceinline__ void exact(const double* v, const int32_t* o, int32_t base, int32_t nmax,
                                      const double* __restrict__ u, double& acc, double& asum) {
    double a[W], g[W];
#pragma unroll
    for (int j = 0; j < W; ++j) a[j] = ld_stream(v + 32 * j);
#pragma unroll
    for (int j = 0; j < W; ++j) g[j] = __ldg(u + min(max(base + __ldg(o + j), 0), nmax));
#pragma unroll
    for (int j = 0; j < W; ++j) {
        acc += a[j] * g[j];
        asum += fabs(a[j]);
    }
}

template <int MINB>
__global__ void __launch_bounds__(256, MINB) ks(View A, Vecs V) {
    const int64_t nslices = (A.n + 31) >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t w0 = ((int64_t)blockIdx.x * 256 + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * 256) >> 5;
    const int32_t nmax = (int32_t)A.n - 1;
    for (int64_t s = w0; s < nslices; s += nw) {
        const uint32_t b0 = __ldg(A.sptr + s);
        const uint32_t w = __ldg(A.sptr + s + 1) - b0;
        const int64_t row = (s << 5) + lane;
        const int32_t base = (int32_t)row;
        const int32_t* o = A.offs + b0;
        const double* v = A.val + (int64_t)b0 * 32 + lane;
        double acc = 0.0, asum = 0.0;
        uint32_t k = 0;
        for (; k + 8 <= w; k += 8) exact<8>(v + 32 * k, o + k, base, nmax, V.u, acc, asum);
        switch (w - k) {
            case 7: exact<7>(v + 32 * k, o + k, base, nmax, V.u, acc, asum); break;
            case 6: exact<6>(v + 32 * k, o + k, base, nmax, V.u, acc, asum); break;
            case 5: exact<5>(v + 32 * k, o + k, base, nmax, V.u, acc, asum); break;
            case 4: exact<4>(v + 32 * k, o + k, base, nmax, V.u, acc, asum); break;
            case 3: exact<3>(v + 32 * k, o + k, base, nmax, V.u, acc, asum); break;
            case 2: exact<2>(v + 32 * k, o + k, base, nmax, V.u, acc, asum); break;
            case 1: exact<1>(v + 32 * k, o + k, base, nmax, V.u, acc, asum); break;
            default: break;
        }
        if (row < A.n) epi(V, row, acc, asum);
    }
}


__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t cnt) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(b)), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(saddr(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT%=;\n}\n" ::"r"(
            saddr(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     saddr(dst)),
                 "l"(src), "r"(bytes), "r"(saddr(bar))
                 : "memory");
}

template <int W>
__device__ __forceinline__ void exact_s(const double* v, const int32_t* o, int32_t base, int32_t nmax,
                                        const double* __restrict__ u, double& acc, double& asum) {
    double a[W], g[W];
#pragma unroll
    for (int j = 0; j < W; ++j) g[j] = __ldg(u + min(max(base + __ldg(o + j), 0), nmax));
#pragma unroll
    for (int j = 0; j < W; ++j) a[j] = v[32 * j];
#pragma unroll
    for (int j = 0; j < W; ++j) {
        acc += a[j] * g[j];
        asum += fabs(a[j]);
    }
}


// library-like variants of ks: PF = L2 prefetch of the epilogue operands before the row, DOT = return
// b_i x'_i, block-reduce, one atomicAdd per block (the library's grid_reduce is a ticketed two-pass)
template <int MINB, bool PF, bool DOT, int CH = 8>
__global__ void __launch_bounds__(256, MINB) ksx(View A, Vecs V, double* dsum) {
    const int64_t nslices = (A.n + 31) >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t w0 = ((int64_t)blockIdx.x * 256 + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * 256) >> 5;
    const int32_t nmax = (int32_t)A.n - 1;
    double d = 0.0;
    for (int64_t s = w0; s < nslices; s += nw) {
        const uint32_t b0 = __ldg(A.sptr + s);
        const uint32_t w = __ldg(A.sptr + s + 1) - b0;
        const int64_t row = (s << 5) + lane;
        if (PF && row < A.n && w <= 16) {
            asm volatile("prefetch.global.L2 [%0];" ::"l"(V.u + row));
            asm volatile("prefetch.global.L2 [%0];" ::"l"(V.r + row));
            asm volatile("prefetch.global.L2 [%0];" ::"l"(V.b + row));
        }
        const int32_t base = (int32_t)row;
        const int32_t* o = A.offs + b0;
        const double* v = A.val + (int64_t)b0 * 32 + lane;
        double acc = 0.0, asum = 0.0;
        uint32_t k = 0;
        for (; k + CH <= w; k += CH) exact<CH>(v + 32 * k, o + k, base, nmax, V.u, acc, asum);
        switch (w - k) {
            case 7: if constexpr (CH > 7) exact<7>(v + 32 * k, o + k, base, nmax, V.u, acc, asum); break;
            case 6: if constexpr (CH > 6) exact<6>(v + 32 * k, o + k, base, nmax, V.u, acc, asum); break;
            case 5: if constexpr (CH > 5) exact<5>(v + 32 * k, o + k, base, nmax, V.u, acc, asum); break;
            case 4: if constexpr (CH > 4) exact<4>(v + 32 * k, o + k, base, nmax, V.u, acc, asum); break;
            case 3: exact<3>(v + 32 * k, o + k, base, nmax, V.u, acc, asum); break;
            case 2: exact<2>(v + 32 * k, o + k, base, nmax, V.u, acc, asum); break;
            case 1: exact<1>(v + 32 * k, o + k, base, nmax, V.u, acc, asum); break;
            default: break;
        }
        if (row < A.n) {
            const double mi = 1.0 / asum, bi = V.b[row];
            const double x = mi * bi + V.u[row] + mi * (V.r[row] - acc);
            V.xo[row] = x;
            if (DOT) d += bi * x;
        }
    }
    if (DOT) {
        __shared__ double part[8];
        for (int o2 = 16; o2 > 0; o2 >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o2);
        if (lane == 0) part[threadIdx.x >> 5] = d;
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = 0.0;
            for (int i = 0; i < 8; ++i) t += part[i];
            atomicAdd(dsum, t);
        }
    }
}

// NC consumer warps + 1 producer warp; S stages of NC slices (<= WMAX entries each)
template <int WMAX, int NC, int S, int MINB>
__global__ void __launch_bounds__((NC + 1) * 32, MINB) kt(View A, Vecs V) {
    extern __shared__ __align__(128) unsigned char smem[];
    constexpr int STAGE = NC * WMAX * 32;  // doubles
    double* ring = (double*)smem;
    uint64_t* full = (uint64_t*)(smem + (size_t)S * STAGE * 8);
    uint64_t* empty = full + S;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t nslices = (A.n + 31) >> 5;
    const int64_t per = ((nslices + gridDim.x - 1) / gridDim.x + NC - 1) / NC * NC;
    const int64_t s0 = (int64_t)blockIdx.x * per, s1 = min(nslices, s0 + per);
    const int64_t nst = s1 > s0 ? (s1 - s0 + NC - 1) / NC : 0;
    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], NC);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == NC) {  // producer
        if (lane == 0) {
            for (int64_t j = 0; j < nst; ++j) {
                const int slot = (int)(j % S);
                const uint32_t ph = (uint32_t)((j / S) & 1);
                mbar_wait(&empty[slot], ph ^ 1u);
                const int64_t ss = s0 + j * NC, se = min(s1, ss + NC);
                const uint32_t k0 = __ldg(A.sptr + ss), k1 = __ldg(A.sptr + se);
                const uint32_t bytes = (k1 - k0) * 256u;
                mbar_expect_tx(&full[slot], bytes);
                bulk_g2s(ring + (size_t)slot * STAGE, A.val + (int64_t)k0 * 32, bytes, &full[slot]);
            }
        }
        return;
    }
    const int32_t nmax = (int32_t)A.n - 1;
    for (int64_t j = 0; j < nst; ++j) {
        const int slot = (int)(j % S);
        const uint32_t ph = (uint32_t)((j / S) & 1);
        const int64_t ss = s0 + j * NC, s = ss + warp;
        // issue this slice's offset loads and prologue before waiting for the values
        uint32_t b0 = 0, w = 0, kb = 0;
        if (s < s1) {
            kb = __ldg(A.sptr + ss);
            b0 = __ldg(A.sptr + s);
            w = __ldg(A.sptr + s + 1) - b0;
        }
        mbar_wait(&full[slot], ph);
        if (s < s1) {
            const int64_t row = (s << 5) + lane;
            const int32_t base = (int32_t)row;
            const int32_t* o = A.offs + b0;
            const double* v = ring + (size_t)slot * STAGE + (size_t)(b0 - kb) * 32 + lane;
            double acc = 0.0, asum = 0.0;
            uint32_t k = 0;
            for (; k + 8 <= w; k += 8) exact_s<8>(v + 32 * k, o + k, base, nmax, V.u, acc, asum);
            switch (w - k) {
                case 7: exact_s<7>(v + 32 * k, o + k, base, nmax, V.u, acc, asum); break;
                case 6: exact_s<6>(v + 32 * k, o + k, base, nmax, V.u, acc, asum); break;
                case 5: exact_s<5>(v + 32 * k, o + k, base, nmax, V.u, acc, asum); break;
                case 4: exact_s<4>(v + 32 * k, o + k, base, nmax, V.u, acc, asum); break;
                case 3: exact_s<3>(v + 32 * k, o + k, base, nmax, V.u, acc, asum); break;
                case 2: exact_s<2>(v + 32 * k, o + k, base, nmax, V.u, acc, asum); break;
                case 1: exact_s<1>(v + 32 * k, o + k, base, nmax, V.u, acc, asum); break;
                default: break;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[slot]);
            if (row < A.n) epi(V, row, acc, asum);
        } else {
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[slot]);
        }
    }
}
// ------------------------------------------------------------------ problems
struct Prob {
    int nx, ny, nz;
    int stencil;  // 7 or 27
};

__global__ void k_fill(Prob P, const uint32_t* sptr, int32_t* offs, double* val, int64_t nsl) {
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= nsl) return;
    const int64_t row0 = s * 32;
    const int64_t nxy = (int64_t)P.nx * P.ny;
    const int x0 = (int)(row0 % P.nx), y = (int)((row0 / P.nx) % P.ny), z = (int)(row0 / nxy);
    const uint32_t b0 = sptr[s];
    int k = 0;
    for (int dz = -1; dz <= 1; ++dz)
        for (int dy = -1; dy <= 1; ++dy)
            for (int dx = -1; dx <= 1; ++dx) {
                const int nnzc = (dx != 0) + (dy != 0) + (dz != 0);
                if (P.stencil == 7 && nnzc > 1) continue;
                if (z + dz < 0 || z + dz >= P.nz || y + dy < 0 || y + dy >= P.ny) continue;
                offs[b0 + k] = (int32_t)(dz * nxy + dy * P.nx + dx);
                for (int l = 0; l < 32; ++l) {
                    const int x = x0 + l;
                    double v = nnzc == 0 ? (double)(P.stencil - 1) : -1.0;
                    if (x + dx < 0 || x + dx >= P.nx) v = 0.0;
                    val[(int64_t)(b0 + k) * 32 + l] = v;
                }
                ++k;
            }
}

__global__ void k_init(double* a, int64_t n, double sc) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        a[i] = sc * (double)((i * 2654435761ull) % 1000) / 1000.0;
}

template <class F>
float timeit(F f, int reps) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    f();
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    for (int i = 0; i < reps; ++i) f();
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms / reps;
}


void run(Prob P, int reps, int nsm) {
    const int64_t N = (int64_t)P.nx * P.ny * P.nz, nsl = N / 32;
    std::vector<uint32_t> sptr(nsl + 1, 0);
    for (int64_t s = 0; s < nsl; ++s) {
        const int64_t row0 = s * 32;
        const int y = (int)((row0 / P.nx) % P.ny), z = (int)(row0 / ((int64_t)P.nx * P.ny));
        int w = 0;
        for (int dz = -1; dz <= 1; ++dz)
            for (int dy = -1; dy <= 1; ++dy)
                for (int dx = -1; dx <= 1; ++dx) {
                    const int nnzc = (dx != 0) + (dy != 0) + (dz != 0);
                    if (P.stencil == 7 && nnzc > 1) continue;
                    if (z + dz < 0 || z + dz >= P.nz || y + dy < 0 || y + dy >= P.ny) continue;
                    ++w;
                }
        sptr[s + 1] = sptr[s] + w;
    }
    const int64_t ne = sptr[nsl];
    uint32_t* d_sptr; int32_t* d_offs; double *d_val, *u, *b, *r, *xo, *xref;
    CK(cudaMalloc(&d_sptr, (nsl + 1) * 4));
    CK(cudaMalloc(&d_offs, ne * 4));
    CK(cudaMalloc(&d_val, ne * 32 * 8));
    CK(cudaMalloc(&u, N * 8)); CK(cudaMalloc(&b, N * 8)); CK(cudaMalloc(&r, N * 8));
    CK(cudaMalloc(&xo, N * 8)); CK(cudaMalloc(&xref, N * 8));
    CK(cudaMemcpy(d_sptr, sptr.data(), (nsl + 1) * 4, cudaMemcpyHostToDevice));
    k_fill<<<(nsl + 255) / 256, 256>>>(P, d_sptr, d_offs, d_val, nsl);
    k_init<<<1184, 256>>>(u, N, 1.0); k_init<<<1184, 256>>>(b, N, 2.0); k_init<<<1184, 256>>>(r, N, 3.0);
    CK(cudaDeviceSynchronize());
    View A{d_sptr, d_offs, d_val, N};
    const double bytes = 8.0 * ne * 32 + 4.0 * ne + 4.0 * (nsl + 1) + 4 * 8.0 * N;
    printf("== %d-point %dx%dx%d: n=%lld, %.2f stored/row, %.3f GB per launch\n", P.stencil, P.nx, P.ny, P.nz,
           (long long)N, (double)ne * 32 / N, bytes / 1e9);
    Vecs Vr{u, b, r, xref}, V{u, b, r, xo};
    std::vector<double> h1(N), h2(N);
    auto report = [&](const char* name, float ms, bool check) {
        double maxd = 0;
        if (check) {
            cudaMemcpy(h1.data(), xo, N * 8, cudaMemcpyDeviceToHost);
            cudaMemcpy(h2.data(), xref, N * 8, cudaMemcpyDeviceToHost);
            for (int64_t i = 0; i < N; ++i) maxd = std::max(maxd, std::fabs(h1[i] - h2[i]));
        }
        printf("%-28s %8.4f ms  %7.1f GB/s  maxdiff %.3g\n", name, ms, bytes / (ms * 1e-3) / 1e9, maxd);
    };
    float t = timeit([&] { ks<8><<<nsm * 8, 256>>>(A, Vr); }, reps);
    report("S (256,8) [library]", t, false);
    double* dsum;
    CK(cudaMalloc(&dsum, 8));
#define X_(NAME, MINB, PF, DOT, CH)                                                   \
    CK(cudaMemset(xo, 0, N * 8));                                                      \
    t = timeit([&] { ksx<MINB, PF, DOT, CH><<<nsm * MINB, 256>>>(A, V, dsum); }, reps);  \
    report(NAME, t, true);
    X_("ksx plain", 8, false, false, 8)
    X_("ksx prefetch(w<=16)", 8, true, false, 8)
    X_("ksx dot", 8, false, true, 8)
    X_("ksx dot minb7", 7, false, true, 8)
    X_("ksx dot minb6", 6, false, true, 8)
    X_("ksx dot minb5", 5, false, true, 8)
    X_("ksx dot minb4", 4, false, true, 8)
    X_("ksx dot ch4", 8, false, true, 4)
    X_("ksx plain minb6", 6, false, false, 8)
    X_("ksx dot pf minb6", 6, true, true, 8)
#define T_(WMAX, NC, S, MINB)                                                                          \
    {                                                                                                  \
        const size_t sm = (size_t)S * NC * WMAX * 32 * 8 + 2 * S * 8;                                   \
        auto kern = kt<WMAX, NC, S, MINB>;                                                             \
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));          \
        int nb = 0;                                                                                    \
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, (NC + 1) * 32, sm);                   \
        CK(cudaMemset(xo, 0, N * 8));                                                                  \
        t = timeit([&] { kern<<<nsm * nb, (NC + 1) * 32, sm>>>(A, V); }, reps);                        \
        char name[64];                                                                                 \
        snprintf(name, 64, "T w%d nc%d s%d (%d/SM, %zuKB)", WMAX, NC, S, nb, sm / 1024);                \
        report(name, t, true);                                                                         \
    }
    if (P.stencil == 7) {
        T_(7, 8, 4, 1) T_(7, 16, 4, 1)
    } else {
        T_(27, 8, 2, 1) T_(27, 16, 1, 1)
    }
    cudaFree(d_sptr); cudaFree(d_offs); cudaFree(d_val); cudaFree(u); cudaFree(b); cudaFree(r);
    cudaFree(xo); cudaFree(xref);
}

int main(int argc, char** argv) {
    const int reps = argc > 1 ? atoi(argv[1]) : 20;
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    run(Prob{256, 256, 256, 7}, reps, nsm);
    run(Prob{256, 256, 256, 27}, reps, nsm);
    return 0;
}
