// spmv_lab.cu — standalone micro-benchmark for the level-0 SDIA-32 sweep kernel
// (the dominant kernel of the c4 V-cycle).  Builds the 256^3 7-point Poisson
// operator in SDIA-32 layout on the device and times variants of the first
// post-sweep  x' = m b + u + m (r - A u),  m_i = 1 / sum_k |a_ik|  (EPost1):
//   K0  the library's current grid-stride warp-per-slice kernel
//   K1  K0 + epilogue operands loaded before the row reduction
//   K2  K1 + two slices per warp iteration
//   K3  bulk-async (cp.async.bulk + mbarrier) staging of values and epilogue
//       vectors into a multi-stage shared-memory ring, 1 producer warp
//   RD  a pure streaming read of the same byte count (read roofline)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o spmv_lab tools/spmv_lab.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

constexpr int NX = 256, NY = 256, NZ = 256;
constexpr int64_t N = (int64_t)NX * NY * NZ;

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

// ---------------------------------------------------------------- fill
__global__ void k_fill(const uint32_t* sptr, int32_t* offs, double* val, int64_t nsl) {
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= nsl) return;
    const int64_t row0 = s * 32;
    const int x0 = (int)(row0 % NX), y = (int)((row0 / NX) % NY), z = (int)(row0 / ((int64_t)NX * NY));
    int32_t o[7];
    int w = 0;
    if (z > 0) o[w++] = -NX * NY;
    if (y > 0) o[w++] = -NX;
    o[w++] = -1;
    o[w++] = 0;
    o[w++] = 1;
    if (y < NY - 1) o[w++] = NX;
    if (z < NZ - 1) o[w++] = NX * NY;
    const uint32_t b0 = sptr[s];
    for (int k = 0; k < w; ++k) {
        offs[b0 + k] = o[k];
        for (int l = 0; l < 32; ++l) {
            const int x = x0 + l;
            double v = (o[k] == 0) ? 6.0 : -1.0;
            if (o[k] == -1 && x == 0) v = 0.0;
            if (o[k] == 1 && x == NX - 1) v = 0.0;
            val[(int64_t)(b0 + k) * 32 + l] = v;
        }
    }
}

__global__ void k_init(double* a, int64_t n, double sc) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        a[i] = sc * (double)((i * 2654435761ull) % 1000) / 1000.0;
}

// ---------------------------------------------------------------- K0
__global__ void __launch_bounds__(256, 8) k0(View A, Vecs V) {
    const int64_t nslices = (A.n + 31) >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t w0 = ((int64_t)blockIdx.x * 256 + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * 256) >> 5;
    for (int64_t s = w0; s < nslices; s += nw) {
        const uint32_t b0 = __ldg(A.sptr + s);
        const uint32_t w = __ldg(A.sptr + s + 1) - b0;
        const int64_t row = (s << 5) + lane;
        const int32_t base = (int32_t)row;
        const int32_t* o = A.offs + b0;
        const double* v = A.val + (int64_t)b0 * 32 + lane;
        double acc = 0.0, asum = 0.0;
#pragma unroll 8
        for (uint32_t k = 0; k < w; ++k) {
            const int32_t c = min(max(base + __ldg(o + k), 0), (int32_t)A.n - 1);
            const double a = ld_stream(v + 32 * k);
            acc += a * __ldg(V.u + c);
            asum += fabs(a);
        }
        if (row < A.n) {
            const double mi = 1.0 / asum, bi = V.b[row];
            V.xo[row] = mi * bi + V.u[row] + mi * (V.r[row] - acc);
        }
    }
}


__device__ __forceinline__ double ld_stream256(const double* p) {
    double r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.f64 %0, [%1];" : "=d"(r) : "l"(p));
    return r;
}
template <bool P256, bool FIX7>
__global__ void __launch_bounds__(256, 8) k6(View A, Vecs V) {
    const int64_t nslices = (A.n + 31) >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t w0 = ((int64_t)blockIdx.x * 256 + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * 256) >> 5;
    for (int64_t s = w0; s < nslices; s += nw) {
        const uint32_t b0 = __ldg(A.sptr + s);
        const uint32_t w = __ldg(A.sptr + s + 1) - b0;
        const int64_t row = (s << 5) + lane;
        const int32_t base = (int32_t)row;
        const int32_t* o = A.offs + b0;
        const double* v = A.val + (int64_t)b0 * 32 + lane;
        double acc = 0.0, asum = 0.0;
        if (FIX7 && w == 7) {
            double a[7], g[7];
#pragma unroll
            for (int k = 0; k < 7; ++k) a[k] = P256 ? ld_stream256(v + 32 * k) : ld_stream(v + 32 * k);
#pragma unroll
            for (int k = 0; k < 7; ++k) {
                const int32_t c = min(max(base + __ldg(o + k), 0), (int32_t)A.n - 1);
                g[k] = __ldg(V.u + c);
            }
#pragma unroll
            for (int k = 0; k < 7; ++k) {
                acc += a[k] * g[k];
                asum += fabs(a[k]);
            }
        } else {
#pragma unroll 8
            for (uint32_t k = 0; k < w; ++k) {
                const int32_t c = min(max(base + __ldg(o + k), 0), (int32_t)A.n - 1);
                const double a = P256 ? ld_stream256(v + 32 * k) : ld_stream(v + 32 * k);
                acc += a * __ldg(V.u + c);
                asum += fabs(a);
            }
        }
        if (row < A.n) {
            const double mi = 1.0 / asum, bi = V.b[row];
            V.xo[row] = mi * bi + V.u[row] + mi * (V.r[row] - acc);
        }
    }
}

// ---------------------------------------------------------------- K1: operands first
__global__ void __launch_bounds__(256, 8) k1(View A, Vecs V) {
    const int64_t nslices = (A.n + 31) >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t w0 = ((int64_t)blockIdx.x * 256 + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * 256) >> 5;
    for (int64_t s = w0; s < nslices; s += nw) {
        const uint32_t b0 = __ldg(A.sptr + s);
        const uint32_t w = __ldg(A.sptr + s + 1) - b0;
        const int64_t row = (s << 5) + lane;
        const bool ok = row < A.n;
        const double bi = ok ? ld_stream(V.b + row) : 0.0;
        const double ri = ok ? ld_stream(V.r + row) : 0.0;
        const int32_t base = (int32_t)row;
        const int32_t* o = A.offs + b0;
        const double* v = A.val + (int64_t)b0 * 32 + lane;
        double acc = 0.0, asum = 0.0, uc = 0.0;
#pragma unroll 8
        for (uint32_t k = 0; k < w; ++k) {
            const int32_t ok_ = __ldg(o + k);
            const int32_t c = min(max(base + ok_, 0), (int32_t)A.n - 1);
            const double a = ld_stream(v + 32 * k);
            const double uj = __ldg(V.u + c);
            if (ok_ == 0) uc = uj;
            acc += a * uj;
            asum += fabs(a);
        }
        if (ok) {
            const double mi = 1.0 / asum;
            V.xo[row] = mi * bi + uc + mi * (ri - acc);
        }
    }
}

// ---------------------------------------------------------------- K2: two slices in flight
__global__ void __launch_bounds__(256, 8) k2(View A, Vecs V) {
    const int64_t nslices = (A.n + 31) >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t w0 = ((int64_t)blockIdx.x * 256 + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * 256) >> 5;
    for (int64_t s = w0; s < nslices; s += 2 * nw) {
        const int64_t sB = s + nw;
        const bool hasB = sB < nslices;
        const uint32_t a0 = __ldg(A.sptr + s), wA = __ldg(A.sptr + s + 1) - a0;
        const uint32_t c0 = hasB ? __ldg(A.sptr + sB) : 0u, wB = hasB ? __ldg(A.sptr + sB + 1) - c0 : 0u;
        const int64_t rowA = (s << 5) + lane, rowB = (sB << 5) + lane;
        const bool okA = rowA < A.n, okB = hasB && rowB < A.n;
        const double bA = okA ? ld_stream(V.b + rowA) : 0.0, rA = okA ? ld_stream(V.r + rowA) : 0.0;
        const double bB = okB ? ld_stream(V.b + rowB) : 0.0, rB = okB ? ld_stream(V.r + rowB) : 0.0;
        double accA = 0.0, asA = 0.0, uA = 0.0, accB = 0.0, asB = 0.0, uB = 0.0;
        const uint32_t wm = max(wA, wB);
#pragma unroll 8
        for (uint32_t k = 0; k < wm; ++k) {
            if (k < wA) {
                const int32_t o = __ldg(A.offs + a0 + k);
                const int32_t c = min(max((int32_t)rowA + o, 0), (int32_t)A.n - 1);
                const double a = ld_stream(A.val + (int64_t)(a0 + k) * 32 + lane);
                const double uj = __ldg(V.u + c);
                if (o == 0) uA = uj;
                accA += a * uj;
                asA += fabs(a);
            }
            if (k < wB) {
                const int32_t o = __ldg(A.offs + c0 + k);
                const int32_t c = min(max((int32_t)rowB + o, 0), (int32_t)A.n - 1);
                const double a = ld_stream(A.val + (int64_t)(c0 + k) * 32 + lane);
                const double uj = __ldg(V.u + c);
                if (o == 0) uB = uj;
                accB += a * uj;
                asB += fabs(a);
            }
        }
        if (okA) {
            const double mi = 1.0 / asA;
            V.xo[rowA] = mi * bA + uA + mi * (rA - accA);
        }
        if (okB) {
            const double mi = 1.0 / asB;
            V.xo[rowB] = mi * bB + uB + mi * (rB - accB);
        }
    }
}

// ---------------------------------------------------------------- K3: bulk-async ring
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t cnt) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(cnt));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n.reg .pred p;\nWAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

template <int KS, int NST, int NCW, int MAXW>
__global__ void __launch_bounds__(32 * (NCW + 1), 1) k3(View A, Vecs V, int64_t nchunks) {
    extern __shared__ __align__(128) unsigned char sm[];
    constexpr int VAL_D = KS * MAXW * 32;  // doubles per stage of values
    double* sval = (double*)sm;                       // [NST][VAL_D]
    double* sb = sval + NST * VAL_D;                  // [NST][KS*32]
    double* sr = sb + NST * KS * 32;                  // [NST][KS*32]
    uint64_t* full = (uint64_t*)(sr + NST * KS * 32); // [NST]
    uint64_t* empty = full + NST;                     // [NST]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < NST; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, NCW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int64_t nslices = (A.n + 31) >> 5;
    if (warp == NCW) {  // producer
        if (lane == 0) {
            int st = 0;
            uint32_t ph = 0;
            for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
                mbar_wait(empty + st, ph ^ 1);
                const int64_t s0 = c * KS, s1 = min(s0 + KS, nslices);
                const uint32_t v0 = __ldg(A.sptr + s0), v1 = __ldg(A.sptr + s1);
                const uint32_t vb = (v1 - v0) * 32u * 8u;
                const int64_t r0 = s0 * 32, r1 = min(s1 * 32, A.n);
                const uint32_t rb = (uint32_t)(r1 - r0) * 8u;
                mbar_expect_tx(full + st, vb + 2 * rb);
                bulk_g2s(sval + st * VAL_D, A.val + (int64_t)v0 * 32, vb, full + st);
                bulk_g2s(sb + st * KS * 32, V.b + r0, rb, full + st);
                bulk_g2s(sr + st * KS * 32, V.r + r0, rb, full + st);
                if (++st == NST) { st = 0; ph ^= 1; }
            }
        }
        return;
    }
    int st = 0;
    uint32_t ph = 0;
    for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
        mbar_wait(full + st, ph);
        const int64_t s0 = c * KS, s1 = min(s0 + KS, nslices);
        const uint32_t v0 = __ldg(A.sptr + s0);
        for (int64_t s = s0 + warp; s < s1; s += NCW) {
            const uint32_t b0 = __ldg(A.sptr + s), w = __ldg(A.sptr + s + 1) - b0;
            const int64_t row = (s << 5) + lane;
            const double* v = sval + st * VAL_D + (int64_t)(b0 - v0) * 32 + lane;
            const int32_t* o = A.offs + b0;
            double acc = 0.0, asum = 0.0, uc = 0.0;
#pragma unroll 8
            for (uint32_t k = 0; k < w; ++k) {
                const int32_t ok_ = __ldg(o + k);
                const int32_t cc = min(max((int32_t)row + ok_, 0), (int32_t)A.n - 1);
                const double a = v[32 * k];
                const double uj = __ldg(V.u + cc);
                if (ok_ == 0) uc = uj;
                acc += a * uj;
                asum += fabs(a);
            }
            if (row < A.n) {
                const int li = (int)(row - s0 * 32);
                const double mi = 1.0 / asum;
                V.xo[row] = mi * sb[st * KS * 32 + li] + uc + mi * (sr[st * KS * 32 + li] - acc);
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + st);
        if (++st == NST) { st = 0; ph ^= 1; }
    }
}

// ---------------------------------------------------------------- read roofline
__global__ void __launch_bounds__(256, 8) k_read(const double* __restrict__ a, int64_t n, double* out) {
    double s = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x; i < n; i += (int64_t)gridDim.x * 256) s += ld_stream(a + i);
    if (s == 123.456) *out = s;
}
__global__ void __launch_bounds__(256, 8) k_copy(const double* __restrict__ a, double* __restrict__ b, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x; i < n; i += (int64_t)gridDim.x * 256) b[i] = ld_stream(a + i);
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

int main(int argc, char** argv) {
    const int reps = argc > 1 ? atoi(argv[1]) : 20;
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const int64_t nsl = N / 32;
    std::vector<uint32_t> sptr(nsl + 1, 0);
    for (int64_t s = 0; s < nsl; ++s) {
        const int64_t row0 = s * 32;
        const int y = (int)((row0 / NX) % NY), z = (int)(row0 / ((int64_t)NX * NY));
        sptr[s + 1] = sptr[s] + 3 + (z > 0) + (y > 0) + (y < NY - 1) + (z < NZ - 1);
    }
    const int64_t ne = sptr[nsl];
    uint32_t* d_sptr; int32_t* d_offs; double *d_val, *u, *b, *r, *xo, *xref, *dummy;
    CK(cudaMalloc(&d_sptr, (nsl + 1) * 4));
    CK(cudaMalloc(&d_offs, ne * 4));
    CK(cudaMalloc(&d_val, ne * 32 * 8));
    CK(cudaMalloc(&u, N * 8)); CK(cudaMalloc(&b, N * 8)); CK(cudaMalloc(&r, N * 8));
    CK(cudaMalloc(&xo, N * 8)); CK(cudaMalloc(&xref, N * 8)); CK(cudaMalloc(&dummy, 8));
    CK(cudaMemcpy(d_sptr, sptr.data(), (nsl + 1) * 4, cudaMemcpyHostToDevice));
    k_fill<<<(nsl + 255) / 256, 256>>>(d_sptr, d_offs, d_val, nsl);
    k_init<<<1184, 256>>>(u, N, 1.0); k_init<<<1184, 256>>>(b, N, 2.0); k_init<<<1184, 256>>>(r, N, 3.0);
    CK(cudaDeviceSynchronize());
    View A{d_sptr, d_offs, d_val, N};
    const double bytes = 8.0 * ne * 32 + 4.0 * ne + 4.0 * (nsl + 1) + 4 * 8.0 * N;  // vals offs sptr u b r xo
    printf("n=%lld stored entries=%lld (%.3f per row) bytes/launch=%.3f GB\n", (long long)N, (long long)(ne * 32),
           (double)ne * 32 / N, bytes / 1e9);
    auto report = [&](const char* name, float ms, bool check) {
        double maxd = 0;
        if (check) {
            std::vector<double> h1(N), h2(N);
            cudaMemcpy(h1.data(), xo, N * 8, cudaMemcpyDeviceToHost);
            cudaMemcpy(h2.data(), xref, N * 8, cudaMemcpyDeviceToHost);
            for (int64_t i = 0; i < N; ++i) maxd = std::max(maxd, std::fabs(h1[i] - h2[i]));
        }
        printf("%-28s %8.4f ms  %7.1f GB/s  maxdiff %.3g\n", name, ms, bytes / (ms * 1e-3) / 1e9, maxd);
    };
    Vecs Vr{u, b, r, xref};
    Vecs V{u, b, r, xo};
    float t = timeit([&] { k0<<<nsm * 8, 256>>>(A, Vr); }, reps);
    report("K0 current", t, false);
    CK(cudaMemset(xo, 0, N * 8));
    t = timeit([&] { k1<<<nsm * 8, 256>>>(A, V); }, reps);
    report("K1 operands-first", t, true);
    CK(cudaMemset(xo, 0, N * 8));
    t = timeit([&] { k2<<<nsm * 8, 256>>>(A, V); }, reps);
    report("K2 two-slices", t, true);
#define RUN3(KS, NST, NCW)                                                                              \
    {                                                                                                   \
        constexpr int MAXW = 7;                                                                         \
        const size_t smem = (size_t)NST * (KS * MAXW * 32 * 8 + 2 * KS * 32 * 8) + 2 * NST * 8;       \
        auto kern = k3<KS, NST, NCW, MAXW>;                                                             \
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));        \
        const int64_t nch = (nsl + KS - 1) / KS;                                                        \
        CK(cudaMemset(xo, 0, N * 8));                                                                   \
        t = timeit([&] { kern<<<nsm, 32 * (NCW + 1), smem>>>(A, V, nch); }, reps);                     \
        char nm[64];                                                                                    \
        snprintf(nm, 64, "K3 bulk KS=%d NST=%d NCW=%d", KS, NST, NCW);                                  \
        report(nm, t, true);                                                                            \
    }
    CK(cudaMemset(xo, 0, N * 8));
    t = timeit([&] { k6<true, false><<<nsm * 8, 256>>>(A, V); }, reps);
    report("K4 L2::256B", t, true);
    CK(cudaMemset(xo, 0, N * 8));
    t = timeit([&] { k6<false, true><<<nsm * 8, 256>>>(A, V); }, reps);
    report("K6 fixed-width-7", t, true);
    CK(cudaMemset(xo, 0, N * 8));
    t = timeit([&] { k6<true, true><<<nsm * 8, 256>>>(A, V); }, reps);
    report("K7 fixed7 + L2::256B", t, true);
    for (int bps : {4, 6, 12, 16}) {
        CK(cudaMemset(xo, 0, N * 8));
        t = timeit([&] { k0<<<nsm * bps, 256>>>(A, V); }, reps);
        char nm[64];
        snprintf(nm, 64, "K0 grid %d/SM", bps);
        report(nm, t, true);
    }
    RUN3(16, 3, 32)
    RUN3(32, 2, 32)
    RUN3(8, 6, 32)
    const int64_t nr = (int64_t)(bytes / 8);
    double* big;
    CK(cudaMalloc(&big, nr * 8 + 8));
    k_init<<<1184, 256>>>(big, nr, 1.0);
    t = timeit([&] { k_read<<<nsm * 8, 256>>>(big, nr, dummy); }, reps);
    report("RD read-only same bytes", t, false);
    t = timeit([&] { k_copy<<<nsm * 8, 256>>>(big, big + nr / 2, nr / 2); }, reps);
    report("CP copy (r+w) same bytes", t, false);
    return 0;
}
