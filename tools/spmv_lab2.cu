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

template <int MINB>
__global__ void __launch_bounds__(256, MINB) k0(View A, Vecs V) {
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
        if (row < A.n) epi(V, row, acc, asum);
    }
}

template <int U>
__device__ __forceinline__ void chunk(const double* v, const int32_t* o, int32_t base, int32_t nmax, uint32_t k0,
                                      uint32_t w, const double* __restrict__ u, double& acc, double& asum) {
    double a[U], g[U];
#pragma unroll
    for (int j = 0; j < U; ++j) a[j] = (k0 + j < w) ? ld_stream(v + 32 * (k0 + j)) : 0.0;
#pragma unroll
    for (int j = 0; j < U; ++j) {
        const int32_t c = (k0 + j < w) ? min(max(base + __ldg(o + k0 + j), 0), nmax) : base < 0 ? 0 : min(base, nmax);
        g[j] = (k0 + j < w) ? __ldg(u + c) : 0.0;
    }
#pragma unroll
    for (int j = 0; j < U; ++j) {
        acc += a[j] * g[j];
        asum += fabs(a[j]);
    }
}

template <int U, int MINB>
__global__ void __launch_bounds__(256, MINB) kc(View A, Vecs V) {
    const int64_t nslices = (A.n + 31) >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t w0 = ((int64_t)blockIdx.x * 256 + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * 256) >> 5;
    for (int64_t s = w0; s < nslices; s += nw) {
        const uint32_t b0 = __ldg(A.sptr + s);
        const uint32_t w = __ldg(A.sptr + s + 1) - b0;
        const int64_t row = (s << 5) + lane;
        const int32_t* o = A.offs + b0;
        const double* v = A.val + (int64_t)b0 * 32 + lane;
        double acc = 0.0, asum = 0.0;
        for (uint32_t k0 = 0; k0 < w; k0 += U) chunk<U>(v, o, (int32_t)row, (int32_t)A.n - 1, k0, w, V.u, acc, asum);
        if (row < A.n) epi(V, row, acc, asum);
    }
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
        printf("%-24s %8.4f ms  %7.1f GB/s  maxdiff %.3g\n", name, ms, bytes / (ms * 1e-3) / 1e9, maxd);
    };
    float t = timeit([&] { k0<8><<<nsm * 8, 256>>>(A, Vr); }, reps);
    report("K0 (256,8)", t, false);
#define V_(NAME, KERN, BPS)                                        \
    CK(cudaMemset(xo, 0, N * 8));                                  \
    t = timeit([&] { KERN<<<nsm * BPS, 256>>>(A, V); }, reps);     \
    report(NAME, t, true);
    V_("C4 (256,8)", (kc<4, 8>), 8)
    V_("C8 (256,8)", (kc<8, 8>), 8)
    V_("C8 (256,6)", (kc<8, 6>), 6)
    V_("C4 (256,6)", (kc<4, 6>), 6)
    V_("S (256,8)", ks<8>, 8)
    V_("S (256,6)", ks<6>, 6)
    V_("S (256,7) grid 7", ks<7>, 7)
    cudaFree(d_sptr); cudaFree(d_offs); cudaFree(d_val); cudaFree(u); cudaFree(b); cudaFree(r);
    cudaFree(xo); cudaFree(xref);
}

int main(int argc, char** argv) {
    const int reps = argc > 1 ? atoi(argv[1]) : 20;
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    run(Prob{256, 256, 256, 7}, reps, nsm);
    run(Prob{128, 128, 128, 27}, reps, nsm);
    return 0;
}
