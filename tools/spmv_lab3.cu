// spmv_lab3.cu — CSR-vector variants for the latency-bound mid/deep levels
// (c2 levels 2-4: 33k x ~150, 4.1k x ~585, 522 x ~520; c5-analogue level 1:
// 893k x ~110).  Kernel: residual y = b - A x (the EResid epilogue).
//   V0  library loop: chunks of 4 per lane + a sequential tail (VW lanes per row)
//   P8  predicated chunks of 8 per lane, no tail loop (masked entries: a = 0, c = 0)
//   P4  predicated chunks of 4
//   B   block (256 threads) per row, predicated chunk 4 (library k_csrb analogue)
// Each is timed L2-warm (back-to-back) and L2-cold (a 256 MB flush between).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o spmv_lab3 tools/spmv_lab3.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

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

struct M {
    const int32_t* rp;
    const int32_t* ci;
    const double* v;
    int64_t n;
};

template <int VW>
__global__ void __launch_bounds__(256) k_v0(M A, const double* __restrict__ x, const double* __restrict__ b,
                                            double* __restrict__ y) {
    const int64_t gid = (int64_t)blockIdx.x * 256 + threadIdx.x;
    const int sub = threadIdx.x % VW;
    const int64_t g0 = gid / VW, ng = ((int64_t)gridDim.x * 256) / VW;
    const int64_t iters = (A.n + ng - 1) / ng;
    for (int64_t it = 0; it < iters; ++it) {
        const int64_t row = g0 + it * ng;
        double acc = 0.0;
        if (row < A.n) {
            int32_t k = __ldg(A.rp + row) + sub;
            const int32_t k1 = __ldg(A.rp + row + 1);
            for (; k + 3 * VW < k1; k += 4 * VW) {
                double a[4], xx[4];
                int32_t c[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) a[j] = ld_stream(A.v + k + j * VW);
#pragma unroll
                for (int j = 0; j < 4; ++j) c[j] = ld_stream(A.ci + k + j * VW);
#pragma unroll
                for (int j = 0; j < 4; ++j) xx[j] = __ldg(x + c[j]);
#pragma unroll
                for (int j = 0; j < 4; ++j) acc += a[j] * xx[j];
            }
            for (; k < k1; k += VW) acc += ld_stream(A.v + k) * __ldg(x + ld_stream(A.ci + k));
        }
#pragma unroll
        for (int o = VW / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o, VW);
        if (sub == 0 && row < A.n) y[row] = b[row] - acc;
    }
}

// V0 + software pipelining across a warp's rows: the next row's pointers and the
// current row's epilogue operand are loaded before the current row's entries
template <int VW>
__global__ void __launch_bounds__(256) k_v0p(M A, const double* __restrict__ x, const double* __restrict__ b,
                                             double* __restrict__ y) {
    const int64_t gid = (int64_t)blockIdx.x * 256 + threadIdx.x;
    const int sub = threadIdx.x % VW;
    const int64_t g0 = gid / VW, ng = ((int64_t)gridDim.x * 256) / VW;
    const int64_t iters = (A.n + ng - 1) / ng;
    int32_t nk0 = 0, nk1 = 0;
    if (g0 < A.n) {
        nk0 = __ldg(A.rp + g0);
        nk1 = __ldg(A.rp + g0 + 1);
    }
    for (int64_t it = 0; it < iters; ++it) {
        const int64_t row = g0 + it * ng;
        const int32_t k0 = nk0, k1 = nk1;
        const int64_t nrow = row + ng;
        if (nrow < A.n) {
            nk0 = __ldg(A.rp + nrow);
            nk1 = __ldg(A.rp + nrow + 1);
        }
        double acc = 0.0, bi = 0.0;
        if (row < A.n) {
            if (sub == 0) bi = b[row];
            int32_t k = k0 + sub;
            for (; k + 3 * VW < k1; k += 4 * VW) {
                double a[4], xx[4];
                int32_t c[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) a[j] = ld_stream(A.v + k + j * VW);
#pragma unroll
                for (int j = 0; j < 4; ++j) c[j] = ld_stream(A.ci + k + j * VW);
#pragma unroll
                for (int j = 0; j < 4; ++j) xx[j] = __ldg(x + c[j]);
#pragma unroll
                for (int j = 0; j < 4; ++j) acc += a[j] * xx[j];
            }
            for (; k < k1; k += VW) acc += ld_stream(A.v + k) * __ldg(x + ld_stream(A.ci + k));
        }
#pragma unroll
        for (int o = VW / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o, VW);
        if (sub == 0 && row < A.n) y[row] = bi - acc;
    }
}

template <int VW, int CH>
__global__ void __launch_bounds__(256) k_p(M A, const double* __restrict__ x, const double* __restrict__ b,
                                           double* __restrict__ y) {
    const int64_t gid = (int64_t)blockIdx.x * 256 + threadIdx.x;
    const int sub = threadIdx.x % VW;
    const int64_t g0 = gid / VW, ng = ((int64_t)gridDim.x * 256) / VW;
    const int64_t iters = (A.n + ng - 1) / ng;
    for (int64_t it = 0; it < iters; ++it) {
        const int64_t row = g0 + it * ng;
        double acc = 0.0;
        if (row < A.n) {
            int32_t k = __ldg(A.rp + row) + sub;
            const int32_t k1 = __ldg(A.rp + row + 1);
            for (; k < k1; k += CH * VW) {
                double a[CH], xx[CH];
                int32_t c[CH];
#pragma unroll
                for (int j = 0; j < CH; ++j) a[j] = (k + j * VW < k1) ? ld_stream(A.v + k + j * VW) : 0.0;
#pragma unroll
                for (int j = 0; j < CH; ++j) c[j] = (k + j * VW < k1) ? ld_stream(A.ci + k + j * VW) : 0;
#pragma unroll
                for (int j = 0; j < CH; ++j) xx[j] = __ldg(x + c[j]);
#pragma unroll
                for (int j = 0; j < CH; ++j) acc += a[j] * xx[j];
            }
        }
#pragma unroll
        for (int o = VW / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o, VW);
        if (sub == 0 && row < A.n) y[row] = b[row] - acc;
    }
}

template <int CH>
__global__ void __launch_bounds__(256) k_b(M A, const double* __restrict__ x, const double* __restrict__ b,
                                           double* __restrict__ y) {
    __shared__ double part[8];
    for (int64_t row = blockIdx.x; row < A.n; row += gridDim.x) {
        int32_t k = __ldg(A.rp + row) + threadIdx.x;
        const int32_t k1 = __ldg(A.rp + row + 1);
        double acc = 0.0;
        for (; k < k1; k += CH * 256) {
            double a[CH], xx[CH];
            int32_t c[CH];
#pragma unroll
            for (int j = 0; j < CH; ++j) a[j] = (k + j * 256 < k1) ? ld_stream(A.v + k + j * 256) : 0.0;
#pragma unroll
            for (int j = 0; j < CH; ++j) c[j] = (k + j * 256 < k1) ? ld_stream(A.ci + k + j * 256) : 0;
#pragma unroll
            for (int j = 0; j < CH; ++j) xx[j] = __ldg(x + c[j]);
#pragma unroll
            for (int j = 0; j < CH; ++j) acc += a[j] * xx[j];
        }
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
        __syncthreads();
        if (threadIdx.x == 0) {
            double s = 0.0;
            for (int w = 0; w < 8; ++w) s += part[w];
            y[row] = b[row] - s;
        }
        __syncthreads();
    }
}

__global__ void k_flush(double* f, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        f[i] = f[i] * 0.5 + 1.0;
}

struct Op {
    const char* name;
    int64_t n;
    int deg;     // mean entries per row
    int spread;  // +- variation of the row length
    int64_t window;
};

static bool load_csr(const char* path, std::vector<int32_t>& rp, std::vector<int32_t>& ci, std::vector<double>& v,
                     int64_t& n) {
    FILE* f = fopen(path, "rb");
    if (!f) return false;
    int64_t hdr[2];
    if (fread(hdr, 8, 2, f) != 2) return false;
    n = hdr[0];
    rp.resize(n + 1);
    ci.resize(hdr[1]);
    v.resize(hdr[1]);
    bool ok = fread(rp.data(), 4, n + 1, f) == (size_t)(n + 1) && fread(ci.data(), 4, hdr[1], f) == (size_t)hdr[1] &&
              fread(v.data(), 8, hdr[1], f) == (size_t)hdr[1];
    fclose(f);
    return ok;
}

int main(int argc, char** argv) {
    std::vector<Op> ops;
    for (int a = 1; a < argc; ++a) ops.push_back(Op{argv[a], 0, 0, 0, -1});
    if (argc < 2) ops = {{"c2_L2 33k x 150", 32866, 150, 40, 8000},
                      {"c2_L3 4.1k x 585", 4147, 585, 150, 4147},
                      {"c2_L4 522 x 500", 522, 500, 20, 522},
                      {"c5_L1 893k x 110", 892552, 110, 40, 40000},
                      {"c4_L2 262k x 60", 262144, 60, 25, 20000}};
    double* flush;
    const int64_t nf = 32 << 20;
    CK(cudaMalloc(&flush, nf * 8));
    CK(cudaMemset(flush, 0, nf * 8));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (Op& op : ops) {
        std::mt19937_64 rng(7);
        std::vector<int32_t> rp(op.n + 1, 0), ci;
        std::vector<double> v;
        if (op.window < 0) {
            int64_t nn;
            if (!load_csr(op.name, rp, ci, v, nn)) { printf("cannot read %s\n", op.name); continue; }
            op.n = nn;
        } else
        for (int64_t i = 0; i < op.n; ++i) {
            int len = op.deg + (int)(rng() % (2 * op.spread + 1)) - op.spread;
            len = std::max(1, std::min<int>(len, (int)op.n));
            std::vector<int32_t> cols;
            for (int t = 0; t < len; ++t) {
                int64_t c = i + (int64_t)(rng() % (2 * op.window + 1)) - op.window;
                c = std::min<int64_t>(std::max<int64_t>(c, 0), op.n - 1);
                cols.push_back((int32_t)c);
            }
            std::sort(cols.begin(), cols.end());
            cols.erase(std::unique(cols.begin(), cols.end()), cols.end());
            for (int32_t c : cols) {
                ci.push_back(c);
                v.push_back(1.0 / (1 + (rng() % 7)));
            }
            rp[i + 1] = (int32_t)ci.size();
        }
        const int64_t nnz = ci.size();
        int32_t *drp, *dci;
        double *dv, *dx, *db, *dy, *dy0;
        CK(cudaMalloc(&drp, (op.n + 1) * 4));
        CK(cudaMalloc(&dci, nnz * 4));
        CK(cudaMalloc(&dv, nnz * 8));
        CK(cudaMalloc(&dx, op.n * 8));
        CK(cudaMalloc(&db, op.n * 8));
        CK(cudaMalloc(&dy, op.n * 8));
        CK(cudaMalloc(&dy0, op.n * 8));
        CK(cudaMemcpy(drp, rp.data(), (op.n + 1) * 4, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dci, ci.data(), nnz * 4, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dv, v.data(), nnz * 8, cudaMemcpyHostToDevice));
        std::vector<double> hx(op.n);
        for (auto& t : hx) t = (double)(rng() % 1000) / 1000.0;
        CK(cudaMemcpy(dx, hx.data(), op.n * 8, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(db, hx.data(), op.n * 8, cudaMemcpyHostToDevice));
        M A{drp, dci, dv, op.n};
        const double bytes = 12.0 * nnz + 4.0 * (op.n + 1) + 24.0 * op.n;
        printf("== %s: nnz %lld (%.1f/row), %.1f MB\n", op.name, (long long)nnz, (double)nnz / op.n, bytes / 1e6);
        auto grid_for = [&](int vw) {
            int64_t thr = op.n * (int64_t)vw;
            return (int)std::max<int64_t>(1, std::min<int64_t>((thr + 255) / 256, 148 * 8));
        };
        auto run = [&](const char* nm, auto launch) {
            for (int mode = 0; mode < 2; ++mode) {
                float tot = 0.f;
                const int reps = 50;
                for (int r = 0; r < reps + 3; ++r) {
                    if (mode) k_flush<<<148 * 8, 256>>>(flush, nf);
                    cudaEventRecord(e0);
                    launch();
                    cudaEventRecord(e1);
                    cudaEventSynchronize(e1);
                    float ms;
                    cudaEventElapsedTime(&ms, e0, e1);
                    if (r >= 3) tot += ms;
                }
                CK(cudaGetLastError());
                const double us = 1e3 * tot / reps;
                std::vector<double> hy(op.n), hy0(op.n);
                CK(cudaMemcpy(hy.data(), dy, op.n * 8, cudaMemcpyDeviceToHost));
                CK(cudaMemcpy(hy0.data(), dy0, op.n * 8, cudaMemcpyDeviceToHost));
                double err = 0;
                for (int64_t i = 0; i < op.n; ++i) err = std::max(err, std::fabs(hy[i] - hy0[i]));
                printf("  %-10s %s %8.2f us  %7.0f GB/s  err %.1e\n", nm, mode ? "cold" : "warm", us, bytes / us / 1e3,
                       err);
            }
        };
        // reference result
        k_v0<32><<<grid_for(32), 256>>>(A, dx, db, dy0);
        CK(cudaDeviceSynchronize());
#define V0(VW) run("V0/" #VW, [&] { k_v0<VW><<<grid_for(VW), 256>>>(A, dx, db, dy); })
#define PV(VW, CH) run("P" #CH "/" #VW, [&] { k_p<VW, CH><<<grid_for(VW), 256>>>(A, dx, db, dy); })
        if (op.n > 1000000 && (double)nnz / op.n < 24) {  // short rows: narrow groups
            V0(1); V0(2); V0(4);
            PV(1, 4); PV(1, 8); PV(2, 4); PV(2, 8); PV(4, 4); PV(4, 8);
        }
        V0(8); V0(16); V0(32);
        run("V0P/8", [&] { k_v0p<8><<<grid_for(8), 256>>>(A, dx, db, dy); });
        run("V0P/16", [&] { k_v0p<16><<<grid_for(16), 256>>>(A, dx, db, dy); });
        run("V0P/32", [&] { k_v0p<32><<<grid_for(32), 256>>>(A, dx, db, dy); });
        PV(8, 4); PV(8, 8); PV(16, 4); PV(16, 8); PV(32, 4); PV(32, 8);
        run("B/4", [&] { k_b<4><<<(int)std::min<int64_t>(op.n, 148 * 8), 256>>>(A, dx, db, dy); });
        run("B/1", [&] { k_b<1><<<(int)std::min<int64_t>(op.n, 148 * 8), 256>>>(A, dx, db, dy); });
        cudaFree(drp); cudaFree(dci); cudaFree(dv); cudaFree(dx); cudaFree(db); cudaFree(dy); cudaFree(dy0);
    }
    return 0;
}
