// setup.hpp — host-side hierarchy construction of the product library.
//
// Built once per matrix (setup on the host; the solve phase runs
// on the GPU).  Independent of oracle/: different algorithms (parallel
// locally-dominant pointer rounds instead of a sorted greedy scan, row-parallel
// SpGEMM with per-thread accumulators) that follow the same canonical arithmetic
// contract so that the aggregate maps are bit-identical.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace amgsetup {

struct Csr {
    int64_t nrows = 0, ncols = 0;
    std::vector<int64_t> rp;   // nrows+1
    std::vector<int32_t> ci;   // ascending within a row
    std::vector<double> v;
    int64_t nnz() const { return (int64_t)rp.size() <= nrows ? 0 : rp[nrows]; }
};

struct Config {
    int sweeps_per_level = 3;
    int smooth_prolongator = 1;
    double prol_omega_scale = 4.0 / 3.0;
    int64_t max_coarse_size = 200;
    int max_levels = 20;
    double min_coarsening_ratio = 1.2;
    int pre_sweeps = 1, post_sweeps = 1;
    int threads = 0;
    int device = 0;  // 1: build on the GPU (setup_gpu.cu, bit-identical results)
};

struct Level {
    Csr A;                    // A_l
    Csr P;                    // smoothed prolongator P-bar_l (n_l x n_{l+1}), empty at coarsest
    Csr R;                    // P-bar_l^T
    std::vector<int32_t> agg; // composite aggregate map (n_l), empty at coarsest
    std::vector<double> w;    // w_l
    std::vector<double> m;    // l1-Jacobi inverse diagonal 1/(sum_j |a_ij|)
    double omega = 0.0;
    int sweeps = 0;
    Csr Wd, Z;                // INVK smoother (smoother == 1): D^{-1} W and Z = W^T
};

// Device-resident operators handed over by the GPU build (raw cudaMalloc'd arrays, freed
// by the consumer with cudaFree): the host Hierarchy then carries only their row pointers.
struct DevCsrRaw {
    int64_t nrows = 0, ncols = 0, nnz = 0;
    int64_t* rp = nullptr;
    int32_t* ci = nullptr;
    double* v = nullptr;
};
struct DeviceKeep {
    std::vector<DevCsrRaw> A, P, R;  // per level (P, R: non-coarsest levels)
    std::vector<double*> m;          // l1-Jacobi inverse diagonals
    void free_all();
};

struct Hierarchy {
    std::vector<Level> lv;
    bool keep_device = false;        // GPU build: keep A_l, P-bar_l, R_l, m_l on the device (dev)
    DeviceKeep dev;
    std::vector<double> coarse_inv;  // dense A_L^{-1}, row-major n_L x n_L
    double setup_s = 0.0;
};

enum { SETUP_OK = 0, SETUP_ERR_ARG = 1, SETUP_ERR_NOT_SPD = 2 };

// Validates A (square, sorted, exactly symmetric, positive diagonal) and w.
int validate(const Csr& A, const std::vector<double>& w, std::string& err);
// Full build.  A0 is moved in.
int build(Csr&& A0, std::vector<double>&& w0, const Config& cfg, Hierarchy& out,
          std::string& err);

// The same build on the current CUDA device (setup_gpu.cu); A0 already validated.
int build_gpu(Csr&& A0, std::vector<double>&& w0, const Config& cfg, Hierarchy& out, std::string& err);
bool dense_inverse_host(const Csr& A, std::vector<double>& inv);
// INVK smoother factors of A: IC(0) = ILU(0) in LDL^T form, W = L^{-1}
// truncated to `fill` levels of positional fill, Wd = D^{-1} W, Z = W^T.  false on a
// non-positive pivot.
bool invk_factors(const Csr& A, int fill, Csr& Wd, Csr& Z);
// The paper's parallel block-Jacobi setting: the matrix whose INVK factors a
// rank uses is its diagonal block A_pp (HINVK) or A_pp + D_l1,p (l1 = true, l1-INVK, Eq. 3.5
// weights of the couplings outside the block).  owner[i] = block of row i (empty: one block).
Csr block_diagonal_part(const Csr& A, const std::vector<int32_t>& owner, bool l1);
// Block of every row of every level: level-0 rows by `bounds0` (nb+1 ascending boundaries), a
// coarse row by the block of its aggregate's minimum member (R18, as the rank partition).
std::vector<std::vector<int32_t>> level_blocks(const Hierarchy& H, const std::vector<int64_t>& bounds0);
void tmark(const char* what);

// Building blocks (exported for the setup self-tests).
Csr spgemm_canonical(const Csr& A, const Csr& Y);
Csr transpose(const Csr& X);
void mirror_drop(Csr& C);
void ld_matching(const Csr& A, const std::vector<double>& w, std::vector<int32_t>& mate);

}  // namespace amgsetup
