// dist_setup.hpp — distributed hierarchy construction.
//
// Every rank holds only its row block of each level and builds the same hierarchy the
// single-process build produces, bit for bit (aggregate maps, A_l, P-bar_l, omega, the
// coarsest inverse), with cross-rank steps only where the method couples rows of
// different ranks:
//  * matching: the locally-dominant matching of PAPER.md:147-150 under the strict order
//    (|c| desc, lo asc, hi asc) — local pointer rounds to a fixed point with the ghosts'
//    state frozen, then an exchange of the boundary vertices' pointers (mutual cross-rank
//    pointers are matched by both sides) and matched flags, repeated until no free vertex
//    has a free neighbour anywhere (the unique LD matching, R5);
//  * coarse numbering: ascending minimum member, i.e. an exclusive scan of the ranks'
//    aggregate counts (R5/R18: every rank owns a contiguous coarse block, the numbering
//    does not depend on np);
//  * Galerkin products: A P rows need the P rows of ghost columns (remote-row gather,
//    PAPER.md:152); P^T (A P) needs, at the owner of each coarse row, the rows i of A P of
//    every fine row with P_iG != 0 in ascending i — remote ones are sent to the owner, so
//    every coarse entry is still summed in the canonical order of C3;
//  * mirroring (C4): a lower entry takes the upper value from the owner of the upper row;
//  * omega: an all-reduce of the maximum (exact, order-free);
//  * the coarsest matrix is all-gathered and inverted on every rank.
// Transport: an abstract all-to-all of byte buffers.  LoopbackComm runs the ranks as
// threads of one process (tests, emulate_ranks); amg_api.cu provides the NCCL transport.
#pragma once
#include <cstdint>
#include <functional>
#include <string>
#include <vector>

#include "partition.hpp"
#include "setup.hpp"

namespace amgsetup {

struct Comm {
    virtual ~Comm() = default;
    virtual int rank() const = 0;
    virtual int size() const = 0;
    // personalised all-to-all: out[q] is delivered to rank q, in[q] receives rank q's buffer
    virtual bool alltoallv(const std::vector<std::vector<char>>& out, std::vector<std::vector<char>>& in) = 0;
};

// One level of the distributed hierarchy on one rank.
struct DistLevel {
    int64_t n = 0;                 // global rows
    std::vector<int64_t> bounds;   // np+1 owned row ranges (R18)
    Csr A;                         // owned rows, GLOBAL column ids, ncols = n
    std::vector<double> w, m;      // owned rows
    Csr P;                         // P-bar owned rows, global coarse ids (non-coarsest)
    Csr R;                         // owned rows of the next level, global fine ids (P-bar^T)
    std::vector<int32_t> agg;      // owned rows -> global coarse id
    double omega = 0.0;
    int sweeps = 0;
    int64_t nnzA = 0, nnzP = 0;    // global counts
};

struct DistHierarchy {
    std::vector<DistLevel> lv;
    std::vector<double> coarse_inv;  // dense A_L^{-1}, replicated
    Csr coarse_A;                    // the whole A_L (replicated)
};

// SPMD build on every rank of `comm`: A_loc holds rows [bounds0[r], bounds0[r+1]) with global
// column ids (validated by the caller), w_loc the same rows of w.
int build_distributed(Comm& comm, const std::vector<int64_t>& bounds0, Csr&& A_loc, std::vector<double>&& w_loc,
                      const Config& cfg, DistHierarchy& out, std::string& err);

// The rank's plan (identical to partition() of the single-process hierarchy for this rank):
// windows, halos, local operators in window frames, replicated levels all-gathered.
bool partition_distributed(Comm& comm, const DistHierarchy& H, int64_t replicate_bytes, RankPlan& plan,
                           std::string& err);

// The checks of validate() on a row-distributed matrix (symmetry through the owners of the
// off-rank couplings); the same error on every rank.
int validate_distributed(Comm& comm, const std::vector<int64_t>& bounds, const Csr& A_loc,
                         const std::vector<double>& w_loc, std::string& err);
int64_t comm_allreduce_sum(Comm& comm, int64_t v);

// Runs fn(comm) on nranks threads of this process, each with its own LoopbackComm.
void run_loopback(int nranks, const std::function<void(Comm&)>& fn);

}  // namespace amgsetup
