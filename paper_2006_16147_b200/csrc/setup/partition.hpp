// partition.hpp — row-block partition of a built hierarchy over np ranks
// (north_star (4)).
//
// Level 0 rows are split into contiguous blocks (z-slabs for the model problems,
// R15).  A coarse row is owned by the rank owning its aggregate's minimum member
// (R18); because coarse ids ascend with the minimum member (R5), every rank owns
// a contiguous coarse block and the hierarchy itself does not depend on np.
// Levels at or below a size threshold (and always the coarsest) are replicated:
// every rank computes all of their rows after one gather of the restricted rhs.
//
// Every level-l vector on a rank is stored as a contiguous WINDOW [win_begin,
// win_end) of the global vector that covers the rows the rank computes and every
// column its local operators reference; column indices are stored in that window
// frame, so (col - row) offsets of stencil-like operators are preserved (SDIA-32
// keeps working per rank).  The referenced window entries owned by other ranks
// form the halo, received before every kernel that gathers the vector.
#pragma once
#include <cstdint>
#include <vector>

#include "setup.hpp"

namespace amgsetup {

struct RankLevel {
    bool replicated = false;
    int64_t n_global = 0;
    int64_t own_begin = 0, own_end = 0;    // owned rows (global ids)
    int64_t comp_begin = 0, comp_end = 0;  // rows this rank computes (owned, or all if replicated)
    int64_t win_begin = 0, win_end = 0;    // vector window held locally
    // rows of R_l (= level l+1 rows) this rank computes: owned rows of l+1, or all if l replicated
    int64_t rst_begin = 0, rst_end = 0;
    // halo of this level's vectors: global ids grouped by owner rank (ascending inside a group)
    std::vector<int64_t> recv_off, recv_ids;  // np+1 offsets
    std::vector<int64_t> send_off, send_ids;  // np+1 offsets; ids owned here, needed by each peer
    Csr A;  // rows [comp_begin, comp_end), columns in the level-l window frame
    Csr P;  // rows [comp_begin, comp_end), columns in the level-(l+1) window frame
    Csr R;  // rows [rst_begin, rst_end) of level l+1, columns in the level-l window frame
    std::vector<double> m;  // l1-Jacobi inverse diagonal over the whole window
    Csr Wd, Z;              // INVK factors (rows [comp_begin, comp_end), block-diagonal: no halo)
};

struct RankPlan {
    int rank = 0, nranks = 1;
    std::vector<RankLevel> lv;  // one per level including the coarsest
};

// Builds the plan of every rank.  row_bounds: np+1 level-0 boundaries.  Level 0 is
// always distributed; a level l >= 1 (and all coarser ones) is replicated when its
// operator bytes (12 nnz(A_l) + 12 nnz(P-bar_l)) are <= replicate_bytes, when some
// rank would own no row, or when it is the coarsest.  Returns false (and sets err) on an invalid partition.
bool partition(const Hierarchy& H, const std::vector<int64_t>& row_bounds, int64_t replicate_bytes,
               std::vector<RankPlan>& plans, std::string& err);

}  // namespace amgsetup
