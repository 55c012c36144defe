// partition.cpp — see partition.hpp.
#include "partition.hpp"

#include <omp.h>

#include <algorithm>
#include <string>

namespace amgsetup {

namespace {

int owner_of(const std::vector<int64_t>& bounds, int64_t id) {
    // bounds: np+1 ascending; owner = g with bounds[g] <= id < bounds[g+1] (skips empty ranks)
    auto it = std::upper_bound(bounds.begin(), bounds.end(), id);
    return (int)(it - bounds.begin()) - 1;
}

// Rows [r0, r1) of M; columns shifted by -col_shift.
Csr slice_rows(const Csr& M, int64_t r0, int64_t r1, int64_t col_shift, int64_t ncols_local) {
    Csr S;
    S.nrows = r1 - r0;
    S.ncols = ncols_local;
    S.rp.resize(S.nrows + 1);
    const int64_t k0 = M.rp[r0];
    for (int64_t i = 0; i <= S.nrows; ++i) S.rp[i] = M.rp[r0 + i] - k0;
    const int64_t nnz = S.rp[S.nrows];
    S.ci.resize(nnz);
    S.v.assign(M.v.begin() + k0, M.v.begin() + k0 + nnz);
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < nnz; ++k) S.ci[k] = (int32_t)((int64_t)M.ci[k0 + k] - col_shift);
    return S;
}

// Scan the columns of rows [r0, r1) of M: update [lo, hi) and collect the ids outside [o0, o1).
void scan_cols(const Csr& M, int64_t r0, int64_t r1, int64_t o0, int64_t o1, int64_t& lo, int64_t& hi,
               std::vector<int64_t>& outside) {
    if (r1 <= r0) return;
    int64_t mn = lo, mx = hi;
    const int nt = omp_get_max_threads();
    std::vector<std::vector<int64_t>> part(nt);
#pragma omp parallel reduction(min : mn) reduction(max : mx)
    {
        auto& mine = part[omp_get_thread_num()];
#pragma omp for schedule(static)
        for (int64_t i = r0; i < r1; ++i)
            for (int64_t k = M.rp[i]; k < M.rp[i + 1]; ++k) {
                const int64_t c = M.ci[k];
                mn = std::min(mn, c);
                mx = std::max(mx, c + 1);
                if (c < o0 || c >= o1) mine.push_back(c);
            }
    }
    lo = mn;
    hi = mx;
    for (auto& p : part) outside.insert(outside.end(), p.begin(), p.end());
}

}  // namespace

bool partition(const Hierarchy& H, const std::vector<int64_t>& rb0, int64_t rep_bytes, std::vector<RankPlan>& plans,
               std::string& err) {
    const int np = (int)rb0.size() - 1;
    const int nl = (int)H.lv.size();
    if (np < 1 || nl < 1) {
        err = "partition: no ranks or no levels";
        return false;
    }
    const int64_t n0 = H.lv[0].A.nrows;
    if (rb0[0] != 0 || rb0[np] != n0) {
        err = "partition: row blocks must cover [0, n)";
        return false;
    }
    for (int g = 0; g < np; ++g)
        if (rb0[g + 1] < rb0[g]) {
            err = "partition: row blocks must be in rank order";
            return false;
        }
    // ---- owned boundaries per level (owner of the minimum member, R18)
    std::vector<std::vector<int64_t>> ob(nl, std::vector<int64_t>(np + 1, 0));
    ob[0] = rb0;
    for (int l = 0; l + 1 < nl; ++l) {
        const auto& agg = H.lv[l].agg;
        const int64_t nc = H.lv[l + 1].A.nrows;
        std::vector<int64_t> minm(nc, -1);
        for (int64_t i = 0; i < (int64_t)agg.size(); ++i)
            if (minm[agg[i]] < 0) minm[agg[i]] = i;
        for (int g = 0; g <= np; ++g)
            ob[l + 1][g] = (int64_t)(std::lower_bound(minm.begin(), minm.end(), ob[l][g]) - minm.begin());
        ob[l + 1][np] = nc;
    }
    // ---- first replicated level
    // level 0 is always distributed (the caller's vectors are row blocks)
    int lrep = nl - 1;
    for (int l = (np > 1 ? 1 : 0); l < nl; ++l) {
        const double bytes = 12.0 * (double)H.lv[l].A.nnz() + 12.0 * (double)H.lv[l].P.nnz();
        bool empty = false;
        for (int g = 0; g < np; ++g) empty |= (ob[l][g + 1] == ob[l][g]);
        if (l == nl - 1 || (np > 1 && (bytes <= (double)rep_bytes || empty))) {
            lrep = l;
            break;
        }
    }
    if (np > 1 && lrep == 0) {
        err = "partition: a single-level hierarchy cannot be distributed (problem too small for the rank count)";
        return false;
    }
    for (int g = 0; np > 1 && g < np; ++g)
        if (ob[0][g + 1] == ob[0][g]) {
            err = "partition: every rank must own at least one level-0 row";
            return false;
        }
    plans.assign(np, RankPlan());
    for (int g = 0; g < np; ++g) {
        RankPlan& P = plans[g];
        P.rank = g;
        P.nranks = np;
        P.lv.resize(nl);
        for (int l = 0; l < nl; ++l) {
            RankLevel& L = P.lv[l];
            L.n_global = H.lv[l].A.nrows;
            L.replicated = (l >= lrep);
            L.own_begin = ob[l][g];
            L.own_end = ob[l][g + 1];
            L.comp_begin = L.replicated ? 0 : L.own_begin;
            L.comp_end = L.replicated ? L.n_global : L.own_end;
            if (l + 1 < nl) {
                L.rst_begin = L.replicated ? 0 : ob[l + 1][g];
                L.rst_end = L.replicated ? H.lv[l + 1].A.nrows : ob[l + 1][g + 1];
            }
        }
        // ---- windows and halos
        std::vector<std::vector<int64_t>> outside(nl);
        std::vector<int64_t> lo(nl), hi(nl);
        for (int l = 0; l < nl; ++l) {
            RankLevel& L = P.lv[l];
            lo[l] = L.comp_begin;
            hi[l] = L.comp_end;
            if (l > 0) {  // outputs of R_{l-1}
                lo[l] = std::min(lo[l], P.lv[l - 1].rst_begin);
                hi[l] = std::max(hi[l], P.lv[l - 1].rst_end);
            }
        }
        for (int l = 0; l < nl; ++l) {
            RankLevel& L = P.lv[l];
            scan_cols(H.lv[l].A, L.comp_begin, L.comp_end, L.own_begin, L.own_end, lo[l], hi[l], outside[l]);
            if (l + 1 < nl) {
                scan_cols(H.lv[l].R, L.rst_begin, L.rst_end, L.own_begin, L.own_end, lo[l], hi[l], outside[l]);
                const RankLevel& C = P.lv[l + 1];
                scan_cols(H.lv[l].P, L.comp_begin, L.comp_end, C.own_begin, C.own_end, lo[l + 1], hi[l + 1],
                          outside[l + 1]);
            }
        }
        for (int l = 0; l < nl; ++l) {
            RankLevel& L = P.lv[l];
            if (L.replicated) {
                L.win_begin = 0;
                L.win_end = L.n_global;
            } else {
                L.win_begin = std::min(lo[l], L.own_begin);
                L.win_end = std::max(hi[l], L.own_end);
            }
            std::vector<int64_t> ids;
            if (L.replicated) {
                if (l > 0 && !P.lv[l - 1].replicated && np > 1) {  // gather after a distributed restriction
                    for (int64_t i = 0; i < L.own_begin; ++i) ids.push_back(i);
                    for (int64_t i = L.own_end; i < L.n_global; ++i) ids.push_back(i);
                }
            } else {
                ids.swap(outside[l]);
                std::sort(ids.begin(), ids.end());
                ids.erase(std::unique(ids.begin(), ids.end()), ids.end());
            }
            L.recv_off.assign(np + 1, 0);
            for (int64_t id : ids) L.recv_off[owner_of(ob[l], id) + 1]++;
            for (int q = 0; q < np; ++q) L.recv_off[q + 1] += L.recv_off[q];
            L.recv_ids = ids;  // ascending ids are already grouped by owner (contiguous blocks)
            // local operators in window frames
            L.A = slice_rows(H.lv[l].A, L.comp_begin, L.comp_end, L.win_begin, L.win_end - L.win_begin);
            // INVK factors are block-diagonal over the owners (HINVK / l1-INVK): their columns stay
            // inside the rows this rank computes, so they need no halo
            if (!H.lv[l].Wd.rp.empty()) {
                L.Wd = slice_rows(H.lv[l].Wd, L.comp_begin, L.comp_end, L.win_begin, L.win_end - L.win_begin);
                L.Z = slice_rows(H.lv[l].Z, L.comp_begin, L.comp_end, L.win_begin, L.win_end - L.win_begin);
            }
            L.m.assign(H.lv[l].m.begin() + L.win_begin, H.lv[l].m.begin() + L.win_end);
        }
        for (int l = 0; l + 1 < nl; ++l) {
            RankLevel& L = P.lv[l];
            const RankLevel& C = P.lv[l + 1];
            L.P = slice_rows(H.lv[l].P, L.comp_begin, L.comp_end, C.win_begin, C.win_end - C.win_begin);
            L.R = slice_rows(H.lv[l].R, L.rst_begin, L.rst_end, L.win_begin, L.win_end - L.win_begin);
        }
    }
    // ---- send lists: what each rank owns and a peer receives from it
    for (int g = 0; g < np; ++g)
        for (int l = 0; l < nl; ++l) {
            RankLevel& L = plans[g].lv[l];
            L.send_off.assign(np + 1, 0);
            L.send_ids.clear();
            for (int q = 0; q < np; ++q) {
                const RankLevel& Q = plans[q].lv[l];
                if (q != g)
                    L.send_ids.insert(L.send_ids.end(), Q.recv_ids.begin() + Q.recv_off[g],
                                      Q.recv_ids.begin() + Q.recv_off[g + 1]);
                L.send_off[q + 1] = (int64_t)L.send_ids.size();
            }
        }
    return true;
}

}  // namespace amgsetup
