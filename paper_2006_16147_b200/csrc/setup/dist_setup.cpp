// dist_setup.cpp — see dist_setup.hpp.  Compiled with -ffp-contract=off (canonical
// arithmetic contract C1); every floating-point expression below is parenthesised exactly as
// in setup.cpp / SURVEY.md §8c O2.1, O2.4, O4, O5, and every sum runs in the order of C3.
#include "dist_setup.hpp"

#include <omp.h>

#include <algorithm>
#include <cmath>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <limits>
#include <mutex>
#include <thread>

namespace amgsetup {

namespace {

// ------------------------------------------------------------------ bytes
struct Wr {
    std::vector<char>& b;
    template <class T>
    void put(const T& v) {
        const char* p = (const char*)&v;
        b.insert(b.end(), p, p + sizeof(T));
    }
    template <class T>
    void putv(const T* p, int64_t n) {
        put<int64_t>(n);
        const char* c = (const char*)p;
        b.insert(b.end(), c, c + n * (int64_t)sizeof(T));
    }
};
struct Rd {
    const std::vector<char>& b;
    size_t pos = 0;
    bool done() const { return pos >= b.size(); }
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
        if (n) std::memcpy(v.data(), b.data() + pos, n * sizeof(T));
        pos += n * sizeof(T);
    }
};

int owner_of(const std::vector<int64_t>& b, int64_t id) {
    return (int)(std::upper_bound(b.begin(), b.end(), id) - b.begin()) - 1;
}

template <class T>
void a2a_vec(Comm& c, const std::vector<std::vector<T>>& out, std::vector<std::vector<T>>& in) {
    const int np = c.size();
    std::vector<std::vector<char>> ob(np), ib;
    for (int q = 0; q < np; ++q) {
        ob[q].resize(out[q].size() * sizeof(T));
        if (!out[q].empty()) std::memcpy(ob[q].data(), out[q].data(), ob[q].size());
    }
    c.alltoallv(ob, ib);
    in.assign(np, {});
    for (int q = 0; q < np; ++q) {
        in[q].resize(ib[q].size() / sizeof(T));
        if (!in[q].empty()) std::memcpy(in[q].data(), ib[q].data(), ib[q].size());
    }
}

template <class T>
std::vector<T> allgatherv(Comm& c, const std::vector<T>& mine) {
    std::vector<std::vector<T>> out(c.size(), mine), in;
    a2a_vec(c, out, in);
    std::vector<T> all;
    for (auto& v : in) all.insert(all.end(), v.begin(), v.end());
    return all;
}
int64_t allreduce_sum(Comm& c, int64_t v) {
    int64_t s = 0;
    for (int64_t x : allgatherv(c, std::vector<int64_t>{v})) s += x;
    return s;
}
double allreduce_max(Comm& c, double v) {
    double m = -std::numeric_limits<double>::infinity();
    for (double x : allgatherv(c, std::vector<double>{v})) m = std::max(m, x);
    return m;
}

// ------------------------------------------------------------------ ghosts
// The non-owned ids a rank references, sorted (hence grouped by owner in rank order), and for
// every peer the owned ids it asked for.
struct GhostPlan {
    std::vector<int64_t> ids;
    std::vector<std::vector<int64_t>> serve;
    int64_t find(int64_t id) const {  // index in ids, or -1
        auto it = std::lower_bound(ids.begin(), ids.end(), id);
        return (it != ids.end() && *it == id) ? (int64_t)(it - ids.begin()) : -1;
    }
};

GhostPlan make_plan(Comm& c, const std::vector<int64_t>& bounds, std::vector<int64_t> ids) {
    const int me = c.rank(), np = c.size();
    std::sort(ids.begin(), ids.end());
    ids.erase(std::unique(ids.begin(), ids.end()), ids.end());
    GhostPlan g;
    std::vector<std::vector<int64_t>> req(np);
    for (int64_t id : ids) {
        const int o = owner_of(bounds, id);
        if (o == me) continue;
        g.ids.push_back(id);
        req[o].push_back(id);
    }
    a2a_vec(c, req, g.serve);
    return g;
}

// values of the plan's ghost ids (aligned with g.ids) from the owners' local arrays
template <class T>
std::vector<T> fetch(Comm& c, const GhostPlan& g, const std::vector<T>& local, int64_t b0) {
    const int np = c.size();
    std::vector<std::vector<T>> out(np), in;
    for (int q = 0; q < np; ++q)
        for (int64_t id : g.serve[q]) out[q].push_back(local[id - b0]);
    a2a_vec(c, out, in);
    std::vector<T> v;
    for (auto& x : in) v.insert(v.end(), x.begin(), x.end());
    return v;
}

// rows of a row-distributed matrix (owned rows, global column ids) for the plan's ghost ids
Csr fetch_rows(Comm& c, const GhostPlan& g, const Csr& M, int64_t b0) {
    const int np = c.size();
    std::vector<std::vector<char>> out(np), in;
    for (int q = 0; q < np; ++q) {
        Wr w{out[q]};
        for (int64_t id : g.serve[q]) {
            const int64_t r = id - b0;
            w.putv(M.ci.data() + M.rp[r], M.rp[r + 1] - M.rp[r]);
            w.putv(M.v.data() + M.rp[r], M.rp[r + 1] - M.rp[r]);
        }
    }
    c.alltoallv(out, in);
    Csr G;
    G.nrows = (int64_t)g.ids.size();
    G.ncols = M.ncols;
    G.rp.assign(1, 0);
    for (int q = 0; q < np; ++q) {
        Rd r{in[q]};
        while (!r.done()) {
            std::vector<int32_t> ci;
            std::vector<double> v;
            r.getv(ci);
            r.getv(v);
            G.ci.insert(G.ci.end(), ci.begin(), ci.end());
            G.v.insert(G.v.end(), v.begin(), v.end());
            G.rp.push_back((int64_t)G.ci.size());
        }
    }
    return G;
}

std::vector<int64_t> col_ids(const Csr& M) {
    std::vector<int64_t> ids(M.ci.begin(), M.ci.end());
    std::sort(ids.begin(), ids.end());
    ids.erase(std::unique(ids.begin(), ids.end()), ids.end());
    return ids;
}

// row of a matrix given as owned rows + ghost rows: (ptr, ptr, len)
struct RowRef {
    const int32_t* ci;
    const double* v;
    int64_t n;
};
RowRef row_of(const Csr& M, int64_t r) { return {M.ci.data() + M.rp[r], M.v.data() + M.rp[r], M.rp[r + 1] - M.rp[r]}; }

// One output row of a canonical product (C3): the products arrive as (column, value) in
// canonical order; each column is summed from +0.0 in arrival order (a stable sort by column
// keeps that order), then the row is emitted with ascending columns.
struct RowAcc {
    std::vector<std::pair<int32_t, double>> prod;
    void clear() { prod.clear(); }
    void add(int32_t K, double p) { prod.emplace_back(K, p); }
    void emit(std::vector<int32_t>& ci, std::vector<double>& v) {
        std::stable_sort(prod.begin(), prod.end(),
                         [](const std::pair<int32_t, double>& a, const std::pair<int32_t, double>& b) {
                             return a.first < b.first;
                         });
        for (size_t k = 0; k < prod.size();) {
            const int32_t K = prod[k].first;
            double acc = 0.0;
            for (; k < prod.size() && prod[k].first == K; ++k) acc += prod[k].second;
            ci.push_back(K);
            v.push_back(acc);
        }
    }
};

// ------------------------------------------------------------------ local helpers
double diag_of(const Csr& A, int64_t r, int64_t gid) {
    const int32_t* b = A.ci.data() + A.rp[r];
    const int32_t* e = A.ci.data() + A.rp[r + 1];
    const int32_t* p = std::lower_bound(b, e, (int32_t)gid);
    return (p != e && *p == gid) ? A.v[p - A.ci.data()] : 0.0;
}

std::vector<double> l1_inv_rows(const Csr& A) {
    std::vector<double> m(A.nrows);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < A.nrows; ++i) {
        double s = 0.0;
        for (int64_t k = A.rp[i]; k < A.rp[i + 1]; ++k) s += std::fabs(A.v[k]);
        m[i] = 1.0 / s;
    }
    return m;
}

// T = A Y for the owned rows of A (global column ids); Y's rows: owned rows (Yown, ids
// [b0, b1)) and ghost rows (Ygh, aligned with g.ids).  Canonical order C3.
Csr spgemm_rows(const Csr& A, int64_t b0, const Csr& Yown, const GhostPlan& g, const Csr& Ygh, int64_t ncols) {
    const int64_t n = A.nrows;
    const int64_t b1 = b0 + Yown.nrows;
    std::vector<std::vector<int32_t>> rc(n);
    std::vector<std::vector<double>> rv(n);
#pragma omp parallel
    {
        RowAcc acc;
#pragma omp for schedule(dynamic, 256)
        for (int64_t i = 0; i < n; ++i) {
            acc.clear();
            for (int64_t k = A.rp[i]; k < A.rp[i + 1]; ++k) {
                const int64_t j = A.ci[k];
                const double a = A.v[k];
                const RowRef y = (j >= b0 && j < b1) ? row_of(Yown, j - b0) : row_of(Ygh, g.find(j));
                for (int64_t t = 0; t < y.n; ++t) acc.add(y.ci[t], a * y.v[t]);
            }
            acc.emit(rc[i], rv[i]);
        }
    }
    Csr T;
    T.nrows = n;
    T.ncols = ncols;
    T.rp.assign(n + 1, 0);
    for (int64_t i = 0; i < n; ++i) T.rp[i + 1] = T.rp[i] + (int64_t)rc[i].size();
    T.ci.resize(T.rp[n]);
    T.v.resize(T.rp[n]);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        std::copy(rc[i].begin(), rc[i].end(), T.ci.begin() + T.rp[i]);
        std::copy(rv[i].begin(), rv[i].end(), T.v.begin() + T.rp[i]);
    }
    return T;
}

// Contributions to the owned coarse rows of X^T T: the entries (G, i, x_iG) of X's owned rows
// whose G is owned by `me`, and from the other ranks the same for their rows, each with the
// row T_i (and w_i for P^T w).  Owner side: per owned G, the contributions sorted by i.
struct Contrib {
    int64_t G, i;
    double x, w;
    RowRef row;
};

// Sends, for every owned fine row i and every entry (G, x) of X_i with G owned by another
// rank, the row T_i (once per destination) with its (G, x) list and w_i; returns all
// contributions to this rank's coarse rows (local ones included), sorted by (G, i).
std::vector<Contrib> gather_contribs(Comm& c, const Csr& X, const Csr& T, const std::vector<double>& w, int64_t b0,
                                     const std::vector<int64_t>& cbounds, std::vector<std::vector<char>>& keep) {
    const int me = c.rank(), np = c.size();
    std::vector<std::vector<char>> out(np);
    std::vector<Contrib> mine;
    for (int64_t r = 0; r < X.nrows; ++r) {
        int last = -1;
        for (int64_t k = X.rp[r]; k < X.rp[r + 1]; ++k) {
            const int64_t G = X.ci[k];
            const int o = owner_of(cbounds, G);
            if (o == me) {
                mine.push_back(Contrib{G, b0 + r, X.v[k], w.empty() ? 0.0 : w[r], row_of(T, r)});
                continue;
            }
            if (o == last) continue;  // this row already went to that owner
            last = o;
            Wr wr{out[o]};
            wr.put<int64_t>(b0 + r);
            wr.put<double>(w.empty() ? 0.0 : w[r]);
            std::vector<int64_t> gs;
            std::vector<double> xs;
            for (int64_t k2 = X.rp[r]; k2 < X.rp[r + 1]; ++k2)
                if (owner_of(cbounds, X.ci[k2]) == o) {
                    gs.push_back(X.ci[k2]);
                    xs.push_back(X.v[k2]);
                }
            wr.putv(gs.data(), (int64_t)gs.size());
            wr.putv(xs.data(), (int64_t)xs.size());
            wr.putv(T.ci.data() + T.rp[r], T.rp[r + 1] - T.rp[r]);
            if ((T.rp[r + 1] - T.rp[r]) & 1) wr.put<int32_t>(0);  // keep the values 8-byte aligned
            wr.putv(T.v.data() + T.rp[r], T.rp[r + 1] - T.rp[r]);
        }
    }
    c.alltoallv(out, keep);
    for (int q = 0; q < np; ++q) {
        const std::vector<char>& b = keep[q];
        size_t pos = 0;
        while (pos < b.size()) {
            int64_t i;
            double wi;
            std::memcpy(&i, b.data() + pos, 8);
            pos += 8;
            std::memcpy(&wi, b.data() + pos, 8);
            pos += 8;
            int64_t ng;
            std::memcpy(&ng, b.data() + pos, 8);
            pos += 8;
            const int64_t* gs = (const int64_t*)(b.data() + pos);
            pos += 8 * ng;
            int64_t nx;
            std::memcpy(&nx, b.data() + pos, 8);
            pos += 8;
            const double* xs = (const double*)(b.data() + pos);
            pos += 8 * nx;
            int64_t nc;
            std::memcpy(&nc, b.data() + pos, 8);
            pos += 8;
            const int32_t* ci = (const int32_t*)(b.data() + pos);
            pos += 4 * nc + ((nc & 1) ? 4 : 0);
            int64_t nv;
            std::memcpy(&nv, b.data() + pos, 8);
            pos += 8;
            const double* vv = (const double*)(b.data() + pos);
            pos += 8 * nv;
            for (int64_t k = 0; k < ng; ++k) {
                double gx, gxw;
                int64_t G;
                std::memcpy(&G, gs + k, 8);
                std::memcpy(&gx, xs + k, 8);
                gxw = wi;
                mine.push_back(Contrib{G, i, gx, gxw, RowRef{ci, vv, nc}});
            }
        }
    }
    std::sort(mine.begin(), mine.end(),
              [](const Contrib& a, const Contrib& b) { return a.G != b.G ? a.G < b.G : a.i < b.i; });
    return mine;
}

// C = X^T T on the owned coarse rows [cb0, cb1): row G sums x_iG * t_iK over i ascending, then
// K ascending, from +0.0 (C3).  Also w_next = X^T w and R = X^T (rows G, (i, x_iG)).
void owner_products(const std::vector<Contrib>& cs, int64_t cb0, int64_t cb1, int64_t ncols, Csr& C,
                    std::vector<double>* wnext, Csr* Rt, int64_t nfine) {
    const int64_t nc = cb1 - cb0;
    std::vector<int64_t> start(nc + 1, 0);
    for (const Contrib& x : cs) start[x.G - cb0 + 1]++;
    for (int64_t g = 0; g < nc; ++g) start[g + 1] += start[g];
    std::vector<std::vector<int32_t>> rc(nc);
    std::vector<std::vector<double>> rv(nc);
#pragma omp parallel
    {
        RowAcc acc;
#pragma omp for schedule(dynamic, 64)
        for (int64_t g = 0; g < nc; ++g) {
            acc.clear();
            for (int64_t q = start[g]; q < start[g + 1]; ++q) {
                const Contrib& x = cs[q];
                for (int64_t t = 0; t < x.row.n; ++t) acc.add(x.row.ci[t], x.x * x.row.v[t]);
            }
            acc.emit(rc[g], rv[g]);
        }
    }
    C = Csr();
    C.nrows = nc;
    C.ncols = ncols;
    C.rp.assign(nc + 1, 0);
    for (int64_t g = 0; g < nc; ++g) C.rp[g + 1] = C.rp[g] + (int64_t)rc[g].size();
    C.ci.resize(C.rp[nc]);
    C.v.resize(C.rp[nc]);
    for (int64_t g = 0; g < nc; ++g) {
        std::copy(rc[g].begin(), rc[g].end(), C.ci.begin() + C.rp[g]);
        std::copy(rv[g].begin(), rv[g].end(), C.v.begin() + C.rp[g]);
    }
    if (wnext) {
        wnext->assign(nc, 0.0);
        for (int64_t g = 0; g < nc; ++g) {
            double s = 0.0;
            for (int64_t q = start[g]; q < start[g + 1]; ++q) s += cs[q].x * cs[q].w;
            (*wnext)[g] = s;
        }
    }
    if (Rt) {
        *Rt = Csr();
        Rt->nrows = nc;
        Rt->ncols = nfine;
        Rt->rp.assign(nc + 1, 0);
        for (int64_t g = 0; g < nc; ++g) Rt->rp[g + 1] = start[g + 1];
        Rt->ci.resize(cs.size());
        Rt->v.resize(cs.size());
        for (size_t q = 0; q < cs.size(); ++q) {
            Rt->ci[q] = (int32_t)cs[q].i;
            Rt->v[q] = cs[q].x;
        }
    }
}

// C4 + C5 on the owned rows [b0, b0 + C.nrows) of a symmetric-pattern product: a lower entry
// (c < r) takes the value of the upper entry (c, r) -- from the owner of row c -- or 0.0 if
// that entry does not exist; exact zeros are dropped.
void mirror_drop_dist(Comm& c, Csr& C, int64_t b0, const std::vector<int64_t>& bounds) {
    const int me = c.rank(), np = c.size();
    const int64_t n = C.nrows;
    std::vector<std::vector<int64_t>> req(np), got;
    for (int64_t r = 0; r < n; ++r)
        for (int64_t k = C.rp[r]; k < C.rp[r + 1]; ++k) {
            const int64_t col = C.ci[k];
            if (col >= b0 + r) break;
            const int o = owner_of(bounds, col);
            if (o != me) {
                req[o].push_back(col);
                req[o].push_back(b0 + r);
            }
        }
    a2a_vec(c, req, got);
    std::vector<std::vector<double>> ans(np), recv;
    auto lookup = [&](int64_t row, int64_t col, double& v) {
        const int64_t r = row - b0;
        const int32_t* b = C.ci.data() + C.rp[r];
        const int32_t* e = C.ci.data() + C.rp[r + 1];
        const int32_t* p = std::lower_bound(b, e, (int32_t)col);
        if (p != e && *p == col) {
            v = C.v[p - C.ci.data()];
            return true;
        }
        return false;
    };
    for (int q = 0; q < np; ++q)
        for (size_t k = 0; k + 1 < got[q].size(); k += 2) {
            double v = 0.0;
            if (!lookup(got[q][k], got[q][k + 1], v)) v = 0.0;
            ans[q].push_back(v);
        }
    a2a_vec(c, ans, recv);
    std::vector<size_t> pos(np, 0);
    std::vector<double> nv(C.nnz());
    for (int64_t r = 0; r < n; ++r)
        for (int64_t k = C.rp[r]; k < C.rp[r + 1]; ++k) {
            const int64_t col = C.ci[k];
            double val = C.v[k];
            if (col < b0 + r) {
                const int o = owner_of(bounds, col);
                if (o == me) {
                    double u;
                    val = lookup(col, b0 + r, u) ? u : 0.0;
                } else {
                    val = recv[o][pos[o]++];
                }
            }
            nv[k] = val;
        }
    Csr D;
    D.nrows = n;
    D.ncols = C.ncols;
    D.rp.assign(n + 1, 0);
    for (int64_t r = 0; r < n; ++r) {
        for (int64_t k = C.rp[r]; k < C.rp[r + 1]; ++k)
            if (nv[k] != 0.0) {
                D.ci.push_back(C.ci[k]);
                D.v.push_back(nv[k]);
            }
        D.rp[r + 1] = (int64_t)D.ci.size();
    }
    C = std::move(D);
}

// ------------------------------------------------------------------ matching
// Distributed locally-dominant matching on the owned rows of A (global ids) with weights w.
// mate[r] = global id of the partner of owned row r, or -1.  Returns false if the rounds stall.
bool dist_matching(Comm& c, const Csr& A, const std::vector<double>& w, int64_t b0, const GhostPlan& g,
                   std::vector<int64_t>& mate) {
    const int64_t nloc = A.nrows, b1 = b0 + nloc;
    const int64_t ng = (int64_t)g.ids.size();
    const int64_t nb = std::lower_bound(g.ids.begin(), g.ids.end(), b0) - g.ids.begin();  // ghosts below
    // local index space: ghosts below | owned rows | ghosts above (monotone in the global id)
    auto lid = [&](int64_t gid) -> int64_t {
        if (gid >= b0 && gid < b1) return nb + (gid - b0);
        const int64_t p = g.find(gid);
        return p < nb ? p : p + nloc;
    };
    auto gid_of = [&](int64_t u) -> int64_t {
        if (u >= nb && u < nb + nloc) return b0 + (u - nb);
        return u < nb ? g.ids[u] : g.ids[u - nloc];
    };
    auto is_own = [&](int64_t u) { return u >= nb && u < nb + nloc; };
    std::vector<double> dl(nloc);
    for (int64_t r = 0; r < nloc; ++r) dl[r] = diag_of(A, r, b0 + r);
    const std::vector<double> dg = fetch(c, g, dl, b0);
    const std::vector<double> wg = fetch(c, g, w, b0);
    auto dval = [&](int64_t gid) { return (gid >= b0 && gid < b1) ? dl[gid - b0] : dg[g.find(gid)]; };
    auto wval = [&](int64_t gid) { return (gid >= b0 && gid < b1) ? w[gid - b0] : wg[g.find(gid)]; };
    // keys (Eq. 3.2, O2.1) and local column indices
    std::vector<double> key(A.nnz());
    std::vector<int64_t> lcol(A.nnz());
#pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t r = 0; r < nloc; ++r) {
        const int64_t i = b0 + r;
        for (int64_t k = A.rp[r]; k < A.rp[r + 1]; ++k) {
            const int64_t j = A.ci[k];
            lcol[k] = lid(j);
            if (j == i) {
                key[k] = -1.0;
                continue;
            }
            const int64_t lo = std::min(i, j), hi = std::max(i, j);
            const double a = A.v[k];
            const double den = (dval(lo) * wval(lo)) * wval(lo) + (dval(hi) * wval(hi)) * wval(hi);
            if (den == 0.0) {
                key[k] = -1.0;
                continue;
            }
            const double cc = 1.0 - (((2.0 * a) * wval(lo)) * wval(hi)) / den;
            key[k] = (cc == 0.0) ? -1.0 : std::fabs(cc);
        }
    }
    const int64_t nu = nloc + ng;
    std::vector<char> matched(nu, 0);
    std::vector<int64_t> ptr(nloc, -1);  // local index of the best free neighbour
    mate.assign(nloc, -1);
    auto best = [&](int64_t r) -> int64_t {
        int64_t b = -1;
        double bk = -1.0;
        for (int64_t k = A.rp[r]; k < A.rp[r + 1]; ++k) {
            const double kk = key[k];
            if (kk < 0.0) continue;
            const int64_t u = lcol[k];
            if (matched[u]) continue;
            if (kk > bk || (kk == bk && u < b)) {
                bk = kk;
                b = u;
            }
        }
        return b;
    };
    // adjacency of owned rows in local indices (for the "who pointed at a matched vertex" pass)
    for (int64_t r = 0; r < nloc; ++r) ptr[r] = best(r);
    std::vector<int64_t> cand(nloc);
    for (int64_t r = 0; r < nloc; ++r) cand[r] = r;
    std::vector<int64_t> stamp(nloc, -1);
    int64_t stampc = 0;
    // serve lists as local rows
    const int np = c.size();
    for (int64_t iter = 0;; ++iter) {
        int64_t nlocal = 0;
        // (1) local pointer rounds to a fixed point, ghosts frozen
        while (!cand.empty()) {
            ++stampc;
            std::vector<std::pair<int64_t, int64_t>> pairs;
            for (int64_t r : cand) {
                if (matched[nb + r]) continue;
                const int64_t t = ptr[r];
                if (t < 0 || !is_own(t) || matched[t]) continue;
                const int64_t tr = t - nb;
                if (ptr[tr] != nb + r) continue;
                const int64_t lo = std::min(r, tr);
                if (stamp[lo] == stampc) continue;
                stamp[lo] = stampc;
                pairs.emplace_back(r, tr);
            }
            if (pairs.empty()) break;
            nlocal += (int64_t)pairs.size();
            std::vector<int64_t> ends;
            for (auto& pr : pairs) {
                matched[nb + pr.first] = matched[nb + pr.second] = 1;
                mate[pr.first] = b0 + pr.second;
                mate[pr.second] = b0 + pr.first;
                ends.push_back(pr.first);
                ends.push_back(pr.second);
            }
            ++stampc;
            std::vector<int64_t> W;
            for (int64_t e : ends)
                for (int64_t k = A.rp[e]; k < A.rp[e + 1]; ++k) {
                    const int64_t u = lcol[k];
                    if (!is_own(u) || matched[u]) continue;
                    const int64_t ur = u - nb;
                    if (!matched[ptr[ur] < 0 ? u : ptr[ur]]) continue;  // its target is still free
                    if (stamp[ur] == stampc) continue;
                    stamp[ur] = stampc;
                    W.push_back(ur);
                }
            for (int64_t ur : W) ptr[ur] = best(ur);
            ++stampc;
            cand.clear();
            for (int64_t ur : W) {
                if (stamp[ur] != stampc) {
                    stamp[ur] = stampc;
                    cand.push_back(ur);
                }
                const int64_t t = ptr[ur];
                if (t >= 0 && is_own(t) && stamp[t - nb] != stampc) {
                    stamp[t - nb] = stampc;
                    cand.push_back(t - nb);
                }
            }
        }
        // (2) the boundary vertices' pointers (global id, -1 if matched / none) to the ranks
        // that ghost them; a mutual cross-rank pointer pair of free vertices is matched by both
        std::vector<std::vector<int64_t>> out(np), in;
        for (int q = 0; q < np; ++q)
            for (int64_t id : g.serve[q]) {
                const int64_t r = id - b0;
                out[q].push_back((matched[nb + r] || ptr[r] < 0) ? -1 : gid_of(ptr[r]));
            }
        a2a_vec(c, out, in);
        std::vector<int64_t> gptr;
        for (auto& v : in) gptr.insert(gptr.end(), v.begin(), v.end());
        int64_t newx = 0;
        for (int64_t r = 0; r < nloc; ++r) {
            if (matched[nb + r]) continue;
            const int64_t t = ptr[r];
            if (t < 0 || is_own(t) || matched[t]) continue;
            const int64_t gi = t < nb ? t : t - nloc;
            if (gptr[gi] != b0 + r) continue;
            matched[nb + r] = matched[t] = 1;
            mate[r] = g.ids[gi];
            ++newx;
        }
        // (3) matched flags of the boundary vertices
        for (int q = 0; q < np; ++q) {
            out[q].clear();
            for (int64_t id : g.serve[q]) out[q].push_back(matched[nb + (id - b0)] ? 1 : 0);
        }
        a2a_vec(c, out, in);
        {
            int64_t gi = 0;
            for (auto& v : in)
                for (int64_t f : v) {
                    const int64_t u = gi < nb ? gi : gi + nloc;
                    if (f) matched[u] = 1;
                    ++gi;
                }
        }
        // (4) re-point the free owned vertices whose target was matched; global progress test
        cand.clear();
        int64_t active = 0;
        for (int64_t r = 0; r < nloc; ++r) {
            if (matched[nb + r]) continue;
            if (ptr[r] >= 0 && matched[ptr[r]]) {
                ptr[r] = best(r);
                cand.push_back(r);
            }
            if (ptr[r] >= 0) {
                ++active;
                if (!is_own(ptr[r])) cand.push_back(r);
            }
        }
        std::sort(cand.begin(), cand.end());
        cand.erase(std::unique(cand.begin(), cand.end()), cand.end());
        const int64_t act = allreduce_sum(c, active);
        const int64_t prog = allreduce_sum(c, newx + nlocal);
        if (act == 0) break;
        // a pass that matched nothing anywhere while free edges remain cannot happen for a strict
        // total order (the heaviest free edge is always mutual): report instead of looping
        if (prog == 0) return false;
    }
    return true;
}

// ------------------------------------------------------------------ one pairwise sweep
struct DistSweep {
    std::vector<int32_t> agg;     // owned rows -> global coarse id
    std::vector<double> pval;     // NaN: no stored entry
    std::vector<int64_t> cbounds; // coarse ownership
    int64_t nc = 0;
};

// Pairs and singletons numbered by ascending minimum member (R5): an exclusive scan of the
// ranks' head counts; a pair whose minimum member is on another rank learns its id from that
// rank.  Values of Eq. 3.3 with the parenthesisation of O2.4.
DistSweep dist_aggregates(Comm& c, const std::vector<int64_t>& mate, const std::vector<double>& w, int64_t b0,
                          const std::vector<int64_t>& bounds, const GhostPlan& g, const std::vector<double>& wg) {
    const int me = c.rank(), np = c.size();
    const int64_t nloc = (int64_t)mate.size(), b1 = b0 + nloc;
    DistSweep s;
    s.agg.assign(nloc, -1);
    s.pval.assign(nloc, 0.0);
    std::vector<int64_t> id(nloc, -1);
    int64_t cnt = 0;
    for (int64_t r = 0; r < nloc; ++r)
        if (mate[r] < 0 || mate[r] > b0 + r) id[r] = cnt++;
    const std::vector<int64_t> counts = allgatherv(c, std::vector<int64_t>{cnt});
    s.cbounds.assign(np + 1, 0);
    for (int q = 0; q < np; ++q) s.cbounds[q + 1] = s.cbounds[q] + counts[q];
    s.nc = s.cbounds[np];
    const int64_t off = s.cbounds[me];
    std::vector<std::vector<int64_t>> out(np), in;
    for (int64_t r = 0; r < nloc; ++r) {
        if (id[r] >= 0) s.agg[r] = (int32_t)(off + id[r]);
        if (id[r] >= 0 && mate[r] >= b1) {
            const int o = owner_of(bounds, mate[r]);
            out[o].push_back(mate[r]);
            out[o].push_back(off + id[r]);
        }
    }
    a2a_vec(c, out, in);
    for (int q = 0; q < np; ++q)
        for (size_t k = 0; k + 1 < in[q].size(); k += 2) s.agg[in[q][k] - b0] = (int32_t)in[q][k + 1];
    for (int64_t r = 0; r < nloc; ++r)
        if (mate[r] >= 0 && mate[r] < b0 + r && mate[r] >= b0) s.agg[r] = (int32_t)(off + id[mate[r] - b0]);
    const double nan = std::numeric_limits<double>::quiet_NaN();
    auto wv = [&](int64_t gid) { return (gid >= b0 && gid < b1) ? w[gid - b0] : wg[g.find(gid)]; };
    for (int64_t r = 0; r < nloc; ++r) {
        const int64_t v = b0 + r, j = mate[r];
        if (j < 0) {
            s.pval[r] = (w[r] == 0.0) ? 1.0 : w[r] / std::fabs(w[r]);
            continue;
        }
        const int64_t lo = std::min(v, j), hi = std::max(v, j);
        const double nrm = std::sqrt((wv(lo) * wv(lo)) + (wv(hi) * wv(hi)));
        if (nrm == 0.0) {
            s.pval[r] = (v == lo) ? 1.0 : nan;
        } else {
            const double pv = w[r] / nrm;
            s.pval[r] = (pv == 0.0) ? nan : pv;
        }
    }
    return s;
}

Csr one_per_row_g(const std::vector<int32_t>& agg, const std::vector<double>& pval, int64_t nc) {
    Csr P;
    const int64_t n = (int64_t)agg.size();
    P.nrows = n;
    P.ncols = nc;
    P.rp.assign(n + 1, 0);
    for (int64_t i = 0; i < n; ++i) {
        if (!std::isnan(pval[i])) {
            P.ci.push_back(agg[i]);
            P.v.push_back(pval[i]);
        }
        P.rp[i + 1] = (int64_t)P.ci.size();
    }
    return P;
}

// Galerkin X^T A X (mirrored, zeros dropped) with X row-distributed like A; the coarse rows
// owned by this rank, plus (optionally) w_next = X^T w and R = X^T.
void galerkin_dist(Comm& c, const Csr& A, const Csr& X, int64_t b0, const GhostPlan& gA,
                   const std::vector<int64_t>& cbounds, int64_t nfine, const std::vector<double>* w, Csr& C,
                   std::vector<double>* wnext, Csr* Rt) {
    const Csr Xg = fetch_rows(c, gA, X, b0);
    const Csr T = spgemm_rows(A, b0, X, gA, Xg, cbounds.back());
    std::vector<std::vector<char>> keep;
    const std::vector<Contrib> cs =
        gather_contribs(c, X, T, w ? *w : std::vector<double>(), b0, cbounds, keep);
    const int me = c.rank();
    owner_products(cs, cbounds[me], cbounds[me + 1], cbounds.back(), C, wnext, Rt, nfine);
    mirror_drop_dist(c, C, cbounds[me], cbounds);
}

}  // namespace

// ====================================================================== build
int build_distributed(Comm& c, const std::vector<int64_t>& bounds0, Csr&& A_loc, std::vector<double>&& w_loc,
                      const Config& cfg, DistHierarchy& out, std::string& err) {
    const int me = c.rank();
    out.lv.clear();
    out.lv.emplace_back();
    {
        DistLevel& L0 = out.lv[0];
        L0.n = bounds0.back();
        L0.bounds = bounds0;
        L0.A = std::move(A_loc);
        L0.w = std::move(w_loc);
    }
    for (int l = 0;; ++l) {
        DistLevel& L = out.lv[l];
        const Csr& A = L.A;
        const int64_t b0 = L.bounds[me];
        L.m = l1_inv_rows(A);  // O7
        L.nnzA = allreduce_sum(c, A.nnz());
        const int64_t n = L.n;
        if (n <= cfg.max_coarse_size || l == cfg.max_levels - 1) break;  // O1
        const GhostPlan gA = make_plan(c, L.bounds, col_ids(A));
        // O2 sweeps; O3 composite map (global ids of the sweep's vertices) and values
        const int64_t nloc = A.nrows;
        std::vector<int32_t> comp_agg(nloc);
        std::vector<double> comp_val(nloc, 1.0);
        for (int64_t r = 0; r < nloc; ++r) comp_agg[r] = (int32_t)(b0 + r);
        Csr As_store;
        const Csr* As = &A;
        std::vector<double> ws = L.w;
        std::vector<int64_t> sb = L.bounds;
        GhostPlan gS = gA;
        int64_t ns = n;
        int done = 0;
        for (int sw = 0; sw < cfg.sweeps_per_level; ++sw) {
            const int64_t sb0 = sb[me];
            std::vector<int64_t> mate;
            if (!dist_matching(c, *As, ws, sb0, gS, mate)) {
                err = "distributed matching stalled";
                return SETUP_ERR_ARG;
            }
            const std::vector<double> wg = fetch(c, gS, ws, sb0);
            DistSweep ds = dist_aggregates(c, mate, ws, sb0, sb, gS, wg);
            if (ds.nc == ns) break;  // no size reduction
            const Csr Ps = one_per_row_g(ds.agg, ds.pval, ds.nc);
            Csr An;
            std::vector<double> wn;
            galerkin_dist(c, *As, Ps, sb0, gS, ds.cbounds, ns, &ws, An, &wn, nullptr);
            // composite map: the sweep's map and value of every level-l row's current vertex
            {
                std::vector<int64_t> ids(comp_agg.begin(), comp_agg.end());
                const GhostPlan gc = make_plan(c, sb, ids);
                std::vector<int32_t> aggc = fetch(c, gc, ds.agg, sb0);
                std::vector<double> pvc = fetch(c, gc, ds.pval, sb0);
                const int64_t sb1 = sb[me + 1];
                for (int64_t r = 0; r < nloc; ++r) {
                    const int64_t a = comp_agg[r];
                    int32_t na;
                    double pv;
                    if (a >= sb0 && a < sb1) {
                        na = ds.agg[a - sb0];
                        pv = ds.pval[a - sb0];
                    } else {
                        const int64_t k = gc.find(a);
                        na = aggc[k];
                        pv = pvc[k];
                    }
                    comp_val[r] = comp_val[r] * pv;
                    comp_agg[r] = na;
                }
            }
            As_store = std::move(An);
            As = &As_store;
            ws.swap(wn);
            sb = ds.cbounds;
            ns = ds.nc;
            gS = make_plan(c, sb, col_ids(*As));
            ++done;
        }
        As_store = Csr();
        if (done == 0 || (double)n / (double)ns < cfg.min_coarsening_ratio) break;  // O1
        const int64_t nc = ns;
        const std::vector<int64_t> cb = sb;  // coarse ownership = the last sweep's
        Csr P = one_per_row_g(comp_agg, comp_val, nc);
        Csr Pb;
        if (cfg.smooth_prolongator) {
            // O4: omega = scale / max_i (sum_j |a_ij|)/a_ii  (max over ranks: exact)
            std::vector<double> d(nloc);
            double mx = 0.0;
            for (int64_t r = 0; r < nloc; ++r) {
                d[r] = diag_of(A, r, b0 + r);
                double s = 0.0;
                for (int64_t k = A.rp[r]; k < A.rp[r + 1]; ++k) s += std::fabs(A.v[k]);
                mx = std::max(mx, s / d[r]);
            }
            mx = allreduce_max(c, mx);
            L.omega = cfg.prol_omega_scale / mx;
            // O5: P-bar[i,G] = P[i,G] - (omega/a_ii) * (A P)[i,G]
            const Csr Pg = fetch_rows(c, gA, P, b0);
            const Csr T = spgemm_rows(A, b0, P, gA, Pg, nc);
            Pb.nrows = nloc;
            Pb.ncols = nc;
            Pb.rp.assign(nloc + 1, 0);
            for (int64_t r = 0; r < nloc; ++r) {
                const double f = L.omega / d[r];
                for (int64_t k = T.rp[r]; k < T.rp[r + 1]; ++k) {
                    const bool own = (P.rp[r + 1] > P.rp[r]) && T.ci[k] == P.ci[P.rp[r]];
                    const double p = own ? P.v[P.rp[r]] : 0.0;
                    const double nv = p - f * T.v[k];
                    if (nv != 0.0) {
                        Pb.ci.push_back(T.ci[k]);
                        Pb.v.push_back(nv);
                    }
                }
                Pb.rp[r + 1] = (int64_t)Pb.ci.size();
            }
        } else {
            L.omega = 0.0;
            Pb = P;
        }
        // O6: A_{l+1} = P-bar^T A P-bar (mirrored), R = P-bar^T; w_{l+1} = P^T w (R6)
        DistLevel next;
        Csr R;
        galerkin_dist(c, A, Pb, b0, gA, cb, n, nullptr, next.A, nullptr, &R);
        {
            // w_{l+1} with the unsmoothed composite P (members in ascending order, C3)
            std::vector<std::vector<char>> keep;
            const Csr empty_rows = [&] {
                Csr E;
                E.nrows = nloc;
                E.ncols = nc;
                E.rp.assign(nloc + 1, 0);
                return E;
            }();
            const std::vector<Contrib> cs = gather_contribs(c, P, empty_rows, L.w, b0, cb, keep);
            Csr dummy;
            owner_products(cs, cb[me], cb[me + 1], nc, dummy, &next.w, nullptr, n);
        }
        next.n = nc;
        next.bounds = cb;
        L.nnzP = allreduce_sum(c, Pb.nnz());
        L.P = std::move(Pb);
        L.R = std::move(R);
        L.agg = std::move(comp_agg);
        L.sweeps = done;
        out.lv.push_back(std::move(next));
    }
    // O8: the coarsest matrix on every rank, its dense inverse
    DistLevel& C = out.lv.back();
    {
        std::vector<int64_t> rl(C.A.nrows);
        for (int64_t r = 0; r < C.A.nrows; ++r) rl[r] = C.A.rp[r + 1] - C.A.rp[r];
        const std::vector<int64_t> lens = allgatherv(c, rl);
        const std::vector<int32_t> ci = allgatherv(c, C.A.ci);
        const std::vector<double> v = allgatherv(c, C.A.v);
        Csr F;
        F.nrows = F.ncols = C.n;
        F.rp.assign(C.n + 1, 0);
        for (int64_t r = 0; r < C.n; ++r) F.rp[r + 1] = F.rp[r] + lens[r];
        F.ci = ci;
        F.v = v;
        out.coarse_A = std::move(F);
    }
    if (!dense_inverse_host(out.coarse_A, out.coarse_inv)) {
        err = "coarsest-level Cholesky failed (matrix not s.p.d.)";
        return SETUP_ERR_NOT_SPD;
    }
    return SETUP_OK;
}


// ====================================================================== plan
namespace {
// all rows of a row-distributed matrix on every rank
Csr allgather_rows(Comm& c, const Csr& M, int64_t nrows_global, int64_t ncols) {
    std::vector<int64_t> rl(M.nrows);
    for (int64_t r = 0; r < M.nrows; ++r) rl[r] = M.rp[r + 1] - M.rp[r];
    const std::vector<int64_t> lens = allgatherv(c, rl);
    Csr F;
    F.nrows = nrows_global;
    F.ncols = ncols;
    F.rp.assign(nrows_global + 1, 0);
    for (int64_t r = 0; r < nrows_global; ++r) F.rp[r + 1] = F.rp[r] + lens[r];
    F.ci = allgatherv(c, M.ci);
    F.v = allgatherv(c, M.v);
    return F;
}
// rows [r0, r1) of M (whose first row is global row m0), columns shifted by -shift
Csr slice_shift(const Csr& M, int64_t m0, int64_t r0, int64_t r1, int64_t shift, int64_t ncols) {
    Csr S;
    S.nrows = r1 - r0;
    S.ncols = ncols;
    S.rp.assign(S.nrows + 1, 0);
    const int64_t k0 = M.rp[r0 - m0];
    for (int64_t i = 0; i <= S.nrows; ++i) S.rp[i] = M.rp[r0 - m0 + i] - k0;
    const int64_t nnz = S.rp[S.nrows];
    S.ci.resize(nnz);
    S.v.assign(M.v.begin() + k0, M.v.begin() + k0 + nnz);
    for (int64_t k = 0; k < nnz; ++k) S.ci[k] = (int32_t)((int64_t)M.ci[k0 + k] - shift);
    return S;
}
void scan(const Csr& M, int64_t o0, int64_t o1, int64_t& lo, int64_t& hi, std::vector<int64_t>& outside) {
    for (int64_t k = 0; k < M.nnz(); ++k) {
        const int64_t c = M.ci[k];
        lo = std::min(lo, c);
        hi = std::max(hi, c + 1);
        if (c < o0 || c >= o1) outside.push_back(c);
    }
}
}  // namespace

bool partition_distributed(Comm& c, const DistHierarchy& H, int64_t rep_bytes, RankPlan& P, std::string& err) {
    const int me = c.rank(), np = c.size();
    const int nl = (int)H.lv.size();
    // first replicated level (as partition(): by the global operator bytes, or an empty rank)
    int lrep = nl - 1;
    for (int l = (np > 1 ? 1 : 0); l < nl; ++l) {
        const double bytes = 12.0 * (double)H.lv[l].nnzA + 12.0 * (double)H.lv[l].nnzP;
        bool empty = false;
        for (int g = 0; g < np; ++g) empty |= (H.lv[l].bounds[g + 1] == H.lv[l].bounds[g]);
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
        if (H.lv[0].bounds[g + 1] == H.lv[0].bounds[g]) {
            err = "partition: every rank must own at least one level-0 row";
            return false;
        }
    P = RankPlan();
    P.rank = me;
    P.nranks = np;
    P.lv.resize(nl);
    // whole operators of the replicated levels (and the coarse rows R of the level above them)
    std::vector<Csr> Af(nl), Pf(nl), Rf(nl);
    std::vector<std::vector<double>> mf(nl);
    for (int l = 0; l < nl; ++l) {
        const DistLevel& D = H.lv[l];
        RankLevel& L = P.lv[l];
        L.n_global = D.n;
        L.replicated = (l >= lrep);
        L.own_begin = D.bounds[me];
        L.own_end = D.bounds[me + 1];
        L.comp_begin = L.replicated ? 0 : L.own_begin;
        L.comp_end = L.replicated ? L.n_global : L.own_end;
        if (l + 1 < nl) {
            L.rst_begin = L.replicated ? 0 : H.lv[l + 1].bounds[me];
            L.rst_end = L.replicated ? H.lv[l + 1].n : H.lv[l + 1].bounds[me + 1];
        }
        if (L.replicated) {
            Af[l] = (l == nl - 1) ? H.coarse_A : allgather_rows(c, D.A, D.n, D.n);
            mf[l] = allgatherv(c, D.m);
            if (l + 1 < nl) {
                Pf[l] = allgather_rows(c, D.P, D.n, H.lv[l + 1].n);
                Rf[l] = allgather_rows(c, D.R, H.lv[l + 1].n, D.n);
            }
        }
    }
    // the computed operators of each level: (matrix, first global row of that storage)
    auto Aop = [&](int l) -> std::pair<const Csr*, int64_t> {
        return P.lv[l].replicated ? std::make_pair(&Af[l], (int64_t)0) : std::make_pair(&H.lv[l].A, P.lv[l].own_begin);
    };
    auto Pop = [&](int l) -> std::pair<const Csr*, int64_t> {
        return P.lv[l].replicated ? std::make_pair(&Pf[l], (int64_t)0) : std::make_pair(&H.lv[l].P, P.lv[l].own_begin);
    };
    auto Rop = [&](int l) -> std::pair<const Csr*, int64_t> {
        return P.lv[l].replicated ? std::make_pair(&Rf[l], (int64_t)0)
                                  : std::make_pair(&H.lv[l].R, H.lv[l + 1].bounds[me]);
    };
    std::vector<std::vector<int64_t>> outside(nl);
    std::vector<int64_t> lo(nl), hi(nl);
    for (int l = 0; l < nl; ++l) {
        RankLevel& L = P.lv[l];
        lo[l] = L.comp_begin;
        hi[l] = L.comp_end;
        if (l > 0) {
            lo[l] = std::min(lo[l], P.lv[l - 1].rst_begin);
            hi[l] = std::max(hi[l], P.lv[l - 1].rst_end);
        }
    }
    for (int l = 0; l < nl; ++l) {
        RankLevel& L = P.lv[l];
        scan(*Aop(l).first, L.own_begin, L.own_end, lo[l], hi[l], outside[l]);
        if (l + 1 < nl) {
            scan(*Rop(l).first, L.own_begin, L.own_end, lo[l], hi[l], outside[l]);
            const RankLevel& C = P.lv[l + 1];
            scan(*Pop(l).first, C.own_begin, C.own_end, lo[l + 1], hi[l + 1], outside[l + 1]);
        }
    }
    for (int l = 0; l < nl; ++l) {
        RankLevel& L = P.lv[l];
        const DistLevel& D = H.lv[l];
        if (L.replicated) {
            L.win_begin = 0;
            L.win_end = L.n_global;
        } else {
            L.win_begin = std::min(lo[l], L.own_begin);
            L.win_end = std::max(hi[l], L.own_end);
        }
        std::vector<int64_t> ids;
        if (L.replicated) {
            if (l > 0 && !P.lv[l - 1].replicated && np > 1) {
                for (int64_t i = 0; i < L.own_begin; ++i) ids.push_back(i);
                for (int64_t i = L.own_end; i < L.n_global; ++i) ids.push_back(i);
            }
        } else {
            ids.swap(outside[l]);
            std::sort(ids.begin(), ids.end());
            ids.erase(std::unique(ids.begin(), ids.end()), ids.end());
        }
        L.recv_off.assign(np + 1, 0);
        for (int64_t id : ids) L.recv_off[owner_of(D.bounds, id) + 1]++;
        for (int q = 0; q < np; ++q) L.recv_off[q + 1] += L.recv_off[q];
        L.recv_ids = ids;
        const auto a = Aop(l);
        L.A = slice_shift(*a.first, a.second, L.comp_begin, L.comp_end, L.win_begin, L.win_end - L.win_begin);
        // l1 diagonal over the whole window: owned values here, the rest from their owners
        if (L.replicated) {
            L.m = mf[l];
        } else {
            std::vector<int64_t> wid;
            for (int64_t i = L.win_begin; i < L.win_end; ++i) wid.push_back(i);
            const GhostPlan gm = make_plan(c, D.bounds, wid);
            const std::vector<double> mg = fetch(c, gm, D.m, L.own_begin);
            L.m.resize(L.win_end - L.win_begin);
            for (int64_t i = L.win_begin; i < L.win_end; ++i)
                L.m[i - L.win_begin] = (i >= L.own_begin && i < L.own_end) ? D.m[i - L.own_begin] : mg[gm.find(i)];
        }
    }
    for (int l = 0; l + 1 < nl; ++l) {
        RankLevel& L = P.lv[l];
        const RankLevel& C = P.lv[l + 1];
        const auto pp = Pop(l);
        L.P = slice_shift(*pp.first, pp.second, L.comp_begin, L.comp_end, C.win_begin, C.win_end - C.win_begin);
        const auto rr = Rop(l);
        L.R = slice_shift(*rr.first, rr.second, L.rst_begin, L.rst_end, L.win_begin, L.win_end - L.win_begin);
    }
    // send lists: what each peer receives from this rank, in peer order
    for (int l = 0; l < nl; ++l) {
        RankLevel& L = P.lv[l];
        std::vector<std::vector<int64_t>> out(np), in;
        for (int q = 0; q < np; ++q)
            out[q].assign(L.recv_ids.begin() + L.recv_off[q], L.recv_ids.begin() + L.recv_off[q + 1]);
        a2a_vec(c, out, in);
        L.send_off.assign(np + 1, 0);
        L.send_ids.clear();
        for (int q = 0; q < np; ++q) {
            if (q != me) L.send_ids.insert(L.send_ids.end(), in[q].begin(), in[q].end());
            L.send_off[q + 1] = (int64_t)L.send_ids.size();
        }
    }
    return true;
}


// ====================================================================== validation
int validate_distributed(Comm& c, const std::vector<int64_t>& bounds, const Csr& A, const std::vector<double>& w,
                         std::string& err) {
    const int me = c.rank(), np = c.size();
    const int64_t b0 = bounds[me], b1 = bounds[me + 1], n = bounds[np];
    int bad = 0;
    int64_t badrow = -1;
    std::vector<std::vector<int64_t>> req(np), got;
    auto lookup = [&](int64_t row, int64_t col, double& v) {
        const int64_t r = row - b0;
        const int32_t* b = A.ci.data() + A.rp[r];
        const int32_t* e = A.ci.data() + A.rp[r + 1];
        const int32_t* p = std::lower_bound(b, e, (int32_t)col);
        if (p != e && *p == col) {
            v = A.v[p - A.ci.data()];
            return true;
        }
        return false;
    };
    for (int64_t r = 0; r < A.nrows && bad < 3; ++r) {
        const int64_t i = b0 + r;
        bool has_d = false;
        for (int64_t k = A.rp[r]; k < A.rp[r + 1]; ++k) {
            const int64_t col = A.ci[k];
            if (col < 0 || col >= n || (k > A.rp[r] && col <= A.ci[k - 1])) {
                bad = 3;
                badrow = i;
                break;
            }
            if (col == i) {
                has_d = true;
                if (!(A.v[k] > 0.0)) bad = std::max(bad, 1), badrow = i;
            }
            if (col >= b0 && col < b1) {
                double t;
                if (!lookup(col, i, t) || t != A.v[k]) bad = std::max(bad, 2), badrow = i;
            } else {
                const int o = owner_of(bounds, col);
                req[o].push_back(col);
                req[o].push_back(i);
            }
        }
        if (!has_d && bad < 3) bad = std::max(bad, 1), badrow = i;
    }
    // the transposed entries of the off-rank couplings, answered by their owners
    std::vector<std::vector<double>> ans(np), vals;
    std::vector<std::vector<int64_t>> hit(np), hits;
    a2a_vec(c, req, got);
    for (int q = 0; q < np; ++q)
        for (size_t k = 0; k + 1 < got[q].size(); k += 2) {
            double v = 0.0;
            const bool f = got[q][k] >= b0 && got[q][k] < b1 && lookup(got[q][k], got[q][k + 1], v);
            ans[q].push_back(v);
            hit[q].push_back(f ? 1 : 0);
        }
    a2a_vec(c, ans, vals);
    a2a_vec(c, hit, hits);
    if (bad < 3) {
        std::vector<size_t> pos(np, 0);
        for (int64_t r = 0; r < A.nrows; ++r)
            for (int64_t k = A.rp[r]; k < A.rp[r + 1]; ++k) {
                const int64_t col = A.ci[k];
                if (col >= b0 && col < b1) continue;
                const int o = owner_of(bounds, col);
                const size_t p = pos[o]++;
                if (!hits[o][p] || vals[o][p] != A.v[k]) bad = std::max(bad, 2), badrow = b0 + r;
            }
    }
    int64_t anyw = 0;
    for (double x : w) anyw |= (x != 0.0);
    const std::vector<int64_t> bads = allgatherv(c, std::vector<int64_t>{bad, badrow});
    int worst = 0;
    int64_t wrow = -1;
    for (int q = 0; q < np; ++q)
        if (bads[2 * q] > worst) worst = (int)bads[2 * q], wrow = bads[2 * q + 1];
    if (worst == 3) {
        err = "column indices must be in range and strictly ascending (row " + std::to_string(wrow) + ")";
        return SETUP_ERR_ARG;
    }
    if (worst == 2) {
        err = "matrix is not exactly symmetric (row " + std::to_string(wrow) + ")";
        return SETUP_ERR_ARG;
    }
    if (worst == 1) {
        err = "non-positive or missing diagonal (row " + std::to_string(wrow) + ")";
        return SETUP_ERR_NOT_SPD;
    }
    if (allreduce_sum(c, anyw) == 0) {
        err = "weight vector w is identically zero";
        return SETUP_ERR_NOT_SPD;
    }
    return SETUP_OK;
}

int64_t comm_allreduce_sum(Comm& c, int64_t v) { return allreduce_sum(c, v); }

// ====================================================================== loopback transport
namespace {
struct Hub {
    int np;
    std::vector<std::vector<std::vector<char>>> box;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    int64_t gen = 0;
    void barrier() {
        std::unique_lock<std::mutex> lk(mu);
        const int64_t g = gen;
        if (++arrived == np) {
            arrived = 0;
            ++gen;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return gen != g; });
        }
    }
};
struct LoopbackComm : Comm {
    Hub* hub;
    int me;
    int rank() const override { return me; }
    int size() const override { return hub->np; }
    bool alltoallv(const std::vector<std::vector<char>>& out, std::vector<std::vector<char>>& in) override {
        const int np = hub->np;
        for (int q = 0; q < np; ++q) hub->box[me][q] = out[q];
        hub->barrier();
        in.assign(np, {});
        for (int q = 0; q < np; ++q) in[q] = hub->box[q][me];
        hub->barrier();
        return true;
    }
};
}  // namespace

void run_loopback(int nranks, const std::function<void(Comm&)>& fn) {
    Hub hub;
    hub.np = nranks;
    hub.box.assign(nranks, std::vector<std::vector<char>>(nranks));
    const int total = omp_get_max_threads();
    std::vector<std::thread> th;
    for (int r = 0; r < nranks; ++r)
        th.emplace_back([&, r] {
            omp_set_num_threads(std::max(1, total / nranks));
            LoopbackComm cm;
            cm.hub = &hub;
            cm.me = r;
            fn(cm);
        });
    for (auto& t : th) t.join();
}

}  // namespace amgsetup
