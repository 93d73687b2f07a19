// bridge.cpp — the matchamg C++ API (include/matchamg/*.hpp, the drop-in for
// /root/reference/proj/include/matchamg) implemented over the mamg C-ABI
// (include/mamg_capi.h). All numerical work runs on the B200; this file only
// validates arguments with the reference's messages, stages host spans to
// device buffers and back, and rethrows the reference's exception types.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <unordered_map>

#include <sys/mman.h>

#include "mamg_capi.h"
#include "matchamg/coarsening.hpp"
#include "matchamg/kernels.hpp"
#include "matchamg/krylov.hpp"
#include "matchamg/matching.hpp"
#include "matchamg/multigrid.hpp"
#include "matchamg/vector_ops.hpp"

namespace matchamg {
namespace detail {

// One process-wide device context (device from $MATCHAMG_DEVICE, default 0).
// The reference is one-solver-per-thread; calls are serialised here.
struct Backend {
    mamg_ctx* ctx = nullptr;
    std::recursive_mutex mu;
    Backend() {
        const char* env = std::getenv("MATCHAMG_DEVICE");
        const int dev = env ? std::atoi(env) : 0;
        if (mamg_ctx_create(dev, &ctx) != MAMG_OK)
            throw std::runtime_error("matchamg: no usable CUDA device (B200 backend)");
    }
    ~Backend() { mamg_ctx_destroy(ctx); }
};

Backend& backend() {
    static Backend b;
    return b;
}

[[noreturn]] void rethrow(int st) {
    mamg_ctx* c = backend().ctx;
    const std::string msg = mamg_last_error(c);
    const index_t idx = mamg_last_error_index(c);
    if (st == MAMG_INVALID_ARGUMENT) throw std::invalid_argument(msg);
    if (st == MAMG_BREAKDOWN) {
        // message is "pcg breakdown at iteration N: <what>"; BreakdownError
        // re-adds the prefix
        const auto colon = msg.find(": ");
        throw BreakdownError(idx, colon == std::string::npos ? msg : msg.substr(colon + 2));
    }
    throw std::runtime_error(msg);
}

inline void ok(int st) {
    if (st != MAMG_OK) rethrow(st);
}

// RAII device vector
struct DVec {
    double* p = nullptr;
    std::size_t n = 0;
    explicit DVec(std::size_t n_) : n(n_) {
        void* q = nullptr;
        ok(mamg_dmalloc(backend().ctx, 8 * (n ? n : 1), &q));
        p = static_cast<double*>(q);
    }
    DVec(std::span<const double> h) : DVec(h.size()) { put(h); }
    ~DVec() { mamg_dfree(backend().ctx, p); }
    DVec(const DVec&) = delete;
    DVec& operator=(const DVec&) = delete;
    void put(std::span<const double> h) {
        if (!h.empty()) ok(mamg_h2d(backend().ctx, p, h.data(), 8 * h.size()));
    }
    void get(std::span<double> h) const {
        if (!h.empty()) ok(mamg_d2h(backend().ctx, h.data(), p, 8 * h.size()));
    }
    std::vector<double> host() const {
        std::vector<double> v(n);
        get(v);
        return v;
    }
};

// RAII device matrix
// Host copies of hierarchy levels (the API returns them in std::vectors):
// large vectors are backed by transparent huge pages (THP "madvise" mode on
// the GPU boxes) so their first touch faults 2 MB pages instead of 4 KB ones
// (measured: the level-0 copy of cfg 2's A took 0.46 s, page faults mostly),
// and large copies run on several threads.
template <class T>
void big_resize(std::vector<T>& v, size_t n) {
    v.clear();
    v.reserve(n);
    const size_t bytes = n * sizeof(T);
    constexpr uintptr_t kHuge = uintptr_t{2} << 20;
    if (bytes >= 4 * kHuge) {
        const uintptr_t b = reinterpret_cast<uintptr_t>(v.data());
        const uintptr_t a = (b + kHuge - 1) & ~(kHuge - 1), e = (b + bytes) & ~(kHuge - 1);
        if (e > a) madvise(reinterpret_cast<void*>(a), e - a, MADV_HUGEPAGE);
    }
    v.resize(n);
}
template <class T>
void par_copy(T* dst, const T* src, size_t n) {
    const size_t per = size_t{1} << 20; // elements per task
    const int T_ = static_cast<int>(std::min<size_t>(16, (n + per - 1) / per));
    if (T_ <= 1) {
        std::copy(src, src + n, dst);
        return;
    }
    std::vector<std::thread> th;
    for (int t = 0; t < T_; ++t)
        th.emplace_back([=] {
            const size_t a = n * static_cast<size_t>(t) / static_cast<size_t>(T_);
            const size_t b = n * static_cast<size_t>(t + 1) / static_cast<size_t>(T_);
            std::copy(src + a, src + b, dst + a);
        });
    for (auto& x : th) x.join();
}
template <class T>
void big_assign(std::vector<T>& dst, const std::vector<T>& src) {
    big_resize(dst, src.size());
    par_copy(dst.data(), src.data(), src.size());
}
CsrMatrix big_copy(const CsrMatrix& A) {
    CsrMatrix B;
    B.nrows = A.nrows;
    B.ncols = A.ncols;
    big_assign(B.row_ptr, A.row_ptr);
    big_assign(B.col_idx, A.col_idx);
    big_assign(B.values, A.values);
    return B;
}

struct DMat {
    mamg_mat* m = nullptr;
    bool owned = true;
    DMat() = default;
    explicit DMat(const CsrMatrix& A) {
        ok(mamg_csr_upload(backend().ctx, A.nrows, A.ncols, A.row_ptr.data(), A.col_idx.data(),
                           A.values.data(), &m));
    }
    static DMat view(const mamg_mat* v) {
        DMat d;
        d.m = const_cast<mamg_mat*>(v);
        d.owned = false;
        return d;
    }
    DMat(DMat&& o) noexcept : m(o.m), owned(o.owned) { o.m = nullptr; }
    ~DMat() {
        if (owned && m) mamg_mat_destroy(m);
    }
    CsrMatrix host() const {
        CsrMatrix A;
        int64_t nr, nc, nz;
        ok(mamg_csr_shape(m, &nr, &nc, &nz));
        A.nrows = nr;
        A.ncols = nc;
        big_resize(A.row_ptr, static_cast<size_t>(nr + 1));
        big_resize(A.col_idx, static_cast<size_t>(nz));
        big_resize(A.values, static_cast<size_t>(nz));
        ok(mamg_csr_download(backend().ctx, m, A.row_ptr.data(), A.col_idx.data(),
                             A.values.data()));
        return A;
    }
};

// ---- several GPUs behind the same API ------------------------------------
// MATCHAMG_DEVICES="0,1,2,3" (read at every build_hierarchy): the hierarchy is
// built row-block partitioned across these devices, one host thread and
// context per device (in-process thread group, mamg_dist_create_group), with
// the Suitor run across the parts (global matching) — so the hierarchy, and
// every pcg_solve preconditioned by it, is bit-identical to the single-device
// (and the reference's) one. A device may be listed twice (tests on one GPU).
struct Multi {
    std::vector<int> devices;
    std::vector<mamg_ctx*> ctxs; // ctxs[r] on devices[r]
    ~Multi() {
        for (auto* c : ctxs) mamg_ctx_destroy(c);
    }
    // the device list of the next build (empty or one device: single-GPU path)
    std::vector<int> requested() const {
        std::vector<int> d;
        const char* e = std::getenv("MATCHAMG_DEVICES");
        if (!e) return d;
        std::string s(e);
        size_t i = 0;
        while (i < s.size()) {
            const size_t j = s.find(',', i);
            const std::string t = s.substr(i, j == std::string::npos ? std::string::npos : j - i);
            if (!t.empty()) d.push_back(std::atoi(t.c_str()));
            if (j == std::string::npos) break;
            i = j + 1;
        }
        return d;
    }
    void ensure(const std::vector<int>& d) {
        for (size_t r = 0; r < d.size(); ++r) {
            if (r < ctxs.size() && devices[r] == d[r]) continue;
            if (r < ctxs.size()) mamg_ctx_destroy(ctxs[r]);
            mamg_ctx* c = nullptr;
            if (mamg_ctx_create(d[r], &c) != MAMG_OK)
                throw std::runtime_error("matchamg: cannot open CUDA device " + std::to_string(d[r]));
            if (r < ctxs.size()) {
                ctxs[r] = c;
                devices[r] = d[r];
            } else {
                ctxs.push_back(c);
                devices.push_back(d[r]);
            }
        }
    }
};

Multi& multi() {
    static Multi m;
    return m;
}

// the reference's exception for a failed call on context c
[[noreturn]] void rethrow_on(mamg_ctx* c, int st) {
    const std::string msg = mamg_last_error(c);
    const index_t idx = mamg_last_error_index(c);
    if (st == MAMG_INVALID_ARGUMENT) throw std::invalid_argument(msg);
    if (st == MAMG_BREAKDOWN) {
        const auto colon = msg.find(": ");
        throw BreakdownError(idx, colon == std::string::npos ? msg : msg.substr(colon + 2));
    }
    throw std::runtime_error(msg);
}

inline void ok_on(mamg_ctx* c, int st) {
    if (st != MAMG_OK) rethrow_on(c, st);
}

// f(rank) on one host thread per rank; the lowest failing rank's error is rethrown
template <class F>
void run_ranks(int world, const std::vector<mamg_ctx*>& ctxs, F&& f) {
    std::vector<int> st(world, MAMG_OK);
    std::vector<std::thread> th;
    for (int r = 0; r < world; ++r) th.emplace_back([&, r] { st[r] = f(r); });
    for (auto& t : th) t.join();
    for (int r = 0; r < world; ++r)
        if (st[r] != MAMG_OK) rethrow_on(ctxs[r], st[r]);
}

struct DeviceHierarchy {
    mamg_hier* h = nullptr;
    // partitioned twin (MATCHAMG_DEVICES): one part per rank
    mamg_group* group = nullptr;
    std::vector<mamg_dist*> parts;
    std::vector<mamg_ctx*> ctxs;
    int64_t n0 = 0;
    // single-device copy for the host-callable cycle operations (lazy)
    std::shared_ptr<DeviceHierarchy> single;
    bool partitioned() const { return !parts.empty(); }
    ~DeviceHierarchy() {
        if (h) mamg_hier_destroy(h);
        for (auto* d : parts) mamg_dist_destroy(d);
        if (group) mamg_group_destroy(group);
    }
};

// device twin of a host hierarchy (uploaded when it was assembled on the host,
// or the single-device copy of a partitioned one for host-callable cycles)
std::shared_ptr<DeviceHierarchy> twin(const Hierarchy& h) {
    if (h.device && !h.device->partitioned()) return h.device;
    if (h.device && h.device->single) return h.device->single;
    const int nl = h.nl();
    std::vector<DMat> A, P, R;
    std::vector<std::unique_ptr<DVec>> l1, w;
    std::vector<mamg_mat*> pa, pp, pr;
    std::vector<const double*> pl, pw;
    for (int k = 0; k < nl; ++k) {
        const Level& L = h.levels[k];
        A.emplace_back(L.A);
        pa.push_back(A.back().m);
        if (k + 1 < nl) {
            P.emplace_back(L.P);
            R.emplace_back(L.R);
            pp.push_back(P.back().m);
            pr.push_back(R.back().m);
        } else {
            pp.push_back(nullptr);
            pr.push_back(nullptr);
        }
        l1.push_back(std::make_unique<DVec>(L.l1_diag));
        pl.push_back(l1.back()->p);
        if (L.w.size() == static_cast<std::size_t>(L.A.nrows)) {
            w.push_back(std::make_unique<DVec>(L.w));
            pw.push_back(w.back()->p);
        } else {
            pw.push_back(nullptr);
        }
    }
    auto d = std::make_shared<DeviceHierarchy>();
    ok(mamg_hier_from_levels(backend().ctx, nl, pa.data(), pp.data(), pr.data(), pl.data(),
                             pw.data(), &d->h));
    if (h.device) h.device->single = d;
    return d;
}

mamg_cycle_cfg ccfg(const CycleConfig& c) {
    return mamg_cycle_cfg{c.cycle == CycleType::W ? 1 : (c.cycle == CycleType::K ? 2 : 0),
                          c.pre_sweeps, c.post_sweeps, c.coarsest_sweeps};
}

} // namespace detail

using detail::backend;
using detail::DMat;
using detail::DVec;
using detail::ok;

// ============================================================== kernels.hpp ==
void spmv_into(const CsrMatrix& A, std::span<const double> x, std::span<double> y,
               LaneGroupPolicy policy) {
    if (static_cast<index_t>(x.size()) != A.ncols)
        throw std::invalid_argument("spmv: x has " + std::to_string(x.size()) + " entries, A has " +
                                    std::to_string(A.ncols) + " columns");
    if (static_cast<index_t>(y.size()) != A.nrows)
        throw std::invalid_argument("spmv: output size mismatch");
    const int g = policy.group_size;
    if (g != 1 && g != 2 && g != 4 && g != 8 && g != 16 && g != 32)
        throw std::invalid_argument("spmv: invalid lane group size " + std::to_string(g));
    std::lock_guard<std::recursive_mutex> lk(backend().mu);
    DMat dA(A);
    DVec dx(x), dy(y.size());
    ok(mamg_spmv(backend().ctx, dA.m, g, dx.p, dy.p));
    dy.get(y);
}

std::vector<double> spmv(const CsrMatrix& A, std::span<const double> x, LaneGroupPolicy policy) {
    std::vector<double> y(A.nrows);
    spmv_into(A, x, y, policy);
    return y;
}

std::vector<double> spmv(const CsrMatrix& A, std::span<const double> x) {
    return spmv(A, x, LaneGroupPolicy::for_matrix(A));
}

void spmv_into(const CsrMatrix& A, std::span<const double> x, std::span<double> y) {
    spmv_into(A, x, y, LaneGroupPolicy::for_matrix(A));
}

// the row-serial baseline is the G = 1 lane tree (a single ordered sum)
std::vector<double> spmv_row_serial(const CsrMatrix& A, std::span<const double> x) {
    if (static_cast<index_t>(x.size()) != A.ncols)
        throw std::invalid_argument("spmv_row_serial: dimension mismatch");
    return spmv(A, x, LaneGroupPolicy{1});
}

CsrMatrix transpose(const CsrMatrix& A) {
    std::lock_guard<std::recursive_mutex> lk(backend().mu);
    DMat dA(A);
    mamg_mat* out = nullptr;
    ok(mamg_transpose(backend().ctx, dA.m, &out));
    DMat r = DMat::view(out);
    r.owned = true;
    return r.host();
}

CsrMatrix spgemm(const CsrMatrix& A, const CsrMatrix& B) {
    if (A.ncols != B.nrows)
        throw std::invalid_argument("spgemm: inner dimensions " + std::to_string(A.ncols) +
                                    " and " + std::to_string(B.nrows) + " differ");
    std::lock_guard<std::recursive_mutex> lk(backend().mu);
    DMat dA(A), dB(B);
    mamg_mat* out = nullptr;
    ok(mamg_spgemm(backend().ctx, dA.m, dB.m, &out));
    DMat r = DMat::view(out);
    r.owned = true;
    return r.host();
}

CsrMatrix galerkin_triple(const CsrMatrix& A, const CsrMatrix& P) {
    if (A.nrows != A.ncols) throw std::invalid_argument("galerkin_triple: A is not square");
    if (A.nrows != P.nrows)
        throw std::invalid_argument("galerkin_triple: A and P row counts differ");
    std::lock_guard<std::recursive_mutex> lk(backend().mu);
    DMat dA(A), dP(P);
    mamg_mat* out = nullptr;
    ok(mamg_galerkin_triple(backend().ctx, dA.m, dP.m, &out));
    DMat r = DMat::view(out);
    r.owned = true;
    return r.host();
}

std::vector<double> l1_diagonal(const CsrMatrix& A) {
    if (A.nrows != A.ncols) throw std::invalid_argument("l1_diagonal: matrix is not square");
    std::lock_guard<std::recursive_mutex> lk(backend().mu);
    DMat dA(A);
    DVec d(A.nrows);
    ok(mamg_l1_diagonal(backend().ctx, dA.m, d.p));
    return d.host();
}

bool has_symmetric_pattern(const CsrMatrix& A) {
    if (A.nrows != A.ncols) return false;
    std::lock_guard<std::recursive_mutex> lk(backend().mu);
    DMat dA(A);
    int out = 0;
    ok(mamg_has_symmetric_pattern(backend().ctx, dA.m, &out));
    return out != 0;
}

// =========================================================== vector_ops.hpp ==
double dot(std::span<const double> x, std::span<const double> y) {
    if (x.size() != y.size()) throw std::invalid_argument("dot: length mismatch");
    std::lock_guard<std::recursive_mutex> lk(backend().mu);
    DVec dx(x), dy(y);
    double r = 0.0;
    ok(mamg_dot(backend().ctx, static_cast<int64_t>(x.size()), dx.p, dy.p, &r));
    return r;
}

double norm2(std::span<const double> x) {
    std::lock_guard<std::recursive_mutex> lk(backend().mu);
    DVec dx(x);
    double r = 0.0;
    ok(mamg_norm2(backend().ctx, static_cast<int64_t>(x.size()), dx.p, &r));
    return r;
}

void axpy(std::span<double> y, double a, std::span<const double> x) {
    if (x.size() != y.size()) throw std::invalid_argument("axpy: length mismatch");
    std::lock_guard<std::recursive_mutex> lk(backend().mu);
    DVec dx(x), dy(std::span<const double>(y.data(), y.size()));
    ok(mamg_axpy(backend().ctx, static_cast<int64_t>(y.size()), dy.p, a, dx.p));
    dy.get(y);
}

TripleDot fused_triple_dot(std::span<const double> w, std::span<const double> r,
                           std::span<const double> v, std::span<const double> q_prev) {
    const std::size_t n = w.size();
    if (r.size() != n || v.size() != n || q_prev.size() != n)
        throw std::invalid_argument("fused_triple_dot: length mismatch");
    std::lock_guard<std::recursive_mutex> lk(backend().mu);
    DVec dw(w), dr(r), dv(v), dq(q_prev);
    double out[3];
    ok(mamg_fused_triple_dot(backend().ctx, static_cast<int64_t>(n), dw.p, dr.p, dv.p, dq.p, out));
    return TripleDot{out[0], out[1], out[2]};
}

void fused_axpy_pair(std::span<double> y1, std::span<double> y2, std::span<const double> x,
                     double a, double b) {
    if (y1.size() != y2.size() || y1.size() != x.size())
        throw std::invalid_argument("fused_axpy_pair: length mismatch");
    std::lock_guard<std::recursive_mutex> lk(backend().mu);
    DVec d1(std::span<const double>(y1.data(), y1.size()));
    DVec d2(std::span<const double>(y2.data(), y2.size()));
    DVec dx(x);
    ok(mamg_fused_axpy_pair(backend().ctx, static_cast<int64_t>(x.size()), d1.p, d2.p, dx.p, a, b));
    d1.get(y1);
    d2.get(y2);
}

// ============================================================= matching.hpp ==
index_t Matching::matched_vertices() const {
    return static_cast<index_t>(
        std::count_if(mate.begin(), mate.end(), [](index_t m) { return m != kUnmatched; }));
}

bool Matching::is_valid() const {
    const index_t n = static_cast<index_t>(mate.size());
    for (index_t i = 0; i < n; ++i) {
        const index_t j = mate[i];
        if (j == kUnmatched) continue;
        if (j < 0 || j >= n || j == i || mate[j] != i) return false;
    }
    return true;
}

WeightedGraph build_weights(const CsrMatrix& A, std::span<const double> w) {
    if (A.nrows != A.ncols) throw std::invalid_argument("build_weights: matrix is not square");
    if (static_cast<index_t>(w.size()) != A.nrows)
        throw std::invalid_argument("build_weights: w length mismatch");
    std::lock_guard<std::recursive_mutex> lk(backend().mu);
    DMat dA(A);
    DVec dw(w);
    mamg_graph* g = nullptr;
    ok(mamg_build_weights(backend().ctx, dA.m, dw.p, &g));
    int64_t n, m, z;
    mamg_graph_shape(g, &n, &m, &z);
    WeightedGraph G;
    G.n = n;
    G.xadj.resize(n + 1);
    G.adjncy.resize(m);
    G.weight.resize(m);
    G.zero_weight_edges = static_cast<long>(z);
    const int st = mamg_graph_download(backend().ctx, g, G.xadj.data(), G.adjncy.data(),
                                       G.weight.data());
    mamg_graph_destroy(g);
    ok(st);
    return G;
}

Matching suitor_match(const WeightedGraph& G) {
    std::lock_guard<std::recursive_mutex> lk(backend().mu);
    mamg_graph* g = nullptr;
    ok(mamg_graph_upload(backend().ctx, G.n, G.xadj.data(), G.adjncy.data(), G.weight.data(), &g));
    Matching M;
    M.mate.assign(G.n, kUnmatched);
    const int st = mamg_suitor_match(backend().ctx, g, M.mate.data());
    mamg_graph_destroy(g);
    ok(st);
    return M;
}

// Exhaustive maximum-weight matching (the reference's test oracle,
// matching.cpp:156-209, same contract and error): a forward sweep over the
// vertices in order. The state after vertex i is the set of vertices > i
// already taken by a partner <= i; vertex i+1 is then either taken (skip),
// left single, or matched to a free neighbour above it. Each layer keeps the
// heaviest path into every reachable state and a back pointer.
Matching exact_match_oracle(const WeightedGraph& G) {
    const index_t n = G.n;
    if (n > 20)
        throw std::invalid_argument("exact_match_oracle: n = " + std::to_string(n) +
                                    " exceeds the exhaustive-search limit of 20");
    std::vector<std::vector<std::pair<index_t, double>>> up(static_cast<std::size_t>(n));
    for (index_t u = 0; u < n; ++u)
        for (index_t k = G.xadj[u]; k < G.xadj[u + 1]; ++k)
            if (G.adjncy[k] > u) up[u].emplace_back(G.adjncy[k], G.weight[k]);
    struct Node {
        double w;
        uint32_t from;  // state before this vertex
        index_t partner; // kUnmatched: single or already taken
    };
    auto relax = [](std::unordered_map<uint32_t, Node>& L, uint32_t key, const Node& cand) {
        auto it = L.find(key);
        if (it == L.end())
            L.emplace(key, cand);
        else if (cand.w > it->second.w)
            it->second = cand;
    };
    std::vector<std::unordered_map<uint32_t, Node>> keep(static_cast<std::size_t>(n) + 1);
    keep[0].emplace(0u, Node{0.0, 0u, kUnmatched});
    for (index_t i = 0; i < n; ++i) {
        const uint32_t bit = 1u << i;
        for (const auto& [key, node] : keep[i]) {
            if (key & bit) {
                relax(keep[i + 1], key & ~bit, Node{node.w, key, kUnmatched});
                continue;
            }
            relax(keep[i + 1], key, Node{node.w, key, kUnmatched});
            for (const auto& [j, w] : up[i])
                if (!(key >> j & 1u)) relax(keep[i + 1], key | (1u << j), Node{node.w + w, key, j});
        }
    }
    Matching M;
    M.mate.assign(static_cast<std::size_t>(n), kUnmatched);
    uint32_t key = 0u;
    for (index_t i = n; i-- > 0;) {
        const Node& nd = keep[i + 1].at(key);
        if (nd.partner != kUnmatched) {
            M.mate[i] = nd.partner;
            M.mate[nd.partner] = i;
        }
        key = nd.from;
    }
    return M;
}

double matching_weight(const WeightedGraph& G, const Matching& M) {
    double total = 0.0;
    for (index_t u = 0; u < G.n; ++u) {
        const index_t v = M.mate[u];
        if (v == kUnmatched || v < u) continue;
        for (index_t k = G.xadj[u]; k < G.xadj[u + 1]; ++k)
            if (G.adjncy[k] == v) {
                total += G.weight[k];
                break;
            }
    }
    return total;
}

// =========================================================== coarsening.hpp ==
Aggregation pairwise_aggregate(const Matching& M, index_t n) {
    if (static_cast<index_t>(M.mate.size()) != n)
        throw std::invalid_argument("pairwise_aggregate: mate length != n");
    if (!M.is_valid()) throw std::invalid_argument("pairwise_aggregate: invalid matching");
    std::lock_guard<std::recursive_mutex> lk(backend().mu);
    Aggregation a;
    a.agg_of.resize(n);
    int64_t cnt[3];
    ok(mamg_pairwise_aggregate(backend().ctx, n, M.mate.data(), a.agg_of.data(), cnt));
    a.n_c = cnt[0];
    a.n_p = cnt[1];
    a.n_s = cnt[2];
    return a;
}

CsrMatrix build_prolongator(const Aggregation& agg, std::span<const double> w) {
    const index_t n = static_cast<index_t>(agg.agg_of.size());
    if (static_cast<index_t>(w.size()) != n)
        throw std::invalid_argument("build_prolongator: w length mismatch");
    std::lock_guard<std::recursive_mutex> lk(backend().mu);
    DVec dw(w);
    mamg_mat* P = nullptr;
    ok(mamg_build_prolongator(backend().ctx, n, agg.n_c, agg.agg_of.data(), dw.p, &P));
    DMat r = DMat::view(P);
    r.owned = true;
    return r.host();
}

std::vector<double> restrict_vector(const CsrMatrix& P, std::span<const double> w) {
    if (static_cast<index_t>(w.size()) != P.nrows)
        throw std::invalid_argument("restrict_vector: length mismatch");
    std::lock_guard<std::recursive_mutex> lk(backend().mu);
    DMat dP(P);
    DVec dw(w), wc(P.ncols);
    ok(mamg_restrict_vector(backend().ctx, dP.m, dw.p, wc.p));
    return wc.host();
}

CsrMatrix galerkin_by_aggregates(const CsrMatrix& A, const CsrMatrix& P) {
    std::lock_guard<std::recursive_mutex> lk(backend().mu);
    DMat dA(A), dP(P);
    mamg_mat* out = nullptr;
    ok(mamg_galerkin_by_aggregates(backend().ctx, dA.m, dP.m, &out));
    DMat r = DMat::view(out);
    r.owned = true;
    return r.host();
}

static CoarseningStep coarsen(const CsrMatrix& A, std::span<const double> w, int mode) {
    if (A.nrows != A.ncols) throw std::invalid_argument("build_weights: matrix is not square");
    if (static_cast<index_t>(w.size()) != A.nrows)
        throw std::invalid_argument("build_weights: w length mismatch");
    std::lock_guard<std::recursive_mutex> lk(backend().mu);
    DMat dA(A);
    DVec dw(w);
    mamg_mat *P = nullptr, *Ac = nullptr;
    double* wc = nullptr;
    int64_t zero = 0;
    ok(mamg_coarsen_step(backend().ctx, dA.m, dw.p, mode, &P, &Ac, &wc, &zero));
    DMat dP = DMat::view(P), dAc = DMat::view(Ac);
    dP.owned = dAc.owned = true;
    CoarseningStep st;
    st.P = dP.host();
    st.A_coarse = dAc.host();
    st.w_coarse.resize(st.A_coarse.nrows);
    const int s2 = mamg_d2h(backend().ctx, st.w_coarse.data(), wc, 8 * st.w_coarse.size());
    mamg_dfree(backend().ctx, wc);
    ok(s2);
    st.zero_weight_edges = static_cast<long>(zero);
    return st;
}

CoarseningStep pairwise_step(const CsrMatrix& A, std::span<const double> w) {
    return coarsen(A, w, 1);
}

CoarseningStep double_pairwise(const CsrMatrix& A, std::span<const double> w) {
    return coarsen(A, w, 2);
}

void SetupConfig::validate() const {
    if (max_levels < 1) throw std::invalid_argument("SetupConfig: max_levels must be >= 1");
    if (!(coarse_factor > 0.0))
        throw std::invalid_argument("SetupConfig: coarse_factor must be > 0");
}

// build_hierarchy across the MATCHAMG_DEVICES (one thread per device): the
// partition-aware setup with global matching, then the host levels gathered
// from the parts (global indices; agglomerated levels come from rank 0)
static Hierarchy build_hierarchy_multi(const CsrMatrix& A, std::span<const double> w,
                                       const mamg_setup_cfg& sc, const std::vector<int>& devs) {
    detail::Multi& M = detail::multi();
    M.ensure(devs);
    const int W = static_cast<int>(devs.size());
    std::vector<mamg_ctx*> ctxs(M.ctxs.begin(), M.ctxs.begin() + W);
    auto dev = std::make_shared<detail::DeviceHierarchy>();
    if (mamg_group_create(W, &dev->group) != MAMG_OK) throw std::runtime_error("matchamg: group");
    dev->parts.assign(W, nullptr);
    dev->ctxs = ctxs;
    dev->n0 = A.nrows;
    static const bool trace = std::getenv("MATCHAMG_TRACE") != nullptr;
    auto t0 = std::chrono::steady_clock::now();
    auto mark = [&](const char* what) {
        if (!trace) return;
        const auto t = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[matchamg] %s %.0f ms\n", what,
                     std::chrono::duration<double, std::milli>(t - t0).count());
        t0 = t;
    };
    detail::run_ranks(W, ctxs, [&](int r) {
        int st = mamg_dist_create_group(ctxs[r], dev->group, r, &dev->parts[r]);
        if (st == MAMG_OK) st = mamg_dist_set_matching(dev->parts[r], 1);
        // one build per load here: the build takes the loaded blocks (one
        // device copy of A, which matters for the matrices routed here by size)
        if (st == MAMG_OK) st = mamg_dist_set_rebuildable(dev->parts[r], 0);
        if (st == MAMG_OK)
            st = mamg_dist_load(dev->parts[r], A.nrows, A.row_ptr.data(), A.col_idx.data(),
                                A.values.data(), w.data());
        return st;
    });
    mark("parts loaded");
    detail::run_ranks(W, ctxs, [&](int r) { return mamg_dist_build(dev->parts[r], &sc); });
    mark("parts built");
    int nl = 0, stalled = 0;
    std::vector<int64_t> ln(64), lz(64);
    int64_t zero = 0;
    mamg_dist_info(dev->parts[0], &nl, ln.data(), lz.data(), &stalled, &zero);
    Hierarchy h;
    h.levels.resize(nl);
    // level data of every part, rows concatenated in rank order
    auto gather = [&](int k, int which, index_t ncols) {
        std::vector<int64_t> nr(W), nz(W);
        int64_t rows = 0, ents = 0;
        for (int r = 0; r < W; ++r) {
            detail::ok_on(ctxs[r], mamg_dist_level_shape(dev->parts[r], r, k, which, &nr[r], &nz[r]));
            rows += nr[r];
            ents += nz[r];
        }
        CsrMatrix M;
        M.nrows = rows;
        M.ncols = ncols;
        detail::big_resize(M.row_ptr, static_cast<size_t>(rows + 1));
        detail::big_resize(M.col_idx, static_cast<size_t>(ents));
        detail::big_resize(M.values, static_cast<size_t>(ents));
        // each part straight into its place; its row pointers (from 0) are
        // shifted by the entries of the parts before it
        int64_t ro = 0, eo = 0;
        for (int r = 0; r < W; ++r) {
            detail::ok_on(ctxs[r], mamg_dist_download(dev->parts[r], r, k, which, M.row_ptr.data() + ro,
                                                      M.col_idx.data() + eo, M.values.data() + eo));
            if (eo) {
                int64_t* p = M.row_ptr.data() + ro;
                const int64_t cnt = nr[r] + 1, base = eo;
                const int T = static_cast<int>(std::min<int64_t>(16, cnt / (int64_t{1} << 20) + 1));
                std::vector<std::thread> th;
                for (int t = 0; t < T; ++t)
                    th.emplace_back([=] {
                        for (int64_t i = cnt * t / T; i < cnt * (t + 1) / T; ++i) p[i] += base;
                    });
                for (auto& x : th) x.join();
            }
            ro += nr[r];
            eo += nz[r];
        }
        return M;
    };
    auto gather_vec = [&](int k, int which) {
        std::vector<int64_t> nr(W);
        int64_t rows = 0;
        for (int r = 0; r < W; ++r) {
            int64_t nz = 0;
            detail::ok_on(ctxs[r], mamg_dist_level_shape(dev->parts[r], r, k, which, &nr[r], &nz));
            rows += nr[r];
        }
        std::vector<double> out;
        detail::big_resize(out, static_cast<size_t>(rows));
        int64_t ro = 0;
        for (int r = 0; r < W; ++r) {
            int64_t rp0[2] = {0, 0}; // (written for parts without rows of a replicated level)
            detail::ok_on(ctxs[r], mamg_dist_download(dev->parts[r], r, k, which, rp0, nullptr,
                                                      out.data() + ro));
            ro += nr[r];
        }
        return out;
    };
    for (int k = 0; k < nl; ++k) {
        Level& L = h.levels[k];
        L.A = k == 0 ? detail::big_copy(A) : gather(k, 0, ln[k]);
        mark("  A");
        if (k + 1 < nl) {
            L.P = gather(k, 1, ln[k + 1]);
            mark("  P");
            L.R = gather(k, 2, ln[k]);
            mark("  R");
        }
        L.l1_diag = gather_vec(k, 3);
        L.w = gather_vec(k, 4);
        mark("  vectors");
        h.stats.level_size.push_back(L.A.nrows);
        h.stats.level_nnz.push_back(L.A.nnz());
    }
    mark("host levels gathered");
    h.stats.stalled = stalled != 0;
    h.stats.zero_weight_edges = static_cast<long>(zero);
    h.device = std::move(dev);
    return h;
}

Hierarchy build_hierarchy(const CsrMatrix& A, std::span<const double> w, const SetupConfig& cfg) {
    cfg.validate();
    if (A.nrows != A.ncols) throw std::invalid_argument("build_hierarchy: matrix is not square");
    if (static_cast<index_t>(w.size()) != A.nrows)
        throw std::invalid_argument("build_hierarchy: w length mismatch");
    std::lock_guard<std::recursive_mutex> lk(backend().mu);
    std::vector<int> devs = detail::multi().requested();
    if (devs.size() < 2) {
        // entry offsets are int32 on the device: a matrix of 2^31 or more
        // entries (the reference's CsrMatrix is int64) is built row-block
        // partitioned on this one device, parts of at most kPartEntries
        // entries each, with global matching — bit-identical to the
        // single-device hierarchy (MATCHAMG_PART_NNZ lowers the cap: tests)
        const char* e = std::getenv("MATCHAMG_PART_NNZ");
        const int64_t cap = e ? std::max<int64_t>(std::atoll(e), 1) : int64_t{2000000000};
        const int64_t nnz = static_cast<int64_t>(A.col_idx.size());
        if (nnz >= cap) {
            const char* d = std::getenv("MATCHAMG_DEVICE");
            const int parts = static_cast<int>(std::max<int64_t>(2, (nnz + cap - 1) / cap));
            devs.assign(static_cast<size_t>(parts), d ? std::atoi(d) : 0);
        }
    }
    if (devs.size() >= 2) {
        const mamg_setup_cfg msc{cfg.max_levels,
                                 cfg.aggregation == AggregationMode::Pairwise ? 1 : 2,
                                 cfg.coarse_factor};
        return build_hierarchy_multi(A, w, msc, devs);
    }
    static const bool trace = std::getenv("MATCHAMG_TRACE") != nullptr;
    auto t0 = std::chrono::steady_clock::now();
    auto mark = [&](const char* what) {
        if (!trace) return;
        const auto t = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[matchamg] %s %.1f ms\n", what,
                     std::chrono::duration<double, std::milli>(t - t0).count());
        t0 = t;
    };
    DMat dA(A);
    DVec dw(w);
    mark("upload");
    const mamg_setup_cfg sc{cfg.max_levels,
                            cfg.aggregation == AggregationMode::Pairwise ? 1 : 2,
                            cfg.coarse_factor};
    auto dev = std::make_shared<detail::DeviceHierarchy>();
    ok(mamg_setup(backend().ctx, dA.m, dw.p, &sc, &dev->h));
    mark("device setup");

    Hierarchy h;
    const int nl = mamg_hier_nl(dev->h);
    h.levels.resize(nl);
    for (int k = 0; k < nl; ++k) {
        Level& L = h.levels[k];
        L.A = k == 0 ? detail::big_copy(A) : DMat::view(mamg_hier_A(dev->h, k)).host();
        mark("  A");
        if (k + 1 < nl) {
            L.P = DMat::view(mamg_hier_P(dev->h, k)).host();
            L.R = DMat::view(mamg_hier_R(dev->h, k)).host();
            mark("  P,R");
        }
        const std::size_t n = static_cast<std::size_t>(L.A.nrows);
        detail::big_resize(L.l1_diag, n);
        detail::big_resize(L.w, n);
        if (n) {
            ok(mamg_d2h(backend().ctx, L.l1_diag.data(), mamg_hier_l1(dev->h, k), 8 * n));
            ok(mamg_d2h(backend().ctx, L.w.data(), mamg_hier_w(dev->h, k), 8 * n));
        }
        h.stats.level_size.push_back(L.A.nrows);
        h.stats.level_nnz.push_back(L.A.nnz());
    }
    int stalled = 0;
    int64_t zero = 0;
    mamg_hier_stats(dev->h, &stalled, &zero);
    h.stats.stalled = stalled != 0;
    h.stats.zero_weight_edges = static_cast<long>(zero);
    h.device = std::move(dev);
    return h;
}

Hierarchy build_hierarchy(const CsrMatrix& A, const SetupConfig& cfg) {
    return build_hierarchy(A, std::vector<double>(A.nrows, 1.0), cfg);
}

HierarchySummary hierarchy_stats(const Hierarchy& h) {
    HierarchySummary s;
    s.nl = h.nl();
    double nnz = 0.0;
    for (const Level& L : h.levels) nnz += static_cast<double>(L.A.nnz());
    s.operator_complexity = nnz / static_cast<double>(h.levels.front().A.nnz());
    double ratio = 0.0;
    for (int k = 1; k < s.nl; ++k)
        ratio += static_cast<double>(h.levels[k - 1].A.nrows) /
                 static_cast<double>(h.levels[k].A.nrows);
    s.coarsening_ratio = ratio / static_cast<double>(s.nl);
    return s;
}

// ============================================================ multigrid.hpp ==
void CycleConfig::validate() const {
    if (pre_sweeps < 0 || post_sweeps < 0)
        throw std::invalid_argument("CycleConfig: sweep counts must be >= 0");
    if (coarsest_sweeps < 1)
        throw std::invalid_argument("CycleConfig: coarsest_sweeps must be >= 1");
}

void l1_jacobi_sweeps(const CsrMatrix& A, std::span<const double> d, std::span<const double> b,
                      std::span<double> x, int k) {
    const index_t n = A.nrows;
    if (A.ncols != n || static_cast<index_t>(d.size()) != n ||
        static_cast<index_t>(b.size()) != n || static_cast<index_t>(x.size()) != n)
        throw std::invalid_argument("l1_jacobi_sweeps: dimension mismatch");
    if (k <= 0) return;
    std::lock_guard<std::recursive_mutex> lk(backend().mu);
    DMat dA(A);
    DVec dd(d), db(b), dx(std::span<const double>(x.data(), x.size()));
    ok(mamg_l1_jacobi(backend().ctx, dA.m, dd.p, db.p, dx.p, k));
    dx.get(x);
}

CycleWorkspace::CycleWorkspace(const Hierarchy& h) {
    const int nl = h.nl();
    scratch_.resize(nl);
    coarse_b_.resize(nl);
    coarse_x_.resize(nl);
    for (int k = 0; k < nl; ++k) {
        scratch_[k].resize(h.levels[k].A.nrows);
        if (k + 1 < nl) {
            coarse_b_[k].resize(h.levels[k + 1].A.nrows);
            coarse_x_[k].resize(h.levels[k + 1].A.nrows);
        }
    }
}

void apply_cycle(const Hierarchy& h, int level, std::span<const double> b, std::span<double> x,
                 const CycleConfig& cfg, CycleWorkspace& ws) {
    (void)ws;
    const int nl = h.nl();
    if (level < 0 || level >= nl)
        throw std::invalid_argument("apply_cycle: level " + std::to_string(level) +
                                    " outside [0, " + std::to_string(nl) + ")");
    const index_t n = h.levels[level].A.nrows;
    if (static_cast<index_t>(b.size()) != n || static_cast<index_t>(x.size()) != n)
        throw std::invalid_argument("apply_cycle: dimension mismatch at level " +
                                    std::to_string(level));
    std::lock_guard<std::recursive_mutex> lk(backend().mu);
    auto dev = detail::twin(h);
    DVec db(b), dx(std::span<const double>(x.data(), x.size()));
    const mamg_cycle_cfg c = detail::ccfg(cfg);
    ok(mamg_apply_cycle(backend().ctx, dev->h, level, &c, db.p, dx.p));
    dx.get(x);
}

static std::vector<double> run_cycle(const Hierarchy& h, int level, std::span<const double> b,
                                     std::span<const double> x0, CycleConfig cfg, CycleType t) {
    cfg.cycle = t;
    cfg.validate();
    std::vector<double> x(x0.begin(), x0.end());
    CycleWorkspace ws;
    apply_cycle(h, level, b, x, cfg, ws);
    return x;
}

std::vector<double> vcycle(const Hierarchy& h, int level, std::span<const double> b,
                           std::span<const double> x0, CycleConfig cfg) {
    return run_cycle(h, level, b, x0, cfg, CycleType::V);
}

std::vector<double> wcycle(const Hierarchy& h, int level, std::span<const double> b,
                           std::span<const double> x0, CycleConfig cfg) {
    return run_cycle(h, level, b, x0, cfg, CycleType::W);
}

MultigridPreconditioner::MultigridPreconditioner(const Hierarchy& h, CycleConfig cfg)
    : h_(&h), cfg_(cfg) {
    cfg.validate();
    std::lock_guard<std::recursive_mutex> lk(backend().mu);
    // a partitioned twin stays partitioned (pcg_solve runs on every device)
    dev_ = h.device && h.device->partitioned() ? h.device : detail::twin(h);
}

void MultigridPreconditioner::apply(std::span<const double> r, std::span<double> z) {
    std::lock_guard<std::recursive_mutex> lk(backend().mu);
    DVec dr(r), dz(z.size());
    const mamg_cycle_cfg c = detail::ccfg(cfg_);
    // one host-callable cycle: the single-device copy of a partitioned twin
    mamg_hier* hh = dev_->partitioned() ? detail::twin(*h_)->h : dev_->h;
    ok(mamg_precond_apply(backend().ctx, hh, &c, dr.p, dz.p));
    dz.get(z);
}

// =============================================================== krylov.hpp ==
void SolveConfig::validate() const {
    if (!(rtol > 0.0)) throw std::invalid_argument("SolveConfig: rtol must be > 0");
    if (itmax < 1) throw std::invalid_argument("SolveConfig: itmax must be >= 1");
}

BreakdownError::BreakdownError(index_t iteration, const std::string& what)
    : std::runtime_error("pcg breakdown at iteration " + std::to_string(iteration) + ": " + what),
      iteration_(iteration) {}

void DevicePrecond::operator()(std::span<const double> r, std::span<double> z) const {
    mg->apply(r, z);
}

PrecondFn device_precond(MultigridPreconditioner& mg) { return PrecondFn(DevicePrecond{&mg}); }

namespace {
struct HostPrecondBox {
    const PrecondFn* fn;
};
void host_precond_trampoline(void* user, const double* r, double* z, int64_t n) {
    const auto* box = static_cast<const HostPrecondBox*>(user);
    (*box->fn)(std::span<const double>(r, static_cast<std::size_t>(n)),
               std::span<double>(z, static_cast<std::size_t>(n)));
}
} // namespace

std::pair<std::vector<double>, SolveReport> pcg_solve(const CsrMatrix& A, const PrecondFn& B,
                                                      std::span<const double> b,
                                                      std::span<const double> u0,
                                                      const SolveConfig& cfg) {
    cfg.validate();
    const index_t n = A.nrows;
    if (A.ncols != n) throw std::invalid_argument("pcg_solve: matrix is not square");
    if (static_cast<index_t>(b.size()) != n || static_cast<index_t>(u0.size()) != n)
        throw std::invalid_argument("pcg_solve: dimension mismatch");
    std::lock_guard<std::recursive_mutex> lk(backend().mu);
    {
        const DevicePrecond* dp = B ? B.target<DevicePrecond>() : nullptr;
        if (dp && dp->mg->device()->partitioned()) {
            // the partitioned PCG on every device of the hierarchy (its level 0
            // is the matrix the hierarchy was built from)
            const auto& D = *dp->mg->device();
            if (D.n0 != n) throw std::invalid_argument("pcg_solve: dimension mismatch");
            const int W = static_cast<int>(D.parts.size());
            const mamg_cycle_cfg c = detail::ccfg(dp->mg->config());
            const mamg_solve_cfg sc{cfg.rtol, cfg.itmax};
            bool zero0 = true;
            for (double x : u0) zero0 = zero0 && x == 0.0;
            std::vector<double> u(static_cast<std::size_t>(n));
            std::vector<std::vector<double>> hist(W, std::vector<double>(static_cast<std::size_t>(cfg.itmax) + 2));
            std::vector<mamg_report> reps(W);
            detail::run_ranks(W, D.ctxs, [&](int r) {
                return mamg_dist_pcg_x0(D.parts[r], b.data(), zero0 ? nullptr : u0.data(), &c, &sc,
                                        u.data(), hist[r].data(), &reps[r]);
            });
            const mamg_report& rep = reps[0];
            SolveReport rr;
            rr.iterations = rep.iterations;
            rr.final_relres = rep.final_relres;
            rr.residual_history.assign(hist[0].begin(), hist[0].begin() + (rep.iterations + 1));
            rr.converged = rep.converged != 0;
            rr.solve_ms = rep.solve_ms;
            rr.audit_checks = rep.audit_checks;
            rr.audit_failures = rep.audit_failures;
            rr.audit_max_rel = rep.audit_max_rel;
            return {std::move(u), std::move(rr)};
        }
    }
    DMat dA(A);
    DVec db(b), du0(u0), du(static_cast<std::size_t>(n));
    const mamg_solve_cfg sc{cfg.rtol, cfg.itmax};
    std::vector<double> hist(static_cast<std::size_t>(cfg.itmax) + 2);
    mamg_report rep{};
    int st;
    const DevicePrecond* dp = B ? B.target<DevicePrecond>() : nullptr;
    if (dp) {
        const mamg_cycle_cfg c = detail::ccfg(dp->mg->config());
        st = mamg_pcg_solve(backend().ctx, dA.m, dp->mg->device()->h, &c, nullptr, nullptr, db.p,
                            du0.p, &sc, du.p, hist.data(), &rep);
    } else if (B) {
        HostPrecondBox box{&B};
        st = mamg_pcg_solve(backend().ctx, dA.m, nullptr, nullptr, host_precond_trampoline, &box,
                            db.p, du0.p, &sc, du.p, hist.data(), &rep);
    } else {
        st = mamg_pcg_solve(backend().ctx, dA.m, nullptr, nullptr, nullptr, nullptr, db.p, du0.p,
                            &sc, du.p, hist.data(), &rep);
    }
    ok(st);
    SolveReport r;
    r.iterations = rep.iterations;
    r.final_relres = rep.final_relres;
    r.residual_history.assign(hist.begin(), hist.begin() + (rep.iterations + 1));
    r.converged = rep.converged != 0;
    r.solve_ms = rep.solve_ms;
    r.audit_checks = rep.audit_checks;
    r.audit_failures = rep.audit_failures;
    r.audit_max_rel = rep.audit_max_rel;
    return {du.host(), std::move(r)};
}

std::pair<std::vector<double>, SolveReport> pcg_solve(const CsrMatrix& A, const PrecondFn& B,
                                                      std::span<const double> b,
                                                      const SolveConfig& cfg) {
    return pcg_solve(A, B, b, std::vector<double>(A.nrows, 0.0), cfg);
}

} // namespace matchamg
