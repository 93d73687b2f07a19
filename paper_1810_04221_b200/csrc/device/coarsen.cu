// coarsen.cu — the setup phase of the matching AMG on sm_100a
// (proj/src/coarsening.cpp): pairwise aggregation, the unit-norm
// piecewise-constant prolongator, the restricted smooth vector, the
// specialised Galerkin product, (double) pairwise steps and the level loop.
#include <cmath>
#include <cstdlib>

#include <chrono>
#include <cstdio>
#include <cstdlib>

#include "ops.cuh"
#include "rowprod.cuh"
#include "dist.cuh"

namespace mamg {
namespace {

constexpr int kBlock = 256;

// ------------------------------------------------------------ aggregation --
// coarsening.cpp:20-32: vertex i leads an aggregate when it is unmatched or
// the smaller end of its pair; aggregate ids follow the leaders in ascending
// order, i.e. an exclusive scan of the leader flags.
__global__ void k_leaders(int64_t n, const int32_t* __restrict__ mate, int32_t* flag,
                          unsigned long long* counts /* pairs, singletons */) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    int f = 0, pair = 0, single = 0;
    if (i < n) {
        const int m = mate[i];
        f = (m < 0 || i < m);
        pair = (m >= 0 && i < m);
        single = m < 0;
        flag[i] = f;
    }
    pair = __syncthreads_count(pair);
    single = __syncthreads_count(single);
    if (threadIdx.x == 0) {
        if (pair) atomicAdd(&counts[0], static_cast<unsigned long long>(pair));
        if (single) atomicAdd(&counts[1], static_cast<unsigned long long>(single));
    }
}

__global__ void k_assign(int64_t n, const int32_t* __restrict__ mate,
                         const int32_t* __restrict__ ids, int32_t* agg_of, int32_t* size) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int m = mate[i];
    const bool lead = m < 0 || i < m;
    agg_of[i] = lead ? ids[i] : ids[m];
    if (lead) size[ids[i]] = m < 0 ? 1 : 2;
}

__global__ void k_members_from_mate(int64_t n, const int32_t* __restrict__ mate,
                                    const int32_t* __restrict__ ids,
                                    const int32_t* __restrict__ mptr, int32_t* members) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int m = mate[i];
    if (!(m < 0 || i < m)) return;
    const int at = mptr[ids[i]];
    members[at] = static_cast<int32_t>(i);
    if (m >= 0) members[at + 1] = m; // m > i: members stay ascending
}

// generic aggregate map -> member lists (counting sort, then per-aggregate
// insertion sort so members are ascending, as build_prolongator and the
// Galerkin product visit them)
__global__ void k_count_agg(int64_t n, int64_t nc, const int32_t* __restrict__ agg,
                            int32_t* cnt, int32_t* bad) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int a = agg[i];
    if (a < 0 || a >= nc) {
        atomicMin(bad, static_cast<int32_t>(i));
        return;
    }
    atomicAdd(&cnt[a], 1);
}

__global__ void k_fill_members(int64_t n, const int32_t* __restrict__ agg, int32_t* cursor,
                               int32_t* members) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    members[atomicAdd(&cursor[agg[i]], 1)] = static_cast<int32_t>(i);
}

__global__ void k_sort_members(int64_t nc, const int32_t* __restrict__ mptr, int32_t* members) {
    const int64_t a = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (a >= nc) return;
    const int lo = mptr[a], hi = mptr[a + 1];
    for (int x = lo + 1; x < hi; ++x) {
        const int32_t key = members[x];
        int y = x - 1;
        while (y >= lo && members[y] > key) {
            members[y + 1] = members[y];
            --y;
        }
        members[y + 1] = key;
    }
}

// ------------------------------------------------------------ prolongator --
// coarsening.cpp:42-60: ||w|_a||^2 summed over members in ascending order
// from 0.0; an aggregate of size > 1 with zero norm is an error.
__global__ void k_agg_norms(int64_t nc, const int32_t* __restrict__ mptr,
                            const int32_t* __restrict__ members, const double* __restrict__ w,
                            double* norm, int32_t* bad) {
    const int64_t a = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (a >= nc) return;
    double s = 0.0;
    const int lo = mptr[a], hi = mptr[a + 1];
    for (int m = lo; m < hi; ++m) {
        const double wi = w[members[m]];
        s = rn_add(s, rn_mul(wi, wi));
    }
    if (s == 0.0 && hi - lo > 1) atomicMin(bad, static_cast<int32_t>(a));
    norm[a] = sqrt(s);
}

// coarsening.cpp:69-74
__global__ void k_pvals(int64_t n, const int32_t* __restrict__ agg, const double* __restrict__ norm,
                        const double* __restrict__ w, int32_t* rp, int32_t* ci, double* pv) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i > n) return;
    rp[i] = static_cast<int32_t>(i);
    if (i == n) return;
    const int a = agg[i];
    const double nr = norm[a];
    ci[i] = a;
    pv[i] = nr == 0.0 ? 1.0 : rn_div(w[i], nr);
}

// coarsening.cpp:78-87: wc[a] = 0.0 + p_i w_i + ... in ascending member order
__global__ void k_restrict_members(int64_t nc, const int32_t* __restrict__ mptr,
                                   const int32_t* __restrict__ members,
                                   const double* __restrict__ pv, const double* __restrict__ w,
                                   double* wc) {
    const int64_t a = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (a >= nc) return;
    double s = 0.0;
    for (int m = mptr[a]; m < mptr[a + 1]; ++m) {
        const int i = members[m];
        s = rn_add(s, rn_mul(pv[i], w[i]));
    }
    wc[a] = s;
}

__global__ void k_restrict_rows(int64_t nc, const int32_t* __restrict__ rp,
                                const int32_t* __restrict__ ci, const double* __restrict__ rv,
                                const double* __restrict__ w, double* wc) {
    const int64_t a = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (a >= nc) return;
    double s = 0.0;
    for (int e = rp[a]; e < rp[a + 1]; ++e) s = rn_add(s, rn_mul(rv[e], w[ci[e]]));
    wc[a] = s;
}

// -------------------------------------------------------------- Galerkin --
// coarsening.cpp:123-146: coarse row I visits its members ascending, each
// member's row in column order; the contribution of a_ik is
// (p_i * a_ik) * p_k into column agg(k).
struct GalerkinProb {
    const int32_t* __restrict__ mptr;
    const int32_t* __restrict__ members;
    const int32_t* __restrict__ rp;
    const int32_t* __restrict__ ci;
    const double* __restrict__ v;
    const int32_t* __restrict__ agg;
    const double* __restrict__ pv;
    struct Outer {
        double pi;
    };
    __device__ int outer_count(int I) const { return mptr[I + 1] - mptr[I]; }
    __device__ Outer outer(int I, int o, int& lo, int& hi) const {
        const int i = members[mptr[I] + o];
        lo = rp[i];
        hi = rp[i + 1];
        return Outer{pv[i]};
    }
    __device__ void contrib(const Outer& ou, int e, int32_t& col, double& val) const {
        const int j = ci[e];
        col = agg[j];
        val = rn_mul(rn_mul(ou.pi, v[e]), pv[j]);
    }
};

__global__ void k_galerkin_ub(int64_t nc, const int32_t* __restrict__ mptr,
                              const int32_t* __restrict__ members, const int32_t* __restrict__ rp,
                              int32_t* ub) {
    const int64_t a = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (a >= nc) return;
    int s = 0;
    for (int m = mptr[a]; m < mptr[a + 1]; ++m) s += rp[members[m] + 1] - rp[members[m]];
    ub[a] = s;
}

// spgemm(P1, P2) for one-entry rows (kernels.cpp:272-281 with a single
// product per row; the first insert assigns): P[i] = p1_i * p2_{a1(i)}
__global__ void k_compose(int64_t n, const int32_t* __restrict__ c1, const double* __restrict__ v1,
                          const int32_t* __restrict__ c2, const double* __restrict__ v2,
                          int32_t* rp, int32_t* ci, double* v) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i > n) return;
    rp[i] = static_cast<int32_t>(i);
    if (i == n) return;
    const int a = c1[i];
    ci[i] = c2[a];
    v[i] = rn_mul(v1[i], v2[a]);
}

__global__ void k_max_row(int64_t n, const int32_t* __restrict__ rp, int32_t* out) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    int m = i < n ? rp[i + 1] - rp[i] : 0;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, off));
    if ((threadIdx.x & 31) == 0 && m > 0) atomicMax(out, m);
}

__global__ void k_fill(int64_t n, double* x, double val) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) x[i] = val;
}

} // namespace

int64_t max_row_nnz(Ctx& c, const DevCsr& A) {
    DBuf<int32_t> m(1, c.stream);
    MAMG_CU(cudaMemsetAsync(m.get(), 0, sizeof(int32_t), c.stream));
    if (A.nrows > 0) {
        k_max_row<<<blocks_for(A.nrows, kBlock), kBlock, 0, c.stream>>>(A.nrows, A.rp.get(), m.get());
        c.count();
        MAMG_LAUNCH_CHECK();
    }
    return read_i32(c, m.get());
}

void fill_f64(Ctx& c, int64_t n, double* dst, double v) {
    if (n <= 0) return;
    k_fill<<<blocks_for(n, kBlock), kBlock, 0, c.stream>>>(n, dst, v);
    c.count();
    MAMG_LAUNCH_CHECK();
}

// ================================================================= host API ==
DevAgg aggregate_from_mate(Ctx& c, int64_t n, const int32_t* mate) {
    DevAgg g;
    g.n = n;
    g.agg_of.alloc(n, c.stream);
    g.members.alloc(n, c.stream);
    // member pointers sized for the upper bound nc <= n: the numbering, the
    // sizes and the member lists are all enqueued before the host needs nc
    g.mptr.alloc(n + 1, c.stream);
    DBuf<int32_t> ids(n + 1, c.stream);
    unsigned long long* counts = reinterpret_cast<unsigned long long*>(c.d_small.get() + 8);
    MAMG_CU(cudaMemsetAsync(counts, 0, 2 * sizeof(unsigned long long), c.stream));
    MAMG_CU(cudaMemsetAsync(g.mptr.get(), 0, sizeof(int32_t) * (n + 1), c.stream));
    if (n > 0) {
        k_leaders<<<blocks_for(n, kBlock), kBlock, 0, c.stream>>>(n, mate, ids.get(), counts);
        c.count();
    }
    exclusive_scan_i32(c, ids.get(), ids.get(), n);
    // pinned slots 16..18: nc, then the pair / singleton counts
    MAMG_CU(cudaMemcpyAsync(c.h_small + 16, ids.get() + n, sizeof(int32_t), cudaMemcpyDeviceToHost,
                            c.stream));
    MAMG_CU(cudaMemcpyAsync(c.h_small + 17, counts, 2 * sizeof(unsigned long long),
                            cudaMemcpyDeviceToHost, c.stream));
    // also raises any deferred check registered before (l1, weights); the
    // aggregate sizes (entries >= nc stay 0), their scan and the member lists
    // run while the host waits for the copies
    sync_checked(c, [&] {
        if (n > 0) {
            k_assign<<<blocks_for(n, kBlock), kBlock, 0, c.stream>>>(n, mate, ids.get(),
                                                                     g.agg_of.get(), g.mptr.get());
            c.count();
        }
        exclusive_scan_i32(c, g.mptr.get(), g.mptr.get(), n);
        if (n > 0) {
            k_members_from_mate<<<blocks_for(n, kBlock), kBlock, 0, c.stream>>>(
                n, mate, ids.get(), g.mptr.get(), g.members.get());
            c.count();
        }
        MAMG_LAUNCH_CHECK();
    });
    g.nc = static_cast<int32_t>(c.h_small[16] & 0xffffffff);
    g.np = c.h_small[17];
    g.ns = c.h_small[18];
    return g;
}

DevAgg aggregate_from_map(Ctx& c, int64_t n, int64_t nc, const int32_t* agg_of) {
    DevAgg g;
    g.n = n;
    g.nc = nc;
    g.agg_of.alloc(n, c.stream);
    g.members.alloc(n, c.stream);
    g.mptr.alloc(nc + 1, c.stream);
    if (n > 0)
        MAMG_CU(cudaMemcpyAsync(g.agg_of.get(), agg_of, sizeof(int32_t) * n,
                                cudaMemcpyDeviceToDevice, c.stream));
    MAMG_CU(cudaMemsetAsync(g.mptr.get(), 0, sizeof(int32_t) * (nc + 1), c.stream));
    int32_t* bad = reinterpret_cast<int32_t*>(c.d_small.get());
    const int32_t init = INT32_MAX;
    MAMG_CU(cudaMemcpyAsync(bad, &init, sizeof(init), cudaMemcpyHostToDevice, c.stream));
    if (n > 0) {
        k_count_agg<<<blocks_for(n, kBlock), kBlock, 0, c.stream>>>(n, nc, g.agg_of.get(),
                                                                    g.mptr.get(), bad);
        c.count();
    }
    const int64_t b = read_i32(c, bad);
    if (b != INT32_MAX)
        invalid("build_prolongator: aggregate id out of range for vertex " + std::to_string(b), b);
    exclusive_scan_i32(c, g.mptr.get(), g.mptr.get(), nc);
    if (n > 0) {
        DBuf<int32_t> cursor(nc + 1, c.stream);
        MAMG_CU(cudaMemcpyAsync(cursor.get(), g.mptr.get(), sizeof(int32_t) * (nc + 1),
                                cudaMemcpyDeviceToDevice, c.stream));
        k_fill_members<<<blocks_for(n, kBlock), kBlock, 0, c.stream>>>(n, g.agg_of.get(),
                                                                       cursor.get(),
                                                                       g.members.get());
        k_sort_members<<<blocks_for(nc, kBlock), kBlock, 0, c.stream>>>(nc, g.mptr.get(),
                                                                        g.members.get());
        c.count(2);
    }
    MAMG_LAUNCH_CHECK();
    return g;
}

DevAgg aggregates_of(Ctx& c, const DevCsr& P) {
    return aggregate_from_map(c, P.nrows, P.ncols, P.ci.get());
}

std::unique_ptr<DevCsr> build_prolongator(Ctx& c, const DevAgg& g, const double* w, bool defer) {
    DBuf<double> norm(g.nc, c.stream);
    auto vanish = [](int, int32_t a) {
        invalid("build_prolongator: smooth vector vanishes on aggregate " + std::to_string(a), a);
    };
    int32_t* bad;
    if (defer) {
        bad = defer_flags(c, 1, vanish);
    } else {
        bad = reinterpret_cast<int32_t*>(c.d_small.get());
        const int32_t init = INT32_MAX;
        MAMG_CU(cudaMemcpyAsync(bad, &init, sizeof(init), cudaMemcpyHostToDevice, c.stream));
    }
    if (g.nc > 0) {
        k_agg_norms<<<blocks_for(g.nc, kBlock), kBlock, 0, c.stream>>>(
            g.nc, g.mptr.get(), g.members.get(), w, norm.get(), bad);
        c.count();
    }
    MAMG_LAUNCH_CHECK();
    if (!defer) {
        const int64_t b = read_i32(c, bad);
        if (b != INT32_MAX) vanish(0, static_cast<int32_t>(b));
    }
    auto P = std::make_unique<DevCsr>();
    P->nrows = g.n;
    P->ncols = g.nc;
    P->nnz = g.n;
    P->rp.alloc(g.n + 1, c.stream);
    P->ci.alloc(g.n, c.stream);
    P->v.alloc(g.n, c.stream);
    k_pvals<<<blocks_for(g.n + 1, kBlock), kBlock, 0, c.stream>>>(
        g.n, g.agg_of.get(), norm.get(), w, P->rp.get(), P->ci.get(), P->v.get());
    c.count();
    MAMG_LAUNCH_CHECK();
    P->single = g.n > 0;
    P->max_tile = 256;
    P->group = lane_policy_from(P->nrows, P->nnz, P->single);
    return P;
}

void restrict_members(Ctx& c, const DevAgg& g, const double* pval, const double* w, double* wc) {
    if (g.nc == 0) return;
    k_restrict_members<<<blocks_for(g.nc, kBlock), kBlock, 0, c.stream>>>(
        g.nc, g.mptr.get(), g.members.get(), pval, w, wc);
    c.count();
    MAMG_LAUNCH_CHECK();
}

void restrict_rows(Ctx& c, const DevCsr& R, const double* w, double* wc) {
    if (R.nrows == 0) return;
    k_restrict_rows<<<blocks_for(R.nrows, kBlock), kBlock, 0, c.stream>>>(
        R.nrows, R.rp.get(), R.ci.get(), R.v.get(), w, wc);
    c.count();
    MAMG_LAUNCH_CHECK();
}

std::unique_ptr<DevCsr> galerkin(Ctx& c, const DevCsr& A, const DevAgg& g, const double* pval,
                                 bool defer_finalize, const std::function<void()>& between) {
    return galerkin_ext(c, A, g, g.agg_of.get(), pval, g.nc, defer_finalize, between);
}

std::unique_ptr<DevCsr> galerkin_ext(Ctx& c, const DevCsr& A, const DevAgg& g,
                                     const int32_t* agg_ext, const double* pv_ext,
                                     int64_t ncols_out, bool defer_finalize,
                                     const std::function<void()>& between) {
    const double* pval = pv_ext;
    DBuf<int32_t> ub(g.nc + 1, c.stream);
    if (g.nc > 0) {
        k_galerkin_ub<<<blocks_for(g.nc, kBlock), kBlock, 0, c.stream>>>(
            g.nc, g.mptr.get(), g.members.get(), A.rp.get(), ub.get());
        c.count();
        MAMG_LAUNCH_CHECK();
    }
    GalerkinProb pb{g.mptr.get(), g.members.get(), A.rp.get(), A.ci.get(),
                    A.v.get(),    agg_ext,         pval};
    // every fine row is a member of exactly one aggregate: the contributions
    // number nnz(A)
    auto Ac = rowprod_run(c, pb, g.nc, ncols_out, ub, A.nnz, defer_finalize, between);
    return Ac;
}

// MAMG_TRACE=1: per-phase host timings of the setup (synchronising; for
// diagnosis only)
namespace {
struct Trace {
    bool on;
    std::chrono::steady_clock::time_point t0;
    Ctx* c;
    explicit Trace(Ctx& cc) : c(&cc) {
        static const bool enabled = std::getenv("MAMG_TRACE") && std::getenv("MAMG_TRACE")[0] == '1';
        on = enabled;
        if (on) {
            c->sync();
            t0 = std::chrono::steady_clock::now();
        }
    }
    void mark(const char* what, int64_t n) {
        if (!on) return;
        c->sync();
        const auto t = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[mamg trace] n=%lld %-12s %8.3f ms\n", static_cast<long long>(n), what,
                     std::chrono::duration<double, std::milli>(t - t0).count());
        t0 = t;
    }
};
} // namespace

DevStep pairwise_step(Ctx& c, const DevCsr& A, const double* w, const WeightsCheck& chk) {
    Trace tr(c);
    DevStep st;
    DBuf<int32_t> mate(A.nrows, c.stream);
    weights_suitor(c, A, w, mate.get(), st.zero_edges, nullptr, 0, chk);
    tr.mark("suitor", A.nrows);
    DevAgg g = aggregate_from_mate(c, A.nrows, mate.get());
    tr.mark("aggregate", A.nrows);
    st.P = build_prolongator(c, g, w, /*defer=*/true); // checked at the Galerkin readback
    tr.mark("prolongator", A.nrows);
    // A_c's flags (finite, longest tile) are read at the next readback: the
    // next step's aggregate count, or the end of the setup
    // the restricted weights need only P: they run while the host waits
    // for A_c's nnz
    st.wc.alloc(g.nc, c.stream);
    st.Ac = galerkin(c, A, g, st.P->v.get(), /*defer_finalize=*/true,
                     [&] { restrict_members(c, g, st.P->v.get(), w, st.wc.get()); });
    tr.mark("galerkin", A.nrows);
    return st;
}

std::unique_ptr<DevCsr> compose_single(Ctx& c, const DevCsr& P1, const DevCsr& P2) {
    const int64_t n = P1.nrows;
    auto P = std::make_unique<DevCsr>();
    P->nrows = n;
    P->ncols = P2.ncols;
    P->nnz = n;
    P->rp.alloc(n + 1, c.stream);
    P->ci.alloc(n, c.stream);
    P->v.alloc(n, c.stream);
    k_compose<<<blocks_for(n + 1, kBlock), kBlock, 0, c.stream>>>(
        n, P1.ci.get(), P1.v.get(), P2.ci.get(), P2.v.get(), P->rp.get(), P->ci.get(), P->v.get());
    c.count();
    MAMG_LAUNCH_CHECK();
    P->single = n > 0;
    P->max_tile = 256;
    P->group = lane_policy_from(P->nrows, P->nnz, P->single);
    return P;
}

DevStep double_pairwise(Ctx& c, const DevCsr& A, const double* w, const WeightsCheck& chk) {
    DevStep first = pairwise_step(c, A, w, chk);
    // a Galerkin product of a pattern-symmetric matrix is pattern-symmetric
    DevStep second = pairwise_step(c, *first.Ac, first.wc.get(), WeightsCheck{false, nullptr});
    DevStep out;
    out.P = compose_single(c, *first.P, *second.P);
    out.Ac = std::move(second.Ac);
    out.wc = std::move(second.wc);
    out.zero_edges = first.zero_edges + second.zero_edges;
    return out;
}

DevHier::~DevHier() = default;

void alloc_workspace(Ctx& c, DevHier& h) {
    const int nl = h.nl();
    // the coarsest level's sweeps in one cluster launch (coarsest.cu) when it fits
    h.coarsest = CoarsestPlan{};
    if (nl >= 1) coarsest_plan(c, *h.lv[nl - 1].A, h.coarsest);
    for (int k = 0; k < nl; ++k) {
        DevLevel& L = h.lv[k];
        const int64_t n = L.A->nrows;
        L.scratch.alloc(n, c.stream);
        L.xw.alloc(n, c.stream);
        if (k + 1 < nl) {
            const int64_t nc = h.lv[k + 1].A->nrows;
            L.cb.alloc(nc, c.stream);
            L.cx.alloc(nc, c.stream);
        }
    }
}

std::unique_ptr<DevHier> build_hierarchy(Ctx& c, const DevCsr& A, const double* w,
                                         const mamg_setup_cfg& cfg) {
    return build_hierarchy_owned(c, A, nullptr, w, cfg);
}

std::unique_ptr<DevHier> build_hierarchy_owned(Ctx& c, const DevCsr& A,
                                               std::unique_ptr<DevCsr> owned, const double* w,
                                               const mamg_setup_cfg& cfg) {
    if (cfg.max_levels < 1) invalid("SetupConfig: max_levels must be >= 1");
    if (!(cfg.coarse_factor > 0.0)) invalid("SetupConfig: coarse_factor must be > 0");
    if (A.nrows != A.ncols) invalid("build_hierarchy: matrix is not square");
    const double bound = cfg.coarse_factor * std::cbrt(static_cast<double>(A.nrows));
    // coarsening.cpp:196: the pattern must be symmetric. When level 0 is
    // coarsened, the weights pass looks up the mirror of every entry anyway:
    // it records the check (a deferred flag registered ahead of every other
    // check, so it is raised first, as in the reference); otherwise the
    // standalone check kernel runs.
    const bool coarsens = static_cast<double>(A.nrows) > bound && cfg.max_levels > 1;
    if (!coarsens && !has_symmetric_pattern(c, A))
        invalid("build_hierarchy: matrix pattern is not symmetric");

    auto h = std::make_unique<DevHier>();
    h->lv.emplace_back();
    DevLevel& L0 = h->lv.back();
    L0.A = owned ? std::move(owned) : csr_clone(c, A); // level 0 owns its copy of A
    L0.l1.alloc(A.nrows, c.stream);
    L0.w.alloc(A.nrows, c.stream);
    if (w) {
        if (A.nrows)
            MAMG_CU(cudaMemcpyAsync(L0.w.get(), w, sizeof(double) * A.nrows,
                                    cudaMemcpyDeviceToDevice, c.stream));
    } else if (A.nrows) {
        k_fill<<<blocks_for(A.nrows, kBlock), kBlock, 0, c.stream>>>(A.nrows, L0.w.get(), 1.0);
        c.count();
    }
    c.pending.clear();
    c.defer_used = 0;
    int32_t* sym_flag = nullptr;
    if (coarsens)
        sym_flag = defer_flags(c, 1, [](int, int32_t) {
            invalid("build_hierarchy: matrix pattern is not symmetric");
        });
    if (A.nrows != A.ncols) invalid("l1_diagonal: matrix is not square");
    l1_diagonal_local(c, *L0.A, L0.l1.get(), /*defer=*/true);
    try {
        grow_hierarchy(c, *h, bound, cfg.max_levels, cfg.aggregation, sym_flag);
    } catch (...) {
        // deferred values may point into matrices being unwound
        c.pending.clear();
        c.defer_used = 0;
        throw;
    }
    return h;
}

// coarsening.cpp:210-238 from the hierarchy's last level (whose A, w, l1
// are set): pairwise steps until the size bound, the level budget or a stall
void grow_hierarchy(Ctx& c, DevHier& hh, double bound, int max_levels, int aggregation,
                    int32_t* sym_flag) {
    DevHier* h = &hh;
    while (static_cast<double>(h->lv.back().A->nrows) > bound && h->nl() < max_levels) {
        DevLevel& fine = h->lv.back();
        // level 0 of build_hierarchy carries its pattern-symmetry check
        // (sym_flag); every coarser level is a Galerkin product: symmetric
        const WeightsCheck chk = h->nl() == 1 && sym_flag ? WeightsCheck{true, sym_flag}
                                                          : WeightsCheck{false, nullptr};
        DevStep st = aggregation == 1 ? pairwise_step(c, *fine.A, fine.w.get(), chk)
                                      : double_pairwise(c, *fine.A, fine.w.get(), chk);
        h->zero_edges += st.zero_edges;
        if (st.Ac->nrows == fine.A->nrows) {
            h->stalled = true;
            sync_checked(c); // st.Ac's deferred flags land before it is dropped
            break;
        }
        fine.P = std::move(st.P);
        fine.R = transpose_agg(c, *fine.P, aggregation == 1 ? 2 : 4);
        DevLevel coarse;
        coarse.A = std::move(st.Ac);
        coarse.l1.alloc(coarse.A->nrows, c.stream);
        coarse.w = std::move(st.wc);
        l1_diagonal_local(c, *coarse.A, coarse.l1.get(), /*defer=*/true);
        h->lv.push_back(std::move(coarse));
    }
    sync_checked(c); // the last level's l1 check
    alloc_workspace(c, *h);
}

std::unique_ptr<DevHier> build_hierarchy_sub(Ctx& c, std::unique_ptr<DevCsr> A, DBuf<double> w,
                                             double bound, int max_levels, int aggregation) {
    auto h = std::make_unique<DevHier>();
    h->lv.emplace_back();
    DevLevel& L0 = h->lv.back();
    L0.A = std::move(A);
    L0.w = std::move(w);
    L0.l1.alloc(L0.A->nrows, c.stream);
    c.pending.clear();
    c.defer_used = 0;
    l1_diagonal_local(c, *L0.A, L0.l1.get(), /*defer=*/true);
    try {
        grow_hierarchy(c, *h, bound, max_levels, aggregation);
    } catch (...) {
        c.pending.clear();
        c.defer_used = 0;
        throw;
    }
    return h;
}

} // namespace mamg
