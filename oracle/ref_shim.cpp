// ref_shim.cpp — TEST INFRASTRUCTURE ONLY (never shipped, never measured as
// the product). A C-ABI veneer over the *unmodified* reference library
// (/root/reference/proj/src/*.cpp compiled by oracle/Makefile into
// oracle/_ref/libmatchamg_ref.so) so that Python tests, the golden-fixture
// generator and bench.py's reference / cpu_baseline legs can call the
// reference's own public API (proj/include/matchamg/*.hpp) through ctypes.
//
// Every entry point catches the reference's exceptions and turns them into a
// status code + message, mirroring the reference's exception classes:
//   0 ok, 1 std::invalid_argument, 2 std::runtime_error, 3 BreakdownError.

#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

#include "matchamg/coarsening.hpp"
#include "matchamg/csr.hpp"
#include "matchamg/kernels.hpp"
#include "matchamg/matrix_market.hpp"
#include "matchamg/krylov.hpp"
#include "matchamg/matching.hpp"
#include "matchamg/multigrid.hpp"
#include "matchamg/problems.hpp"
#include "matchamg/vector_ops.hpp"

using namespace matchamg;

namespace {

thread_local std::string g_err;
thread_local int64_t g_err_iter = -1;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const BreakdownError& e) {
        g_err = e.what();
        g_err_iter = e.iteration();
        return 3;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}

CsrMatrix* as_csr(void* p) { return static_cast<CsrMatrix*>(p); }
const CsrMatrix* as_csr(const void* p) { return static_cast<const CsrMatrix*>(p); }

struct StepBox {
    CoarseningStep step;
};

CycleConfig make_cycle(int cycle, int pre, int post, int coarsest) {
    CycleConfig c;
    c.cycle = cycle == 1 ? CycleType::W : CycleType::V;
    c.pre_sweeps = pre;
    c.post_sweeps = post;
    c.coarsest_sweeps = coarsest;
    return c;
}

} // namespace

extern "C" {

struct mref_report {
    int64_t iterations;
    double final_relres;
    int32_t converged;
    int32_t pad;
    double solve_ms;
    int64_t audit_checks;
    int64_t audit_failures;
    double audit_max_rel;
    int64_t breakdown_iteration;
};

const char* mref_last_error(void) { return g_err.c_str(); }
int64_t mref_last_error_iteration(void) { return g_err_iter; }

void mref_set_threads(int t) {
#ifdef _OPENMP
    if (t > 0) omp_set_num_threads(t);
#else
    (void)t;
#endif
}

int mref_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

// ---- CsrMatrix handles ----------------------------------------------------
void* mref_csr_from_arrays(int64_t nrows, int64_t ncols, const int64_t* rp,
                           const int64_t* ci, const double* v) {
    auto* A = new CsrMatrix;
    A->nrows = nrows;
    A->ncols = ncols;
    A->row_ptr.assign(rp, rp + nrows + 1);
    const int64_t nnz = rp[nrows];
    A->col_idx.assign(ci, ci + nnz);
    A->values.assign(v, v + nnz);
    return A;
}

void* mref_csr_from_triplets(int64_t nrows, int64_t ncols, int64_t nt,
                             const int64_t* r, const int64_t* c,
                             const double* v) {
    void* out = nullptr;
    const int st = guarded([&] {
        std::vector<Triplet> t(nt);
        for (int64_t k = 0; k < nt; ++k) t[k] = Triplet{r[k], c[k], v[k]};
        out = new CsrMatrix(CsrMatrix::from_triplets(nrows, ncols, std::move(t)));
    });
    return st == 0 ? out : nullptr;
}

void mref_csr_free(void* A) { delete as_csr(A); }

void mref_csr_shape(const void* A, int64_t* nrows, int64_t* ncols, int64_t* nnz) {
    *nrows = as_csr(A)->nrows;
    *ncols = as_csr(A)->ncols;
    *nnz = as_csr(A)->nnz();
}

void mref_csr_export(const void* A, int64_t* rp, int64_t* ci, double* v) {
    const CsrMatrix& M = *as_csr(A);
    std::memcpy(rp, M.row_ptr.data(), sizeof(int64_t) * M.row_ptr.size());
    std::memcpy(ci, M.col_idx.data(), sizeof(int64_t) * M.col_idx.size());
    std::memcpy(v, M.values.data(), sizeof(double) * M.values.size());
}

int mref_csr_validate(const void* A) { return guarded([&] { as_csr(A)->validate(); }); }

// ---- generators (proj/src/problems.cpp) -----------------------------------
void* mref_gen_poisson2d(int64_t nx, int64_t ny) {
    void* out = nullptr;
    guarded([&] { out = new CsrMatrix(gen_poisson_2d(nx, ny)); });
    return out;
}

void* mref_gen_aniso2d(int64_t nx, int64_t ny, double eps, double theta) {
    void* out = nullptr;
    guarded([&] {
        AniSpec s;
        s.nx = nx;
        s.ny = ny;
        s.epsilon = eps;
        s.theta = theta;
        out = new CsrMatrix(gen_anisotropic_2d(s));
    });
    return out;
}

void* mref_gen_randk3d(int64_t nx, int64_t ny, int64_t nz, double sigma,
                       uint64_t seed) {
    void* out = nullptr;
    guarded([&] {
        RandPermSpec s;
        s.nx = nx;
        s.ny = ny;
        s.nz = nz;
        s.sigma = sigma;
        s.seed = seed;
        out = new CsrMatrix(gen_poisson_3d_randk(s));
    });
    return out;
}

// ---- MatrixMarket I/O (proj/src/matrix_market.cpp) --------------------------
void* mref_read_mm(const char* path) {
    void* out = nullptr;
    guarded([&] { out = new CsrMatrix(read_matrix_market(path)); });
    return out;
}

int mref_write_mm(const void* A, const char* path, int symmetric) {
    return guarded([&] { write_matrix_market(*as_csr(A), path, symmetric != 0); });
}

// ---- sparse kernels (proj/src/kernels.cpp, csr.cpp) -----------------------
int mref_lane_policy(const void* A) {
    return LaneGroupPolicy::for_matrix(*as_csr(A)).group_size;
}

int mref_spmv(const void* A, int group, const double* x, double* y) {
    return guarded([&] {
        const CsrMatrix& M = *as_csr(A);
        std::span<const double> xs(x, M.ncols);
        std::span<double> ys(y, M.nrows);
        if (group <= 0)
            spmv_into(M, xs, ys);
        else
            spmv_into(M, xs, ys, LaneGroupPolicy::fixed(group));
    });
}

int mref_l1_diagonal(const void* A, double* d) {
    return guarded([&] {
        const std::vector<double> r = l1_diagonal(*as_csr(A));
        std::memcpy(d, r.data(), sizeof(double) * r.size());
    });
}

int mref_diagonal(const void* A, double* d) {
    return guarded([&] {
        const std::vector<double> r = diagonal(*as_csr(A));
        std::memcpy(d, r.data(), sizeof(double) * r.size());
    });
}

int mref_has_symmetric_pattern(const void* A) {
    return has_symmetric_pattern(*as_csr(A)) ? 1 : 0;
}

int mref_transpose(const void* A, void** out) {
    return guarded([&] { *out = new CsrMatrix(transpose(*as_csr(A))); });
}

int mref_spgemm(const void* A, const void* B, void** out) {
    return guarded([&] { *out = new CsrMatrix(spgemm(*as_csr(A), *as_csr(B))); });
}

int mref_galerkin_triple(const void* A, const void* P, void** out) {
    return guarded(
        [&] { *out = new CsrMatrix(galerkin_triple(*as_csr(A), *as_csr(P))); });
}

// ---- matching (proj/src/matching.cpp) -------------------------------------
// Graph arrays are caller-owned; capacity of adjncy/weight must be >= nnz(A).
int mref_build_weights(const void* A, const double* w, int64_t* xadj,
                       int64_t* adjncy, double* weight, int64_t* zero_edges) {
    return guarded([&] {
        const CsrMatrix& M = *as_csr(A);
        const WeightedGraph G = build_weights(M, std::span<const double>(w, M.nrows));
        std::memcpy(xadj, G.xadj.data(), sizeof(int64_t) * G.xadj.size());
        std::memcpy(adjncy, G.adjncy.data(), sizeof(int64_t) * G.adjncy.size());
        std::memcpy(weight, G.weight.data(), sizeof(double) * G.weight.size());
        *zero_edges = G.zero_weight_edges;
    });
}

static WeightedGraph graph_from(int64_t n, const int64_t* xadj,
                                const int64_t* adjncy, const double* weight) {
    WeightedGraph G;
    G.n = n;
    G.xadj.assign(xadj, xadj + n + 1);
    G.adjncy.assign(adjncy, adjncy + xadj[n]);
    G.weight.assign(weight, weight + xadj[n]);
    return G;
}

int mref_suitor(int64_t n, const int64_t* xadj, const int64_t* adjncy,
                const double* weight, int64_t* mate) {
    return guarded([&] {
        const Matching M = suitor_match(graph_from(n, xadj, adjncy, weight));
        std::memcpy(mate, M.mate.data(), sizeof(int64_t) * n);
    });
}

int mref_exact_match(int64_t n, const int64_t* xadj, const int64_t* adjncy,
                     const double* weight, int64_t* mate) {
    return guarded([&] {
        const Matching M = exact_match_oracle(graph_from(n, xadj, adjncy, weight));
        std::memcpy(mate, M.mate.data(), sizeof(int64_t) * n);
    });
}

double mref_matching_weight(int64_t n, const int64_t* xadj, const int64_t* adjncy,
                            const double* weight, const int64_t* mate) {
    Matching M;
    M.mate.assign(mate, mate + n);
    return matching_weight(graph_from(n, xadj, adjncy, weight), M);
}

// ---- coarsening (proj/src/coarsening.cpp) ---------------------------------
int mref_pairwise_aggregate(int64_t n, const int64_t* mate, int64_t* agg_of,
                            int64_t* counts /* n_c, n_p, n_s */) {
    return guarded([&] {
        Matching M;
        M.mate.assign(mate, mate + n);
        const Aggregation a = pairwise_aggregate(M, n);
        std::memcpy(agg_of, a.agg_of.data(), sizeof(int64_t) * n);
        counts[0] = a.n_c;
        counts[1] = a.n_p;
        counts[2] = a.n_s;
    });
}

int mref_build_prolongator(int64_t n, int64_t n_c, const int64_t* agg_of,
                           const double* w, void** out) {
    return guarded([&] {
        Aggregation a;
        a.agg_of.assign(agg_of, agg_of + n);
        a.n_c = n_c;
        *out = new CsrMatrix(build_prolongator(a, std::span<const double>(w, n)));
    });
}

int mref_restrict_vector(const void* P, const double* w, double* wc) {
    return guarded([&] {
        const CsrMatrix& M = *as_csr(P);
        const std::vector<double> r =
            restrict_vector(M, std::span<const double>(w, M.nrows));
        std::memcpy(wc, r.data(), sizeof(double) * r.size());
    });
}

int mref_galerkin_by_aggregates(const void* A, const void* P, void** out) {
    return guarded([&] {
        *out = new CsrMatrix(galerkin_by_aggregates(*as_csr(A), *as_csr(P)));
    });
}

// mode 1 = pairwise_step, 2 = double_pairwise
int mref_coarsen_step(const void* A, const double* w, int mode, void** out) {
    return guarded([&] {
        const CsrMatrix& M = *as_csr(A);
        std::span<const double> ws(w, M.nrows);
        auto* box = new StepBox;
        box->step = mode == 2 ? double_pairwise(M, ws) : pairwise_step(M, ws);
        *out = box;
    });
}
const void* mref_step_P(const void* s) { return &static_cast<const StepBox*>(s)->step.P; }
const void* mref_step_Ac(const void* s) { return &static_cast<const StepBox*>(s)->step.A_coarse; }
void mref_step_wc(const void* s, double* wc) {
    const auto& v = static_cast<const StepBox*>(s)->step.w_coarse;
    std::memcpy(wc, v.data(), sizeof(double) * v.size());
}
int64_t mref_step_zero_edges(const void* s) {
    return static_cast<const StepBox*>(s)->step.zero_weight_edges;
}
void mref_step_free(void* s) { delete static_cast<StepBox*>(s); }

// mode 1 = Pairwise, 2 = DoublePairwise; w == NULL means ones
int mref_build_hierarchy(const void* A, const double* w, int max_levels,
                         double coarse_factor, int mode, void** out,
                         double* setup_ms) {
    return guarded([&] {
        const CsrMatrix& M = *as_csr(A);
        SetupConfig cfg;
        cfg.max_levels = max_levels;
        cfg.coarse_factor = coarse_factor;
        cfg.aggregation =
            mode == 1 ? AggregationMode::Pairwise : AggregationMode::DoublePairwise;
        std::vector<double> wv = w ? std::vector<double>(w, w + M.nrows)
                                   : std::vector<double>(M.nrows, 1.0);
        const auto t0 = std::chrono::steady_clock::now();
        auto* h = new Hierarchy(build_hierarchy(M, wv, cfg));
        if (setup_ms)
            *setup_ms = std::chrono::duration<double, std::milli>(
                            std::chrono::steady_clock::now() - t0)
                            .count();
        *out = h;
    });
}

void mref_hier_free(void* h) { delete static_cast<Hierarchy*>(h); }
int mref_hier_nl(const void* h) { return static_cast<const Hierarchy*>(h)->nl(); }
const void* mref_hier_A(const void* h, int k) {
    return &static_cast<const Hierarchy*>(h)->levels[k].A;
}
const void* mref_hier_P(const void* h, int k) {
    return &static_cast<const Hierarchy*>(h)->levels[k].P;
}
const void* mref_hier_R(const void* h, int k) {
    return &static_cast<const Hierarchy*>(h)->levels[k].R;
}
void mref_hier_l1(const void* h, int k, double* out) {
    const auto& v = static_cast<const Hierarchy*>(h)->levels[k].l1_diag;
    std::memcpy(out, v.data(), sizeof(double) * v.size());
}
void mref_hier_w(const void* h, int k, double* out) {
    const auto& v = static_cast<const Hierarchy*>(h)->levels[k].w;
    std::memcpy(out, v.data(), sizeof(double) * v.size());
}
void mref_hier_stats(const void* h, int32_t* stalled, int64_t* zero_edges,
                     double* opcx, double* cratio) {
    const Hierarchy& H = *static_cast<const Hierarchy*>(h);
    *stalled = H.stats.stalled ? 1 : 0;
    *zero_edges = H.stats.zero_weight_edges;
    const HierarchySummary s = hierarchy_stats(H);
    *opcx = s.operator_complexity;
    *cratio = s.coarsening_ratio;
}

// Assemble a reference Hierarchy from given levels (partition-aware oracle:
// levels built by composing the reference's own functions). A/P/R handles
// are copied; l1 and w arrays hold the level sizes.
int mref_hier_from_levels(int nl, void* const* A, void* const* P, void* const* R,
                          const double* const* l1, const double* const* w, void** out) {
    return guarded([&] {
        auto* h = new Hierarchy;
        for (int k = 0; k < nl; ++k) {
            Level L;
            L.A = *as_csr(A[k]);
            if (k + 1 < nl) {
                L.P = *as_csr(P[k]);
                L.R = *as_csr(R[k]);
            }
            const auto n = static_cast<std::size_t>(L.A.nrows);
            L.l1_diag.assign(l1[k], l1[k] + n);
            L.w.assign(w[k], w[k] + n);
            h->levels.push_back(std::move(L));
        }
        for (const Level& lvl : h->levels) {
            h->stats.level_size.push_back(lvl.A.nrows);
            h->stats.level_nnz.push_back(lvl.A.nnz());
        }
        *out = h;
    });
}

// ---- multigrid (proj/src/multigrid.cpp) -----------------------------------
int mref_l1_jacobi(const void* A, const double* d, const double* b, double* x,
                   int k) {
    return guarded([&] {
        const CsrMatrix& M = *as_csr(A);
        const auto n = static_cast<std::size_t>(M.nrows);
        l1_jacobi_sweeps(M, std::span<const double>(d, n),
                         std::span<const double>(b, n), std::span<double>(x, n), k);
    });
}

int mref_apply_cycle(const void* h, int level, const double* b, double* x,
                     int cycle, int pre, int post, int coarsest) {
    return guarded([&] {
        const Hierarchy& H = *static_cast<const Hierarchy*>(h);
        const CycleConfig cfg = make_cycle(cycle, pre, post, coarsest);
        cfg.validate();
        CycleWorkspace ws(H);
        const auto n = static_cast<std::size_t>(H.levels.at(level).A.nrows);
        apply_cycle(H, level, std::span<const double>(b, n), std::span<double>(x, n),
                    cfg, ws);
    });
}

int mref_precond_apply(const void* h, int cycle, int pre, int post, int coarsest,
                       const double* r, double* z) {
    return guarded([&] {
        const Hierarchy& H = *static_cast<const Hierarchy*>(h);
        MultigridPreconditioner M(H, make_cycle(cycle, pre, post, coarsest));
        const auto n = static_cast<std::size_t>(H.levels[0].A.nrows);
        M.apply(std::span<const double>(r, n), std::span<double>(z, n));
    });
}

// ---- Krylov (proj/src/krylov.cpp) -----------------------------------------
// h == NULL runs unpreconditioned CG; u0 == NULL is the zero guess; hist must
// hold itmax + 1 doubles.
int mref_pcg(const void* A, const void* h, int cycle, int pre, int post,
             int coarsest, const double* b, const double* u0, double rtol,
             int64_t itmax, double* u, double* hist, mref_report* rep) {
    std::memset(rep, 0, sizeof(*rep));
    rep->breakdown_iteration = -1;
    const int st = guarded([&] {
        const CsrMatrix& M = *as_csr(A);
        const auto n = static_cast<std::size_t>(M.nrows);
        SolveConfig sc;
        sc.rtol = rtol;
        sc.itmax = itmax;
        PrecondFn B;
        std::unique_ptr<MultigridPreconditioner> mg;
        if (h) {
            mg = std::make_unique<MultigridPreconditioner>(
                *static_cast<const Hierarchy*>(h), make_cycle(cycle, pre, post, coarsest));
            B = [&](std::span<const double> r, std::span<double> z) { mg->apply(r, z); };
        }
        std::vector<double> zero;
        std::span<const double> u0s;
        if (u0) {
            u0s = std::span<const double>(u0, n);
        } else {
            zero.assign(n, 0.0);
            u0s = zero;
        }
        auto [sol, r] = pcg_solve(M, B, std::span<const double>(b, n), u0s, sc);
        std::memcpy(u, sol.data(), sizeof(double) * n);
        std::memcpy(hist, r.residual_history.data(),
                    sizeof(double) * r.residual_history.size());
        rep->iterations = r.iterations;
        rep->final_relres = r.final_relres;
        rep->converged = r.converged ? 1 : 0;
        rep->solve_ms = r.solve_ms;
        rep->audit_checks = r.audit_checks;
        rep->audit_failures = r.audit_failures;
        rep->audit_max_rel = r.audit_max_rel;
    });
    if (st == 3) rep->breakdown_iteration = g_err_iter;
    return st;
}

// cli::run_solve (proj/src/cli.cpp:242-328) on a matrix already held by the
// reference (no marshalling inside the timers): w = b = ones, setup_ms = wall
// time around build_hierarchy (cli.cpp:273-275), solve_ms = the reference's
// own SolveReport::solve_ms (krylov.cpp:54-64); wall_ms also counts the
// MultigridPreconditioner construction. u may be NULL.
int mref_run_solve(const void* A, int threads, int max_levels, double coarse_factor, int mode,
                   int cycle, int pre, int post, int coarsest, double rtol, int64_t itmax,
                   double* setup_ms, double* solve_ms, double* wall_ms, int64_t* iterations,
                   double* relres, int* nl, double* u) {
    return guarded([&] {
        mref_set_threads(threads);
        const CsrMatrix& M = *as_csr(A);
        const std::vector<double> w(static_cast<std::size_t>(M.nrows), 1.0);
        SetupConfig setup;
        setup.max_levels = max_levels;
        setup.coarse_factor = coarse_factor;
        setup.aggregation = mode == 1 ? AggregationMode::Pairwise : AggregationMode::DoublePairwise;
        const auto t0 = std::chrono::steady_clock::now();
        Hierarchy h = build_hierarchy(M, w, setup);
        const auto t1 = std::chrono::steady_clock::now();
        CycleConfig cyc = make_cycle(cycle, pre, post, coarsest);
        SolveConfig sc;
        sc.rtol = rtol;
        sc.itmax = itmax;
        const std::vector<double> b(static_cast<std::size_t>(M.nrows), 1.0);
        cyc.validate();
        sc.validate();
        MultigridPreconditioner precond(h, cyc);
        auto result = pcg_solve(
            M, [&precond](std::span<const double> r, std::span<double> z) { precond.apply(r, z); },
            b, sc);
        const auto t2 = std::chrono::steady_clock::now();
        *setup_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
        *solve_ms = result.second.solve_ms;
        *wall_ms = std::chrono::duration<double, std::milli>(t2 - t0).count();
        *iterations = result.second.iterations;
        *relres = result.second.final_relres;
        *nl = h.nl();
        if (u) std::memcpy(u, result.first.data(), sizeof(double) * result.first.size());
    });
}

// ---- vector ops (proj/src/vector_ops.cpp) ---------------------------------
double mref_dot(int64_t n, const double* x, const double* y) {
    return dot(std::span<const double>(x, n), std::span<const double>(y, n));
}
double mref_norm2(int64_t n, const double* x) {
    return norm2(std::span<const double>(x, n));
}
void mref_axpy(int64_t n, double* y, double a, const double* x) {
    axpy(std::span<double>(y, n), a, std::span<const double>(x, n));
}
void mref_triple_dot(int64_t n, const double* w, const double* r, const double* v,
                     const double* q, double* out3) {
    const TripleDot t = fused_triple_dot(
        std::span<const double>(w, n), std::span<const double>(r, n),
        std::span<const double>(v, n), std::span<const double>(q, n));
    out3[0] = t.wr;
    out3[1] = t.wv;
    out3[2] = t.wq;
}
void mref_axpy_pair(int64_t n, double* y1, double* y2, const double* x, double a,
                    double b) {
    fused_axpy_pair(std::span<double>(y1, n), std::span<double>(y2, n),
                    std::span<const double>(x, n), a, b);
}

} // extern "C"
