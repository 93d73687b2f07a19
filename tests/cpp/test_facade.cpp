// test_facade.cpp — the reference's own test idioms (proj/tests/*.cpp),
// compiled against OUR include/matchamg/*.hpp and linked only with
// libmatchamg.so + libmamg_cuda.so: source written for the reference builds
// unchanged and produces the reference's known answers on the B200.
// Run by tests/test_cpp_facade.py (-m gpu). Prints one line per check.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <algorithm>
#include <tuple>
#include <vector>

#include "matchamg/coarsening.hpp"
#include "matchamg/csr.hpp"
#include "matchamg/kernels.hpp"
#include "matchamg/krylov.hpp"
#include "matchamg/matching.hpp"
#include "matchamg/matrix_market.hpp"
#include "matchamg/multigrid.hpp"
#include "matchamg/problems.hpp"
#include "matchamg/vector_ops.hpp"

using namespace matchamg;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                                               \
    do {                                                                          \
        if (cond) {                                                               \
            ++g_pass;                                                             \
        } else {                                                                  \
            ++g_fail;                                                             \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);           \
        }                                                                         \
    } while (0)

template <class E, class F>
static std::string throws(F&& f) {
    try {
        f();
    } catch (const E& e) {
        return e.what();
    } catch (...) {
        return "<other exception>";
    }
    return "<no exception>";
}

static CsrMatrix small_2x2() {
    return CsrMatrix::from_triplets(2, 2, {{0, 0, 2.0}, {0, 1, -1.0}, {1, 0, -1.0}, {1, 1, 2.0}});
}

static CsrMatrix poisson_1d(index_t n) {
    std::vector<Triplet> t;
    for (index_t i = 0; i < n; ++i) {
        if (i > 0) t.push_back({i, i - 1, -1.0});
        t.push_back({i, i, 2.0});
        if (i + 1 < n) t.push_back({i, i + 1, -1.0});
    }
    return CsrMatrix::from_triplets(n, n, std::move(t));
}

int main() {
    std::setvbuf(stdout, nullptr, _IONBF, 0);
    // --- sparse core (test_sparse_core.cpp) ---
    {
        const CsrMatrix I = CsrMatrix::identity(3);
        CHECK((spmv(I, std::vector<double>{1.0, 2.0, 3.0}) == std::vector<double>{1.0, 2.0, 3.0}));
        CHECK((spmv(small_2x2(), std::vector<double>{1.0, 1.0}) == std::vector<double>{1.0, 1.0}));
        for (int g : LaneGroupPolicy::kAdmissible)
            CHECK((spmv(small_2x2(), std::vector<double>{1.0, 1.0}, LaneGroupPolicy::fixed(g)) ==
                   std::vector<double>{1.0, 1.0}));
        CHECK(throws<std::invalid_argument>([] { LaneGroupPolicy::fixed(3); }) != "<no exception>");
        CHECK(throws<std::invalid_argument>([] { spmv(small_2x2(), std::vector<double>(3, 0.0)); }) ==
              "spmv: x has 3 entries, A has 2 columns");
        CHECK((l1_diagonal(small_2x2()) == std::vector<double>{3.0, 3.0}));
        CHECK((l1_diagonal(poisson_1d(5)) == std::vector<double>{3.0, 4.0, 4.0, 4.0, 3.0}));
        const CsrMatrix Z = CsrMatrix::from_triplets(
            2, 2, {{0, 0, 1.0}, {0, 1, 1.0}, {1, 0, 1.0}, {1, 1, 0.0}});
        CHECK(throws<std::invalid_argument>([&] { l1_diagonal(Z); }) ==
              "l1_diagonal: zero or missing diagonal entry in row 1");
        const CsrMatrix T = transpose(transpose(poisson_1d(7)));
        CHECK(T.col_idx == poisson_1d(7).col_idx && T.values == poisson_1d(7).values);
        CHECK(has_symmetric_pattern(poisson_1d(9)));
    }
    // --- matching (test_matching.cpp) ---
    {
        const WeightedGraph G = build_weights(small_2x2(), std::vector<double>{1.0, 1.0});
        CHECK(G.xadj[2] == 2 && G.weight[0] == 1.5 && G.weight[1] == 1.5 && G.zero_weight_edges == 0);
        WeightedGraph path;
        path.n = 3;
        path.xadj = {0, 1, 3, 4};
        path.adjncy = {1, 0, 2, 1};
        path.weight = {1.0, 1.0, 2.0, 2.0};
        const Matching M = suitor_match(path);
        CHECK((M.mate == std::vector<index_t>{kUnmatched, 2, 1}));
        CHECK(std::abs(matching_weight(path, M) - 2.0) < 1e-15);
        CHECK(std::abs(matching_weight(path, exact_match_oracle(path)) - 2.0) < 1e-15);
        CHECK(M.is_valid() && M.matched_vertices() == 2);
        // exact oracle hand cases (test_matching.cpp:162-182)
        auto from_edges = [](index_t n, std::vector<std::tuple<index_t, index_t, double>> e) {
            std::vector<std::vector<std::pair<index_t, double>>> adj(n);
            for (auto [u, v, w] : e) {
                adj[u].push_back({v, w});
                adj[v].push_back({u, w});
            }
            WeightedGraph g;
            g.n = n;
            g.xadj.assign(n + 1, 0);
            for (index_t u = 0; u < n; ++u) {
                std::sort(adj[u].begin(), adj[u].end());
                for (auto [v, w] : adj[u]) {
                    g.adjncy.push_back(v);
                    g.weight.push_back(w);
                }
                g.xadj[u + 1] = static_cast<index_t>(g.adjncy.size());
            }
            return g;
        };
        const WeightedGraph tri = from_edges(3, {{0, 1, 3.0}, {1, 2, 2.0}, {0, 2, 1.0}});
        CHECK(matching_weight(tri, exact_match_oracle(tri)) == 3.0);
        const WeightedGraph empty = from_edges(4, {});
        CHECK(exact_match_oracle(empty).matched_vertices() == 0);
        const WeightedGraph cyc = from_edges(4, {{0, 1, 1.0}, {1, 2, 1.0}, {2, 3, 1.0}, {0, 3, 1.0}});
        CHECK(matching_weight(cyc, exact_match_oracle(cyc)) == 2.0);
        // a heavy middle edge loses to the two outer ones: 2 + 2 > 3
        const WeightedGraph p4 = from_edges(4, {{0, 1, 2.0}, {1, 2, 3.0}, {2, 3, 2.0}});
        const Matching E4 = exact_match_oracle(p4);
        CHECK(E4.is_valid() && matching_weight(p4, E4) == 4.0 && E4.mate[1] == 0);
        // exact >= suitor >= exact / 2 on a random graph of 18 vertices
        {
            std::vector<std::tuple<index_t, index_t, double>> e;
            uint64_t st = 12345;
            auto rnd = [&st] {
                st = st * 6364136223846793005ull + 1442695040888963407ull;
                return static_cast<double>(st >> 11) * (1.0 / 9007199254740992.0);
            };
            for (index_t u = 0; u < 18; ++u)
                for (index_t v = u + 1; v < 18; ++v)
                    if (rnd() < 0.3) e.push_back({u, v, 0.1 + rnd()});
            const WeightedGraph g = from_edges(18, e);
            const double ex = matching_weight(g, exact_match_oracle(g));
            const double su = matching_weight(g, suitor_match(g));
            CHECK(exact_match_oracle(g).is_valid() && ex >= su - 1e-12 && su >= 0.5 * ex - 1e-12);
        }
        WeightedGraph big;
        big.n = 21;
        big.xadj.assign(22, 0);
        bool threw = false;
        try {
            exact_match_oracle(big);
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        CHECK(threw);
    }
    // --- coarsening (test_coarsening.cpp) ---
    {
        Matching m;
        m.mate = {kUnmatched, 2, 1, kUnmatched};
        const Aggregation a = pairwise_aggregate(m, 4);
        CHECK((a.agg_of == std::vector<index_t>{0, 1, 1, 2}) && a.n_c == 3 && a.n_p == 1 && a.n_s == 2);
        Aggregation pair;
        pair.agg_of = {0, 0};
        pair.n_c = 1;
        pair.n_p = 1;
        const CsrMatrix P = build_prolongator(pair, std::vector<double>{1.0, 1.0});
        CHECK(std::abs(P.values[0] - 1.0 / std::sqrt(2.0)) < 1e-15);
        CHECK(throws<std::invalid_argument>([&] {
                  build_prolongator(pair, std::vector<double>{0.0, 0.0});
              }) == "build_prolongator: smooth vector vanishes on aggregate 0");
        CHECK(std::abs(restrict_vector(P, std::vector<double>{1.0, 1.0})[0] - std::sqrt(2.0)) < 1e-15);
        const CsrMatrix Ac = galerkin_by_aggregates(small_2x2(), P);
        CHECK(Ac.nrows == 1 && std::abs(Ac.values[0] - 1.0) < 1e-15);
        const CsrMatrix A64 = gen_poisson_2d(64, 64);
        const Hierarchy h = build_hierarchy(A64, SetupConfig{});
        CHECK(h.nl() >= 3 && h.nl() <= 4 && h.device != nullptr);
        const HierarchySummary s = hierarchy_stats(h);
        CHECK(s.operator_complexity > 1.0 && s.operator_complexity < 1.7);
        for (int k = 0; k + 1 < h.nl(); ++k) {
            const CsrMatrix PtP = spgemm(transpose(h.levels[k].P), h.levels[k].P);
            double err = 0.0;
            for (index_t i = 0; i < PtP.nrows; ++i)
                for (index_t q = PtP.row_begin(i); q < PtP.row_end(i); ++q)
                    err = std::max(err, std::abs(PtP.values[q] - (PtP.col_idx[q] == i ? 1.0 : 0.0)));
            CHECK(err <= 1e-13);
        }
        std::vector<Triplet> dt;
        for (index_t i = 0; i < 300; ++i) dt.push_back({i, i, 1.0 + i});
        const Hierarchy hd = build_hierarchy(CsrMatrix::from_triplets(300, 300, dt), SetupConfig{});
        CHECK(hd.stats.stalled && hd.nl() == 1);
        const CsrMatrix asym = CsrMatrix::from_triplets(2, 2, {{0, 0, 2.0}, {0, 1, 1.0}, {1, 1, 2.0}});
        CHECK(throws<std::invalid_argument>([&] { build_hierarchy(asym, SetupConfig{}); }) ==
              "build_hierarchy: matrix pattern is not symmetric");
    }
    // --- multigrid + krylov (test_multigrid.cpp, test_krylov.cpp) ---
    {
        const TripleDot t = fused_triple_dot(std::vector<double>{1, 2, 3}, std::vector<double>{2, 3, 1},
                                             std::vector<double>{3, 4, 2}, std::vector<double>{4, 5, 3});
        CHECK(t.wr == 11.0 && t.wv == 17.0 && t.wq == 23.0);
        std::vector<double> x{0.0, 0.0};
        l1_jacobi_sweeps(small_2x2(), std::vector<double>{3.0, 3.0}, std::vector<double>{1.0, 1.0}, x, 1);
        CHECK(std::abs(x[0] - 1.0 / 3.0) < 1e-16 && std::abs(x[1] - 1.0 / 3.0) < 1e-16);

        const CsrMatrix A = gen_poisson_2d(64, 64);
        const Hierarchy h = build_hierarchy(A, SetupConfig{});
        MultigridPreconditioner M(h, CycleConfig{});
        const std::vector<double> b(A.nrows, 1.0);
        // the reference idiom: a host lambda (staged through the host)
        auto [u1, r1] = pcg_solve(A, [&](std::span<const double> r, std::span<double> z) { M.apply(r, z); },
                                  b, SolveConfig{});
        // the device-resident form
        auto [u2, r2] = pcg_solve(A, device_precond(M), b, SolveConfig{});
        CHECK(r1.converged && r2.converged && r1.iterations < 50 && r1.audit_failures == 0);
        CHECK(r1.iterations == r2.iterations && r1.residual_history == r2.residual_history && u1 == u2);
        std::printf("info poisson64 iterations=%lld relres=%.6e\n",
                    static_cast<long long>(r2.iterations), r2.final_relres);
        // a host-built hierarchy (no device twin) goes through an upload
        Hierarchy hc = h;
        hc.device.reset();
        MultigridPreconditioner M2(hc, CycleConfig{});
        auto [u3, r3] = pcg_solve(A, device_precond(M2), b, SolveConfig{});
        CHECK(u3 == u2);
        // W-cycle and vcycle/wcycle wrappers
        CycleConfig wc;
        wc.cycle = CycleType::W;
        const std::vector<double> zv = vcycle(h, 0, b, std::vector<double>(A.nrows, 0.0), CycleConfig{});
        std::vector<double> zp(A.nrows);
        M.apply(b, zp);
        CHECK(zv == zp);
        const std::vector<double> zw = wcycle(h, 0, b, std::vector<double>(A.nrows, 0.0), wc);
        CHECK(zw.size() == static_cast<size_t>(A.nrows));
        // degenerate cases
        auto [ui, ri] = pcg_solve(CsrMatrix::identity(4), PrecondFn{}, std::vector<double>{1, 2, 3, 4}, SolveConfig{});
        CHECK(ri.iterations == 1 && ri.converged);
        auto [u0, r0] = pcg_solve(A, PrecondFn{}, std::vector<double>(A.nrows, 0.0), SolveConfig{});
        CHECK(r0.iterations == 0 && r0.converged && r0.residual_history == std::vector<double>{0.0});
        const CsrMatrix D = CsrMatrix::from_triplets(3, 3, {{0, 0, 1.0}, {1, 1, -1.0}, {2, 2, 2.0}});
        index_t bd_it = -1;
        try {
            pcg_solve(D, PrecondFn{}, std::vector<double>{1.0, 1.0, 0.0}, SolveConfig{});
        } catch (const BreakdownError& e) {
            bd_it = e.iteration();
            CHECK(std::string(e.what()).rfind("pcg breakdown at iteration 0: rho_0 = ", 0) == 0);
        }
        CHECK(bd_it == 0);
        SolveConfig bad;
        bad.rtol = 0.0;
        CHECK(throws<std::invalid_argument>([&] { bad.validate(); }) == "SolveConfig: rtol must be > 0");
    }
    // --- problems (test_problems_io.cpp) ---
    {
        const CsrMatrix R = gen_poisson_3d_randk({8, 8, 8, 0.0, 0});
        CHECK(R.nrows == 512 && R.nnz() == 512 * 7 - 6 * 64);
        CHECK(has_symmetric_pattern(R) && symmetry_gap(R) == 0.0);
        // MatrixMarket round trip (test_problems_io.cpp:184-211), symmetric storage
        const std::string path = "/tmp/mamg_facade_rt.mtx";
        write_matrix_market(R, path, /*symmetric=*/true);
        const CsrMatrix Q = read_matrix_market(path);
        CHECK(Q.row_ptr == R.row_ptr && Q.col_idx == R.col_idx && Q.values == R.values);
        std::remove(path.c_str());
        CHECK(throws<std::runtime_error>([&] { read_matrix_market("/nonexistent/missing.mtx"); })
                  .rfind("cannot open matrix file", 0) == 0);
        // BASELINE cfg 3-5 generators: symmetric patterns, expected sizes
        const CsrMatrix Q1 = gen_anisotropic_3d_q1({6, 6, 6, 1.0, 1.0, 1e-2});
        const CsrMatrix J = gen_jump_3d({8, 8, 8, 4, 1, 1e-3, 1e3});
        const CsrMatrix E = gen_elasticity_3d({4, 4, 4, 0.42, 1.7});
        CHECK(Q1.nrows == 216 && J.nrows == 512 && E.nrows == 192);
        CHECK(symmetry_gap(Q1) == 0.0 && symmetry_gap(J) == 0.0 && symmetry_gap(E) == 0.0);
    }
    // --- K-cycle (CycleType::K, the north star's K-cycle driver) ---
    {
        const CsrMatrix A = gen_poisson_2d(128, 128);
        const Hierarchy h = build_hierarchy(A, SetupConfig{});
        CycleConfig kc;
        kc.cycle = CycleType::K;
        MultigridPreconditioner MV(h, CycleConfig{}), MK(h, kc);
        const std::vector<double> b(A.nrows, 1.0);
        auto [uv, rv] = pcg_solve(A, device_precond(MV), b, SolveConfig{});
        auto [uk, rk] = pcg_solve(A, device_precond(MK), b, SolveConfig{});
        CHECK(rv.converged && rk.converged && rk.iterations < rv.iterations);
        std::printf("info poisson128 V iterations=%lld K iterations=%lld\n",
                    static_cast<long long>(rv.iterations), static_cast<long long>(rk.iterations));
    }
    // --- several devices behind the same API (MATCHAMG_DEVICES) ---
    // ranks as threads, here all on device 0 ("0,0", "0,0,0"): the hierarchy
    // (global matching across the parts) and the preconditioned pcg_solve
    // must equal the single-device ones bit for bit
    {
        RandPermSpec rs;
        rs.nx = rs.ny = rs.nz = 24;
        rs.sigma = 1.0;
        const CsrMatrix probs[2] = {gen_poisson_2d(96, 96), gen_poisson_3d_randk(rs)};
        for (const CsrMatrix& A : probs) {
            unsetenv("MATCHAMG_DEVICES");
            const Hierarchy h1 = build_hierarchy(A, SetupConfig{});
            MultigridPreconditioner mg1(h1, CycleConfig{});
            const std::vector<double> b(A.nrows, 1.0);
            const auto r1 = pcg_solve(A, device_precond(mg1), b, SolveConfig{});
            for (const char* devs : {"0,0", "0,0,0"}) {
                setenv("MATCHAMG_DEVICES", devs, 1);
                const Hierarchy hm = build_hierarchy(A, SetupConfig{});
                unsetenv("MATCHAMG_DEVICES");
                bool same = hm.nl() == h1.nl();
                for (int k = 0; same && k < h1.nl(); ++k) {
                    const Level &a = h1.levels[k], &m = hm.levels[k];
                    same = a.A.row_ptr == m.A.row_ptr && a.A.col_idx == m.A.col_idx &&
                           a.A.values == m.A.values && a.l1_diag == m.l1_diag && a.w == m.w;
                    if (same && k + 1 < h1.nl())
                        same = a.P.row_ptr == m.P.row_ptr && a.P.col_idx == m.P.col_idx &&
                               a.P.values == m.P.values && a.R.col_idx == m.R.col_idx &&
                               a.R.values == m.R.values;
                }
                CHECK(same);
                CHECK(hm.device != nullptr);
                MultigridPreconditioner mgm(hm, CycleConfig{});
                const auto rm = pcg_solve(A, device_precond(mgm), b, SolveConfig{});
                CHECK(rm.second.iterations == r1.second.iterations);
                CHECK(rm.first == r1.first);
                CHECK(rm.second.residual_history == r1.second.residual_history);
                // from a nonzero initial guess
                std::vector<double> u0(A.nrows);
                for (index_t i = 0; i < A.nrows; ++i) u0[i] = 0.001 * static_cast<double>(i % 7);
                const auto s1 = pcg_solve(A, device_precond(mg1), b, u0, SolveConfig{});
                const auto sm = pcg_solve(A, device_precond(mgm), b, u0, SolveConfig{});
                CHECK(sm.first == s1.first && sm.second.iterations == s1.second.iterations);
                // a host-callable cycle on the partitioned hierarchy (its single-device copy)
                std::vector<double> z1(A.nrows), zm(A.nrows);
                mg1.apply(b, z1);
                mgm.apply(b, zm);
                CHECK(z1 == zm);
            }
        }
    }
    // --- matrices of 2^31 or more entries: auto-partitioned on one device ---
    // (the cap is lowered here with MATCHAMG_PART_NNZ: ~90k entries -> 3 parts)
    {
        RandPermSpec rs;
        rs.nx = rs.ny = rs.nz = 24;
        rs.sigma = 1.0;
        const CsrMatrix A = gen_poisson_3d_randk(rs);
        unsetenv("MATCHAMG_DEVICES");
        unsetenv("MATCHAMG_PART_NNZ");
        const Hierarchy h1 = build_hierarchy(A, SetupConfig{});
        MultigridPreconditioner mg1(h1, CycleConfig{});
        const std::vector<double> b(A.nrows, 1.0);
        const auto r1 = pcg_solve(A, device_precond(mg1), b, SolveConfig{});
        const std::string cap = std::to_string(A.nnz() / 3 + 1);
        setenv("MATCHAMG_PART_NNZ", cap.c_str(), 1);
        const Hierarchy hp = build_hierarchy(A, SetupConfig{});
        unsetenv("MATCHAMG_PART_NNZ");
        bool same = hp.nl() == h1.nl();
        for (int k = 0; same && k < h1.nl(); ++k)
            same = h1.levels[k].A.col_idx == hp.levels[k].A.col_idx &&
                   h1.levels[k].A.values == hp.levels[k].A.values;
        CHECK(same);
        MultigridPreconditioner mgp(hp, CycleConfig{});
        const auto rp = pcg_solve(A, device_precond(mgp), b, SolveConfig{});
        CHECK(rp.second.iterations == r1.second.iterations && rp.first == r1.first);
    }
    std::printf("facade checks: %d passed, %d failed\n", g_pass, g_fail);
    return g_fail == 0 ? 0 : 1;
}
