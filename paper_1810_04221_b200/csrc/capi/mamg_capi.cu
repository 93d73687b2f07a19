// mamg_capi.cu — the C-ABI of include/mamg_capi.h over the internal sm_100a
// implementation. Each entry point translates internal exceptions into a
// status code + message (the message text follows the reference's exception
// wording, so the C++ facade can rethrow the same std::invalid_argument).
#include <chrono>
#include <exception>
#include <thread>
#include <cstring>
#include <vector>

#include "../device/dist.cuh"
#include "../device/ops.cuh"

struct mamg_ctx {
    mamg::Ctx c;
};
struct mamg_mat {
    std::unique_ptr<mamg::DevCsr> m;
    const mamg::DevCsr* view = nullptr; // borrowed (hierarchy level) when m is empty
    const mamg::DevCsr& get() const { return m ? *m : *view; }
};
struct mamg_dist {
    mamg_ctx* ctx = nullptr;
    std::shared_ptr<mamg::ThreadGroup> group; // keeps a thread group's memory alive
    mamg::DistHier d;
};
struct mamg_group {
    std::shared_ptr<mamg::ThreadGroup> g;
};
struct mamg_graph {
    std::unique_ptr<mamg::DevGraph> g;
};
struct mamg_hier {
    std::unique_ptr<mamg::DevHier> h;
    std::vector<mamg_mat> A, P, R; // borrowed views
    void refresh() {
        const int nl = h->nl();
        A.resize(nl);
        P.resize(nl);
        R.resize(nl);
        for (int k = 0; k < nl; ++k) {
            A[k].view = h->lv[k].A.get();
            P[k].view = h->lv[k].P.get();
            R[k].view = h->lv[k].R.get();
        }
    }
};

namespace {

using mamg::Error;

template <class F>
int guard(mamg_ctx* ctx, F&& f) {
    if (!ctx) return MAMG_INVALID_ARGUMENT;
    // a failed call leaves no deferred value behind: its targets may be gone
    struct DropPending {
        mamg::Ctx& c;
        bool ok = false;
        ~DropPending() {
            if (!ok) {
                c.pending.clear();
                c.defer_used = 0;
            }
        }
    } drop{ctx->c};
    try {
        ctx->c.err.clear();
        ctx->c.err_index = -1;
        MAMG_CU(cudaSetDevice(ctx->c.device));
        f();
        drop.ok = true;
        return MAMG_OK;
    } catch (const Error& e) {
        ctx->c.err = e.what();
        ctx->c.err_index = e.index;
        return e.status;
    } catch (const std::bad_alloc&) {
        ctx->c.err = "out of host memory";
        return MAMG_RUNTIME;
    } catch (const std::exception& e) {
        ctx->c.err = e.what();
        return MAMG_RUNTIME;
    }
}

void need(bool ok, const char* what) {
    if (!ok) mamg::invalid(what);
}

} // namespace

extern "C" {

const char* mamg_version(void) { return "matchamg-b200 0.1 (sm_100a)"; }

int mamg_ctx_create(int device, mamg_ctx** out) {
    if (!out) return MAMG_INVALID_ARGUMENT;
    *out = nullptr;
    auto* ctx = new mamg_ctx;
    ctx->c.device = device;
    try {
        MAMG_CU(cudaSetDevice(device));
        MAMG_CU(cudaStreamCreateWithFlags(&ctx->c.stream, cudaStreamNonBlocking));
        mamg::big_stream_live(ctx->c.stream, true);
        MAMG_CU(cudaDeviceGetAttribute(&ctx->c.num_sms, cudaDevAttrMultiProcessorCount, device));
        // keep freed blocks in the stream-ordered pool across setups
        cudaMemPool_t pool;
        MAMG_CU(cudaDeviceGetDefaultMemPool(&pool, device));
        uint64_t thr = UINT64_MAX;
        MAMG_CU(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
        MAMG_CU(cudaMallocHost(reinterpret_cast<void**>(&ctx->c.h_small), 64 * sizeof(int64_t)));
        ctx->c.d_small.alloc(64, ctx->c.stream);
        MAMG_CU(cudaStreamSynchronize(ctx->c.stream));
    } catch (const std::exception& e) {
        delete ctx;
        return MAMG_CUDA;
    }
    *out = ctx;
    return MAMG_OK;
}

void mamg_ctx_destroy(mamg_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->c.device);
    cudaStreamSynchronize(ctx->c.stream);
    ctx->c.release_scratch();
    if (ctx->c.d_defer) cudaFree(ctx->c.d_defer);
    if (ctx->c.ev_read) cudaEventDestroy(ctx->c.ev_read);
    ctx->c.d_small.release();
    mamg::big_stream_live(ctx->c.stream, false); // frees its cached large blocks
    cudaStreamSynchronize(ctx->c.stream);
    if (ctx->c.staging_free) ctx->c.staging_free(ctx->c.staging);
    if (ctx->c.h_small) cudaFreeHost(ctx->c.h_small);
    cudaStreamDestroy(ctx->c.stream);
    delete ctx;
}

// errors of the context-less entry points (mamg_shm_allgather)
static thread_local std::string g_noctx_err = "no context";
const char* mamg_last_error(const mamg_ctx* ctx) { return ctx ? ctx->c.err.c_str() : g_noctx_err.c_str(); }
int64_t mamg_last_error_index(const mamg_ctx* ctx) { return ctx ? ctx->c.err_index : -1; }
int64_t mamg_kernel_launches(const mamg_ctx* ctx) { return ctx ? ctx->c.launches : 0; }

int mamg_synchronize(mamg_ctx* ctx) {
    return guard(ctx, [&] { ctx->c.sync(); });
}

int mamg_dmalloc(mamg_ctx* ctx, size_t bytes, void** d_out) {
    return guard(ctx, [&] {
        MAMG_CU(cudaMallocAsync(d_out, bytes ? bytes : 8, ctx->c.stream));
        ctx->c.sync();
    });
}
int mamg_dfree(mamg_ctx* ctx, void* d_ptr) {
    return guard(ctx, [&] {
        if (d_ptr) MAMG_CU(cudaFreeAsync(d_ptr, ctx->c.stream));
        ctx->c.sync();
    });
}
int mamg_h2d(mamg_ctx* ctx, void* d_dst, const void* h_src, size_t bytes) {
    return guard(ctx, [&] {
        if (bytes)
            MAMG_CU(cudaMemcpyAsync(d_dst, h_src, bytes, cudaMemcpyHostToDevice, ctx->c.stream));
        ctx->c.sync();
    });
}
int mamg_d2h(mamg_ctx* ctx, void* h_dst, const void* d_src, size_t bytes) {
    return guard(ctx, [&] {
        if (bytes)
            MAMG_CU(cudaMemcpyAsync(h_dst, d_src, bytes, cudaMemcpyDeviceToHost, ctx->c.stream));
        ctx->c.sync();
    });
}

// ---------------------------------------------------------------- matrices --
int mamg_csr_upload(mamg_ctx* ctx, int64_t nrows, int64_t ncols, const int64_t* h_rp,
                    const int64_t* h_ci, const double* h_v, mamg_mat** out) {
    return guard(ctx, [&] {
        need(out && h_rp, "mamg_csr_upload: null argument");
        auto* m = new mamg_mat;
        try {
            m->m = mamg::csr_upload(ctx->c, nrows, ncols, h_rp, h_ci, h_v);
        } catch (...) {
            delete m;
            throw;
        }
        *out = m;
    });
}

// ---- generators assembled on the device (problems.hpp, bit-identical) ----
extern "C++" {
template <class F>
static int gen_into(mamg_ctx* ctx, mamg_mat** out, F&& make) {
    return guard(ctx, [&] {
        need(out != nullptr, "generator: null output");
        auto* m = new mamg_mat;
        try {
            m->m = make();
        } catch (...) {
            delete m;
            throw;
        }
        *out = m;
    });
}
} // extern "C++"

int mamg_gen_poisson2d_dev(mamg_ctx* ctx, int64_t nx, int64_t ny, mamg_mat** out) {
    return gen_into(ctx, out, [&] { return mamg::gen_nine_point_dev(ctx->c, nx, ny, 1.0, 1.0, 0.0); });
}

int mamg_gen_aniso2d_dev(mamg_ctx* ctx, int64_t nx, int64_t ny, double epsilon, double theta,
                         mamg_mat** out) {
    return gen_into(ctx, out, [&] {
        need(epsilon > 0.0, "gen_anisotropic_2d: epsilon must be > 0");
        const double co = std::cos(theta), si = std::sin(theta);
        return mamg::gen_nine_point_dev(ctx->c, nx, ny, epsilon + co * co, epsilon + si * si, co * si);
    });
}

int mamg_gen_randk3d_dev(mamg_ctx* ctx, int64_t nx, int64_t ny, int64_t nz, double sigma,
                         uint64_t seed, mamg_mat** out) {
    return gen_into(ctx, out, [&] { return mamg::gen_randk3d_dev(ctx->c, nx, ny, nz, sigma, seed); });
}

int mamg_gen_jump3d_dev(mamg_ctx* ctx, int64_t nx, int64_t ny, int64_t nz, int64_t block,
                        uint64_t seed, double lo, double hi, mamg_mat** out) {
    return gen_into(ctx, out,
                    [&] { return mamg::gen_jump3d_dev(ctx->c, nx, ny, nz, block, seed, lo, hi); });
}

int mamg_gen_aniso27_dev(mamg_ctx* ctx, int64_t nx, int64_t ny, int64_t nz, double kx, double ky,
                         double kz, mamg_mat** out) {
    return gen_into(ctx, out, [&] { return mamg::gen_aniso27_dev(ctx->c, nx, ny, nz, kx, ky, kz); });
}

int mamg_gen_elast3d_dev(mamg_ctx* ctx, int64_t nx, int64_t ny, int64_t nz, double mu,
                         double lambda, mamg_mat** out) {
    return gen_into(ctx, out, [&] { return mamg::gen_elast3d_dev(ctx->c, nx, ny, nz, mu, lambda); });
}

int mamg_csr_shape(const mamg_mat* A, int64_t* nrows, int64_t* ncols, int64_t* nnz) {
    if (!A) return MAMG_INVALID_ARGUMENT;
    const auto& M = A->get();
    if (nrows) *nrows = M.nrows;
    if (ncols) *ncols = M.ncols;
    if (nnz) *nnz = M.nnz;
    return MAMG_OK;
}

int mamg_csr_download(mamg_ctx* ctx, const mamg_mat* A, int64_t* h_rp, int64_t* h_ci,
                      double* h_v) {
    return guard(ctx, [&] {
        need(A != nullptr, "mamg_csr_download: null matrix");
        mamg::csr_download(ctx->c, A->get(), h_rp, h_ci, h_v);
    });
}

void mamg_mat_destroy(mamg_mat* A) { delete A; }

int mamg_lane_policy(const mamg_mat* A) { return A ? A->get().group : -1; }

int mamg_has_symmetric_pattern(mamg_ctx* ctx, const mamg_mat* A, int* out) {
    return guard(ctx, [&] { *out = mamg::has_symmetric_pattern(ctx->c, A->get()) ? 1 : 0; });
}

int mamg_spmv(mamg_ctx* ctx, const mamg_mat* A, int group, const double* d_x, double* d_y) {
    return guard(ctx, [&] {
        const auto& M = A->get();
        const int G = group <= 0 ? M.group : group;
        if (G != 1 && G != 2 && G != 4 && G != 8 && G != 16 && G != 32)
            mamg::invalid("LaneGroupPolicy: group size " + std::to_string(G) +
                          " not in {1,2,4,8,16,32}");
        mamg::spmv(ctx->c, M, G, d_x, d_y);
        ctx->c.sync();
    });
}

int mamg_l1_diagonal(mamg_ctx* ctx, const mamg_mat* A, double* d_out) {
    return guard(ctx, [&] { mamg::l1_diagonal(ctx->c, A->get(), d_out); });
}

int mamg_transpose(mamg_ctx* ctx, const mamg_mat* A, mamg_mat** out) {
    return guard(ctx, [&] {
        auto* m = new mamg_mat;
        m->m = mamg::transpose(ctx->c, A->get());
        *out = m;
    });
}

int mamg_spgemm(mamg_ctx* ctx, const mamg_mat* A, const mamg_mat* B, mamg_mat** out) {
    return guard(ctx, [&] {
        auto C = mamg::spgemm(ctx->c, A->get(), B->get());
        auto* m = new mamg_mat;
        m->m = std::move(C);
        *out = m;
    });
}

int mamg_galerkin_triple(mamg_ctx* ctx, const mamg_mat* A, const mamg_mat* P, mamg_mat** out) {
    return guard(ctx, [&] {
        const auto& Am = A->get();
        const auto& Pm = P->get();
        if (Am.nrows != Am.ncols) mamg::invalid("galerkin_triple: A is not square");
        if (Am.nrows != Pm.nrows) mamg::invalid("galerkin_triple: A and P row counts differ");
        auto AP = mamg::spgemm(ctx->c, Am, Pm);
        auto Pt = mamg::transpose(ctx->c, Pm);
        auto* m = new mamg_mat;
        m->m = mamg::spgemm(ctx->c, *Pt, *AP);
        *out = m;
    });
}

// ---------------------------------------------------------------- matching --
int mamg_build_weights(mamg_ctx* ctx, const mamg_mat* A, const double* d_w, mamg_graph** out) {
    return guard(ctx, [&] {
        const auto& M = A->get();
        mamg::DBuf<double> wt;
        int64_t zero = 0;
        mamg::build_weights_aligned(ctx->c, M, d_w, wt, zero);
        auto* g = new mamg_graph;
        g->g = mamg::graph_from_aligned(ctx->c, M, wt.get(), zero);
        ctx->c.sync();
        *out = g;
    });
}

int mamg_graph_upload(mamg_ctx* ctx, int64_t n, const int64_t* h_xadj, const int64_t* h_adjncy,
                      const double* h_weight, mamg_graph** out) {
    return guard(ctx, [&] {
        auto* g = new mamg_graph;
        // a WeightedGraph has CSR shape: reuse the CSR upload path
        auto csr = mamg::csr_upload(ctx->c, n, n, h_xadj, h_adjncy, h_weight);
        g->g = std::make_unique<mamg::DevGraph>();
        g->g->n = n;
        g->g->nedges = csr->nnz;
        g->g->xadj = std::move(csr->rp);
        g->g->adj = std::move(csr->ci);
        g->g->wt = std::move(csr->v);
        *out = g;
    });
}

int mamg_graph_shape(const mamg_graph* G, int64_t* n, int64_t* nedges, int64_t* zero_edges) {
    if (!G) return MAMG_INVALID_ARGUMENT;
    if (n) *n = G->g->n;
    if (nedges) *nedges = G->g->nedges;
    if (zero_edges) *zero_edges = G->g->zero_edges;
    return MAMG_OK;
}

int mamg_graph_download(mamg_ctx* ctx, const mamg_graph* G, int64_t* h_xadj, int64_t* h_adjncy,
                        double* h_weight) {
    return guard(ctx, [&] {
        mamg::DevCsr tmp; // borrow the buffers through a CSR view for download
        const auto& g = *G->g;
        std::vector<int32_t> xa(g.n + 1), ad(g.nedges);
        MAMG_CU(cudaMemcpyAsync(xa.data(), g.xadj.get(), sizeof(int32_t) * (g.n + 1),
                                cudaMemcpyDeviceToHost, ctx->c.stream));
        if (g.nedges) {
            MAMG_CU(cudaMemcpyAsync(ad.data(), g.adj.get(), sizeof(int32_t) * g.nedges,
                                    cudaMemcpyDeviceToHost, ctx->c.stream));
            MAMG_CU(cudaMemcpyAsync(h_weight, g.wt.get(), sizeof(double) * g.nedges,
                                    cudaMemcpyDeviceToHost, ctx->c.stream));
        }
        ctx->c.sync();
        for (int64_t i = 0; i <= g.n; ++i) h_xadj[i] = xa[i];
        for (int64_t k = 0; k < g.nedges; ++k) h_adjncy[k] = ad[k];
    });
}

void mamg_graph_destroy(mamg_graph* G) { delete G; }

int mamg_suitor_match(mamg_ctx* ctx, const mamg_graph* G, int64_t* h_mate) {
    return guard(ctx, [&] {
        const auto& g = *G->g;
        mamg::DBuf<int32_t> mate(g.n, ctx->c.stream);
        mamg::suitor(ctx->c, g.n, g.nedges, g.xadj.get(), g.adj.get(), g.wt.get(), mate.get());
        std::vector<int32_t> hm(g.n);
        if (g.n)
            MAMG_CU(cudaMemcpyAsync(hm.data(), mate.get(), sizeof(int32_t) * g.n,
                                    cudaMemcpyDeviceToHost, ctx->c.stream));
        ctx->c.sync();
        for (int64_t i = 0; i < g.n; ++i) h_mate[i] = hm[i];
    });
}

// -------------------------------------------------------------- coarsening --
int mamg_pairwise_aggregate(mamg_ctx* ctx, int64_t n, const int64_t* h_mate, int64_t* h_agg_of,
                            int64_t* h_counts) {
    return guard(ctx, [&] {
        // Matching::is_valid (matching.cpp:18-26), checked on the host input
        for (int64_t i = 0; i < n; ++i) {
            const int64_t j = h_mate[i];
            if (j == -1) continue;
            if (j < 0 || j >= n || j == i || h_mate[j] != i)
                mamg::invalid("pairwise_aggregate: invalid matching");
        }
        std::vector<int32_t> m32(h_mate, h_mate + n);
        mamg::DBuf<int32_t> dm(n, ctx->c.stream);
        if (n)
            MAMG_CU(cudaMemcpyAsync(dm.get(), m32.data(), sizeof(int32_t) * n,
                                    cudaMemcpyHostToDevice, ctx->c.stream));
        mamg::DevAgg g = mamg::aggregate_from_mate(ctx->c, n, dm.get());
        std::vector<int32_t> ha(n);
        if (n)
            MAMG_CU(cudaMemcpyAsync(ha.data(), g.agg_of.get(), sizeof(int32_t) * n,
                                    cudaMemcpyDeviceToHost, ctx->c.stream));
        ctx->c.sync();
        for (int64_t i = 0; i < n; ++i) h_agg_of[i] = ha[i];
        h_counts[0] = g.nc;
        h_counts[1] = g.np;
        h_counts[2] = g.ns;
    });
}

static std::vector<int32_t> narrow(const int64_t* p, int64_t n) {
    return std::vector<int32_t>(p, p + n);
}

int mamg_build_prolongator(mamg_ctx* ctx, int64_t n, int64_t n_c, const int64_t* h_agg_of,
                           const double* d_w, mamg_mat** out_P) {
    return guard(ctx, [&] {
        for (int64_t i = 0; i < n; ++i)
            if (h_agg_of[i] < 0 || h_agg_of[i] >= n_c)
                mamg::invalid("build_prolongator: aggregate id out of range for vertex " +
                                  std::to_string(i),
                              i);
        auto a32 = narrow(h_agg_of, n);
        mamg::DBuf<int32_t> da(n, ctx->c.stream);
        if (n)
            MAMG_CU(cudaMemcpyAsync(da.get(), a32.data(), sizeof(int32_t) * n,
                                    cudaMemcpyHostToDevice, ctx->c.stream));
        mamg::DevAgg g = mamg::aggregate_from_map(ctx->c, n, n_c, da.get());
        auto* m = new mamg_mat;
        m->m = mamg::build_prolongator(ctx->c, g, d_w);
        ctx->c.sync();
        *out_P = m;
    });
}

int mamg_restrict_vector(mamg_ctx* ctx, const mamg_mat* P, const double* d_w, double* d_wc) {
    return guard(ctx, [&] {
        // wc = P^T w in P's row order == R's rows (ascending sources) from 0.0
        auto R = mamg::transpose(ctx->c, P->get());
        mamg::restrict_rows(ctx->c, *R, d_w, d_wc);
        ctx->c.sync();
    });
}

int mamg_galerkin_by_aggregates(mamg_ctx* ctx, const mamg_mat* A, const mamg_mat* P,
                                mamg_mat** out) {
    return guard(ctx, [&] {
        const auto& Am = A->get();
        const auto& Pm = P->get();
        if (Am.nrows != Am.ncols || Am.nrows != Pm.nrows)
            mamg::invalid("galerkin_by_aggregates: shape mismatch");
        std::vector<int32_t> rp(Pm.nrows + 1);
        MAMG_CU(cudaMemcpyAsync(rp.data(), Pm.rp.get(), sizeof(int32_t) * (Pm.nrows + 1),
                                cudaMemcpyDeviceToHost, ctx->c.stream));
        ctx->c.sync();
        for (int64_t i = 0; i < Pm.nrows; ++i)
            if (rp[i + 1] - rp[i] != 1)
                mamg::invalid("galerkin_by_aggregates: row " + std::to_string(i) + " of P has " +
                                  std::to_string(rp[i + 1] - rp[i]) + " nonzeros, expected 1",
                              i);
        mamg::DevAgg g = mamg::aggregates_of(ctx->c, Pm);
        auto* m = new mamg_mat;
        m->m = mamg::galerkin(ctx->c, Am, g, Pm.v.get());
        *out = m;
    });
}

int mamg_coarsen_step(mamg_ctx* ctx, const mamg_mat* A, const double* d_w, int mode,
                      mamg_mat** out_P, mamg_mat** out_Ac, double** out_d_wc,
                      int64_t* zero_edges) {
    return guard(ctx, [&] {
        const auto& Am = A->get();
        if (Am.nrows != Am.ncols) mamg::invalid("build_weights: matrix is not square");
        mamg::DevStep st = mode == 2 ? mamg::double_pairwise(ctx->c, Am, d_w)
                                     : mamg::pairwise_step(ctx->c, Am, d_w);
        auto* P = new mamg_mat;
        P->m = std::move(st.P);
        auto* Ac = new mamg_mat;
        Ac->m = std::move(st.Ac);
        *out_P = P;
        *out_Ac = Ac;
        mamg::sync_checked(ctx->c); // A_c's deferred flags (galerkin in the step)
        *out_d_wc = st.wc.release_ownership();
        *zero_edges = st.zero_edges;
    });
}

// --------------------------------------------------------------- hierarchy --
int mamg_setup(mamg_ctx* ctx, const mamg_mat* A, const double* d_w, const mamg_setup_cfg* cfg,
               mamg_hier** out) {
    return guard(ctx, [&] {
        mamg_setup_cfg def{40, 2, 40.0};
        auto* hh = new mamg_hier;
        try {
            hh->h = mamg::build_hierarchy(ctx->c, A->get(), d_w, cfg ? *cfg : def);
        } catch (...) {
            delete hh;
            throw;
        }
        hh->refresh();
        ctx->c.sync();
        *out = hh;
    });
}

int mamg_hier_from_levels(mamg_ctx* ctx, int nl, mamg_mat* const* A, mamg_mat* const* P,
                          mamg_mat* const* R, const double* const* d_l1,
                          const double* const* d_w, mamg_hier** out) {
    return guard(ctx, [&] {
        need(nl >= 1, "mamg_hier_from_levels: need at least one level");
        auto h = std::make_unique<mamg::DevHier>();
        for (int k = 0; k < nl; ++k) {
            mamg::DevLevel L;
            L.A = mamg::csr_clone(ctx->c, A[k]->get());
            if (k + 1 < nl) {
                L.P = mamg::csr_clone(ctx->c, P[k]->get());
                L.R = mamg::csr_clone(ctx->c, R[k]->get());
            }
            const int64_t n = L.A->nrows;
            L.l1.alloc(n, ctx->c.stream);
            L.w.alloc(n, ctx->c.stream);
            if (n) {
                MAMG_CU(cudaMemcpyAsync(L.l1.get(), d_l1[k], sizeof(double) * n,
                                        cudaMemcpyDeviceToDevice, ctx->c.stream));
                if (d_w && d_w[k])
                    MAMG_CU(cudaMemcpyAsync(L.w.get(), d_w[k], sizeof(double) * n,
                                            cudaMemcpyDeviceToDevice, ctx->c.stream));
            }
            h->lv.push_back(std::move(L));
        }
        mamg::alloc_workspace(ctx->c, *h);
        auto* hh = new mamg_hier;
        hh->h = std::move(h);
        hh->refresh();
        ctx->c.sync();
        *out = hh;
    });
}

void mamg_hier_destroy(mamg_hier* h) { delete h; }
int mamg_hier_nl(const mamg_hier* h) { return h ? h->h->nl() : 0; }
int mamg_hier_stats(const mamg_hier* h, int* stalled, int64_t* zero_edges) {
    if (!h) return MAMG_INVALID_ARGUMENT;
    if (stalled) *stalled = h->h->stalled ? 1 : 0;
    if (zero_edges) *zero_edges = h->h->zero_edges;
    return MAMG_OK;
}
const mamg_mat* mamg_hier_A(const mamg_hier* h, int k) {
    return (h && k >= 0 && k < h->h->nl()) ? &h->A[k] : nullptr;
}
const mamg_mat* mamg_hier_P(const mamg_hier* h, int k) {
    return (h && k >= 0 && k + 1 < h->h->nl()) ? &h->P[k] : nullptr;
}
const mamg_mat* mamg_hier_R(const mamg_hier* h, int k) {
    return (h && k >= 0 && k + 1 < h->h->nl()) ? &h->R[k] : nullptr;
}
const double* mamg_hier_l1(const mamg_hier* h, int k) {
    return (h && k >= 0 && k < h->h->nl()) ? h->h->lv[k].l1.get() : nullptr;
}
const double* mamg_hier_w(const mamg_hier* h, int k) {
    return (h && k >= 0 && k < h->h->nl()) ? h->h->lv[k].w.get() : nullptr;
}

// --------------------------------------------------------------- multigrid --
int mamg_l1_jacobi(mamg_ctx* ctx, const mamg_mat* A, const double* d_d, const double* d_b,
                   double* d_x, int sweeps) {
    return guard(ctx, [&] {
        const auto& M = A->get();
        if (M.ncols != M.nrows) mamg::invalid("l1_jacobi_sweeps: dimension mismatch");
        mamg::l1_jacobi(ctx->c, M, d_d, d_b, d_x, sweeps);
        ctx->c.sync();
    });
}

int mamg_apply_cycle(mamg_ctx* ctx, mamg_hier* h, int level, const mamg_cycle_cfg* cfg,
                     const double* d_b, double* d_x) {
    return guard(ctx, [&] {
        mamg::apply_cycle(ctx->c, *h->h, level, *cfg, d_b, d_x, false);
        ctx->c.sync();
    });
}

int mamg_precond_apply(mamg_ctx* ctx, mamg_hier* h, const mamg_cycle_cfg* cfg, const double* d_r,
                       double* d_z) {
    return guard(ctx, [&] {
        mamg::apply_cycle(ctx->c, *h->h, 0, *cfg, d_r, d_z, true);
        ctx->c.sync();
    });
}

// ------------------------------------------------------------------ vectors --
int mamg_dot(mamg_ctx* ctx, int64_t n, const double* d_x, const double* d_y, double* h_out) {
    return guard(ctx, [&] { *h_out = mamg::dot(ctx->c, n, d_x, d_y); });
}
int mamg_norm2(mamg_ctx* ctx, int64_t n, const double* d_x, double* h_out) {
    return guard(ctx, [&] { *h_out = std::sqrt(mamg::dot(ctx->c, n, d_x, d_x)); });
}
int mamg_axpy(mamg_ctx* ctx, int64_t n, double* d_y, double a, const double* d_x) {
    return guard(ctx, [&] {
        mamg::axpy(ctx->c, n, d_y, a, d_x);
        ctx->c.sync();
    });
}
int mamg_fused_triple_dot(mamg_ctx* ctx, int64_t n, const double* d_w, const double* d_r,
                          const double* d_v, const double* d_q, double* h_out3) {
    return guard(ctx, [&] { mamg::triple_dot(ctx->c, n, d_w, d_r, d_v, d_q, h_out3); });
}
int mamg_fused_axpy_pair(mamg_ctx* ctx, int64_t n, double* d_y1, double* d_y2, const double* d_x,
                         double a, double b) {
    return guard(ctx, [&] {
        mamg::axpy_pair(ctx->c, n, d_y1, d_y2, d_x, a, b);
        ctx->c.sync();
    });
}

// ------------------------------------------------------------------- Krylov --
int mamg_pcg_solve(mamg_ctx* ctx, const mamg_mat* A, mamg_hier* hier, const mamg_cycle_cfg* cycle,
                   mamg_host_precond host_prec, void* user, const double* d_b, const double* d_u0,
                   const mamg_solve_cfg* cfg, double* d_u, double* h_hist, mamg_report* rep) {
    int st = MAMG_OK;
    const int g = guard(ctx, [&] {
        mamg_solve_cfg def{1e-6, 5000};
        st = mamg::pcg_solve(ctx->c, A->get(), hier ? hier->h.get() : nullptr, cycle, host_prec,
                             user, d_b, d_u0, cfg ? *cfg : def, d_u, h_hist, rep);
        if (st == MAMG_BREAKDOWN) {
            ctx->c.err = "pcg breakdown at iteration " + std::to_string(rep->breakdown_iteration) +
                         ": " +
                         (rep->breakdown_iteration == 0 ? "rho_0 = " : "rho = ") +
                         std::to_string(rep->breakdown_rho);
            ctx->c.err_index = rep->breakdown_iteration;
        }
    });
    return g != MAMG_OK ? g : st;
}

int mamg_solve_host(mamg_ctx* ctx, int64_t nrows, const int64_t* h_rp, const int64_t* h_ci,
                    const double* h_v, const double* h_w, const double* h_b,
                    const mamg_setup_cfg* scfg, const mamg_cycle_cfg* ccfg,
                    const mamg_solve_cfg* cfg, double* h_u, double* h_hist, mamg_report* rep,
                    int* h_nl, double* h_times) {
    int st = MAMG_OK;
    const int g = guard(ctx, [&] {
        using clock = std::chrono::steady_clock;
        auto& c = ctx->c;
        const auto t_up = clock::now();
        mamg::DBuf<double> w, b, u;
        if (h_w) w.alloc(nrows, c.stream);
        b.alloc(nrows, c.stream);
        u.alloc(nrows, c.stream);
        std::vector<mamg::UpSeg> extra;
        if (!h_b) mamg::fill_f64(c, nrows, b.get(), 1.0); // b = ones (cli default), made on the device
        if (h_w)
            extra.push_back(mamg::UpSeg{mamg::UpSeg::F64, w.get(), h_w, static_cast<size_t>(nrows), 0, 0});
        // one staged pass: A's row_ptr / col_idx / values and w (the setup's inputs)
        auto A = mamg::csr_upload(c, nrows, nrows, h_rp, h_ci, h_v, extra);
        const double up_ms =
            std::chrono::duration<double, std::milli>(clock::now() - t_up).count();
        const auto t_setup = clock::now();
        // b is needed only by the solve: its staged upload (the staging pool's
        // own threads and streams) overlaps the setup's kernels
        c.sync(); // b's allocation is complete before another stream writes it
        std::thread b_up;
        std::exception_ptr b_err;
        if (h_b && nrows > 0)
            b_up = std::thread([&] {
                try {
                    mamg::upload_f64(c, b.get(), h_b, static_cast<size_t>(nrows));
                } catch (...) {
                    b_err = std::current_exception();
                }
            });
        struct Join {
            std::thread& t;
            ~Join() {
                if (t.joinable()) t.join();
            }
        } join_b{b_up};
        mamg_setup_cfg sdef{40, 2, 40.0};
        // the hierarchy's level 0 takes A itself (no device copy of the matrix)
        const mamg::DevCsr& Aref = *A;
        auto H = mamg::build_hierarchy_owned(c, Aref, std::move(A), h_w ? w.get() : nullptr,
                                             scfg ? *scfg : sdef);
        c.sync();
        if (b_up.joinable()) b_up.join();
        if (b_err) std::rethrow_exception(b_err);
        const double setup_ms =
            std::chrono::duration<double, std::milli>(clock::now() - t_setup).count();
        mamg_cycle_cfg cdef{0, 1, 1, 20};
        mamg_solve_cfg def{1e-6, 5000};
        st = mamg::pcg_solve(c, *H->lv[0].A, H.get(), ccfg ? ccfg : &cdef, nullptr, nullptr, b.get(),
                             nullptr, cfg ? *cfg : def, u.get(), h_hist, rep);
        const auto t_down = clock::now();
        mamg::download_f64(c, h_u, u.get(), static_cast<size_t>(nrows));
        const double down_ms =
            std::chrono::duration<double, std::milli>(clock::now() - t_down).count();
        if (h_nl) *h_nl = H->nl();
        if (h_times) {
            h_times[0] = setup_ms;
            h_times[1] = rep->solve_ms;
            h_times[2] = up_ms;
            h_times[3] = down_ms;
        }
        if (st == MAMG_BREAKDOWN) {
            c.err = "pcg breakdown at iteration " + std::to_string(rep->breakdown_iteration);
            c.err_index = rep->breakdown_iteration;
        }
    });
    return g != MAMG_OK ? g : st;
}

// ------------------------------------------------------------------- timing --
static thread_local cudaEvent_t g_t0 = nullptr, g_t1 = nullptr;

int mamg_timer_start(mamg_ctx* ctx) {
    return guard(ctx, [&] {
        if (!g_t0) {
            MAMG_CU(cudaEventCreate(&g_t0));
            MAMG_CU(cudaEventCreate(&g_t1));
        }
        MAMG_CU(cudaEventRecord(g_t0, ctx->c.stream));
    });
}

int mamg_timer_stop(mamg_ctx* ctx, double* ms) {
    return guard(ctx, [&] {
        MAMG_CU(cudaEventRecord(g_t1, ctx->c.stream));
        MAMG_CU(cudaEventSynchronize(g_t1));
        float f = 0.f;
        MAMG_CU(cudaEventElapsedTime(&f, g_t0, g_t1));
        *ms = f;
    });
}

} // extern "C"

template <class F>
static double time_reps(mamg::Ctx& c, int reps, F&& launch) {
    cudaEvent_t a, b;
    MAMG_CU(cudaEventCreate(&a));
    MAMG_CU(cudaEventCreate(&b));
    launch(); // warm-up
    c.sync();
    MAMG_CU(cudaEventRecord(a, c.stream));
    for (int r = 0; r < reps; ++r) launch();
    MAMG_CU(cudaEventRecord(b, c.stream));
    MAMG_CU(cudaEventSynchronize(b));
    float f = 0.f;
    MAMG_CU(cudaEventElapsedTime(&f, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return static_cast<double>(f) / reps;
}

extern "C" {

int mamg_time_smoother(mamg_ctx* ctx, mamg_hier* h, int level, int reps, double* ms) {
    return guard(ctx, [&] {
        auto& L = h->h->lv.at(level);
        const int64_t n = L.A->nrows;
        mamg::DBuf<double> b(n, ctx->c.stream), x0(n, ctx->c.stream), x1(n, ctx->c.stream);
        MAMG_CU(cudaMemsetAsync(b.get(), 0, 8 * n, ctx->c.stream));
        MAMG_CU(cudaMemsetAsync(x0.get(), 0, 8 * n, ctx->c.stream));
        int flip = 0;
        *ms = time_reps(ctx->c, reps, [&] {
            double* src = flip ? x1.get() : x0.get();
            double* dst = flip ? x0.get() : x1.get();
            mamg::smooth_sweep(ctx->c, *L.A, L.l1.get(), b.get(), src, dst);
            flip ^= 1;
        });
    });
}

int mamg_time_spmv(mamg_ctx* ctx, mamg_hier* h, int level, int reps, double* ms) {
    return guard(ctx, [&] {
        auto& L = h->h->lv.at(level);
        const int64_t n = L.A->nrows;
        mamg::DBuf<double> x(n, ctx->c.stream), y(n, ctx->c.stream);
        MAMG_CU(cudaMemsetAsync(x.get(), 0, 8 * n, ctx->c.stream));
        *ms = time_reps(ctx->c, reps,
                        [&] { mamg::spmv(ctx->c, *L.A, L.A->group, x.get(), y.get()); });
    });
}

int mamg_time_precond(mamg_ctx* ctx, mamg_hier* h, const mamg_cycle_cfg* cfg, int reps,
                      double* ms) {
    return guard(ctx, [&] {
        const int64_t n = h->h->lv[0].A->nrows;
        mamg::DBuf<double> r(n, ctx->c.stream), z(n, ctx->c.stream);
        MAMG_CU(cudaMemsetAsync(r.get(), 0, 8 * n, ctx->c.stream));
        *ms = time_reps(ctx->c, reps,
                        [&] { mamg::apply_cycle(ctx->c, *h->h, 0, *cfg, r.get(), z.get(), true); });
    });
}

// ------------------------------------------------------------ partitioned --
int mamg_nccl_unique_id(void* out128) { return mamg::nccl_unique_id(out128); }

int mamg_dist_create(mamg_ctx* ctx, int world, int rank, const void* nccl_uid, mamg_dist** out) {
    return guard(ctx, [&] {
        need(world >= 1, "mamg_dist_create: world must be >= 1");
        need(rank >= -1 && rank < world, "mamg_dist_create: rank out of range");
        auto* d = new mamg_dist;
        d->ctx = ctx;
        try {
            if (rank < 0)
                d->d.comm = mamg::make_loopback_comm(world);
            else {
                need(nccl_uid != nullptr, "mamg_dist_create: NCCL unique id required");
                d->d.comm = mamg::make_nccl_comm(ctx->c, rank, world, nccl_uid);
            }
        } catch (...) {
            delete d;
            throw;
        }
        *out = d;
    });
}

int mamg_dist_create_shm(mamg_ctx* ctx, int world, int rank, const char* shm_name, mamg_dist** out) {
    return guard(ctx, [&] {
        need(world >= 1, "mamg_dist_create_shm: world must be >= 1");
        need(rank >= 0 && rank < world, "mamg_dist_create_shm: rank out of range");
        need(shm_name != nullptr && shm_name[0] != '\0', "mamg_dist_create_shm: segment name required");
        auto* d = new mamg_dist;
        d->ctx = ctx;
        try {
            d->d.comm = mamg::make_shm_comm(ctx->c, rank, world, shm_name);
        } catch (...) {
            delete d;
            throw;
        }
        *out = d;
    });
}

void mamg_dist_destroy(mamg_dist* d) { delete d; }

int mamg_group_create(int world, mamg_group** out) {
    if (world < 1 || !out) return MAMG_INVALID_ARGUMENT;
    try {
        *out = new mamg_group{std::make_shared<mamg::ThreadGroup>(world)};
    } catch (...) {
        return MAMG_RUNTIME;
    }
    return MAMG_OK;
}

void mamg_group_destroy(mamg_group* g) { delete g; }

int mamg_dist_create_group(mamg_ctx* ctx, mamg_group* g, int rank, mamg_dist** out) {
    return guard(ctx, [&] {
        need(g != nullptr && out != nullptr, "mamg_dist_create_group: null argument");
        need(rank >= 0 && rank < g->g->world, "mamg_dist_create_group: rank out of range");
        auto* d = new mamg_dist;
        d->ctx = ctx;
        d->group = g->g;
        try {
            d->d.comm = mamg::make_thread_comm(ctx->c, rank, *g->g);
        } catch (...) {
            delete d;
            throw;
        }
        *out = d;
    });
}

int mamg_dist_time(mamg_dist* d, int what, const mamg_cycle_cfg* cyc, int reps, double* ms) {
    return guard(d->ctx, [&] { *ms = mamg::dist_time(d->ctx->c, d->d, what, *cyc, reps); });
}

int mamg_dist_last_solve(const mamg_dist* d, int* flags4) {
    if (!d || !flags4) return MAMG_INVALID_ARGUMENT;
    for (int i = 0; i < 4; ++i) flags4[i] = d->d.last_solve[i];
    return MAMG_OK;
}

int mamg_shm_allgather(const char* shm_name, int world, int rank, const int64_t* mine, int64_t len,
                       int64_t* out) {
    if (!shm_name || !shm_name[0] || world < 1 || rank < 0 || rank >= world || len < 0)
        return MAMG_INVALID_ARGUMENT;
    try {
        const auto all = mamg::shm_allgather_once(shm_name, world, rank, mine, len);
        std::copy(all.begin(), all.end(), out);
    } catch (const mamg::Error& e) {
        g_noctx_err = e.what();
        return e.status;
    }
    return MAMG_OK;
}

int mamg_dist_set_rebuildable(mamg_dist* d, int keep) {
    if (!d) return MAMG_INVALID_ARGUMENT;
    d->d.consume_level0 = keep == 0;
    return MAMG_OK;
}

int mamg_dist_set_matching(mamg_dist* d, int mode) {
    return guard(d->ctx, [&] {
        need(mode == 0 || mode == 1, "mamg_dist_set_matching: mode must be 0 (local) or 1 (global)");
        d->d.matching = mode;
    });
}

int mamg_dist_set_agglomeration(mamg_dist* d, int64_t rows) {
    return guard(d->ctx, [&] {
        need(rows >= 0, "mamg_dist_set_agglomeration: rows must be >= 0");
        d->d.agglom_rows = rows;
    });
}

int mamg_dist_bounds(int64_t n, int world, int64_t* h_bounds) {
    if (world < 1 || n < 0) return MAMG_INVALID_ARGUMENT;
    const auto b = mamg::dist_bounds(n, world);
    std::copy(b.begin(), b.end(), h_bounds);
    return MAMG_OK;
}

int mamg_dist_setup(mamg_dist* d, int64_t n, const int64_t* h_rp, const int64_t* h_ci,
                    const double* h_v, const double* h_w, const mamg_setup_cfg* cfg) {
    return guard(d->ctx, [&] {
        mamg_setup_cfg def{40, 2, 40.0};
        mamg::dist_setup(d->ctx->c, d->d, n, h_rp, h_ci, h_v, h_w, cfg ? *cfg : def);
    });
}

int mamg_dist_load(mamg_dist* d, int64_t n, const int64_t* h_rp, const int64_t* h_ci,
                   const double* h_v, const double* h_w) {
    return guard(d->ctx, [&] { mamg::dist_load(d->ctx->c, d->d, n, h_rp, h_ci, h_v, h_w); });
}

int mamg_dist_build(mamg_dist* d, const mamg_setup_cfg* cfg) {
    return guard(d->ctx, [&] {
        mamg_setup_cfg def{40, 2, 40.0};
        mamg::dist_build(d->ctx->c, d->d, cfg ? *cfg : def);
    });
}

int mamg_dist_info(const mamg_dist* d, int* nl, int64_t* level_n, int64_t* level_nnz, int* stalled,
                   int64_t* zero_edges) {
    if (!d) return MAMG_INVALID_ARGUMENT;
    if (nl) *nl = d->d.nl;
    for (int k = 0; k < d->d.nl && k < 64; ++k) {
        if (level_n) level_n[k] = d->d.level_n[k];
        if (level_nnz) level_nnz[k] = d->d.level_nnz[k];
    }
    if (stalled) *stalled = d->d.stalled ? 1 : 0;
    if (zero_edges) *zero_edges = d->d.zero_edges;
    return MAMG_OK;
}

// agglomerated levels (replicated on every process) are reported as owned by
// rank 0: bounds [0, n, ..., n], downloads from the other ranks are empty
static bool replicated(const mamg_dist* d, int level) {
    return d->d.agg_level >= 0 && level >= d->d.agg_level;
}

int mamg_dist_level_bounds(const mamg_dist* d, int level, int64_t* h_bounds) {
    if (!d || d->d.parts.empty() || level < 0 || level >= d->d.nl) return MAMG_INVALID_ARGUMENT;
    if (replicated(d, level)) {
        h_bounds[0] = 0;
        for (int r = 1; r <= d->d.comm->world; ++r) h_bounds[r] = d->d.level_n[level];
        return MAMG_OK;
    }
    const auto& b = d->d.parts[0].lv[level].bounds;
    std::copy(b.begin(), b.end(), h_bounds);
    return MAMG_OK;
}

static const mamg::Part* find_part(const mamg_dist* d, int rank) {
    for (const auto& p : d->d.parts)
        if (p.rank == rank) return &p;
    return nullptr;
}

int mamg_dist_level_shape(const mamg_dist* d, int rank, int level, int which, int64_t* nrows,
                          int64_t* nnz) {
    const mamg::Part* p = d ? find_part(d, rank) : nullptr;
    if (!p || level < 0 || level >= d->d.nl) return MAMG_INVALID_ARGUMENT;
    if (replicated(d, level)) {
        const mamg::DevLevel& R = d->d.rep->lv[level - d->d.agg_level];
        const mamg::DevCsr* M = which == 1 ? R.P.get() : which == 2 ? R.R.get() : R.A.get();
        if (!M) return MAMG_INVALID_ARGUMENT;
        *nrows = rank == 0 ? M->nrows : 0;
        *nnz = rank == 0 ? (which >= 3 ? M->nrows : M->nnz) : 0;
        return MAMG_OK;
    }
    const mamg::PLevel& L = p->lv[level];
    const mamg::DevCsr* M = which == 0 ? L.A.get() : which == 1 ? L.P.get() : which == 2 ? L.R.get() : L.A.get();
    if (!M) return MAMG_INVALID_ARGUMENT;
    *nrows = M->nrows;
    *nnz = which >= 3 ? M->nrows : M->nnz;
    return MAMG_OK;
}

int mamg_dist_download(mamg_dist* d, int rank, int level, int which, int64_t* h_rp, int64_t* h_ci,
                       double* h_v) {
    return guard(d->ctx, [&] {
        const mamg::Part* p = find_part(d, rank);
        need(p != nullptr && level >= 0 && level < d->d.nl, "mamg_dist_download: bad part/level");
        auto& c = d->ctx->c;
        if (replicated(d, level)) {
            if (rank != 0) {
                if (h_rp) h_rp[0] = 0;
                return;
            }
            const mamg::DevLevel& R = d->d.rep->lv[level - d->d.agg_level];
            if (which >= 3) {
                const double* src = which == 3 ? R.l1.get() : R.w.get();
                if (R.A->nrows)
                    MAMG_CU(cudaMemcpyAsync(h_v, src, sizeof(double) * R.A->nrows,
                                            cudaMemcpyDeviceToHost, c.stream));
                c.sync();
                return;
            }
            const mamg::DevCsr* M = which == 0 ? R.A.get() : which == 1 ? R.P.get() : R.R.get();
            need(M != nullptr, "mamg_dist_download: no such matrix on this level");
            mamg::csr_download(c, *M, h_rp, h_ci, h_v);
            return;
        }
        const mamg::PLevel& L = p->lv[level];
        if (which >= 3) {
            const double* src = which == 3 ? L.l1.get() : L.w.get();
            if (L.A->nrows)
                MAMG_CU(cudaMemcpyAsync(h_v, src, sizeof(double) * L.A->nrows,
                                        cudaMemcpyDeviceToHost, c.stream));
            c.sync();
            return;
        }
        const mamg::DevCsr* M = which == 0 ? L.A.get() : which == 1 ? L.P.get() : L.R.get();
        need(M != nullptr, "mamg_dist_download: no such matrix on this level");
        mamg::csr_download(c, *M, h_rp, h_ci, h_v);
        if (which == 0) { // global column ids
            std::vector<int32_t> cg(M->nnz);
            if (M->nnz)
                MAMG_CU(cudaMemcpyAsync(cg.data(), L.cg.get(), sizeof(int32_t) * M->nnz,
                                        cudaMemcpyDeviceToHost, c.stream));
            c.sync();
            for (int64_t k = 0; k < M->nnz; ++k) h_ci[k] = cg[k];
        } else if (which == 1 ? L.Pg.get() != nullptr : L.Rg.get() != nullptr) {
            // stored global ids (global matching; P above an agglomeration)
            const mamg::DBuf<int32_t>& g = which == 1 ? L.Pg : L.Rg;
            std::vector<int32_t> cg(M->nnz);
            if (M->nnz)
                MAMG_CU(cudaMemcpyAsync(cg.data(), g.get(), sizeof(int32_t) * M->nnz,
                                        cudaMemcpyDeviceToHost, c.stream));
            c.sync();
            for (int64_t k = 0; k < M->nnz; ++k) h_ci[k] = cg[k];
        } else if (which == 1) { // local coarse -> global coarse
            const int64_t off = p->lv[level + 1].bounds[rank];
            for (int64_t k = 0; k < M->nnz; ++k) h_ci[k] += off;
        } else { // R columns: local fine -> global fine
            const int64_t off = L.bounds[rank];
            for (int64_t k = 0; k < M->nnz; ++k) h_ci[k] += off;
        }
    });
}

int mamg_dist_pcg_x0(mamg_dist* d, const double* h_b, const double* h_u0, const mamg_cycle_cfg* cyc,
                     const mamg_solve_cfg* cfg, double* h_u, double* h_hist, mamg_report* rep) {
    int st = MAMG_OK;
    const int g = guard(d->ctx, [&] {
        mamg_cycle_cfg cdef{0, 1, 1, 20};
        mamg_solve_cfg sdef{1e-6, 5000};
        st = mamg::dist_pcg(d->ctx->c, d->d, cyc ? *cyc : cdef, h_b, cfg ? *cfg : sdef, h_u,
                            h_hist, rep, h_u0);
        if (st == MAMG_BREAKDOWN) {
            d->ctx->c.err = "pcg breakdown at iteration " + std::to_string(rep->breakdown_iteration);
            d->ctx->c.err_index = rep->breakdown_iteration;
        }
    });
    return g != MAMG_OK ? g : st;
}

int mamg_dist_pcg(mamg_dist* d, const double* h_b, const mamg_cycle_cfg* cyc,
                  const mamg_solve_cfg* cfg, double* h_u, double* h_hist, mamg_report* rep) {
    return mamg_dist_pcg_x0(d, h_b, nullptr, cyc, cfg, h_u, h_hist, rep);
}

} // extern "C"
