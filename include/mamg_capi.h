/* mamg_capi.h — the thin C-ABI between the host C++ `matchamg` API
 * (include/matchamg/*.hpp, the drop-in for /root/reference/proj/include) and the
 * B200 (sm_100a) CUDA implementation in libmamg_cuda.so.
 *
 * Conventions
 *  - Every entry point returns an mamg_status; on failure mamg_last_error(ctx)
 *    holds the message (worded like the reference's exception text) and
 *    mamg_last_error_index(ctx) the offending row / aggregate / iteration.
 *  - Host pointers (const int64_t*, const double* named h_*) are borrowed for
 *    the duration of the call and copied. Device pointers (named d_*) are
 *    caller-owned device memory on the context's device.
 *  - Handles (mamg_mat, mamg_hier, mamg_graph) own device memory.
 *  - One context = one device + one CUDA stream; a context is not thread-safe
 *    (one solver per host thread, as the reference's README requires of its
 *    CycleWorkspace). All work is ordered on the context stream.
 *  - API index type is int64 (proj/include/matchamg/csr.hpp:14); the device
 *    stores int32 row pointers/columns, so nnz and n must be < 2^31.
 *  - Arithmetic is IEEE binary64 in the reference's evaluation order: results
 *    are bit-identical to the reference CPU library.
 */
#ifndef MAMG_CAPI_H
#define MAMG_CAPI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    MAMG_OK = 0,
    MAMG_INVALID_ARGUMENT = 1, /* std::invalid_argument in the reference */
    MAMG_RUNTIME = 2,          /* std::runtime_error */
    MAMG_BREAKDOWN = 3,        /* matchamg::BreakdownError (krylov.hpp:52-59) */
    MAMG_CUDA = 4,             /* CUDA runtime failure */
    MAMG_NCCL = 5              /* collective failure (partitioned path) */
} mamg_status;

typedef struct mamg_ctx mamg_ctx;
typedef struct mamg_mat mamg_mat;     /* device CSR (int32 rp/ci, fp64 values) */
typedef struct mamg_graph mamg_graph; /* device weighted graph (WeightedGraph) */
typedef struct mamg_hier mamg_hier;   /* device-resident multigrid hierarchy */

/* ---- context --------------------------------------------------------------- */
int mamg_ctx_create(int device, mamg_ctx** out);
void mamg_ctx_destroy(mamg_ctx* ctx);
const char* mamg_last_error(const mamg_ctx* ctx);
int64_t mamg_last_error_index(const mamg_ctx* ctx);
int mamg_synchronize(mamg_ctx* ctx);
/* number of kernels this context has launched (incl. graph nodes replayed) */
int64_t mamg_kernel_launches(const mamg_ctx* ctx);
const char* mamg_version(void);

/* ---- device memory helpers (for callers without their own allocator) -------- */
int mamg_dmalloc(mamg_ctx* ctx, size_t bytes, void** d_out);
int mamg_dfree(mamg_ctx* ctx, void* d_ptr);
int mamg_h2d(mamg_ctx* ctx, void* d_dst, const void* h_src, size_t bytes);
int mamg_d2h(mamg_ctx* ctx, void* h_dst, const void* d_src, size_t bytes);

/* ---- CsrMatrix (proj/include/matchamg/csr.hpp:30-57) ------------------------- */
int mamg_csr_upload(mamg_ctx* ctx, int64_t nrows, int64_t ncols, const int64_t* h_rp,
                    const int64_t* h_ci, const double* h_v, mamg_mat** out);
/* The problem generators of problems.hpp assembled directly on the device
 * (SURVEY.md §8f rank 3): the same matrices bit for bit as gen_poisson_2d /
 * gen_anisotropic_2d / gen_poisson_3d_randk (proj/src/problems.cpp:67-193)
 * and the cfg 3-5 generators, without a host CSR or an upload. */
int mamg_gen_poisson2d_dev(mamg_ctx* ctx, int64_t nx, int64_t ny, mamg_mat** out);
int mamg_gen_aniso2d_dev(mamg_ctx* ctx, int64_t nx, int64_t ny, double epsilon, double theta,
                         mamg_mat** out);
int mamg_gen_randk3d_dev(mamg_ctx* ctx, int64_t nx, int64_t ny, int64_t nz, double sigma,
                         uint64_t seed, mamg_mat** out);
int mamg_gen_jump3d_dev(mamg_ctx* ctx, int64_t nx, int64_t ny, int64_t nz, int64_t block,
                        uint64_t seed, double lo, double hi, mamg_mat** out);
int mamg_gen_aniso27_dev(mamg_ctx* ctx, int64_t nx, int64_t ny, int64_t nz, double kx, double ky,
                         double kz, mamg_mat** out);
int mamg_gen_elast3d_dev(mamg_ctx* ctx, int64_t nx, int64_t ny, int64_t nz, double mu,
                         double lambda, mamg_mat** out);
int mamg_csr_shape(const mamg_mat* A, int64_t* nrows, int64_t* ncols, int64_t* nnz);
int mamg_csr_download(mamg_ctx* ctx, const mamg_mat* A, int64_t* h_rp, int64_t* h_ci,
                      double* h_v);
void mamg_mat_destroy(mamg_mat* A);
/* LaneGroupPolicy::for_matrix (proj/src/kernels.cpp:11-24) as cached on A */
int mamg_lane_policy(const mamg_mat* A);
/* has_symmetric_pattern (proj/src/csr.cpp:106-112) -> *out 0/1 */
int mamg_has_symmetric_pattern(mamg_ctx* ctx, const mamg_mat* A, int* out);

/* ---- sparse kernels (proj/include/matchamg/kernels.hpp:21-49) ---------------- */
/* group 0 = LaneGroupPolicy::for_matrix; else one of {1,2,4,8,16,32} */
int mamg_spmv(mamg_ctx* ctx, const mamg_mat* A, int group, const double* d_x, double* d_y);
int mamg_l1_diagonal(mamg_ctx* ctx, const mamg_mat* A, double* d_out);
int mamg_transpose(mamg_ctx* ctx, const mamg_mat* A, mamg_mat** out);
int mamg_spgemm(mamg_ctx* ctx, const mamg_mat* A, const mamg_mat* B, mamg_mat** out);
int mamg_galerkin_triple(mamg_ctx* ctx, const mamg_mat* A, const mamg_mat* P, mamg_mat** out);

/* ---- matching (proj/include/matchamg/matching.hpp:27-65) --------------------- */
int mamg_build_weights(mamg_ctx* ctx, const mamg_mat* A, const double* d_w, mamg_graph** out);
int mamg_graph_upload(mamg_ctx* ctx, int64_t n, const int64_t* h_xadj, const int64_t* h_adjncy,
                      const double* h_weight, mamg_graph** out);
/* sizes: *n, *nedges (= xadj[n]), *zero_weight_edges */
int mamg_graph_shape(const mamg_graph* G, int64_t* n, int64_t* nedges, int64_t* zero_edges);
int mamg_graph_download(mamg_ctx* ctx, const mamg_graph* G, int64_t* h_xadj, int64_t* h_adjncy,
                        double* h_weight);
void mamg_graph_destroy(mamg_graph* G);
/* suitor_match: h_mate[n] (int64, -1 = unmatched) */
int mamg_suitor_match(mamg_ctx* ctx, const mamg_graph* G, int64_t* h_mate);

/* ---- coarsening (proj/include/matchamg/coarsening.hpp:17-58) ----------------- */
/* pairwise_aggregate: h_counts = {n_c, n_p, n_s} */
int mamg_pairwise_aggregate(mamg_ctx* ctx, int64_t n, const int64_t* h_mate, int64_t* h_agg_of,
                            int64_t* h_counts);
int mamg_build_prolongator(mamg_ctx* ctx, int64_t n, int64_t n_c, const int64_t* h_agg_of,
                           const double* d_w, mamg_mat** out_P);
int mamg_restrict_vector(mamg_ctx* ctx, const mamg_mat* P, const double* d_w, double* d_wc);
int mamg_galerkin_by_aggregates(mamg_ctx* ctx, const mamg_mat* A, const mamg_mat* P,
                                mamg_mat** out);
/* pairwise_step (mode 1) / double_pairwise (mode 2): P, A_coarse, d_wc (device,
 * allocated by the call; free with mamg_dfree), zero-weight-edge count */
int mamg_coarsen_step(mamg_ctx* ctx, const mamg_mat* A, const double* d_w, int mode,
                      mamg_mat** out_P, mamg_mat** out_Ac, double** out_d_wc,
                      int64_t* zero_edges);

typedef struct {
    int32_t max_levels;   /* 40 */
    int32_t aggregation;  /* 1 = Pairwise, 2 = DoublePairwise (default) */
    double coarse_factor; /* 40.0 */
} mamg_setup_cfg;

/* build_hierarchy (proj/src/coarsening.cpp:194-238). d_w NULL = ones. A is
 * copied into level 0 (the caller keeps ownership of A). */
int mamg_setup(mamg_ctx* ctx, const mamg_mat* A, const double* d_w, const mamg_setup_cfg* cfg,
               mamg_hier** out);
/* assemble a device hierarchy from host levels (MultigridPreconditioner over a
 * host-built Hierarchy): nl levels of A, nl-1 of P and R, l1 and w per level */
int mamg_hier_from_levels(mamg_ctx* ctx, int nl, mamg_mat* const* A, mamg_mat* const* P,
                          mamg_mat* const* R, const double* const* d_l1,
                          const double* const* d_w, mamg_hier** out);
void mamg_hier_destroy(mamg_hier* h);
int mamg_hier_nl(const mamg_hier* h);
/* stats: stalled flag and zero-weight edges (HierarchyStats, coarsening.hpp:82-87) */
int mamg_hier_stats(const mamg_hier* h, int* stalled, int64_t* zero_edges);
/* borrowed views (valid while h lives); P/R are NULL on the coarsest level */
const mamg_mat* mamg_hier_A(const mamg_hier* h, int level);
const mamg_mat* mamg_hier_P(const mamg_hier* h, int level);
const mamg_mat* mamg_hier_R(const mamg_hier* h, int level);
const double* mamg_hier_l1(const mamg_hier* h, int level);
const double* mamg_hier_w(const mamg_hier* h, int level);

/* ---- multigrid (proj/include/matchamg/multigrid.hpp:15-77) ------------------- */
typedef struct {
    int32_t cycle; /* 0 = V, 1 = W, 2 = K (K-cycle extension; single-device path) */
    int32_t pre_sweeps;
    int32_t post_sweeps;
    int32_t coarsest_sweeps;
} mamg_cycle_cfg;

int mamg_l1_jacobi(mamg_ctx* ctx, const mamg_mat* A, const double* d_d, const double* d_b,
                   double* d_x, int sweeps);
/* apply_cycle at `level`, x updated in place */
int mamg_apply_cycle(mamg_ctx* ctx, mamg_hier* h, int level, const mamg_cycle_cfg* cfg,
                     const double* d_b, double* d_x);
/* MultigridPreconditioner::apply: z = B(r), one cycle from z = 0 */
int mamg_precond_apply(mamg_ctx* ctx, mamg_hier* h, const mamg_cycle_cfg* cfg, const double* d_r,
                       double* d_z);

/* ---- vector ops (proj/include/matchamg/vector_ops.hpp:16-39) ----------------- */
int mamg_dot(mamg_ctx* ctx, int64_t n, const double* d_x, const double* d_y, double* h_out);
int mamg_norm2(mamg_ctx* ctx, int64_t n, const double* d_x, double* h_out);
int mamg_axpy(mamg_ctx* ctx, int64_t n, double* d_y, double a, const double* d_x);
int mamg_fused_triple_dot(mamg_ctx* ctx, int64_t n, const double* d_w, const double* d_r,
                          const double* d_v, const double* d_q, double* h_out3);
int mamg_fused_axpy_pair(mamg_ctx* ctx, int64_t n, double* d_y1, double* d_y2,
                         const double* d_x, double a, double b);

/* ---- Krylov (proj/include/matchamg/krylov.hpp:29-74) ------------------------- */
typedef struct {
    double rtol;   /* 1e-6 */
    int64_t itmax; /* 5000 */
} mamg_solve_cfg;

typedef struct {
    int64_t iterations;
    double final_relres;
    int32_t converged;
    int32_t pad;
    double solve_ms;
    int64_t audit_checks;
    int64_t audit_failures;
    double audit_max_rel;
    int64_t breakdown_iteration; /* -1 unless MAMG_BREAKDOWN */
    double breakdown_rho;        /* the offending rho on breakdown */
} mamg_report;

/* Host preconditioner callback (PrecondFn, krylov.hpp:62): z = B(r) on HOST
 * buffers of length n. */
typedef void (*mamg_host_precond)(void* user, const double* h_r, double* h_z, int64_t n);

/* pcg_solve (proj/src/krylov.cpp:43-141) on device vectors. Preconditioner:
 * hier != NULL -> device multigrid cycle (cfg); else host_prec != NULL -> the
 * host callback (staged copies); else unpreconditioned CG. d_u0 NULL = zero
 * guess. h_hist (may be NULL) receives itmax + 1 residual norms. */
int mamg_pcg_solve(mamg_ctx* ctx, const mamg_mat* A, mamg_hier* hier,
                   const mamg_cycle_cfg* cycle, mamg_host_precond host_prec, void* user,
                   const double* d_b, const double* d_u0, const mamg_solve_cfg* cfg,
                   double* d_u, double* h_hist, mamg_report* rep);

/* End-to-end cli::run_solve path (proj/src/cli.cpp:242-328) on HOST buffers:
 * upload A, setup, solve A u = b, download u. Times: h_times[0] = setup ms
 * (device build_hierarchy, as cli.cpp:273-275), [1] = solve ms (as
 * krylov.cpp:54), [2] = upload ms, [3] = download ms. h_w / h_b NULL = ones. */
int mamg_solve_host(mamg_ctx* ctx, int64_t nrows, const int64_t* h_rp, const int64_t* h_ci,
                    const double* h_v, const double* h_w, const double* h_b,
                    const mamg_setup_cfg* scfg, const mamg_cycle_cfg* ccfg,
                    const mamg_solve_cfg* cfg, double* h_u, double* h_hist, mamg_report* rep,
                    int* h_nl, double* h_times);

/* ---- row-block partitioned path --------------------------------
 * The matrix is split into `world` contiguous row blocks (level-0 boundaries
 * on multiples of 2048 rows, mamg_dist_bounds); matching runs on each block's
 * local graph; halos move ghost values; dot partials are allgathered so every
 * dot product equals the unpartitioned one bit for bit. Parity target: the
 * partition-aware composition of the reference's functions (oracle/partition.py).
 *   rank >= 0: this process owns part `rank`; NCCL transport, `nccl_uid` from
 *              mamg_nccl_unique_id() on rank 0 (broadcast by the caller).
 *   rank == -1: all `world` parts live in this context (in-process loopback
 *              transport on one device). */
typedef struct mamg_dist mamg_dist;
int mamg_nccl_unique_id(void* out128);
int mamg_dist_create(mamg_ctx* ctx, int world, int rank, const void* nccl_uid, mamg_dist** out);
/* this process owns part `rank` of `world`, without NCCL: host collectives
 * through the POSIX shared-memory segment `shm_name` (every rank passes the
 * same, fresh name; rank 0 unlinks it once all ranks have attached), device
 * data through CUDA-IPC blocks. One node; ranks may share a GPU. The solve's
 * peer paths (IPC mailboxes, peer reductions, peer-memory Suitor) are the
 * same as with NCCL; its collectives wait on the host, so no iteration graph. */
int mamg_dist_create_shm(mamg_ctx* ctx, int world, int rank, const char* shm_name, mamg_dist** out);
void mamg_dist_destroy(mamg_dist* d);
/* device ms (CUDA events, mean over reps) of this process's parts: what 0 =
 * one level-0 fused l1-Jacobi sweep of the local rows (kernel alone), what 1
 * = one preconditioner application from zero with halos. Collective: every
 * rank calls it. */
int mamg_dist_time(mamg_dist* d, int what, const mamg_cycle_cfg* cyc, int reps, double* ms);
/* ranks as THREADS of one process (one rank per device; several ranks may
 * share a device, then the solve keeps the Comm's halos / allgathers): every
 * rank's thread calls mamg_dist_create_group with the same group, its own
 * context (device) and rank; the group must outlive nothing — each dist keeps
 * it alive. Host collectives through the group's memory, device data through
 * directly shared blocks with peer access. */
typedef struct mamg_group mamg_group;
int mamg_group_create(int world, mamg_group** out);
void mamg_group_destroy(mamg_group* g);
int mamg_dist_create_group(mamg_ctx* ctx, mamg_group* g, int rank, mamg_dist** out);
/* how the last mamg_dist_pcg ran: flags4[0] dot partials through peer memory,
 * [1] halos through the peer mailboxes, [2] halo/interior overlap on a second
 * stream, [3] iteration CUDA graphs replayed */
int mamg_dist_last_solve(const mamg_dist* d, int* flags4);
/* the shm transport's host collective alone (no GPU needed): attach to the
 * segment `shm_name`, allgather `len` int64 per rank into out[world * len]
 * (rank-major), detach. Every rank passes the same fresh name. */
int mamg_shm_allgather(const char* shm_name, int world, int rank, const int64_t* mine, int64_t len,
                       int64_t* out);
/* matching mode of the following builds: 0 = on each part's local graph block
 * (default; aggregates never straddle parts), 1 = global Suitor across parts
 * (cross-part aggregates; hierarchy and PCG bit-identical to the
 * unpartitioned build at any part count). Replaces the
 * reference's single-process suitor_match (proj/src/matching.cpp:117-154). */
int mamg_dist_set_matching(mamg_dist* d, int mode);
/* keep = 1 (default): mamg_dist_build works on a copy of the loaded level-0
 * blocks, so the hierarchy can be rebuilt from one load. keep = 0: the next
 * build consumes them (one device copy of A instead of two — matrices near
 * the device memory; a later build needs a new mamg_dist_load). */
int mamg_dist_set_rebuildable(mamg_dist* d, int keep);
/* agglomeration of the following builds: the first level below the finest
 * with at most `rows` rows, and every coarser level, are replicated on all
 * ranks and cycled by the single-device code (one allgather per visit instead
 * of per-sweep halos). 0 = off; default 262144. Levels at and below it are
 * reported as owned by rank 0 (mamg_dist_level_bounds / _download). */
int mamg_dist_set_agglomeration(mamg_dist* d, int64_t rows);
int mamg_dist_bounds(int64_t n, int world, int64_t* h_bounds /* world + 1 */);
/* every process passes the FULL host matrix and keeps its own rows; d_w NULL = ones */
int mamg_dist_setup(mamg_dist* d, int64_t n, const int64_t* h_rp, const int64_t* h_ci,
                    const double* h_v, const double* h_w, const mamg_setup_cfg* cfg);
/* the two halves of mamg_dist_setup: load = H2D of the local row blocks (kept
 * device-resident), build = the partition-aware build_hierarchy on the device */
int mamg_dist_load(mamg_dist* d, int64_t n, const int64_t* h_rp, const int64_t* h_ci,
                   const double* h_v, const double* h_w);
int mamg_dist_build(mamg_dist* d, const mamg_setup_cfg* cfg);
/* global level sizes (arrays of capacity 64) */
int mamg_dist_info(const mamg_dist* d, int* nl, int64_t* level_n, int64_t* level_nnz, int* stalled,
                   int64_t* zero_edges);
int mamg_dist_level_bounds(const mamg_dist* d, int level, int64_t* h_bounds);
/* level data of a local part with GLOBAL indices: which 0 = A (its rows),
 * 1 = P (its fine rows), 2 = R (its coarse rows), 3 = l1, 4 = w. Sizes first
 * (nrows, nnz), then the arrays (h_rp: nrows + 1, h_ci / h_v: nnz; vectors
 * use h_v only). */
int mamg_dist_level_shape(const mamg_dist* d, int rank, int level, int which, int64_t* nrows,
                          int64_t* nnz);
int mamg_dist_download(mamg_dist* d, int rank, int level, int which, int64_t* h_rp, int64_t* h_ci,
                       double* h_v);
/* partitioned pcg_solve with the device cycle; h_b: full rhs (NULL = ones,
 * generated on the device); h_u: full-length host vector (NULL = keep on the
 * device), the rows of the local parts are written */
int mamg_dist_pcg(mamg_dist* d, const double* h_b, const mamg_cycle_cfg* cyc,
                  const mamg_solve_cfg* cfg, double* h_u, double* h_hist, mamg_report* rep);
/* the same from the initial guess h_u0 (full-length host vector; NULL = 0),
 * pcg_solve's u0 (proj/src/krylov.cpp:73-84) */
int mamg_dist_pcg_x0(mamg_dist* d, const double* h_b, const double* h_u0, const mamg_cycle_cfg* cyc,
                     const mamg_solve_cfg* cfg, double* h_u, double* h_hist, mamg_report* rep);

/* ---- device-event timing (bench.py) ----------------------------------------
 * Stream-ordered CUDA events on the context stream. */
int mamg_timer_start(mamg_ctx* ctx);
int mamg_timer_stop(mamg_ctx* ctx, double* ms);
/* average device time of one launch of the fused l1-Jacobi sweep kernel
 * (SpMV + update, the dominant solve kernel) on `level`, over `reps` launches */
int mamg_time_smoother(mamg_ctx* ctx, mamg_hier* h, int level, int reps, double* ms_per_launch);
/* average device time of one plain SpMV y = A x on `level` */
int mamg_time_spmv(mamg_ctx* ctx, mamg_hier* h, int level, int reps, double* ms_per_launch);
/* average device time of one preconditioner application (cycle from z = 0) */
int mamg_time_precond(mamg_ctx* ctx, mamg_hier* h, const mamg_cycle_cfg* cfg, int reps,
                      double* ms_per_apply);

#ifdef __cplusplus
}
#endif
#endif
