// ops.cuh — internal host-side interface between the .cu translation units
// of libmamg_cuda.so. Everything here runs on Ctx::stream.
#pragma once

#include <memory>
#include <vector>

#include "common.cuh"

namespace mamg {

// ------------------------------------------------------------------ scan.cu --
// Exclusive prefix sum of in[0..n) into out[0..n]; out[n] = total. In-place
// (in == out) is allowed when out has room for n + 1 entries.
void exclusive_scan_i32(Ctx& c, const int32_t* in, int32_t* out, int64_t n);
// Blocking readback of one device int32.
int64_t read_i32(Ctx& c, const int32_t* d);

// ---- deferred checks (Ctx::pending) --------------------------------------
constexpr int32_t kNoViolation = 0x7f7f7f7f; // flag slots start here (memset 0x7f)
// k consecutive int32 flag slots (atomicMin of the offending index); `fail`
// runs at the next sync_checked with slot j's value if it is not kNoViolation
int32_t* defer_flags(Ctx& c, int k, std::function<void(int, int32_t)> fail);
// k int32 slots initialised from `init` (host); take(j, value) runs for every
// slot at the next sync_checked (values, not checks: it must not throw)
int32_t* defer_values(Ctx& c, int k, const int32_t* init, std::function<void(int, int32_t)> take);
// a uint64 counter (zeroed); `take` receives its value at the next sync_checked
unsigned long long* defer_counter(Ctx& c, std::function<void(int64_t)> take);
// enqueue the pending readbacks, synchronise, run the checks in order
// between: stream work that does not depend on the values read back; it is
// enqueued after the readback copies, and the host waits for the copies only
// (so the GPU keeps running while the host turns around)
void sync_checked(Ctx& c, const std::function<void()>& between = {});

// -------------------------------------------------------------- transfer.cu --
// Staged host->device copies through pinned buffers on host worker threads.
void upload_f64(Ctx& c, double* dst, const double* src, size_t n);
// one staged H2D pass over several host arrays (no pipeline drain between
// them); kinds: F64 copy, INDEX int64 -> int32 with lo <= a < hi, ROW_PTR
// int64 -> int32 monotone from 0 to hi (= nnz). Returns validity per segment.
struct UpSeg {
    enum Kind { F64, INDEX, ROW_PTR } kind;
    void* dst;
    const void* src;
    size_t n;
    int64_t lo, hi;
};
std::vector<bool> upload_many(Ctx& c, const std::vector<UpSeg>& segs);
// int64 -> int32 with lo <= a < hi; returns false on a violation
bool upload_index(Ctx& c, int32_t* dst, const int64_t* src, size_t n, int64_t lo, int64_t hi);
// CSR row pointers: monotone, [0] == 0, [n] == nnz
bool upload_row_ptr(Ctx& c, int32_t* dst, const int64_t* src, size_t n_plus_1, int64_t nnz);
void download_f64(Ctx& c, double* dst, const double* src, size_t n);
// x[0..n) = v on the context stream
void fill_f64(Ctx& c, int64_t n, double* dst, double v);
// longest row of A (blocking readback)
int64_t max_row_nnz(Ctx& c, const DevCsr& A);

// ---------------------------------------------------------------- sparse.cu --
// `extra`: further host arrays (already allocated device destinations) sent in
// the same staged pass as the matrix
std::unique_ptr<DevCsr> csr_upload(Ctx& c, int64_t nrows, int64_t ncols, const int64_t* rp,
                                   const int64_t* ci, const double* v,
                                   std::vector<UpSeg> extra = {});
void csr_download(Ctx& c, const DevCsr& A, int64_t* rp, int64_t* ci, double* v);
std::unique_ptr<DevCsr> csr_clone(Ctx& c, const DevCsr& A);
// recompute `single`, `group` and `finite` from device data (one readback)
void csr_finalize(Ctx& c, DevCsr& A);
// the same flags, read at the next sync_checked instead of now (the setup's
// Galerkin outputs: nothing before the next readback needs them). A must
// stay alive until then; rows == nnz falls back to csr_finalize (the lane
// policy depends on the `single` flag there).
void csr_finalize_deferred(Ctx& c, DevCsr& A);

// y = A x with lane group G (1,2,4,8,16,32); kernels return early when
// gate != nullptr && *gate != 0 (device-side loop termination).
void spmv(Ctx& c, const DevCsr& A, int G, const double* x, double* y, const int* gate = nullptr);
// r = b - A x
void residual(Ctx& c, const DevCsr& A, const double* b, const double* x, double* r,
              const int* gate = nullptr);
// l1-Jacobi sweep: xo = xi + (b - A xi) / d   (xi != xo)
void smooth_sweep(Ctx& c, const DevCsr& A, const double* d, const double* b, const double* xi,
                  double* xo, const int* gate = nullptr);
// the same three on rows [r0, r1) only (the partitioned cycle's interior /
// boundary split; every row's arithmetic unchanged)
void spmv_rows(Ctx& c, const DevCsr& A, int G, const double* x, double* y, const int* gate,
               int64_t r0, int64_t r1);
void residual_rows(Ctx& c, const DevCsr& A, const double* b, const double* x, double* r,
                   const int* gate, int64_t r0, int64_t r1);
void smooth_sweep_rows(Ctx& c, const DevCsr& A, const double* d, const double* b, const double* xi,
                       double* xo, const int* gate, int64_t r0, int64_t r1);
// first sweep from x = 0:  x = 0 + b / d
void smooth_from_zero(Ctx& c, int64_t n, const double* d, const double* b, double* x,
                      const int* gate = nullptr);
// x += 1.0 * (P xc) for a one-entry-per-row P
void prolong_correct(Ctx& c, const DevCsr& P, const double* xc, double* x,
                     const int* gate = nullptr);
void l1_diagonal(Ctx& c, const DevCsr& A, double* d); // throws like the reference
// l1 diagonal of a row block (local rows, local/ghost columns): no squareness
// check; the error index is the local row
void l1_diagonal_local(Ctx& c, const DevCsr& A, double* d, bool defer = false);
bool has_symmetric_pattern(Ctx& c, const DevCsr& A);
std::unique_ptr<DevCsr> transpose(Ctx& c, const DevCsr& A);
// transpose of a one-entry-per-row prolongator whose aggregates have at most
// max_members members: no csr_finalize readback (flags known on the host)
std::unique_ptr<DevCsr> transpose_agg(Ctx& c, const DevCsr& P, int max_members);
std::unique_ptr<DevCsr> spgemm(Ctx& c, const DevCsr& A, const DevCsr& B);

// -------------------------------------------------------------- matching.cu --
// Edge weights c_ij aligned with A's entries (diagonal slots hold -1, which
// Suitor never proposes along). Throws like build_weights.
// Partitioned matrices pass cg (global column ids) and g0 (global id of local
// row 0); columns >= nrows (ghosts) are masked out of the graph.
void build_weights_aligned(Ctx& c, const DevCsr& A, const double* w, DBuf<double>& wt,
                           int64_t& zero_edges, const int32_t* cg = nullptr, int64_t g0 = 0);
// the same into caller storage of A.nnz doubles
void build_weights_into(Ctx& c, const DevCsr& A, const double* w, double* wt,
                        int64_t& zero_edges, const int32_t* cg = nullptr, int64_t g0 = 0);
// build_weights + Suitor of a pairwise step, fused (the weights feed the
// candidate ranking directly); same checks/messages as build_weights, but
// DEFERRED to the next sync_checked — zero_edges must stay valid until then.
// Partitioned levels pass cg / g0 as for build_weights_aligned (ghost
// columns masked).
// pattern checks of the weights pass: check_upper = also verify the mirror
// of upper entries (lower entries always need theirs, for the value); a
// sym_flag replaces build_weights' asymmetry flag (build_hierarchy's own
// "matrix pattern is not symmetric" check, registered ahead of the others)
struct WeightsCheck {
    bool check_upper = true;
    int32_t* sym_flag = nullptr;
};
void weights_suitor(Ctx& c, const DevCsr& A, const double* w, int32_t* mate, int64_t& zero_edges,
                    const int32_t* cg = nullptr, int64_t g0 = 0, const WeightsCheck& chk = WeightsCheck{});
// Parallel Suitor over any CSR graph (rp, ci, wt); mate[v] = u or -1.
void suitor(Ctx& c, int64_t n, int64_t nnz, const int32_t* rp, const int32_t* ci, const double* wt,
            int32_t* mate);

// ---- global (cross-partition) matching, SURVEY.md §8f rank 1 (matching.cu) --
// The Suitor state of every part lives in one device block per part:
// [suitor words (16 B x n) | candidates (16 B x nnz) | rp (n + 1) | ncand (n)].
// A kernel of part `me` sees all parts' blocks through a pointer table (the
// same device for the loopback transport, NVLink peer mappings for NCCL).
constexpr int kMaxWorld = 16;
struct SuitorBlock {
    size_t s_off = 0, cand_off = 0, rp_off = 0, ncand_off = 0, bytes = 0;
};
SuitorBlock suitor_block(int64_t n, int64_t nnz);
struct SuitorView {
    int world = 1;
    int bounds[kMaxWorld + 1] = {}; // global row blocks of the level
    void* S[kMaxWorld] = {};
    const void* cand[kMaxWorld] = {};
    const int32_t* rp[kMaxWorld] = {};
    const int32_t* ncand[kMaxWorld] = {};
};
// diagonal of the owned rows (k_diag), positivity violations -> flag[0]
void diag_owned(Ctx& c, const DevCsr& A, const int32_t* cg, int64_t g0, double* dg, int32_t* flag);
// Edge weights of the owned rows over the extended column space (dg / w hold
// owned + ghost values). Entries to a LOWER part are not written (their
// weight is computed by that part from its upper entry and exchanged);
// flags: [asymmetric, non-finite]; zeros counted once per edge (lower end).
void weights_global(Ctx& c, const DevCsr& A, const int32_t* cg, int64_t g0, const double* dg,
                    const double* w, double* wt, int32_t* flags, unsigned long long* zeros);
// sorted admissible candidates of every row (ids = global vertex ids)
void candidates_into(Ctx& c, int64_t n, int64_t nnz, const int32_t* rp, const int32_t* ids,
                     const double* wt, void* cand, int32_t* ncand);
void suitor_global_init(Ctx& c, void* S, int64_t n);
// proposals of part `me`'s vertices; chains follow dislodged vertices of any
// part. sys = system-scope atomics (peer memory of other GPUs).
void suitor_global(Ctx& c, const SuitorView& g, int me, bool sys);
// mate (GLOBAL id, -1 unmatched) of part `me`'s vertices
void mate_global(Ctx& c, const SuitorView& g, int me, bool sys, int32_t* mate);

struct DevGraph {
    int64_t n = 0, nedges = 0, zero_edges = 0;
    DBuf<int32_t> xadj, adj;
    DBuf<double> wt;
};
// compact the aligned weights into a WeightedGraph (drops the diagonal)
std::unique_ptr<DevGraph> graph_from_aligned(Ctx& c, const DevCsr& A, const double* wt,
                                             int64_t zero_edges);

// -------------------------------------------------------------- coarsen.cu --
// Aggregates with member lists in ascending fine index (the rows of R = P^T).
struct DevAgg {
    int64_t n = 0, nc = 0, np = 0, ns = 0;
    DBuf<int32_t> agg_of;  // n
    DBuf<int32_t> mptr;    // >= nc + 1 entries (aggregate_from_mate: n + 1)
    DBuf<int32_t> members; // n
};
DevAgg aggregate_from_mate(Ctx& c, int64_t n, const int32_t* mate);
DevAgg aggregate_from_map(Ctx& c, int64_t n, int64_t nc, const int32_t* agg_of);
std::unique_ptr<DevCsr> build_prolongator(Ctx& c, const DevAgg& g, const double* w,
                                          bool defer = false);
// wc = P^T w with members of each aggregate in ascending order
void restrict_members(Ctx& c, const DevAgg& g, const double* pval, const double* w, double* wc);
// defer_finalize: the output's flags arrive at the next sync_checked (the
// setup's pairwise steps, which always reach one while the output lives)
std::unique_ptr<DevCsr> galerkin(Ctx& c, const DevCsr& A, const DevAgg& g, const double* pval,
                                 bool defer_finalize = false,
                                 const std::function<void()>& between = {});
// Galerkin with column data over A's (extended) column space: agg_ext / pv_ext
// give the global coarse id and p value of every local column (owned and
// ghost); members are local rows; the output has ncols_out (global) columns.
std::unique_ptr<DevCsr> galerkin_ext(Ctx& c, const DevCsr& A, const DevAgg& g,
                                     const int32_t* agg_ext, const double* pv_ext,
                                     int64_t ncols_out, bool defer_finalize = false,
                                     const std::function<void()>& between = {});
// wc[a] = 0.0 + sum over R's row a of R_ae * w_e (restrict_vector for any P)
void restrict_rows(Ctx& c, const DevCsr& R, const double* w, double* wc);
// P (one entry per row) -> member structure
DevAgg aggregates_of(Ctx& c, const DevCsr& P);

struct DevStep {
    std::unique_ptr<DevCsr> P, Ac;
    DBuf<double> wc;
    int64_t zero_edges = 0;
};
DevStep pairwise_step(Ctx& c, const DevCsr& A, const double* w, const WeightsCheck& chk = WeightsCheck{});
DevStep double_pairwise(Ctx& c, const DevCsr& A, const double* w, const WeightsCheck& chk = WeightsCheck{});

struct KWork; // K-cycle workspace of a level (solve.cu), allocated on first use

// one-launch coarsest solve (coarsest.cu); cs == 0 -> not applicable
// (per-sweep kernels).
// MAMG_COARSEST=0 keeps the per-sweep kernels.
struct CoarsestPlan {
    int cs = 0, rpc = 0, width = 0; // cluster size, rows per CTA, ELL width
    size_t smem = 0;                // dynamic shared memory per CTA
    DBuf<uint32_t> readers;         // per row: bitmask of the CTAs that read x_i
};
bool coarsest_plan(Ctx& c, const DevCsr& A, CoarsestPlan& p);
void coarsest_launch(Ctx& c, const DevCsr& A, const double* l1, const CoarsestPlan& p,
                     const double* b, double* x_out, int k, const int* gate);

struct DevLevel {
    std::unique_ptr<DevCsr> A, P, R;
    DBuf<double> l1, w;
    // cycle workspace: working x and scratch (n_k), coarse b / x (n_{k+1})
    DBuf<double> xw, scratch, cb, cx;
    std::shared_ptr<KWork> kw;
};

struct DevHier {
    std::vector<DevLevel> lv;
    bool stalled = false;
    int64_t zero_edges = 0;
    CoarsestPlan coarsest; // plan of the one-launch coarsest solve (last level)
    ~DevHier();
    int nl() const { return static_cast<int>(lv.size()); }
};

std::unique_ptr<DevHier> build_hierarchy(Ctx& c, const DevCsr& A, const double* w,
                                         const mamg_setup_cfg& cfg);
// the same, level 0 taking `owned` (== A's storage) instead of a copy of A
std::unique_ptr<DevHier> build_hierarchy_owned(Ctx& c, const DevCsr& A,
                                               std::unique_ptr<DevCsr> owned, const double* w,
                                               const mamg_setup_cfg& cfg);
void alloc_workspace(Ctx& c, DevHier& h);
// continue a hierarchy from its last level (A, w, l1 set) with an explicit
// stop bound / level budget (the agglomerated tail of the partitioned path)
void grow_hierarchy(Ctx& c, DevHier& h, double bound, int max_levels, int aggregation,
                    int32_t* sym_flag = nullptr);
// a hierarchy whose level 0 is (A, w) but whose stop rule is `bound`,
// `max_levels` (the levels below the partitioned path's agglomeration point)
std::unique_ptr<DevHier> build_hierarchy_sub(Ctx& c, std::unique_ptr<DevCsr> A, DBuf<double> w,
                                             double bound, int max_levels, int aggregation);

// ----------------------------------------------------------- generators.cu --
// The BASELINE generators assembled on the device, bit-identical to the host
// ones (csrc/host/problems.cpp); sigma > 0 draws the permeability on the host.
std::unique_ptr<DevCsr> gen_nine_point_dev(Ctx& c, int64_t nx, int64_t ny, double a, double b,
                                           double cc);
std::unique_ptr<DevCsr> gen_randk3d_dev(Ctx& c, int64_t nx, int64_t ny, int64_t nz, double sigma,
                                        uint64_t seed);
std::unique_ptr<DevCsr> gen_jump3d_dev(Ctx& c, int64_t nx, int64_t ny, int64_t nz, int64_t block,
                                       uint64_t seed, double lo, double hi);
std::unique_ptr<DevCsr> gen_aniso27_dev(Ctx& c, int64_t nx, int64_t ny, int64_t nz, double kx,
                                        double ky, double kz);
std::unique_ptr<DevCsr> gen_elast3d_dev(Ctx& c, int64_t nx, int64_t ny, int64_t nz, double mu,
                                        double lambda);

// ---------------------------------------------------------------- solve.cu --
void apply_cycle(Ctx& c, DevHier& h, int level, const mamg_cycle_cfg& cfg, const double* b,
                 double* x, bool x_is_zero, const int* gate = nullptr);
void l1_jacobi(Ctx& c, const DevCsr& A, const double* d, const double* b, double* x, int k);

// blocked deterministic reductions (proj/src/vector_ops.cpp:12-46)
double dot(Ctx& c, int64_t n, const double* x, const double* y);
void triple_dot(Ctx& c, int64_t n, const double* w, const double* r, const double* v,
                const double* q, double* out3);
void axpy(Ctx& c, int64_t n, double* y, double a, const double* x, const int* gate = nullptr);
void axpy_pair(Ctx& c, int64_t n, double* y1, double* y2, const double* x, double a, double b);

int pcg_solve(Ctx& c, const DevCsr& A, DevHier* h, const mamg_cycle_cfg* cyc,
              mamg_host_precond hp, void* user, const double* b, const double* u0,
              const mamg_solve_cfg& cfg, double* u, double* hist, mamg_report* rep);

// Warp-wide bitonic sort network over 32 Q register-held elements, element
// q of a lane at position Q lane + q: the strides below Q pair elements of
// the same lane (register swaps), the others exchange element q with lane
// lane ^ (j / Q) — log2(Q) of every merge's stages need no shuffle (15
// shuffle stages for Q = 4 or 8 instead of 25 / 30 with position lane + 32 q).
// first(a, b): a sorts before b (a strict total order).
template <int Q, class T, class First, class Shfl>
__device__ __forceinline__ void warp_bitonic(T (&x)[Q], int lane, First first, Shfl shfl) {
    constexpr int N = 32 * Q;
#pragma unroll
    for (int k = 2; k <= N; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (j < Q) {
#pragma unroll
                for (int q = 0; q < Q; ++q) {
                    const int qp = q ^ j;
                    if (qp > q) {
                        const bool asc = ((Q * lane + q) & k) == 0;
                        if (first(x[qp], x[q]) == asc) {
                            const T t = x[q];
                            x[q] = x[qp];
                            x[qp] = t;
                        }
                    }
                }
            } else {
                const bool lower = (lane & (j / Q)) == 0;
#pragma unroll
                for (int q = 0; q < Q; ++q) {
                    const T o = shfl(x[q], j / Q);
                    const bool asc = ((Q * lane + q) & k) == 0;
                    // the lower position of an ascending pair keeps the one that comes first
                    if (first(o, x[q]) == (asc == lower)) x[q] = o;
                }
            }
        }
    }
}

} // namespace mamg
