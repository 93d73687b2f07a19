// dist.cuh — row-block partitioned hierarchy and solve.
//
// Every level is split into contiguous row blocks ("parts", one per rank).
// A part stores its rows with LOCAL column ids: owned columns first
// (0..nowned), then ghost columns (nowned..nowned+nghost) in ascending global
// order, so a row keeps the reference's entry order (and hence its exact
// summation tree) while its gathers stay local. Matching runs on the local
// graph block only; Galerkin, prolongation and smoothing use the full rows.
// Ghost values travel through a per-level halo plan built locally: the
// pattern is structurally symmetric, so the rows part q must send to part r
// are exactly q's rows with a column owned by r (verified by exchanging the
// counts). Level-0 blocks start at multiples of 2048 rows, so the
// rank-ordered concatenation of the parts' block partials IS the
// unpartitioned partial array and every dot product is bit-identical.
//
// The transport (Comm) is NCCL for one rank per process / GPU, or a loopback
// that keeps all parts in this process (used to verify the partitioned
// numerics on a single device against the partition-aware oracle). The
// setup's exchanges go through it (send-recv halos, allgathers); the solve
// loop at world > 1 uses peer memory instead (shared_blocks: CUDA IPC over
// NVLink): halo mailboxes (peer_halo.cu), dot partials stored into every
// rank's buffer (solve.cu k_blockdot peer mode), the agglomeration gather.
// Optional: matching across parts (dist_global.cu), agglomeration of the
// small coarse levels onto every rank (DistHier::rep).
#pragma once

#include <memory>
#include <string>
#include <vector>

#include "ops.cuh"

namespace mamg {

constexpr int64_t kPartAlign = 2048; // level-0 block boundary alignment (= dot block)

struct Halo {
    int64_t nowned = 0, nghost = 0;
    std::vector<int64_t> send_off; // world + 1 offsets into send_idx, by destination rank
    std::vector<int64_t> recv_off; // world + 1 offsets into the ghost region, by source rank
    DBuf<int32_t> send_idx;        // owned rows to pack, grouped by destination
    DBuf<double> send_f64;
    DBuf<int32_t> send_i32;
};

struct PLevel {
    int64_t g0 = 0;                  // global id of local row 0
    int64_t nglob = 0, nnzglob = 0;  // global level size / nnz
    std::vector<int64_t> bounds;     // global block boundaries (world + 1)
    std::unique_ptr<DevCsr> A;       // local rows; ci = local ids, ncols = nowned + nghost
    DBuf<int32_t> cg;                // A's global column ids (entry-aligned)
    DBuf<int32_t> ghost_g;           // global id of every ghost slot
    std::unique_ptr<DevCsr> P, R;    // local fine rows -> local coarse columns
    DBuf<double> l1, w;
    Halo halo;
    // global matching mode (aggregates may straddle parts): R's columns are
    // owned rows + rhalo slots (fine values of remote members, received
    // before the restriction), P's columns own coarse rows + phalo slots
    // (coarse values of remote aggregates, received before the
    // prolongation); Pg / Rg hold their global column ids
    Halo rhalo, phalo;
    DBuf<int32_t> Pg, Rg;
    // interior rows [ia, ib): the longest run of rows without a ghost column
    // (computed per build for the overlap of halos with the interior rows)
    int64_t ia = 0, ib = 0;
    int interior_gen = -1;
    DBuf<double> xw, scratch, cb, cx; // cycle workspace (xw, scratch, cx hold ghost room)
};

struct Part {
    int rank = 0;
    std::vector<PLevel> lv;
};

class Comm {
public:
    virtual ~Comm() = default;
    int world = 1;
    std::vector<int> ranks; // ranks of the parts living in this process (ascending)

    // Fill the ghost region x[nowned .. nowned + nghost) of every local part.
    virtual void halo_f64(Ctx& c, const std::vector<Halo*>& h, const std::vector<double*>& x) = 0;
    virtual void halo_i32(Ctx& c, const std::vector<Halo*>& h, const std::vector<int32_t*>& x) = 0;
    // Host allgather: one value per local part -> `world` values in rank order.
    virtual std::vector<int64_t> allgather(Ctx& c, const std::vector<int64_t>& mine) = 0;
    // The same with `len` values per part (mine: part-major) -> world x len,
    // rank-major: one collective instead of `len`.
    virtual std::vector<int64_t> allgather_n(Ctx& c, const std::vector<int64_t>& mine, int len) = 0;
    // Device allgather: rank q contributes counts[q] doubles (src of its part);
    // every local part receives the rank-ordered concatenation in dst.
    virtual void allgather_f64(Ctx& c, const std::vector<const double*>& src,
                               const std::vector<int64_t>& counts,
                               const std::vector<double*>& dst) = 0;
    virtual void allgather_i32(Ctx& c, const std::vector<const int32_t*>& src,
                               const std::vector<int64_t>& counts,
                               const std::vector<int32_t*>& dst) = 0;
    // equal-count allgather (one collective): rank q's `count` doubles land at
    // dst + q * count (parts sharing one dst pointer are filled once)
    virtual void allgather_equal_f64(Ctx& c, const std::vector<const double*>& src, int64_t count,
                                     const std::vector<double*>& dst) = 0;
    // Device memory every rank can address: each local part asks for
    // `bytes[i]`; returns the `world` block pointers (rank order) valid in
    // this process's kernels — the parts' own blocks for the loopback, NVLink
    // peer mappings (CUDA IPC) of the other ranks' blocks for NCCL. Blocks are
    // kept and grown across calls; pointers stay valid until the next call.
    // `slot` selects an independent set of blocks (0: global Suitor, 1: the
    // partitioned PCG's peer reductions, 2: the peer halo mailboxes).
    virtual std::vector<void*> shared_blocks(Ctx& c, const std::vector<size_t>& bytes,
                                             int slot = 0) = 0;
    // stream-ordered barrier: work queued after it on c.stream starts after
    // every rank's work queued before it has completed
    virtual void barrier(Ctx& c) = 0;
    virtual bool peer_memory() const { return false; } // blocks of other GPUs
    // the collectives may be captured into a CUDA graph (stream-ordered, no
    // host-side wait); false: the partitioned PCG replays no graphs
    virtual bool capturable() const { return true; }
};

// One CUDA-IPC mapped device block per rank (Comm::shared_blocks of the
// multi-process transports): grown on demand, handles exchanged through the
// Comm's host allgather; pointers valid until the next get().
struct IpcBlocks {
    void* mine = nullptr;
    size_t cap = 0;
    std::vector<void*> peers;
    std::vector<void*> get(Ctx& c, Comm& comm, size_t bytes);
    void close_peers();
    void release();
};

// Run f — local work that may raise a check failure (mamg::Error) and
// contains no collective — at a point every rank reaches: a failure on any
// rank is raised on every rank (the failing rank with its own message), so no
// process is left waiting in a later collective.
template <class F>
void on_all_ranks(Ctx& c, Comm& comm, F&& f) {
    int code = 0;
    std::string msg;
    int64_t idx = -1;
    try {
        f();
    } catch (const Error& e) {
        code = e.status;
        msg = e.what();
        idx = e.index;
    }
    const auto all = comm.allgather(c, std::vector<int64_t>(comm.ranks.size(), code));
    if (code) throw Error(code, msg, idx);
    for (int r = 0; r < comm.world; ++r)
        if (all[r])
            throw Error(static_cast<int>(all[r]),
                        "partitioned build: a check failed on rank " + std::to_string(r), -1);
}

std::unique_ptr<Comm> make_loopback_comm(int world);
std::unique_ptr<Comm> make_nccl_comm(Ctx& c, int rank, int world, const void* unique_id);
// one rank per process on ONE node without NCCL (shm_comm.cu): host
// collectives through a POSIX shared-memory segment `name` (every rank passes
// the same name), device data through CUDA-IPC blocks. Ranks may share a GPU.
std::unique_ptr<Comm> make_shm_comm(Ctx& c, int rank, int world, const char* name);
// ranks as threads of ONE process (one rank per device, or several on one
// device for tests): host collectives through the group's memory, device data
// through directly shared cudaMalloc blocks (peer access across devices)
struct ThreadGroup {
    explicit ThreadGroup(int world);
    int world;
    std::vector<int64_t> mem; // the collective segment (zeroed)
};
std::unique_ptr<Comm> make_thread_comm(Ctx& c, int rank, ThreadGroup& g);
// the shm transport's host collective alone (no CUDA): attach, allgather, detach
std::vector<int64_t> shm_allgather_once(const char* name, int world, int rank, const int64_t* mine,
                                        int64_t len);
int nccl_unique_id(void* out128);

// Peer-memory halo exchange of the partitioned cycle (peer_halo.cu): per
// partitioned level, every part owns a mailbox (two parities x its ghost
// count) plus arrival / epoch / error counters in a slot-2 shared block;
// senders store boundary values straight into the receivers' mailboxes.
struct PeerDest {
    int64_t start, cnt;             // segment of the part's send list
    double* mbox;                   // receiver's mailbox (parity 0)
    int64_t seg, ng;                // my slot offset there, its ghost count
    unsigned long long* arrive;     // receiver's arrival counter
};
struct PeerHaloLevel {
    int64_t ng = 0;
    double* mbox = nullptr;
    unsigned long long* ctrs = nullptr; // [arrive, epoch, err]
    int nsrc = 0, ndst = 0;
    DBuf<PeerDest> dests;
    DBuf<unsigned> cta; // last-CTA counter of the push kernel
};
struct PeerHalo {
    bool on = false;
    int gen = -1;                               // build generation it was set up for
    uint64_t layout = 0;                        // fingerprint of the halo layouts it encodes
    std::vector<std::vector<PeerHaloLevel>> lv; // [part][level]
    // allgather of the restricted residual into the agglomerated levels:
    // the same push/unpack with every rank a destination ("mailbox" =
    // the full coarse vector) and the own rows repeated once per rank
    std::vector<PeerHaloLevel> ag;              // [part]
    std::vector<DBuf<int32_t>> ag_idx;          // [part] own rows x world
};

struct DistHier {
    std::unique_ptr<Comm> comm;
    PeerHalo peer;
    int gen = 0; // incremented by every dist_build
    // 0: matching on each part's local graph block (north star); 1: global
    // Suitor across parts, aggregates may straddle parts -> hierarchy and
    // solve bit-identical to the unpartitioned build
    int matching = 0;
    // Agglomeration: the first level k >= 1 with at most `agglom_rows` rows is
    // gathered onto every rank (one copy per process) and it and all coarser
    // levels are built and cycled by the single-device code (`rep`, its level
    // 0 = level agg_level): one allgather per visit replaces the per-sweep
    // halos of small, latency-bound levels. 0 disables.
    int64_t agglom_rows = 262144;
    int agg_level = -1;
    std::unique_ptr<DevHier> rep;
    DBuf<double> rep_b, rep_x; // full-size right-hand side / iterate of rep's level 0
    std::vector<Part> parts; // parts of this process, rank order
    int nl = 0;
    bool stalled = false;
    int64_t zero_edges = 0;
    std::vector<int64_t> level_n, level_nnz; // global sizes per level
    // level-0 input kept device-resident (dist_load) so dist_build can rerun
    std::vector<std::unique_ptr<DevCsr>> A0; // the loaded level-0 blocks
    std::vector<DBuf<double>> w0;
    bool consume_level0 = false; // the next build takes A0 / w0 (no copy)
    int64_t n0 = 0, nnz0 = 0;
    // how the last dist_pcg ran: [0] peer reductions, [1] peer halos,
    // [2] halo/interior overlap, [3] iteration graphs replayed
    int last_solve[4] = {0, 0, 0, 0};
};

// level-0 block boundaries (multiples of kPartAlign, the last one n)
std::vector<int64_t> dist_bounds(int64_t n, int world);

// Upload this process's row blocks of the full host matrix (every process
// passes the same matrix and keeps its own rows).
void dist_load(Ctx& c, DistHier& d, int64_t n, const int64_t* rp, const int64_t* ci,
               const double* v, const double* w);
// Partition-aware build_hierarchy from the loaded (device-resident) blocks.
void dist_build(Ctx& c, DistHier& d, const mamg_setup_cfg& cfg);
// dist_load + dist_build
void dist_setup(Ctx& c, DistHier& d, int64_t n, const int64_t* rp, const int64_t* ci,
                const double* v, const double* w, const mamg_setup_cfg& cfg);

// Partitioned PCG with the device V/W cycle. h_b: full right-hand side (or
// null = ones); h_u0: full initial guess (null = zero); h_u receives the
// owned rows of the local parts.
int dist_pcg(Ctx& c, DistHier& d, const mamg_cycle_cfg& cyc, const double* h_b,
             const mamg_solve_cfg& cfg, double* h_u, double* hist, mamg_report* rep,
             const double* h_u0 = nullptr);

// device ms of one partitioned level-0 sweep (what 0, no halo) or one
// preconditioner application with halos (what 1), mean over reps (solve.cu)
double dist_time(Ctx& c, DistHier& d, int what, const mamg_cycle_cfg& cyc, int reps);

// --- global matching mode (dist_global.cu) ---
// build the next level of every local part with the global Suitor: sets the
// fine level's P, R, Pg, Rg, rhalo, phalo and returns the coarse levels
// (GLOBAL columns, not yet localized) with their w; cbounds = coarse blocks.
// Returns false on a stall (no level appended).
bool dist_step_global(Ctx& c, DistHier& d, int k, int aggregation, std::vector<PLevel>& coarse,
                      int64_t& zero_edges);
// Turn a part's level matrix (local rows, GLOBAL columns in A->ci) into the
// local-column form and build its halo plan (dist.cu)
void localize(Ctx& c, int world, int rank, PLevel& L);
void set_policy(DevCsr& M, int64_t nrows_glob, int64_t nnz_glob, bool single);
int64_t sum_all(const std::vector<int64_t>& v);
std::vector<int64_t> prefix_of(const std::vector<int64_t>& counts);

// Set up (once per build) and reset (every solve) the peer halo mailboxes of
// levels [0, nlev); returns false (NCCL / loopback halos stay in use) when
// disabled (MAMG_DIST_NCCL_HALO=1) or when any rank cannot map its peers.
bool peer_halo_prepare(Ctx& c, DistHier& d, int nlev);
// halo exchange of level k's vectors x (one per local part) through the mailboxes
void peer_halo_exchange(Ctx& c, DistHier& d, int k, const std::vector<double*>& x);
// interior row ranges of the partitioned levels [0, nlev) (once per build)
void interior_ranges(Ctx& c, DistHier& d, int nlev);
// allgather of every part's own rows of the agglomeration level (cb) into out
// (the full vector; out may be shared by the in-process parts)
void peer_agg_gather(Ctx& c, DistHier& d, const std::vector<const double*>& cb, double* out);
// any bounded wait of this solve timed out (collective protocol fault)
bool peer_halo_failed(Ctx& c, DistHier& d);

// one-entry-per-row product P1 * P2 (kernels.cpp:272-281 for 1-entry rows)
std::unique_ptr<DevCsr> compose_single(Ctx& c, const DevCsr& P1, const DevCsr& P2);

} // namespace mamg
