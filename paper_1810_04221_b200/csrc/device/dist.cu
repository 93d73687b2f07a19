// dist.cu — partitioned setup (partition-aware build_hierarchy) and the two
// transports. See dist.cuh for the data layout and the parity argument.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>

#include <nccl.h>

#include "dist.cuh"

namespace mamg {
namespace {

constexpr int kBlock = 256;

// ------------------------------------------------------------- localize --
__global__ void k_mark_ghosts(int64_t n, int64_t g0, const int32_t* __restrict__ rp,
                              const int32_t* __restrict__ cg, int32_t* marker) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    for (int k = rp[i]; k < rp[i + 1]; ++k) {
        const int64_t j = cg[k];
        if (j < g0 || j >= g0 + n) marker[j] = 1;
    }
}

// after the exclusive scan: slot[j] = ghost slot of global column j
__global__ void k_ghost_list(int64_t nglob, const int32_t* __restrict__ slot, int32_t* ghost_g) {
    const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= nglob) return;
    if (slot[j + 1] != slot[j]) ghost_g[slot[j]] = static_cast<int32_t>(j);
}

__global__ void k_localize(int64_t n, int64_t g0, const int32_t* __restrict__ rp,
                           const int32_t* __restrict__ cg, const int32_t* __restrict__ slot,
                           int32_t* ci) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    for (int k = rp[i]; k < rp[i + 1]; ++k) {
        const int64_t j = cg[k];
        ci[k] = (j >= g0 && j < g0 + n) ? static_cast<int32_t>(j - g0)
                                        : static_cast<int32_t>(n + slot[j]);
    }
}

// rows of this part with a column in [lo, hi) (global) -> flag
__global__ void k_touches(int64_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ cg,
                          int64_t lo, int64_t hi, int32_t* flag) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int f = 0;
    for (int k = rp[i]; k < rp[i + 1]; ++k) f |= (cg[k] >= lo && cg[k] < hi);
    flag[i] = f;
}

__global__ void k_compact_rows(int64_t n, const int32_t* __restrict__ pos, int32_t* out) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (pos[i + 1] != pos[i]) out[pos[i]] = static_cast<int32_t>(i);
}

// local pattern symmetry among owned entries (csr.cpp:106-112 restricted
// to the block; cross-block symmetry is checked through the halo counts)
__global__ void k_sym_owned(int64_t n, int64_t g0, const int32_t* __restrict__ rp,
                            const int32_t* __restrict__ cg, int32_t* ok) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int gi = static_cast<int>(g0 + i);
    for (int k = rp[i]; k < rp[i + 1]; ++k) {
        const int64_t j = cg[k] - g0;
        if (j < 0 || j >= n) continue;
        int lo = rp[j], hi = rp[j + 1];
        while (lo < hi) {
            const int mid = lo + ((hi - lo) >> 1); // no int32 overflow past 2^30 entries
            if (cg[mid] < gi)
                lo = mid + 1;
            else
                hi = mid;
        }
        if (lo >= rp[j + 1] || cg[lo] != gi) {
            *ok = 0;
            return;
        }
    }
}

// owned part of the extended column arrays: global coarse id and p value
__global__ void k_ext_owned(int64_t n, const int32_t* __restrict__ agg, int64_t coff,
                            const double* __restrict__ p, int32_t* agg_ext, double* pv_ext) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    agg_ext[i] = static_cast<int32_t>(agg[i] + coff);
    pv_ext[i] = p[i];
}

__global__ void k_fill_ones(int64_t n, double* x) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) x[i] = 1.0;
}

template <class T>
__global__ void k_pack(int64_t m, const int32_t* __restrict__ idx, const T* __restrict__ x, T* out) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t < m) out[t] = x[idx[t]];
}

template <class T>
void pack(Ctx& c, Halo& h, const T* x, T* out) {
    const int64_t m = h.send_off.empty() ? 0 : h.send_off.back();
    if (m == 0) return;
    k_pack<<<blocks_for(m, kBlock), kBlock, 0, c.stream>>>(m, h.send_idx.get(), x, out);
    c.count();
}

// ------------------------------------------------------------ loopback --
class LoopbackComm : public Comm {
public:
    explicit LoopbackComm(int w) {
        world = w;
        for (int r = 0; r < w; ++r) ranks.push_back(r);
    }
    template <class T>
    void halo(Ctx& c, const std::vector<Halo*>& h, const std::vector<T*>& x, bool dbl) {
        for (int r = 0; r < world; ++r) {
            T* buf = dbl ? reinterpret_cast<T*>(h[r]->send_f64.get())
                         : reinterpret_cast<T*>(h[r]->send_i32.get());
            pack<T>(c, *h[r], x[r], buf);
        }
        for (int r = 0; r < world; ++r)
            for (int q = 0; q < world; ++q) {
                if (q == r) continue;
                const int64_t cnt = h[r]->recv_off[q + 1] - h[r]->recv_off[q];
                if (!cnt) continue;
                const T* src = dbl ? reinterpret_cast<const T*>(h[q]->send_f64.get())
                                   : reinterpret_cast<const T*>(h[q]->send_i32.get());
                MAMG_CU(cudaMemcpyAsync(x[r] + h[r]->nowned + h[r]->recv_off[q],
                                        src + h[q]->send_off[r], cnt * sizeof(T),
                                        cudaMemcpyDeviceToDevice, c.stream));
            }
    }
    void halo_f64(Ctx& c, const std::vector<Halo*>& h, const std::vector<double*>& x) override {
        halo<double>(c, h, x, true);
    }
    void halo_i32(Ctx& c, const std::vector<Halo*>& h, const std::vector<int32_t*>& x) override {
        halo<int32_t>(c, h, x, false);
    }
    std::vector<int64_t> allgather(Ctx&, const std::vector<int64_t>& mine) override { return mine; }
    std::vector<int64_t> allgather_n(Ctx&, const std::vector<int64_t>& mine, int) override {
        return mine;
    }
    std::vector<void*> shared_blocks(Ctx& c, const std::vector<size_t>& bytes, int slot) override {
        auto& bl = blocks_[slot % 3];
        bl.resize(world);
        std::vector<void*> out(world);
        for (int r = 0; r < world; ++r) {
            if (bl[r].size() < bytes[r]) bl[r].alloc(bytes[r] + bytes[r] / 8, c.stream);
            out[r] = bl[r].get();
        }
        return out;
    }
    void barrier(Ctx&) override {} // one stream: program order
    template <class T>
    void gather(Ctx& c, const std::vector<const T*>& src, const std::vector<int64_t>& counts,
                const std::vector<T*>& dst) {
        for (int r = 0; r < world; ++r) {
            if (r > 0 && dst[r] == dst[0]) continue; // one shared destination
            int64_t off = 0;
            for (int q = 0; q < world; ++q) {
                if (counts[q])
                    MAMG_CU(cudaMemcpyAsync(dst[r] + off, src[q], counts[q] * sizeof(T),
                                            cudaMemcpyDeviceToDevice, c.stream));
                off += counts[q];
            }
        }
    }
    void allgather_f64(Ctx& c, const std::vector<const double*>& src,
                       const std::vector<int64_t>& counts, const std::vector<double*>& dst) override {
        gather<double>(c, src, counts, dst);
    }
    void allgather_i32(Ctx& c, const std::vector<const int32_t*>& src,
                       const std::vector<int64_t>& counts, const std::vector<int32_t*>& dst) override {
        gather<int32_t>(c, src, counts, dst);
    }
    void allgather_equal_f64(Ctx& c, const std::vector<const double*>& src, int64_t count,
                             const std::vector<double*>& dst) override {
        gather<double>(c, src, std::vector<int64_t>(world, count), dst);
    }

private:
    std::vector<DBuf<char>> blocks_[3];
};

// ---------------------------------------------------------------- NCCL --
#define MAMG_NCCL(x)                                                                   \
    do {                                                                               \
        ncclResult_t r_ = (x);                                                         \
        if (r_ != ncclSuccess)                                                         \
            throw Error(MAMG_NCCL, std::string("NCCL error ") + ncclGetErrorString(r_) + \
                                       " in " #x);                                     \
    } while (0)

class NcclComm : public Comm {
public:
    NcclComm(Ctx& c, int rank, int w, const void* uid) {
        world = w;
        ranks.push_back(rank);
        ncclUniqueId id;
        std::memcpy(&id, uid, sizeof(id));
        MAMG_NCCL(ncclCommInitRank(&comm_, w, id, rank));
        tmp_.alloc(2 * static_cast<size_t>(w), c.stream);
    }
    ~NcclComm() override {
        for (auto& sh : sh_) sh.release();
        if (comm_) ncclCommDestroy(comm_);
    }
    bool peer_memory() const override { return world > 1; }
    void barrier(Ctx& c) override {
        MAMG_NCCL(ncclAllReduce(tmp_.get(), tmp_.get(), 1, ncclInt64, ncclSum, comm_, c.stream));
    }
    std::vector<void*> shared_blocks(Ctx& c, const std::vector<size_t>& bytes, int slot) override {
        return sh_[slot % 3].get(c, *this, bytes[0]);
    }
    template <class T>
    void halo(Ctx& c, Halo& h, T* x, T* buf, ncclDataType_t ty) {
        pack<T>(c, h, x, buf);
        const int me = ranks[0];
        MAMG_NCCL(ncclGroupStart());
        for (int q = 0; q < world; ++q) {
            if (q == me) continue;
            const int64_t sc = h.send_off[q + 1] - h.send_off[q];
            const int64_t rc = h.recv_off[q + 1] - h.recv_off[q];
            if (sc) MAMG_NCCL(ncclSend(buf + h.send_off[q], sc, ty, q, comm_, c.stream));
            if (rc) MAMG_NCCL(ncclRecv(x + h.nowned + h.recv_off[q], rc, ty, q, comm_, c.stream));
        }
        MAMG_NCCL(ncclGroupEnd());
    }
    void halo_f64(Ctx& c, const std::vector<Halo*>& h, const std::vector<double*>& x) override {
        halo<double>(c, *h[0], x[0], h[0]->send_f64.get(), ncclDouble);
    }
    void halo_i32(Ctx& c, const std::vector<Halo*>& h, const std::vector<int32_t*>& x) override {
        halo<int32_t>(c, *h[0], x[0], h[0]->send_i32.get(), ncclInt32);
    }
    std::vector<int64_t> allgather(Ctx& c, const std::vector<int64_t>& mine) override {
        std::vector<int64_t> all(world);
        MAMG_CU(cudaMemcpyAsync(tmp_.get(), mine.data(), sizeof(int64_t), cudaMemcpyHostToDevice,
                                c.stream));
        MAMG_NCCL(ncclAllGather(tmp_.get(), tmp_.get() + world, 1, ncclInt64, comm_, c.stream));
        MAMG_CU(cudaMemcpyAsync(all.data(), tmp_.get() + world, sizeof(int64_t) * world,
                                cudaMemcpyDeviceToHost, c.stream));
        c.sync();
        return all;
    }
    std::vector<int64_t> allgather_n(Ctx& c, const std::vector<int64_t>& mine, int len) override {
        std::vector<int64_t> all(static_cast<size_t>(world) * len);
        if (len <= 0) return all;
        if (tmpn_.size() < static_cast<size_t>(world + 1) * len)
            tmpn_.alloc(static_cast<size_t>(world + 1) * len, c.stream);
        MAMG_CU(cudaMemcpyAsync(tmpn_.get(), mine.data(), sizeof(int64_t) * len,
                                cudaMemcpyHostToDevice, c.stream));
        MAMG_NCCL(ncclAllGather(tmpn_.get(), tmpn_.get() + len, len, ncclInt64, comm_, c.stream));
        MAMG_CU(cudaMemcpyAsync(all.data(), tmpn_.get() + len, sizeof(int64_t) * all.size(),
                                cudaMemcpyDeviceToHost, c.stream));
        c.sync();
        return all;
    }
    template <class T>
    void gather(Ctx& c, const T* src, const std::vector<int64_t>& counts, T* dst,
                ncclDataType_t ty) {
        const int me = ranks[0];
        int64_t off = 0;
        MAMG_NCCL(ncclGroupStart());
        for (int q = 0; q < world; ++q) {
            if (counts[q])
                MAMG_NCCL(ncclBroadcast(q == me ? src : dst + off, dst + off, counts[q], ty, q,
                                        comm_, c.stream));
            off += counts[q];
        }
        MAMG_NCCL(ncclGroupEnd());
    }
    void allgather_f64(Ctx& c, const std::vector<const double*>& src,
                       const std::vector<int64_t>& counts, const std::vector<double*>& dst) override {
        gather<double>(c, src[0], counts, dst[0], ncclDouble);
    }
    void allgather_i32(Ctx& c, const std::vector<const int32_t*>& src,
                       const std::vector<int64_t>& counts, const std::vector<int32_t*>& dst) override {
        gather<int32_t>(c, src[0], counts, dst[0], ncclInt32);
    }
    void allgather_equal_f64(Ctx& c, const std::vector<const double*>& src, int64_t count,
                             const std::vector<double*>& dst) override {
        if (count) MAMG_NCCL(ncclAllGather(src[0], dst[0], count, ncclDouble, comm_, c.stream));
    }

private:
    ncclComm_t comm_ = nullptr;
    DBuf<int64_t> tmp_, tmpn_;
    IpcBlocks sh_[3];
};

} // namespace

// ------------------------------------------------------ IPC shared blocks --
// Each rank cudaMallocs its block (IPC needs a plain allocation), publishes
// the handle through the Comm's host allgather and opens every peer's with
// lazy peer access (NVLink across GPUs; the same device across processes).
// Re-published only when some rank had to grow.
std::vector<void*> IpcBlocks::get(Ctx& c, Comm& comm, size_t bytes) {
    const int me = comm.ranks[0], world = comm.world;
    const int grow = bytes > cap ? 1 : 0;
    const auto g = comm.allgather(c, {grow});
    bool any = peers.empty();
    for (auto x : g) any = any || x != 0;
    if (!any) return peers;
    c.sync(); // my kernels are done with the old blocks
    close_peers();
    comm.allgather(c, {0}); // every rank has unmapped the old blocks
    if (grow) {
        if (mine) MAMG_CU(cudaFree(mine));
        mine = nullptr;
        cap = std::max<size_t>(bytes + bytes / 8, 1 << 20);
        MAMG_CU(cudaMalloc(&mine, cap));
    }
    cudaIpcMemHandle_t h;
    MAMG_CU(cudaIpcGetMemHandle(&h, mine));
    static_assert(sizeof(h) == 64, "IPC handle size");
    std::vector<int64_t> words(8);
    std::memcpy(words.data(), &h, sizeof(h));
    const auto all = comm.allgather_n(c, words, 8);
    peers.assign(world, nullptr);
    for (int r = 0; r < world; ++r) {
        if (r == me) {
            peers[r] = mine;
            continue;
        }
        cudaIpcMemHandle_t hr;
        std::memcpy(&hr, all.data() + static_cast<size_t>(r) * 8, sizeof(hr));
        MAMG_CU(cudaIpcOpenMemHandle(&peers[r], hr, cudaIpcMemLazyEnablePeerAccess));
    }
    return peers;
}

void IpcBlocks::close_peers() {
    for (size_t r = 0; r < peers.size(); ++r)
        if (peers[r] && peers[r] != mine) cudaIpcCloseMemHandle(peers[r]);
    peers.clear();
}

void IpcBlocks::release() {
    close_peers();
    if (mine) cudaFree(mine);
    mine = nullptr;
    cap = 0;
}

// ----------------------------------------------------------- helpers --
int64_t sum_all(const std::vector<int64_t>& v) {
    int64_t s = 0;
    for (auto x : v) s += x;
    return s;
}

std::vector<int64_t> prefix_of(const std::vector<int64_t>& counts) {
    std::vector<int64_t> b(counts.size() + 1, 0);
    for (size_t q = 0; q < counts.size(); ++q) b[q + 1] = b[q] + counts[q];
    return b;
}

// Turn a part's level matrix (local rows, GLOBAL columns in A->ci) into the
// local-column form and build its halo plan.
void localize(Ctx& c, int world, int rank, PLevel& L) {
    DevCsr& A = *L.A;
    const int64_t n = A.nrows;
    L.g0 = L.bounds[rank];
    L.cg = std::move(A.ci);
    A.ci.alloc(A.nnz, c.stream);
    DBuf<int32_t> slot(L.nglob + 1, c.stream);
    MAMG_CU(cudaMemsetAsync(slot.get(), 0, sizeof(int32_t) * (L.nglob + 1), c.stream));
    if (n) {
        k_mark_ghosts<<<blocks_for(n, kBlock), kBlock, 0, c.stream>>>(n, L.g0, A.rp.get(),
                                                                      L.cg.get(), slot.get());
        c.count();
    }
    exclusive_scan_i32(c, slot.get(), slot.get(), L.nglob);
    const int64_t nghost = read_i32(c, slot.get() + L.nglob);
    L.ghost_g.alloc(nghost, c.stream);
    if (L.nglob) {
        k_ghost_list<<<blocks_for(L.nglob, kBlock), kBlock, 0, c.stream>>>(L.nglob, slot.get(),
                                                                           L.ghost_g.get());
        c.count();
    }
    if (n) {
        k_localize<<<blocks_for(n, kBlock), kBlock, 0, c.stream>>>(n, L.g0, A.rp.get(), L.cg.get(),
                                                                   slot.get(), A.ci.get());
        c.count();
    }
    A.ncols = n + nghost;
    Halo& h = L.halo;
    h.nowned = n;
    h.nghost = nghost;
    // receive layout: ghosts are sorted, so each source rank owns one run
    std::vector<int32_t> gg(nghost);
    if (nghost)
        MAMG_CU(cudaMemcpyAsync(gg.data(), L.ghost_g.get(), sizeof(int32_t) * nghost,
                                cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    h.recv_off.assign(world + 1, 0);
    for (int q = 0; q <= world; ++q)
        h.recv_off[q] = std::lower_bound(gg.begin(), gg.end(), L.bounds[q]) - gg.begin();
    // send lists: my rows with a column owned by q (pattern symmetry)
    h.send_off.assign(world + 1, 0);
    std::vector<DBuf<int32_t>> lists(world);
    DBuf<int32_t> flag(n + 1, c.stream);
    for (int q = 0; q < world; ++q) {
        h.send_off[q + 1] = h.send_off[q];
        if (q == rank || !n) continue;
        k_touches<<<blocks_for(n, kBlock), kBlock, 0, c.stream>>>(n, A.rp.get(), L.cg.get(),
                                                                  L.bounds[q], L.bounds[q + 1],
                                                                  flag.get());
        c.count();
        exclusive_scan_i32(c, flag.get(), flag.get(), n);
        const int64_t m = read_i32(c, flag.get() + n);
        lists[q].alloc(m, c.stream);
        if (m) {
            k_compact_rows<<<blocks_for(n, kBlock), kBlock, 0, c.stream>>>(n, flag.get(),
                                                                           lists[q].get());
            c.count();
        }
        h.send_off[q + 1] += m;
    }
    h.send_idx.alloc(h.send_off[world], c.stream);
    for (int q = 0; q < world; ++q) {
        const int64_t m = h.send_off[q + 1] - h.send_off[q];
        if (m)
            MAMG_CU(cudaMemcpyAsync(h.send_idx.get() + h.send_off[q], lists[q].get(),
                                    sizeof(int32_t) * m, cudaMemcpyDeviceToDevice, c.stream));
    }
    h.send_f64.alloc(h.send_off[world], c.stream);
    h.send_i32.alloc(h.send_off[world], c.stream);
    c.sync();
}

// localize every local part of level k and verify the cross-part pattern
// symmetry through the halo counts (send r->q must equal recv q<-r)
void localize_level(Ctx& c, DistHier& d, int k) {
    const int world = d.comm->world;
    for (auto& p : d.parts) localize(c, world, p.rank, p.lv[k]);
    // pairwise consistency: gather the full world x world matrices (one
    // collective: every part's [send counts | receive counts])
    std::vector<int64_t> S(world * world), R(world * world), mine;
    for (auto& p : d.parts) {
        const Halo& h = p.lv[k].halo;
        for (int q = 0; q < world; ++q) mine.push_back(h.send_off[q + 1] - h.send_off[q]); // me -> q
        for (int q = 0; q < world; ++q) mine.push_back(h.recv_off[q + 1] - h.recv_off[q]); // me <- q
    }
    const auto all = d.comm->allgather_n(c, mine, 2 * world);
    for (int r = 0; r < world; ++r)
        for (int q = 0; q < world; ++q) {
            S[r * world + q] = all[static_cast<size_t>(r) * 2 * world + q];
            R[r * world + q] = all[static_cast<size_t>(r) * 2 * world + world + q];
        }
    for (int r = 0; r < world; ++r)
        for (int q = 0; q < world; ++q)
            if (r != q && S[r * world + q] != R[q * world + r])
                invalid("build_hierarchy: matrix pattern is not symmetric");
}

void set_policy(DevCsr& M, int64_t nrows_glob, int64_t nnz_glob, bool single) {
    M.single = single;
    M.group = lane_policy_from(nrows_glob, nnz_glob, single);
}

namespace {

struct PStep {
    std::unique_ptr<DevCsr> P, Ac; // P local->local coarse; Ac local rows, GLOBAL cols
    DBuf<double> wc;
};

// partition-aware pairwise step on level data L (already localized) of
// every local part; returns per-part results, coarse bounds and zero edges
void pairwise_step_dist(Ctx& c, DistHier& d, std::vector<PLevel*>& L,
                        std::vector<const double*>& w, std::vector<PStep>& out,
                        std::vector<int64_t>& cbounds, int64_t& zero_edges) {
    const size_t np = d.parts.size();
    out.clear();
    out.resize(np);
    std::vector<DevAgg> agg(np);
    std::vector<int64_t> ncs, zeros;
    on_all_ranks(c, *d.comm, [&] {
    for (size_t i = 0; i < np; ++i) {
        PLevel& lv = *L[i];
        int64_t z = 0;
        DBuf<int32_t> mate(lv.A->nrows, c.stream);
        try {
            // fused weights + candidates + Suitor on the local graph block;
            // its checks are raised here (local rows -> global in the message)
            weights_suitor(c, *lv.A, w[i], mate.get(), z, lv.cg.get(), lv.g0);
            sync_checked(c);
        } catch (const Error& e) {
            if (e.index < 0) throw;
            std::string msg = e.what();
            const size_t at = msg.rfind(' ');
            if (at != std::string::npos) msg = msg.substr(0, at + 1) + std::to_string(e.index + lv.g0);
            throw Error(e.status, msg, e.index + lv.g0);
        }
        agg[i] = aggregate_from_mate(c, lv.A->nrows, mate.get());
        out[i].P = build_prolongator(c, agg[i], w[i]);
        ncs.push_back(agg[i].nc);
        zeros.push_back(z);
    }
    });
    const auto all_nc = d.comm->allgather(c, ncs);
    zero_edges = sum_all(d.comm->allgather(c, zeros));
    cbounds = prefix_of(all_nc);
    const int64_t nc_glob = cbounds.back();
    // extended column data (global coarse id, p) over owned + ghost columns
    std::vector<DBuf<int32_t>> aggx(np);
    std::vector<DBuf<double>> pvx(np);
    std::vector<int32_t*> ax;
    std::vector<double*> px;
    for (size_t i = 0; i < np; ++i) {
        PLevel& lv = *L[i];
        const int64_t n = lv.A->nrows, ext = n + lv.halo.nghost;
        aggx[i].alloc(ext, c.stream);
        pvx[i].alloc(ext, c.stream);
        if (n) {
            k_ext_owned<<<blocks_for(n, kBlock), kBlock, 0, c.stream>>>(
                n, agg[i].agg_of.get(), cbounds[d.parts[i].rank], out[i].P->v.get(),
                aggx[i].get(), pvx[i].get());
            c.count();
        }
        ax.push_back(aggx[i].get());
        px.push_back(pvx[i].get());
    }
    std::vector<Halo*> hs;
    for (auto* lv : L) hs.push_back(&lv->halo);
    d.comm->halo_i32(c, hs, ax);
    d.comm->halo_f64(c, hs, px);
    for (size_t i = 0; i < np; ++i) {
        out[i].Ac = galerkin_ext(c, *L[i]->A, agg[i], aggx[i].get(), pvx[i].get(), nc_glob);
        out[i].wc.alloc(agg[i].nc, c.stream);
        restrict_members(c, agg[i], out[i].P->v.get(), w[i], out[i].wc.get());
    }
}

} // namespace

std::unique_ptr<Comm> make_loopback_comm(int world) {
    return std::make_unique<LoopbackComm>(world);
}

std::unique_ptr<Comm> make_nccl_comm(Ctx& c, int rank, int world, const void* unique_id) {
    return std::make_unique<NcclComm>(c, rank, world, unique_id);
}

int nccl_unique_id(void* out128) {
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return MAMG_NCCL;
    std::memcpy(out128, &id, sizeof(id));
    return MAMG_OK;
}

std::vector<int64_t> dist_bounds(int64_t n, int world) {
    std::vector<int64_t> b{0};
    for (int r = 1; r < world; ++r) {
        const double ideal = static_cast<double>(r) * static_cast<double>(n) / world / kPartAlign;
        int64_t cut = static_cast<int64_t>(std::llround(ideal)) * kPartAlign;
        cut = std::min(std::max(cut, b.back()), n);
        b.push_back(cut);
    }
    b.push_back(n);
    return b;
}

void dist_load(Ctx& c, DistHier& d, int64_t n, const int64_t* rp, const int64_t* ci,
               const double* v, const double* w) {
    const int world = d.comm->world;
    const auto bounds0 = dist_bounds(n, world);
    d.parts.clear();
    d.nl = 0;
    // the loaded level-0 blocks (d.A0 / d.w0): every build starts from them
    d.A0.clear();
    d.w0.clear();
    for (int r : d.comm->ranks) {
        Part p;
        p.rank = r;
        const int64_t g0 = bounds0[r], g1 = bounds0[r + 1], nl = g1 - g0;
        // rows [g0, g1) with global column ids
        std::vector<int64_t> lrp(nl + 1);
        for (int64_t i = 0; i <= nl; ++i) lrp[i] = rp[g0 + i] - rp[g0];
        d.A0.push_back(csr_upload(c, nl, n, lrp.data(), ci + rp[g0], v + rp[g0]));
        DBuf<double> wl(nl, c.stream);
        if (w) {
            if (nl) upload_f64(c, wl.get(), w + g0, static_cast<size_t>(nl));
        } else if (nl) {
            k_fill_ones<<<blocks_for(nl, kBlock), kBlock, 0, c.stream>>>(nl, wl.get());
            c.count();
        }
        d.w0.push_back(std::move(wl));
        d.parts.push_back(std::move(p));
    }
    d.n0 = n;
    d.nnz0 = rp[n];
    c.sync();
}

void dist_setup(Ctx& c, DistHier& d, int64_t n, const int64_t* rp, const int64_t* ci,
                const double* v, const double* w, const mamg_setup_cfg& cfg) {
    dist_load(c, d, n, rp, ci, v, w);
    dist_build(c, d, cfg);
}

namespace {
__global__ void k_rowlen_d(int64_t n, const int32_t* __restrict__ rp, int32_t* out) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) out[i] = rp[i + 1] - rp[i];
}
__global__ void k_add_i32(int64_t n, int32_t* x, int32_t v) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) x[i] += v;
}

// Gather level k (every part's rows, global columns) onto every process and
// build it and the coarser levels with the single-device code (DistHier::rep).
// Level k-1's P then reads the full iterate: its columns become global.
void agglomerate(Ctx& c, DistHier& d, int k, const mamg_setup_cfg& cfg, double bound) {
    Comm& comm = *d.comm;
    const int W = comm.world;
    const size_t np = d.parts.size();
    const int64_t n = d.level_n[k], nnz = d.level_nnz[k];
    const std::vector<int64_t> b = d.parts[0].lv[k].bounds;
    std::vector<int64_t> rows(W), nnzs;
    for (int r = 0; r < W; ++r) rows[r] = b[r + 1] - b[r];
    for (auto& p : d.parts) nnzs.push_back(p.lv[k].A->nnz);
    const auto all_nnz = comm.allgather(c, nnzs);
    auto A = std::make_unique<DevCsr>();
    A->nrows = n;
    A->ncols = n;
    A->nnz = nnz;
    A->rp.alloc(n + 1, c.stream);
    A->ci.alloc(nnz, c.stream);
    A->v.alloc(nnz, c.stream);
    DBuf<double> w(n, c.stream);
    std::vector<DBuf<int32_t>> lens(np);
    std::vector<const int32_t*> ls, cgs;
    std::vector<const double*> vs, ws;
    for (size_t i = 0; i < np; ++i) {
        PLevel& L = d.parts[i].lv[k];
        const int64_t m = L.A->nrows;
        lens[i].alloc(m, c.stream);
        if (m) {
            k_rowlen_d<<<blocks_for(m, kBlock), kBlock, 0, c.stream>>>(m, L.A->rp.get(), lens[i].get());
            c.count();
        }
        ls.push_back(lens[i].get());
        cgs.push_back(L.cg.get());
        vs.push_back(L.A->v.get());
        ws.push_back(L.w.get());
    }
    comm.allgather_i32(c, ls, rows, std::vector<int32_t*>(np, A->rp.get()));
    exclusive_scan_i32(c, A->rp.get(), A->rp.get(), n);
    comm.allgather_i32(c, cgs, all_nnz, std::vector<int32_t*>(np, A->ci.get()));
    comm.allgather_f64(c, vs, all_nnz, std::vector<double*>(np, A->v.get()));
    comm.allgather_f64(c, ws, rows, std::vector<double*>(np, w.get()));
    csr_finalize(c, *A);
    d.rep = build_hierarchy_sub(c, std::move(A), std::move(w), bound, cfg.max_levels - k,
                                cfg.aggregation);
    d.agg_level = k;
    for (int j = 1; j < d.rep->nl(); ++j) {
        d.level_n.push_back(d.rep->lv[j].A->nrows);
        d.level_nnz.push_back(d.rep->lv[j].A->nnz);
    }
    d.stalled = d.rep->stalled;
    d.zero_edges += d.rep->zero_edges;
    for (auto& p : d.parts) {
        PLevel& F = p.lv[k - 1];
        const int64_t m = F.P->nrows;
        if (d.matching == 1) {
            if (m)
                MAMG_CU(cudaMemcpyAsync(F.P->ci.get(), F.Pg.get(), sizeof(int32_t) * m,
                                        cudaMemcpyDeviceToDevice, c.stream));
        } else {
            if (m) {
                k_add_i32<<<blocks_for(m, kBlock), kBlock, 0, c.stream>>>(
                    m, F.P->ci.get(), static_cast<int32_t>(b[p.rank]));
                c.count();
            }
            F.Pg.alloc(m, c.stream);
            if (m)
                MAMG_CU(cudaMemcpyAsync(F.Pg.get(), F.P->ci.get(), sizeof(int32_t) * m,
                                        cudaMemcpyDeviceToDevice, c.stream));
        }
        F.P->ncols = n;
        F.phalo = Halo{};
    }
    d.rep_b.alloc(n, c.stream);
    d.rep_x.alloc(n, c.stream);
    MAMG_LAUNCH_CHECK();
}
} // namespace

void dist_build(Ctx& c, DistHier& d, const mamg_setup_cfg& cfg) {
    if (cfg.max_levels < 1) invalid("SetupConfig: max_levels must be >= 1");
    if (!(cfg.coarse_factor > 0.0)) invalid("SetupConfig: coarse_factor must be > 0");
    if (d.A0.size() != d.parts.size() || (!d.A0.empty() && !d.A0[0]))
        invalid("mamg_dist_build: no matrix loaded");
    const int64_t n = d.n0;
    const auto bounds0 = dist_bounds(n, d.comm->world);
    // reset to level 0 from the pristine copies
    for (size_t i = 0; i < d.parts.size(); ++i) {
        Part& p = d.parts[i];
        p.lv.clear();
        p.lv.emplace_back();
        PLevel& L = p.lv.back();
        L.bounds = bounds0;
        L.nglob = n;
        L.nnzglob = d.nnz0;
        if (d.consume_level0) {
            L.A = std::move(d.A0[i]);
            L.w = std::move(d.w0[i]);
        } else {
            L.A = csr_clone(c, *d.A0[i]);
            L.w.alloc(L.A->nrows, c.stream);
            if (L.A->nrows)
                MAMG_CU(cudaMemcpyAsync(L.w.get(), d.w0[i].get(), sizeof(double) * L.A->nrows,
                                        cudaMemcpyDeviceToDevice, c.stream));
        }
    }
    // level-0 symmetry among owned entries (cross-part: via halo counts)
    {
        int32_t* ok = reinterpret_cast<int32_t*>(c.d_small.get());
        const int32_t one = 1;
        MAMG_CU(cudaMemcpyAsync(ok, &one, sizeof(one), cudaMemcpyHostToDevice, c.stream));
        for (auto& p : d.parts) {
            PLevel& L = p.lv[0];
            if (L.A->nrows)
                k_sym_owned<<<blocks_for(L.A->nrows, kBlock), kBlock, 0, c.stream>>>(
                    L.A->nrows, L.bounds[p.rank], L.A->rp.get(), L.A->ci.get(), ok);
        }
        on_all_ranks(c, *d.comm, [&] {
            if (read_i32(c, ok) != 1) invalid("build_hierarchy: matrix pattern is not symmetric");
        });
    }
    localize_level(c, d, 0);
    const double bound = cfg.coarse_factor * std::cbrt(static_cast<double>(n));
    d.level_n = {n};
    d.level_nnz = {d.nnz0};
    d.stalled = false;
    d.zero_edges = 0;
    on_all_ranks(c, *d.comm, [&] {
        for (auto& p : d.parts) {
            PLevel& L = p.lv[0];
            set_policy(*L.A, n, d.nnz0, false);
            L.l1.alloc(L.A->nrows, c.stream);
            try {
                l1_diagonal_local(c, *L.A, L.l1.get());
            } catch (const Error& e) {
                throw Error(e.status,
                            "l1_diagonal: zero or missing diagonal entry in row " +
                                std::to_string(e.index + L.g0),
                            e.index + L.g0);
            }
        }
    });
    d.rep.reset();
    ++d.gen; // invalidates the peer halo mailboxes of the previous build
    d.agg_level = -1;
    int k = 0;
    while (static_cast<double>(d.level_n[k]) > bound && k + 1 < cfg.max_levels) {
        if (k >= 1 && d.agglom_rows > 0 && d.level_n[k] <= d.agglom_rows) {
            agglomerate(c, d, k, cfg, bound);
            break;
        }
        if (d.matching == 1) {
            std::vector<PLevel> coarse;
            int64_t z = 0;
            const bool ok = dist_step_global(c, d, k, cfg.aggregation, coarse, z);
            d.zero_edges += z;
            if (!ok) {
                d.stalled = true;
                break;
            }
            const int64_t nc_glob = coarse[0].nglob, nnz_c = coarse[0].nnzglob;
            for (size_t i = 0; i < d.parts.size(); ++i) d.parts[i].lv.push_back(std::move(coarse[i]));
            ++k;
            d.level_n.push_back(nc_glob);
            d.level_nnz.push_back(nnz_c);
            localize_level(c, d, k);
            on_all_ranks(c, *d.comm, [&] {
                for (auto& p : d.parts) {
                    PLevel& L = p.lv[k];
                    set_policy(*L.A, nc_glob, nnz_c, false);
                    L.l1.alloc(L.A->nrows, c.stream);
                    l1_diagonal_local(c, *L.A, L.l1.get());
                }
            });
            continue;
        }
        std::vector<PLevel*> Ls;
        std::vector<const double*> ws;
        for (auto& p : d.parts) {
            Ls.push_back(&p.lv[k]);
            ws.push_back(p.lv[k].w.get());
        }
        std::vector<PStep> s1;
        std::vector<int64_t> cb1;
        int64_t z1 = 0;
        pairwise_step_dist(c, d, Ls, ws, s1, cb1, z1);
        std::vector<PStep>* fin = &s1;
        std::vector<int64_t> cbf = cb1;
        int64_t zsum = z1;
        std::vector<PStep> s2;
        std::vector<PLevel> tmp(d.parts.size());
        if (cfg.aggregation != 1) {
            // second pairwise step on the first coarse level (its own halo)
            std::vector<PLevel*> Ts;
            std::vector<const double*> tws;
            std::vector<int64_t> nnzs;
            for (size_t i = 0; i < d.parts.size(); ++i) {
                tmp[i].bounds = cb1;
                tmp[i].nglob = cb1.back();
                tmp[i].A = std::move(s1[i].Ac);
                nnzs.push_back(tmp[i].A->nnz);
            }
            const int64_t nnz1 = sum_all(d.comm->allgather(c, nnzs));
            for (size_t i = 0; i < d.parts.size(); ++i) {
                localize(c, d.comm->world, d.parts[i].rank, tmp[i]);
                set_policy(*tmp[i].A, cb1.back(), nnz1, false);
                Ts.push_back(&tmp[i]);
                tws.push_back(s1[i].wc.get());
            }
            std::vector<int64_t> cb2;
            int64_t z2 = 0;
            pairwise_step_dist(c, d, Ts, tws, s2, cb2, z2);
            for (size_t i = 0; i < d.parts.size(); ++i)
                s2[i].P = compose_single(c, *s1[i].P, *s2[i].P);
            fin = &s2;
            cbf = cb2;
            zsum += z2;
        }
        d.zero_edges += zsum;
        const int64_t nc_glob = cbf.back();
        if (nc_glob == d.level_n[k]) {
            d.stalled = true;
            break;
        }
        std::vector<int64_t> nnzs;
        for (auto& st : *fin) nnzs.push_back(st.Ac->nnz);
        const int64_t nnz_c = sum_all(d.comm->allgather(c, nnzs));
        for (size_t i = 0; i < d.parts.size(); ++i) {
            Part& p = d.parts[i];
            PLevel& fine = p.lv[k];
            PStep& st = (*fin)[i];
            fine.P = std::move(st.P);
            fine.P->ncols = cbf[p.rank + 1] - cbf[p.rank];
            set_policy(*fine.P, d.level_n[k], d.level_n[k], true);
            fine.R = transpose(c, *fine.P);
            set_policy(*fine.R, nc_glob, d.level_n[k], false);
            PLevel coarse;
            coarse.bounds = cbf;
            coarse.nglob = nc_glob;
            coarse.nnzglob = nnz_c;
            coarse.A = std::move(st.Ac);
            coarse.w = std::move(st.wc);
            p.lv.push_back(std::move(coarse));
        }
        ++k;
        d.level_n.push_back(nc_glob);
        d.level_nnz.push_back(nnz_c);
        localize_level(c, d, k);
        on_all_ranks(c, *d.comm, [&] {
            for (auto& p : d.parts) {
                PLevel& L = p.lv[k];
                set_policy(*L.A, nc_glob, nnz_c, false);
                L.l1.alloc(L.A->nrows, c.stream);
                l1_diagonal_local(c, *L.A, L.l1.get());
            }
        });
    }
    d.nl = d.agg_level >= 0 ? d.agg_level + d.rep->nl() : k + 1;
    // levels cycled partitioned (the agglomerated ones run on `rep`)
    const int npl = d.agg_level >= 0 ? d.agg_level : d.nl;
    // cycle workspace: vectors read by a SpMV carry the ghost region
    for (auto& p : d.parts)
        for (int j = 0; j < npl; ++j) {
            PLevel& L = p.lv[j];
            // ghost room also takes the restriction's remote members (rhalo)
            const int64_t ext = L.A->nrows + std::max(L.halo.nghost, L.rhalo.nghost);
            L.xw.alloc(ext, c.stream);
            L.scratch.alloc(ext, c.stream);
            if (j + 1 < d.nl) {
                const PLevel& C = p.lv[j + 1];
                L.cb.alloc(C.A->nrows, c.stream);
                // ... and the prolongation's remote aggregates (phalo); the
                // level above the agglomeration reads rep_x instead
                if (j + 1 != d.agg_level)
                    L.cx.alloc(C.A->nrows + std::max(C.halo.nghost, L.phalo.nghost), c.stream);
            }
        }
    c.sync();
}

} // namespace mamg
