// shm_comm.cu — the multi-process transport without NCCL.
//
// One rank per process on one node; ranks may share a GPU (NCCL refuses two
// ranks on one device, so this is the transport that runs the partitioned
// path's cross-process protocol — IPC mailboxes, system-scope arrival
// counters, peer reductions, the peer-memory Suitor — on a single B200).
//
//  * host collectives (allgather, barrier): a POSIX shared-memory segment
//    holding a sense-reversing barrier and one data slot per rank;
//  * device data (setup halos, allgathers): every rank stages its outgoing
//    values in its own CUDA-IPC exchange block, the receivers copy them out
//    of the peers' blocks (mapped with cudaIpcOpenMemHandle);
//  * shared_blocks: the same CUDA-IPC blocks the NCCL transport publishes.
//
// Every collective first drains the caller's stream and then meets the other
// ranks on the host, so collectives are not graph-capturable (capturable()
// false: the partitioned PCG runs eagerly with this transport). Host waits
// are bounded (MAMG_SHM_TIMEOUT seconds, default 300): a rank that died makes
// the others fail loudly instead of hanging.
#include <fcntl.h>
#include <sched.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <string>

#include "dist.cuh"

namespace mamg {
namespace {

constexpr int kBlock = 256;
constexpr size_t kSlotWords = 4096; // int64 words per rank and round of an allgather

struct ShmHeader {
    uint64_t arrived;
    uint64_t gen;
    uint64_t world;
    uint64_t pad[5];
};

template <class T>
__global__ void k_pack_shm(int64_t m, const int32_t* __restrict__ idx, const T* __restrict__ x,
                           T* out) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t < m) out[t] = x[idx[t]];
}

// The host half: a POSIX shared-memory segment with a sense-reversing
// barrier and one data slot per rank (no CUDA). Every rank passes the same
// fresh name; rank 0 unlinks it once all ranks have attached.
class ShmSegment {
public:
    ShmSegment(int rank, int world, const char* name, double timeout_s)
        : me_(rank), world_(world), timeout_s_(timeout_s) {
        bytes_ = sizeof(ShmHeader) + sizeof(int64_t) * kSlotWords * static_cast<size_t>(world);
        const std::string nm = name[0] == '/' ? std::string(name) : "/" + std::string(name);
        const int fd = shm_open(nm.c_str(), O_CREAT | O_RDWR, 0600);
        if (fd < 0) throw Error(MAMG_RUNTIME, "shm transport: shm_open(" + nm + ") failed", -1);
        // every rank sizes the (zero-filled) segment identically: idempotent
        if (ftruncate(fd, static_cast<off_t>(bytes_)) != 0) {
            close(fd);
            throw Error(MAMG_RUNTIME, "shm transport: ftruncate failed", -1);
        }
        void* p = mmap(nullptr, bytes_, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
        close(fd);
        if (p == MAP_FAILED) throw Error(MAMG_RUNTIME, "shm transport: mmap failed", -1);
        hdr_ = static_cast<ShmHeader*>(p);
        data_ = reinterpret_cast<int64_t*>(hdr_ + 1);
        try {
            barrier(); // every rank has mapped the segment
        } catch (...) {
            munmap(hdr_, bytes_);
            if (rank == 0) shm_unlink(nm.c_str());
            throw;
        }
        if (rank == 0) shm_unlink(nm.c_str());
    }
    // attach to process-local memory (the in-process thread group): every
    // rank passes the same zero-initialised region of bytes_for(world)
    ShmSegment(int rank, int world, void* mem, double timeout_s)
        : me_(rank), world_(world), timeout_s_(timeout_s), owned_(false) {
        bytes_ = bytes_for(world);
        hdr_ = static_cast<ShmHeader*>(mem);
        data_ = reinterpret_cast<int64_t*>(hdr_ + 1);
    }
    static size_t bytes_for(int world) {
        return sizeof(ShmHeader) + sizeof(int64_t) * kSlotWords * static_cast<size_t>(world);
    }
    ~ShmSegment() {
        if (hdr_ && owned_) munmap(hdr_, bytes_);
    }
    ShmSegment(const ShmSegment&) = delete;
    ShmSegment& operator=(const ShmSegment&) = delete;

    // sense-reversing barrier (GCC atomics on the shared mapping)
    void barrier() {
        const uint64_t g = __atomic_load_n(&hdr_->gen, __ATOMIC_ACQUIRE);
        if (__atomic_add_fetch(&hdr_->arrived, 1, __ATOMIC_ACQ_REL) == static_cast<uint64_t>(world_)) {
            __atomic_store_n(&hdr_->arrived, 0, __ATOMIC_RELAXED);
            __atomic_store_n(&hdr_->gen, g + 1, __ATOMIC_RELEASE);
            return;
        }
        const auto t0 = std::chrono::steady_clock::now();
        for (uint64_t spins = 0; __atomic_load_n(&hdr_->gen, __ATOMIC_ACQUIRE) == g; ++spins) {
            if ((spins & 1023) == 1023) {
                sched_yield();
                const double s =
                    std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
                if (s > timeout_s_)
                    throw Error(MAMG_RUNTIME,
                                "shm transport: rank " + std::to_string(me_) +
                                    " timed out in a collective (a peer process died or diverged)",
                                -1);
            }
        }
    }

    // `len` values per rank -> world x len, rank-major
    std::vector<int64_t> allgather_n(const int64_t* mine, int64_t len) {
        std::vector<int64_t> all(static_cast<size_t>(world_) * len);
        for (int64_t off = 0; off < len; off += static_cast<int64_t>(kSlotWords)) {
            const int64_t m = std::min<int64_t>(len - off, static_cast<int64_t>(kSlotWords));
            volatile int64_t* slot = data_ + static_cast<size_t>(me_) * kSlotWords;
            for (int64_t j = 0; j < m; ++j) slot[j] = mine[off + j];
            barrier(); // published
            for (int r = 0; r < world_; ++r) {
                const volatile int64_t* s = data_ + static_cast<size_t>(r) * kSlotWords;
                for (int64_t j = 0; j < m; ++j) all[static_cast<size_t>(r) * len + off + j] = s[j];
            }
            barrier(); // read: the slots may be overwritten
        }
        return all;
    }

private:
    int me_ = 0, world_ = 1;
    double timeout_s_ = 300.0;
    bool owned_ = true;
    size_t bytes_ = 0;
    ShmHeader* hdr_ = nullptr;
    int64_t* data_ = nullptr;
};

// Shared device blocks of ranks living in ONE process (threads): plain
// cudaMalloc'd blocks, raw pointers published through the host allgather
// (unified addressing), readable across devices through peer access.
struct DirectBlocks {
    void* mine = nullptr;
    size_t cap = 0;
    std::vector<void*> peers;
    std::vector<void*> get(Ctx& c, Comm& comm, size_t bytes) {
        const int grow = bytes > cap ? 1 : 0;
        const auto g = comm.allgather(c, {grow});
        bool any = peers.empty();
        for (auto x : g) any = any || x != 0;
        if (!any) return peers;
        c.sync();              // my kernels are done with the old blocks
        comm.allgather(c, {0}); // so are everyone's
        if (grow) {
            if (mine) MAMG_CU(cudaFree(mine));
            mine = nullptr;
            cap = std::max<size_t>(bytes + bytes / 8, 1 << 20);
            MAMG_CU(cudaMalloc(&mine, cap));
        }
        const auto all = comm.allgather(c, {static_cast<int64_t>(reinterpret_cast<intptr_t>(mine))});
        peers.assign(all.size(), nullptr);
        for (size_t r = 0; r < all.size(); ++r) peers[r] = reinterpret_cast<void*>(static_cast<intptr_t>(all[r]));
        return peers;
    }
    void release() {
        if (mine) cudaFree(mine);
        mine = nullptr;
        cap = 0;
        peers.clear();
    }
};

double shm_timeout() {
    const char* t = std::getenv("MAMG_SHM_TIMEOUT");
    return t ? std::atof(t) : 300.0;
}

// One rank of a multi-rank group without NCCL: host collectives through a
// ShmSegment (POSIX shared memory across processes, or process memory across
// threads), device data through shared blocks (CUDA IPC or direct pointers).
template <class Blocks>
class HostComm : public Comm {
public:
    // across processes: POSIX shared memory `name`
    HostComm(Ctx&, int rank, int w, const char* name)
        : me_(rank), seg_(rank, w, name, shm_timeout()) {
        world = w;
        ranks.push_back(rank);
    }
    // across threads of this process: the group's memory; enables peer
    // access to the other ranks' devices
    HostComm(Ctx& c, int rank, int w, void* mem) : me_(rank), seg_(rank, w, mem, shm_timeout()) {
        world = w;
        ranks.push_back(rank);
        const auto devs = allgather(c, {c.device});
        for (int q = 0; q < w; ++q) {
            if (q == rank) continue;
            const int d = static_cast<int>(devs[q]);
            if (d == c.device) {
                shares_device_ = true;
                continue;
            }
            int can = 0;
            cudaDeviceCanAccessPeer(&can, c.device, d);
            if (!can) {
                no_p2p_ = true;
                continue;
            }
            const cudaError_t e = cudaDeviceEnablePeerAccess(d, 0);
            if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) no_p2p_ = true;
            cudaGetLastError();
        }
    }
    ~HostComm() override {
        for (auto& b : blocks_) b.release();
        exchange_.release();
    }
    // ranks of one process sharing a device keep the Comm's halos and
    // allgathers: the peer paths' waiting kernels (reduction folds, halo
    // unpacks) would need the partner's kernels co-resident on that device
    bool peer_memory() const override { return world > 1 && !shares_device_ && !no_p2p_; }
    bool capturable() const override { return false; }

    void barrier(Ctx& c) override {
        c.sync();
        host_barrier();
    }
    // slot 0 (the global Suitor: lock-free, no waiting kernel) works on a
    // shared device; slots 1-2 (peer reductions, halo mailboxes) are refused
    // there, and everywhere without peer access — every rank then falls back
    std::vector<void*> shared_blocks(Ctx& c, const std::vector<size_t>& bytes, int slot) override {
        if (no_p2p_) throw Error(MAMG_RUNTIME, "shared blocks: no peer access between the ranks' devices", -1);
        if (shares_device_ && slot % 3 != 0)
            throw Error(MAMG_RUNTIME, "shared blocks: ranks share a device (peer paths off)", -1);
        return blocks_[slot % 3].get(c, *this, bytes[0]);
    }
    std::vector<int64_t> allgather(Ctx& c, const std::vector<int64_t>& mine) override {
        return allgather_n(c, mine, 1);
    }
    std::vector<int64_t> allgather_n(Ctx&, const std::vector<int64_t>& mine, int len) override {
        return seg_.allgather_n(mine.data(), len);
    }

    void halo_f64(Ctx& c, const std::vector<Halo*>& h, const std::vector<double*>& x) override {
        halo<double>(c, *h[0], x[0]);
    }
    void halo_i32(Ctx& c, const std::vector<Halo*>& h, const std::vector<int32_t*>& x) override {
        halo<int32_t>(c, *h[0], x[0]);
    }
    void allgather_f64(Ctx& c, const std::vector<const double*>& src,
                       const std::vector<int64_t>& counts, const std::vector<double*>& dst) override {
        gather<double>(c, src[0], counts, dst[0]);
    }
    void allgather_i32(Ctx& c, const std::vector<const int32_t*>& src,
                       const std::vector<int64_t>& counts, const std::vector<int32_t*>& dst) override {
        gather<int32_t>(c, src[0], counts, dst[0]);
    }
    void allgather_equal_f64(Ctx& c, const std::vector<const double*>& src, int64_t count,
                             const std::vector<double*>& dst) override {
        gather<double>(c, src[0], std::vector<int64_t>(world, count), dst[0]);
    }

private:
    void host_barrier() { seg_.barrier(); }

    // setup halo: pack my send list into my exchange block, meet, copy each
    // source's segment for me out of its block, meet again (blocks reusable)
    template <class T>
    void halo(Ctx& c, Halo& h, T* x) {
        const int64_t m = h.send_off.empty() ? 0 : h.send_off.back();
        const auto offs = allgather_n(c, h.send_off, world + 1);
        auto ex = exchange_.get(c, *this, sizeof(T) * static_cast<size_t>(std::max<int64_t>(m, 1)));
        if (m) {
            k_pack_shm<T><<<blocks_for(m, kBlock), kBlock, 0, c.stream>>>(
                m, h.send_idx.get(), x, static_cast<T*>(ex[me_]));
            c.count();
        }
        c.sync();
        host_barrier();
        for (int q = 0; q < world; ++q) {
            if (q == me_) continue;
            const int64_t cnt = h.recv_off[q + 1] - h.recv_off[q];
            const int64_t* oq = offs.data() + static_cast<size_t>(q) * (world + 1);
            if (cnt != oq[me_ + 1] - oq[me_])
                invalid("build_hierarchy: matrix pattern is not symmetric");
            if (!cnt) continue;
            MAMG_CU(cudaMemcpyAsync(x + h.nowned + h.recv_off[q], static_cast<const T*>(ex[q]) + oq[me_],
                                    sizeof(T) * cnt, cudaMemcpyDefault, c.stream));
        }
        c.sync();
        host_barrier();
    }

    // allgather: stage my counts[me] values, meet, copy every rank's run
    template <class T>
    void gather(Ctx& c, const T* src, const std::vector<int64_t>& counts, T* dst) {
        const int64_t mine = counts[me_];
        auto ex = exchange_.get(c, *this, sizeof(T) * static_cast<size_t>(std::max<int64_t>(mine, 1)));
        if (mine)
            MAMG_CU(cudaMemcpyAsync(ex[me_], src, sizeof(T) * mine, cudaMemcpyDeviceToDevice, c.stream));
        c.sync();
        host_barrier();
        int64_t off = 0;
        for (int q = 0; q < world; ++q) {
            if (counts[q])
                MAMG_CU(cudaMemcpyAsync(dst + off, ex[q], sizeof(T) * counts[q], cudaMemcpyDefault,
                                        c.stream));
            off += counts[q];
        }
        c.sync();
        host_barrier();
    }

    int me_ = 0;
    ShmSegment seg_;
    Blocks blocks_[3]; // shared_blocks slots 0-2
    Blocks exchange_;  // staging of the setup collectives
    bool shares_device_ = false, no_p2p_ = false;
};

} // namespace

std::unique_ptr<Comm> make_shm_comm(Ctx& c, int rank, int world, const char* name) {
    return std::make_unique<HostComm<IpcBlocks>>(c, rank, world, name);
}

ThreadGroup::ThreadGroup(int w) : world(w), mem(ShmSegment::bytes_for(w) / sizeof(int64_t) + 1, 0) {}

std::unique_ptr<Comm> make_thread_comm(Ctx& c, int rank, ThreadGroup& g) {
    return std::make_unique<HostComm<DirectBlocks>>(c, rank, g.world, g.mem.data());
}

std::vector<int64_t> shm_allgather_once(const char* name, int world, int rank, const int64_t* mine,
                                        int64_t len) {
    ShmSegment seg(rank, world, name, shm_timeout());
    return seg.allgather_n(mine, len);
}

} // namespace mamg
