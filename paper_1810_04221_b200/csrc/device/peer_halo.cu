// peer_halo.cu — halo exchange of the partitioned cycle over peer memory
// (NVLink stores instead of NCCL send/recv).
//
// Per partitioned level every part owns a mailbox of two parities x its ghost
// count and three counters (arrival, epoch = completed exchanges, error), in
// one slot-2 shared block per part (CUDA IPC mappings for NCCL, the parts'
// own blocks for the loopback). An exchange is two kernels per part:
//  * push: the part's send list (its Halo, grouped by destination) is read
//    from x and stored straight into each receiver's mailbox, at the segment
//    the receiver's ghost layout gives this sender (parity = epoch mod 2);
//    the last CTA fences (system scope) and increments each receiver's
//    arrival counter;
//  * unpack: wait (acquire, bounded) until every source of this part has
//    signalled this exchange, copy the mailbox into the ghost region of x,
//    advance the epoch.
// Every rank runs the same exchanges, so epochs agree. Two parities suffice:
// the halo pattern is symmetric (a part's sources are its destinations), so
// a sender can only reach exchange j+2 after receiving exchange j+1 from the
// receiver, which the receiver pushes after unpacking exchange j.
#include <algorithm>
#include <cstdlib>

#include "dist.cuh"

namespace mamg {
namespace {

constexpr int kPushThreads = 256;
constexpr int kUnpackThreads = 1024;

__global__ void __launch_bounds__(kPushThreads)
k_halo_push(int64_t m, const int32_t* __restrict__ idx, const double* __restrict__ x,
            const PeerDest* __restrict__ dst, int ndst, const unsigned long long* epoch,
            unsigned* cta) {
    __shared__ bool last;
    const int64_t par = static_cast<int64_t>(*epoch & 1ull);
    // grid-stride (at most one CTA per SM): one fence + one counter update
    // per CTA instead of per 256 elements
    for (int64_t t = static_cast<int64_t>(blockIdx.x) * kPushThreads + threadIdx.x; t < m;
         t += static_cast<int64_t>(gridDim.x) * kPushThreads) {
        int d = 0;
        while (d + 1 < ndst && t >= dst[d + 1].start) ++d;
        const PeerDest& q = dst[d];
        q.mbox[par * q.ng + q.seg + (t - q.start)] = x[idx[t]];
    }
    // the CTA barrier orders every thread's stores before thread 0's
    // system-scope fence, which is cumulative: one fence per CTA
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        last = atomicAdd(cta, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (last && threadIdx.x == 0) {
        __threadfence_system();
        for (int d = 0; d < ndst; ++d) atomicAdd_system(dst[d].arrive, 1ull);
        *cta = 0u;
    }
}

// multi-CTA unpack: every CTA waits for the arrivals, copies its slice; the
// last CTA to finish advances the epoch (all CTAs read it before that)
__global__ void __launch_bounds__(kUnpackThreads)
k_halo_unpack(int64_t ng, const double* mbox, double* xg, unsigned long long* ctrs, int nsrc,
              unsigned* cta) {
    __shared__ unsigned long long ep;
    __shared__ bool last;
    if (threadIdx.x == 0) {
        ep = ctrs[1];
        const unsigned long long target = (ep + 1) * static_cast<unsigned long long>(nsrc);
        long long spins = 0;
        for (;;) {
            unsigned long long a;
            asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(a) : "l"(ctrs) : "memory");
            if (a >= target) break;
            if (++spins > (1ll << 26)) { // ~7 s: a protocol fault, not a hang
                atomicExch(ctrs + 2, 1ull);
                break;
            }
            __nanosleep(100);
        }
    }
    __syncthreads();
    const double* src = mbox + static_cast<int64_t>(ep & 1ull) * ng;
    for (int64_t t = static_cast<int64_t>(blockIdx.x) * kUnpackThreads + threadIdx.x; t < ng;
         t += static_cast<int64_t>(gridDim.x) * kUnpackThreads)
        xg[t] = __ldcg(src + t);
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(cta, 1u) == gridDim.x - 1;
    __syncthreads();
    if (last && threadIdx.x == 0) {
        ctrs[1] = ep + 1;
        *cta = 0u;
    }
}

size_t align256(size_t b) { return (b + 255) & ~size_t{255}; }

// interior range of a part: first / last row without a ghost column
// (atomics), then the ghost rows strictly between them (zero = one contiguous
// interior run, the slab case; otherwise no overlap at this level)
__global__ void k_interior_ends(int64_t n, const int32_t* __restrict__ rp,
                                const int32_t* __restrict__ ci, int* ends) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    bool ghost = false;
    for (int k = rp[i]; k < rp[i + 1]; ++k) ghost |= ci[k] >= n;
    if (!ghost) {
        atomicMin(&ends[0], static_cast<int>(i));
        atomicMax(&ends[1], static_cast<int>(i));
    }
}

__global__ void k_interior_holes(int64_t n, const int32_t* __restrict__ rp,
                                 const int32_t* __restrict__ ci, int* ends) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n || i <= ends[0] || i >= ends[1]) return;
    bool ghost = false;
    for (int k = rp[i]; k < rp[i + 1]; ++k) ghost |= ci[k] >= n;
    if (ghost) atomicAdd(&ends[2], 1);
}

} // namespace

bool peer_halo_prepare(Ctx& c, DistHier& d, int nlev) {
    const bool off = std::getenv("MAMG_DIST_NCCL_HALO") != nullptr;
    const bool force = std::getenv("MAMG_DIST_PEER") != nullptr;
    PeerHalo& ph = d.peer;
    Comm& comm = *d.comm;
    const int W = comm.world;
    const size_t np = d.parts.size();
    if (off || W > kMaxWorld || nlev <= 0 || (W == 1 && !force)) {
        ph.on = false;
        return false;
    }
    // a rebuild of the same matrix keeps every halo layout: reuse the plan
    // when every rank's layout fingerprint is unchanged (one allgather)
    uint64_t fp = 1469598103934665603ull;
    auto mix = [&fp](int64_t v) {
        fp ^= static_cast<uint64_t>(v);
        fp *= 1099511628211ull;
    };
    mix(nlev);
    mix(d.agg_level);
    for (auto& p : d.parts)
        for (int k = 0; k < nlev; ++k) {
            const Halo& h = p.lv[k].halo;
            mix(h.nghost);
            for (auto v : h.send_off) mix(v);
            for (auto v : h.recv_off) mix(v);
        }
    if (d.agg_level >= 1)
        for (auto v : d.parts[0].lv[d.agg_level].bounds) mix(v);
    if (ph.gen != d.gen && ph.gen >= 0) {
        bool same = true;
        const int64_t mine = fp == ph.layout ? 1 : 0;
        for (auto v : comm.allgather(c, std::vector<int64_t>(np, mine))) same = same && v != 0;
        if (same) ph.gen = d.gen;
    }
    if (ph.gen != d.gen) {
        // per part: level offsets inside its block
        std::vector<std::vector<size_t>> off_l(np, std::vector<size_t>(nlev + 1, 0));
        std::vector<size_t> bytes(np);
        for (size_t i = 0; i < np; ++i) {
            for (int k = 0; k < nlev; ++k) {
                const int64_t ng = d.parts[i].lv[k].halo.nghost;
                off_l[i][k + 1] = off_l[i][k] + align256(sizeof(double) * 2 * ng) + 256;
            }
            bytes[i] = off_l[i][nlev];
            if (d.agg_level >= 1)
                bytes[i] += align256(sizeof(double) * 2 * d.level_n[d.agg_level]) + 256;
        }
        int64_t ok = 1;
        std::vector<void*> blocks;
        try {
            blocks = comm.shared_blocks(c, bytes, 2);
        } catch (const Error&) {
            ok = 0;
        }
        bool all_ok = true;
        for (auto v : comm.allgather(c, std::vector<int64_t>(np, ok))) all_ok = all_ok && v != 0;
        if (!all_ok) {
            ph.on = false;
            return false;
        }
        ph.lv.clear();
        ph.lv.resize(np);
        for (auto& v : ph.lv) v.resize(nlev);
        for (int k = 0; k < nlev; ++k) {
            // every rank's level offset, ghost count and ghost layout (one collective)
            std::vector<int64_t> mine;
            for (size_t i = 0; i < np; ++i) {
                const Halo& h = d.parts[i].lv[k].halo;
                mine.push_back(static_cast<int64_t>(off_l[i][k]));
                mine.push_back(h.nghost);
                for (int q = 0; q < W; ++q) mine.push_back(h.recv_off[q]);
            }
            const auto all = comm.allgather_n(c, mine, W + 2);
            std::vector<int64_t> all_off(W), all_ng(W);
            std::vector<std::vector<int64_t>> recv_at(W, std::vector<int64_t>(W, 0)); // [rank][src]
            for (int r = 0; r < W; ++r) {
                const int64_t* a = all.data() + static_cast<size_t>(r) * (W + 2);
                all_off[r] = a[0];
                all_ng[r] = a[1];
                for (int q = 0; q < W; ++q) recv_at[r][q] = a[2 + q];
            }
            for (size_t i = 0; i < np; ++i) {
                const int me = d.parts[i].rank;
                const Halo& h = d.parts[i].lv[k].halo;
                PeerHaloLevel& pl = ph.lv[i][k];
                char* mine = static_cast<char*>(blocks[me]) + off_l[i][k];
                pl.ng = h.nghost;
                pl.mbox = reinterpret_cast<double*>(mine);
                pl.ctrs = reinterpret_cast<unsigned long long*>(mine + align256(sizeof(double) * 2 * h.nghost));
                pl.nsrc = 0;
                for (int q = 0; q < W; ++q) pl.nsrc += h.recv_off[q + 1] > h.recv_off[q];
                std::vector<PeerDest> ds;
                for (int q = 0; q < W; ++q) {
                    const int64_t cnt = h.send_off[q + 1] - h.send_off[q];
                    if (!cnt) continue;
                    char* qb = static_cast<char*>(blocks[q]) + all_off[q];
                    PeerDest pd;
                    pd.start = h.send_off[q];
                    pd.cnt = cnt;
                    pd.mbox = reinterpret_cast<double*>(qb);
                    pd.seg = recv_at[q][me];
                    pd.ng = all_ng[q];
                    pd.arrive = reinterpret_cast<unsigned long long*>(qb + align256(sizeof(double) * 2 * all_ng[q]));
                    ds.push_back(pd);
                }
                pl.ndst = static_cast<int>(ds.size());
                pl.dests.alloc(ds.size(), c.stream);
                if (!ds.empty())
                    MAMG_CU(cudaMemcpyAsync(pl.dests.get(), ds.data(), sizeof(PeerDest) * ds.size(),
                                            cudaMemcpyHostToDevice, c.stream));
                pl.cta.alloc(2, c.stream); // [push, unpack] last-CTA counters
            }
        }
        ph.ag.clear();
        ph.ag_idx.clear();
        if (d.agg_level >= 1) {
            // coarse blocks of the agglomeration level: rank q's rows
            const std::vector<int64_t>& cb = d.parts[0].lv[d.agg_level].bounds;
            const int64_t na = d.level_n[d.agg_level];
            std::vector<int64_t> mo;
            for (size_t i = 0; i < np; ++i) mo.push_back(static_cast<int64_t>(off_l[i][nlev]));
            const auto all_off = comm.allgather(c, mo);
            // every rank signals every exchange, also one owning no rows
            // (else it would not be waited for, and the two-parity argument
            // needs every destination to be a source)
            const int nsrc = W;
            ph.ag.resize(np);
            ph.ag_idx.resize(np);
            for (size_t i = 0; i < np; ++i) {
                const int me = d.parts[i].rank;
                const int64_t nown = cb[me + 1] - cb[me];
                PeerHaloLevel& pl = ph.ag[i];
                char* mine = static_cast<char*>(blocks[me]) + off_l[i][nlev];
                pl.ng = na;
                pl.mbox = reinterpret_cast<double*>(mine);
                pl.ctrs = reinterpret_cast<unsigned long long*>(mine + align256(sizeof(double) * 2 * na));
                pl.nsrc = nsrc;
                std::vector<PeerDest> ds;
                std::vector<int32_t> idx;
                for (int q = 0; q < W; ++q) {
                    char* qb = static_cast<char*>(blocks[q]) + all_off[q];
                    PeerDest pd;
                    pd.start = static_cast<int64_t>(q) * nown;
                    pd.cnt = nown;
                    pd.mbox = reinterpret_cast<double*>(qb);
                    pd.seg = cb[me];
                    pd.ng = na;
                    pd.arrive = reinterpret_cast<unsigned long long*>(qb + align256(sizeof(double) * 2 * na));
                    ds.push_back(pd);
                    for (int64_t t = 0; t < nown; ++t) idx.push_back(static_cast<int32_t>(t));
                }
                pl.ndst = static_cast<int>(ds.size());
                pl.dests.alloc(ds.size(), c.stream);
                ph.ag_idx[i].alloc(idx.size(), c.stream);
                if (!ds.empty())
                    MAMG_CU(cudaMemcpyAsync(pl.dests.get(), ds.data(), sizeof(PeerDest) * ds.size(),
                                            cudaMemcpyHostToDevice, c.stream));
                if (!idx.empty())
                    MAMG_CU(cudaMemcpyAsync(ph.ag_idx[i].get(), idx.data(), sizeof(int32_t) * idx.size(),
                                            cudaMemcpyHostToDevice, c.stream));
                pl.cta.alloc(2, c.stream);
            }
            c.sync();
        }
        ph.gen = d.gen;
        ph.layout = fp;
    }
    // every solve starts from zeroed counters on every rank
    auto zero = [&](PeerHaloLevel& pl) {
        MAMG_CU(cudaMemsetAsync(pl.ctrs, 0, 3 * sizeof(unsigned long long), c.stream));
        MAMG_CU(cudaMemsetAsync(pl.cta.get(), 0, 2 * sizeof(unsigned), c.stream));
    };
    for (auto& lvs : ph.lv)
        for (auto& pl : lvs) zero(pl);
    for (auto& pl : ph.ag) zero(pl);
    comm.barrier(c);
    c.sync();
    ph.on = true;
    return true;
}

void peer_halo_exchange(Ctx& c, DistHier& d, int k, const std::vector<double*>& x) {
    PeerHalo& ph = d.peer;
    for (size_t i = 0; i < d.parts.size(); ++i) {
        const Halo& h = d.parts[i].lv[k].halo;
        PeerHaloLevel& pl = ph.lv[i][k];
        const int64_t m = h.send_off.empty() ? 0 : h.send_off.back();
        if (m == 0) continue;
        k_halo_push<<<std::min<unsigned>(c.num_sms, blocks_for(m, kPushThreads)), kPushThreads, 0,
                      c.stream>>>(m, h.send_idx.get(), x[i], pl.dests.get(), pl.ndst, pl.ctrs + 1,
                                  pl.cta.get());
        c.count();
    }
    for (size_t i = 0; i < d.parts.size(); ++i) {
        PeerHaloLevel& pl = ph.lv[i][k];
        if (pl.nsrc == 0) continue;
        const int grid = static_cast<int>(std::min<int64_t>(c.num_sms, (pl.ng + kUnpackThreads - 1) / kUnpackThreads));
        k_halo_unpack<<<grid, kUnpackThreads, 0, c.stream>>>(
            pl.ng, pl.mbox, x[i] + d.parts[i].lv[k].halo.nowned, pl.ctrs, pl.nsrc,
            pl.cta.get() + 1);
        c.count();
    }
    MAMG_LAUNCH_CHECK();
}

void interior_ranges(Ctx& c, DistHier& d, int nlev) {
    for (auto& p : d.parts)
        for (int k = 0; k < nlev && k < static_cast<int>(p.lv.size()); ++k) {
            PLevel& L = p.lv[k];
            if (L.interior_gen == d.gen) continue;
            const int64_t n = L.A->nrows;
            L.ia = L.ib = 0;
            if (n > 0 && L.halo.nghost > 0) {
                DBuf<int> ends(3, c.stream);
                const int init[3] = {INT32_MAX, -1, 0};
                MAMG_CU(cudaMemcpyAsync(ends.get(), init, sizeof(init), cudaMemcpyHostToDevice,
                                        c.stream));
                k_interior_ends<<<blocks_for(n, kPushThreads), kPushThreads, 0, c.stream>>>(
                    n, L.A->rp.get(), L.A->ci.get(), ends.get());
                k_interior_holes<<<blocks_for(n, kPushThreads), kPushThreads, 0, c.stream>>>(
                    n, L.A->rp.get(), L.A->ci.get(), ends.get());
                c.count(2);
                int h[3];
                MAMG_CU(cudaMemcpyAsync(h, ends.get(), sizeof(h), cudaMemcpyDeviceToHost, c.stream));
                c.sync();
                if (h[1] >= 0 && h[2] == 0) {
                    L.ia = h[0];
                    L.ib = static_cast<int64_t>(h[1]) + 1;
                }
            }
            L.interior_gen = d.gen;
        }
}

void peer_agg_gather(Ctx& c, DistHier& d, const std::vector<const double*>& cb, double* out) {
    PeerHalo& ph = d.peer;
    for (size_t i = 0; i < d.parts.size(); ++i) {
        PeerHaloLevel& pl = ph.ag[i];
        const int64_t m = static_cast<int64_t>(ph.ag_idx[i].size());
        if (pl.ndst == 0) continue;
        // m == 0 (no own rows): one CTA that only signals
        k_halo_push<<<std::max(1u, std::min<unsigned>(c.num_sms, blocks_for(m, kPushThreads))), kPushThreads, 0,
                      c.stream>>>(m, ph.ag_idx[i].get(), cb[i], pl.dests.get(), pl.ndst, pl.ctrs + 1,
                                  pl.cta.get());
        c.count();
    }
    for (size_t i = 0; i < d.parts.size(); ++i) {
        PeerHaloLevel& pl = ph.ag[i];
        if (pl.nsrc == 0) continue;
        const int grid = static_cast<int>(std::min<int64_t>(c.num_sms, (pl.ng + kUnpackThreads - 1) / kUnpackThreads));
        k_halo_unpack<<<grid, kUnpackThreads, 0, c.stream>>>(pl.ng, pl.mbox, out, pl.ctrs, pl.nsrc,
                                                             pl.cta.get() + 1);
        c.count();
    }
    MAMG_LAUNCH_CHECK();
}

bool peer_halo_failed(Ctx& c, DistHier& d) {
    if (!d.peer.on) return false;
    c.sync();
    auto bad = [&](PeerHaloLevel& pl) {
        unsigned long long e = 0;
        MAMG_CU(cudaMemcpy(&e, pl.ctrs + 2, sizeof(e), cudaMemcpyDeviceToHost));
        return e != 0;
    };
    for (auto& lvs : d.peer.lv)
        for (auto& pl : lvs)
            if (bad(pl)) return true;
    for (auto& pl : d.peer.ag)
        if (bad(pl)) return true;
    return false;
}

} // namespace mamg
