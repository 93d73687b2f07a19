// dist_global.cu — global (cross-part) matching for the row-block partitioned
// hierarchy.
//
// With matching on each part's local graph block (the north-star default,
// dist.cu) aggregates never straddle parts and the hierarchy depends on the
// partition (cfg 2: +2..3 PCG iterations at 2..8 parts). Here the Suitor runs
// on the WHOLE graph: every part proposes along all of its edges, including
// those to other parts' vertices, through suitor words addressed across parts
// (loopback transport: one device; NCCL: CUDA-IPC NVLink peer mappings and
// system-scope 128-bit CAS, matching.cu k_suitor_glob). The Suitor fixed
// point is unique (proj/include/matchamg/matching.hpp:51-57), so the mate
// array — and with it every aggregate, P, Galerkin product and coarse level —
// is bit-identical to the unpartitioned build at any part count.
//
// Aggregates then straddle parts. An aggregate (coarse row) belongs to the
// part of its leader, the smallest member (coarsening.cpp:20-32), so coarse
// blocks stay contiguous in the global numbering. Cross-part pieces:
//  * weights (matching.cpp:60-79): an edge's weight is evaluated by the part
//    holding the upper entry A(min, max) and sent to the other endpoint's part
//    in that part's (ghost column, row) order — the "tplan";
//  * a follower whose leader is remote sends its Galerkin contributions
//    (p_f a_fk) p_k -> agg(k) — the very products the reference forms,
//    coarsening.cpp:125-138 — with p_f and w_f to the leader's part, which
//    replays them after the leader's own row (members ascending);
//  * the level's final P / R get two halo plans: rhalo brings the fine
//    residual of remote members to the aggregate's part before the
//    restriction, phalo the coarse correction back before the prolongation.
// Every exchange is a Halo (dist.cuh) moved by the part's Comm.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <string>

#include "dist.cuh"
#include "rowprod.cuh"

namespace mamg {
namespace {

constexpr int kBlock = 256;

__device__ __forceinline__ int lower_bound_i32(const int32_t* a, int n, int key) {
    int lo = 0, hi = n;
    while (lo < hi) {
        const int mid = lo + ((hi - lo) >> 1); // no int32 overflow past 2^30 entries
        if (a[mid] < key)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}

__global__ void k_iota(int64_t n, int32_t base, int32_t* out) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) out[i] = base + static_cast<int32_t>(i);
}

__global__ void k_rowlen(int64_t n, const int32_t* __restrict__ rp, int32_t* out) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) out[i] = rp[i + 1] - rp[i];
}

__global__ void k_key_in(int64_t n, const int32_t* __restrict__ key, int64_t lo, int64_t hi,
                         int32_t* flag) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) flag[i] = key[i] >= lo && key[i] < hi;
}

__global__ void k_compact(int64_t n, const int32_t* __restrict__ pos, int32_t* out) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n && pos[i + 1] != pos[i]) out[pos[i]] = static_cast<int32_t>(i);
}

__global__ void k_scatter_pos(int64_t m, const int32_t* __restrict__ list, int32_t* out) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t < m) out[list[t]] = static_cast<int32_t>(t);
}

__global__ void k_scatter_f64(int64_t m, const int32_t* __restrict__ list,
                              const double* __restrict__ src, double* dst) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t < m) dst[list[t]] = src[t];
}

__global__ void k_fill_i32(int64_t n, int32_t* x, int32_t v) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) x[i] = v;
}

__global__ void k_gather_i32(int64_t m, const int32_t* __restrict__ idx,
                             const int32_t* __restrict__ src, int32_t* dst) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t < m) dst[t] = src[idx[t]];
}

__global__ void k_sub_i32(int64_t n, const int32_t* __restrict__ a, int32_t off, int32_t* out) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) out[i] = a[i] - off;
}

// tplan receiver: entries whose column lies in a LOWER part, grouped by ghost
// slot (= ascending global column), ascending entry (= row) inside a slot
__global__ void k_low_count(int64_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                            const int32_t* __restrict__ cg, int g0, int32_t* cnt) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    for (int k = rp[i]; k < rp[i + 1]; ++k)
        if (cg[k] < g0) atomicAdd(&cnt[ci[k] - n], 1);
}

__global__ void k_low_fill(int64_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                           const int32_t* __restrict__ cg, int g0, int32_t* cursor, int32_t* list) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    for (int k = rp[i]; k < rp[i + 1]; ++k)
        if (cg[k] < g0) list[atomicAdd(&cursor[ci[k] - n], 1)] = k;
}

// insertion sort of every segment [off[s], off[s+1]) (short segments)
__global__ void k_sort_segments(int64_t nseg, const int32_t* __restrict__ off, int32_t* a) {
    const int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (s >= nseg) return;
    const int lo = off[s], hi = off[s + 1];
    for (int x = lo + 1; x < hi; ++x) {
        const int32_t key = a[x];
        int y = x - 1;
        while (y >= lo && a[y] > key) {
            a[y + 1] = a[y];
            --y;
        }
        a[y + 1] = key;
    }
}

// ------------------------------------------------------------ aggregation --
__global__ void k_leaders_g(int64_t n, int g0, const int32_t* __restrict__ mate, int32_t* flag) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int m = mate[i];
    flag[i] = m < 0 || g0 + static_cast<int>(i) < m;
}

// global aggregate of leaders and local followers; remote followers -1 (their
// leader's part fills the ghost slot); mslot = local (extended) column of the
// mate, found in the row (a matched pair is an edge of A)
__global__ void k_agg_first(int64_t n, int g0, const int32_t* __restrict__ rp,
                            const int32_t* __restrict__ ci, const int32_t* __restrict__ cg,
                            const int32_t* __restrict__ mate, const int32_t* __restrict__ ids,
                            int cbme, int32_t* aggx, int32_t* mslot) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int m = mate[i], I = g0 + static_cast<int>(i);
    int slot = -1;
    if (m >= 0) {
        if (m >= g0 && m < g0 + n) {
            slot = m - g0;
        } else {
            int lo = rp[i], hi = rp[i + 1];
            while (lo < hi) {
                const int mid = lo + ((hi - lo) >> 1); // no int32 overflow past 2^30 entries
                if (cg[mid] < m)
                    lo = mid + 1;
                else
                    hi = mid;
            }
            slot = ci[lo];
        }
    }
    mslot[i] = slot;
    if (m < 0 || I < m)
        aggx[i] = cbme + ids[i];
    else if (m >= g0 && m < g0 + n)
        aggx[i] = cbme + ids[m - g0];
    else
        aggx[i] = -1;
}

__global__ void k_agg_remote(int64_t n, const int32_t* __restrict__ mslot, int32_t* aggx) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n && aggx[i] < 0) aggx[i] = aggx[mslot[i]];
}

// coarsening.cpp:42-74 per row: ||w|_a||^2 = 0.0 + w_lead^2 (+ w_follow^2),
// p_i = w_i / sqrt(.), 1.0 for a zero-norm singleton; a pair with zero norm
// is flagged (by the leader's part) with its global aggregate id
__global__ void k_pvals_g(int64_t n, int g0, const int32_t* __restrict__ mate,
                          const int32_t* __restrict__ mslot, const double* __restrict__ wx,
                          const int32_t* __restrict__ aggx, double* pv, int32_t* bad) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int m = mate[i], I = g0 + static_cast<int>(i);
    const double wi = wx[i];
    double s;
    if (m < 0) {
        s = rn_add(0.0, rn_mul(wi, wi));
    } else {
        const double wm = wx[mslot[i]];
        s = I < m ? rn_add(rn_add(0.0, rn_mul(wi, wi)), rn_mul(wm, wm))
                  : rn_add(rn_add(0.0, rn_mul(wm, wm)), rn_mul(wi, wi));
        if (s == 0.0 && I < m) atomicMin(bad, aggx[i]);
    }
    const double nr = sqrt(s);
    pv[i] = nr == 0.0 ? 1.0 : rn_div(wi, nr);
}

// contributions of the followers sent to their leader's part, in entry order
__global__ void k_payload(int64_t nexp, const int32_t* __restrict__ exp,
                          const int32_t* __restrict__ off, const int32_t* __restrict__ rp,
                          const int32_t* __restrict__ ci, const double* __restrict__ v,
                          const int32_t* __restrict__ aggx, const double* __restrict__ pvx,
                          int32_t* PJ, double* PV) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= nexp) return;
    const int i = exp[t];
    const double pi = pvx[i];
    int o = off[t];
    for (int k = rp[i]; k < rp[i + 1]; ++k, ++o) {
        const int j = ci[k];
        PJ[o] = aggx[j];
        PV[o] = rn_mul(rn_mul(pi, v[k]), pvx[j]);
    }
}

__global__ void k_agg_size_g(int64_t n, int g0, const int32_t* __restrict__ mate,
                             const int32_t* __restrict__ ids, int32_t* size) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int m = mate[i];
    if (m < 0 || g0 + static_cast<int>(i) < m) size[ids[i]] = m < 0 ? 1 : 2;
}

// members (augmented index: owned row x, imported follower n + t) ascending
__global__ void k_members_g(int64_t n, int g0, const int32_t* __restrict__ mate,
                            const int32_t* __restrict__ ids, const int32_t* __restrict__ mptr,
                            const int32_t* __restrict__ imp_gid, int nimp, int32_t* members,
                            int32_t* imp_agg, int32_t* bad) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int m = mate[i];
    if (!(m < 0 || g0 + static_cast<int>(i) < m)) return;
    const int at = mptr[ids[i]];
    members[at] = static_cast<int32_t>(i);
    if (m < 0) return;
    if (m < g0 + n) {
        members[at + 1] = m - g0;
    } else {
        const int t = lower_bound_i32(imp_gid, nimp, m);
        if (t >= nimp || imp_gid[t] != m) {
            atomicMin(bad, static_cast<int32_t>(i));
            return;
        }
        members[at + 1] = static_cast<int32_t>(n) + t;
        imp_agg[t] = ids[i];
    }
}

__global__ void k_gal_ub_g(int64_t nc, const int32_t* __restrict__ mptr,
                           const int32_t* __restrict__ members, const int32_t* __restrict__ rp,
                           int64_t n, const int32_t* __restrict__ ioff, int32_t* ub) {
    const int64_t a = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (a >= nc) return;
    int s = 0;
    for (int m = mptr[a]; m < mptr[a + 1]; ++m) {
        const int x = members[m];
        s += x < n ? rp[x + 1] - rp[x] : ioff[x - n + 1] - ioff[x - n];
    }
    ub[a] = s;
}

// coarse row I: members ascending; an owned member's row is multiplied here
// ((p_i a_ik) p_k, column agg(k)), an imported follower's contributions were
// formed by its own part (same products, same order)
struct GalerkinG {
    const int32_t* __restrict__ mptr;
    const int32_t* __restrict__ members;
    const int32_t* __restrict__ rp;
    const int32_t* __restrict__ ci;
    const double* __restrict__ v;
    const int32_t* __restrict__ aggx;
    const double* __restrict__ pvx;
    int n;
    const int32_t* __restrict__ ioff;
    const int32_t* __restrict__ PJ;
    const double* __restrict__ PV;
    struct Outer {
        double pi;
        int imported;
    };
    __device__ int outer_count(int I) const { return mptr[I + 1] - mptr[I]; }
    __device__ Outer outer(int I, int o, int& lo, int& hi) const {
        const int x = members[mptr[I] + o];
        if (x < n) {
            lo = rp[x];
            hi = rp[x + 1];
            return Outer{pvx[x], 0};
        }
        lo = ioff[x - n];
        hi = ioff[x - n + 1];
        return Outer{0.0, 1};
    }
    __device__ void contrib(const Outer& ou, int e, int32_t& col, double& val) const {
        if (ou.imported) {
            col = PJ[e];
            val = PV[e];
            return;
        }
        const int j = ci[e];
        col = aggx[j];
        val = rn_mul(rn_mul(ou.pi, v[e]), pvx[j]);
    }
};

// composition P = P1 * P2 (kernels.cpp:272-281, one entry per row): the
// coarse-1 aggregate of a row is owned (local id) or remote (its P2 entry
// arrived in the reverse plan's slot for this row)
__global__ void k_compose_g(int64_t n, const int32_t* __restrict__ pc1, const double* __restrict__ pv1,
                            const int32_t* __restrict__ exp_pos, int cb1me, int nc1own,
                            const int32_t* __restrict__ x2c, const double* __restrict__ x2v,
                            int32_t* pc, double* pv) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int e = exp_pos[i];
    const int t = e < 0 ? pc1[i] - cb1me : nc1own + e;
    pc[i] = x2c[t];
    pv[i] = rn_mul(pv1[i], x2v[t]);
}

// ------------------------------------------------------- final operators --
// R rows (own aggregates) over the augmented fine index (owned rows, then
// the rhalo slots of remote members), members ascending by global id
__global__ void k_r_count(int64_t n, int64_t nrecv, const int32_t* __restrict__ pc,
                          const int32_t* __restrict__ pcr, int cbme, int ncown, int32_t* cnt) {
    const int64_t x = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (x >= n + nrecv) return;
    const int a = (x < n ? pc[x] : pcr[x - n]) - cbme;
    if (a >= 0 && a < ncown) atomicAdd(&cnt[a], 1);
}

__global__ void k_r_fill(int64_t n, int64_t nrecv, const int32_t* __restrict__ pc,
                         const int32_t* __restrict__ pcr, int cbme, int ncown, int32_t* cursor,
                         int32_t* rci) {
    const int64_t x = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (x >= n + nrecv) return;
    const int a = (x < n ? pc[x] : pcr[x - n]) - cbme;
    if (a >= 0 && a < ncown) rci[atomicAdd(&cursor[a], 1)] = static_cast<int32_t>(x);
}

__device__ __forceinline__ int aug_gid(int x, int64_t n, int g0, const int32_t* gidr) {
    return x < n ? g0 + x : gidr[x - n];
}

__global__ void k_r_sort(int64_t nrows, const int32_t* __restrict__ rp, int64_t n, int g0,
                         const int32_t* __restrict__ gidr, const double* __restrict__ pv,
                         const double* __restrict__ pvr, int32_t* rci, double* rv, int32_t* rg) {
    const int64_t a = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (a >= nrows) return;
    const int lo = rp[a], hi = rp[a + 1];
    for (int x = lo + 1; x < hi; ++x) {
        const int32_t key = rci[x];
        const int kg = aug_gid(key, n, g0, gidr);
        int y = x - 1;
        while (y >= lo && aug_gid(rci[y], n, g0, gidr) > kg) {
            rci[y + 1] = rci[y];
            --y;
        }
        rci[y + 1] = key;
    }
    for (int e = lo; e < hi; ++e) {
        const int x = rci[e];
        rv[e] = x < n ? pv[x] : pvr[x - n];
        rg[e] = aug_gid(x, n, g0, gidr);
    }
}

__global__ void k_p_local(int64_t n, const int32_t* __restrict__ pc, const double* __restrict__ pv,
                          const int32_t* __restrict__ rem_pos, int cbme, int ncown, int32_t* rp,
                          int32_t* ci, double* v) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i > n) return;
    rp[i] = static_cast<int32_t>(i);
    if (i == n) return;
    const int r = rem_pos[i];
    ci[i] = r < 0 ? pc[i] - cbme : ncown + r;
    v[i] = pv[i];
}

// ============================================================ host side ==
void d2d(Ctx& c, void* dst, const void* src, size_t bytes) {
    if (bytes) MAMG_CU(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, c.stream));
}

// counts[i][q] = elements local part i sends to rank q -> what each local
// part receives from every rank
std::vector<std::vector<int64_t>> exchange_counts(Ctx& c, Comm& comm,
                                                  const std::vector<std::vector<int64_t>>& send) {
    const int W = comm.world;
    std::vector<int64_t> mine;
    for (const auto& v : send) mine.insert(mine.end(), v.begin(), v.end());
    const auto all = comm.allgather_n(c, mine, W); // all[r * W + q] = count r -> q
    std::vector<std::vector<int64_t>> recv(send.size(), std::vector<int64_t>(W, 0));
    for (size_t i = 0; i < send.size(); ++i) {
        const int me = comm.ranks[i];
        for (int r = 0; r < W; ++r) recv[i][r] = all[static_cast<size_t>(r) * W + me];
    }
    return recv;
}

// positions i in [0, n) with key[i] in rank q's block, for every q != me in
// [qlo, qhi), grouped by q, ascending inside a group
DBuf<int32_t> group_by_owner(Ctx& c, int64_t n, const int32_t* key, const std::vector<int64_t>& b,
                             int me, int qlo, int qhi, std::vector<int64_t>& counts) {
    const int W = static_cast<int>(b.size()) - 1;
    counts.assign(W, 0);
    std::vector<DBuf<int32_t>> lists(W);
    DBuf<int32_t> flag(n + 1, c.stream);
    int64_t total = 0;
    for (int q = 0; q < W; ++q) {
        if (q == me || q < qlo || q >= qhi || n == 0 || b[q] == b[q + 1]) continue;
        k_key_in<<<blocks_for(n, kBlock), kBlock, 0, c.stream>>>(n, key, b[q], b[q + 1], flag.get());
        c.count();
        exclusive_scan_i32(c, flag.get(), flag.get(), n);
        const int64_t m = read_i32(c, flag.get() + n);
        counts[q] = m;
        total += m;
        if (m) {
            lists[q].alloc(m, c.stream);
            k_compact<<<blocks_for(n, kBlock), kBlock, 0, c.stream>>>(n, flag.get(), lists[q].get());
            c.count();
        }
    }
    DBuf<int32_t> out(total, c.stream);
    int64_t at = 0;
    for (int q = 0; q < W; ++q) {
        d2d(c, out.get() + at, lists[q].get(), sizeof(int32_t) * counts[q]);
        at += counts[q];
    }
    MAMG_LAUNCH_CHECK();
    return out;
}

Halo make_halo(Ctx& c, int64_t nowned, DBuf<int32_t>&& send_idx, const std::vector<int64_t>& scnt,
               const std::vector<int64_t>& rcnt) {
    Halo h;
    const size_t W = scnt.size();
    h.nowned = nowned;
    h.send_off.assign(W + 1, 0);
    h.recv_off.assign(W + 1, 0);
    for (size_t q = 0; q < W; ++q) {
        h.send_off[q + 1] = h.send_off[q] + scnt[q];
        h.recv_off[q + 1] = h.recv_off[q] + rcnt[q];
    }
    h.nghost = h.recv_off[W];
    h.send_idx = std::move(send_idx);
    h.send_f64.alloc(h.send_off[W], c.stream);
    h.send_i32.alloc(h.send_off[W], c.stream);
    return h;
}

std::vector<int64_t> counts_of(const std::vector<int64_t>& off) {
    std::vector<int64_t> c(off.size() - 1);
    for (size_t q = 0; q + 1 < off.size(); ++q) c[q] = off[q + 1] - off[q];
    return c;
}

template <class T>
std::vector<T*> ptrs(std::vector<DBuf<T>>& v) {
    std::vector<T*> out;
    for (auto& b : v) out.push_back(b.get());
    return out;
}

std::vector<Halo*> hptrs(std::vector<Halo>& v) {
    std::vector<Halo*> out;
    for (auto& h : v) out.push_back(&h);
    return out;
}


int64_t total_of(const std::vector<int64_t>& v) {
    int64_t s = 0;
    for (auto x : v) s += x;
    return s;
}

// one pairwise step with the global Suitor (per local part)
struct GStep {
    DBuf<int32_t> pc;           // per owned fine row: global coarse id
    DBuf<double> pv;            // and its P value
    std::unique_ptr<DevCsr> Ac; // own coarse rows, GLOBAL columns
    DBuf<double> wc;
    int64_t nc_own = 0;
    Halo fw;               // followers -> their leader's part (fine side)
    DBuf<int32_t> imp_agg; // per imported follower: local coarse id
    DBuf<int32_t> exp_pos; // per owned fine row: slot in fw's send list, -1
};

// L: the level's local parts (localized, with halo plans); w their smooth
// vectors. Fills out[i] per local part, cb = coarse blocks (world + 1).
void gstep(Ctx& c, DistHier& d, std::vector<PLevel*>& L, std::vector<const double*>& w,
           std::vector<GStep>& out, std::vector<int64_t>& cb, int64_t& zero_edges) {
    static const bool trace_on = std::getenv("MAMG_TRACE_DIST") != nullptr;
    auto tstart = std::chrono::steady_clock::now();
    auto gmark = [&](const char* what) {
        if (!trace_on) return;
        c.sync();
        std::fprintf(stderr, "[gstep rank %d n=%lld] %s %.0f ms\n", d.parts[0].rank,
                     static_cast<long long>(L[0]->A->nrows), what,
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tstart).count());
    };

    Comm& comm = *d.comm;
    const int W = comm.world;
    const size_t np = L.size();
    out.clear();
    out.resize(np);
    std::vector<int64_t> zs(np, 0);
    std::vector<int32_t*> flags(np);
    std::vector<unsigned long long*> zc(np);
    std::vector<Halo*> lh;
    for (auto* lv : L) lh.push_back(&lv->halo);
    // ---- 1. diagonal and w over owned + ghost columns
    std::vector<DBuf<double>> dgx(np), wx(np);
    for (size_t i = 0; i < np; ++i) {
        PLevel& lv = *L[i];
        const int64_t n = lv.A->nrows, ext = n + lv.halo.nghost;
        const int64_t g0 = lv.g0;
        flags[i] = defer_flags(c, 3, [g0](int j, int32_t row) {
            const int64_t r = row + g0;
            if (j == 0) invalid("build_weights: non-positive diagonal in row " + std::to_string(r), r);
            if (j == 1)
                invalid("build_weights: pattern not symmetric, offending row " + std::to_string(r), r);
            invalid("build_weights: non-finite weight produced in row " + std::to_string(r), r);
        });
        int64_t* zdst = &zs[i];
        zc[i] = defer_counter(c, [zdst](int64_t v) { *zdst = v; });
        dgx[i].alloc(ext, c.stream);
        wx[i].alloc(ext, c.stream);
        diag_owned(c, *lv.A, lv.cg.get(), g0, dgx[i].get(), flags[i]);
        d2d(c, wx[i].get(), w[i], sizeof(double) * n);
    }
    comm.halo_f64(c, lh, ptrs(dgx));
    comm.halo_f64(c, lh, ptrs(wx));
    gmark("2. tplan");
    // ---- 2. tplan: weights of edges to lower parts arrive from those parts
    std::vector<Halo> tp(np);
    std::vector<DBuf<int32_t>> trecv(np);
    std::vector<std::vector<int64_t>> tsend(np), trcnt(np);
    for (size_t i = 0; i < np; ++i) {
        PLevel& lv = *L[i];
        const DevCsr& A = *lv.A;
        const int me = d.parts[i].rank;
        const int64_t n = A.nrows;
        const int64_t nlow = lv.halo.recv_off[me]; // ghost slots of lower parts
        DBuf<int32_t> cnt(nlow + 1, c.stream);
        MAMG_CU(cudaMemsetAsync(cnt.get(), 0, sizeof(int32_t) * (nlow + 1), c.stream));
        if (n && nlow) {
            k_low_count<<<blocks_for(n, kBlock), kBlock, 0, c.stream>>>(
                n, A.rp.get(), A.ci.get(), lv.cg.get(), static_cast<int>(lv.g0), cnt.get());
            c.count();
        }
        exclusive_scan_i32(c, cnt.get(), cnt.get(), nlow);
        std::vector<int32_t> off(nlow + 1);
        MAMG_CU(cudaMemcpyAsync(off.data(), cnt.get(), sizeof(int32_t) * (nlow + 1),
                                cudaMemcpyDeviceToHost, c.stream));
        c.sync();
        const int64_t nrecv = off[nlow];
        trecv[i].alloc(nrecv, c.stream);
        if (nrecv) {
            DBuf<int32_t> cursor(nlow + 1, c.stream);
            d2d(c, cursor.get(), cnt.get(), sizeof(int32_t) * (nlow + 1));
            k_low_fill<<<blocks_for(n, kBlock), kBlock, 0, c.stream>>>(
                n, A.rp.get(), A.ci.get(), lv.cg.get(), static_cast<int>(lv.g0), cursor.get(),
                trecv[i].get());
            k_sort_segments<<<blocks_for(nlow, kBlock), kBlock, 0, c.stream>>>(nlow, cnt.get(),
                                                                               trecv[i].get());
            c.count(2);
        }
        trcnt[i].assign(W, 0);
        for (int q = 0; q < me; ++q)
            trcnt[i][q] = off[lv.halo.recv_off[q + 1]] - off[lv.halo.recv_off[q]];
        DBuf<int32_t> sl = group_by_owner(c, A.nnz, lv.cg.get(), lv.bounds, me, me + 1, W, tsend[i]);
        tp[i] = make_halo(c, A.nnz, std::move(sl), tsend[i], trcnt[i]);
    }
    {
        const auto got = exchange_counts(c, comm, tsend);
        for (size_t i = 0; i < np; ++i)
            if (got[i] != trcnt[i]) invalid("build_hierarchy: matrix pattern is not symmetric");
    }
    gmark("3. weights");
    // ---- 3. weights (own upper entries), exchange, scatter
    std::vector<DBuf<double>> wt(np);
    for (size_t i = 0; i < np; ++i) {
        PLevel& lv = *L[i];
        wt[i].alloc(lv.A->nnz + tp[i].nghost, c.stream);
        weights_global(c, *lv.A, lv.cg.get(), lv.g0, dgx[i].get(), wx[i].get(), wt[i].get(),
                       flags[i] + 1, zc[i]);
    }
    comm.halo_f64(c, hptrs(tp), ptrs(wt));
    for (size_t i = 0; i < np; ++i) {
        const int64_t m = tp[i].nghost;
        if (m) {
            k_scatter_f64<<<blocks_for(m, kBlock), kBlock, 0, c.stream>>>(
                m, trecv[i].get(), wt[i].get() + L[i]->A->nnz, wt[i].get());
            c.count();
        }
    }
    gmark("4. candidates");
    // ---- 4. candidates into the shared Suitor blocks, 5. global Suitor
    if (W > kMaxWorld) invalid("global matching: at most 16 parts");
    std::vector<int64_t> my_nnz;
    for (auto* lv : L) my_nnz.push_back(lv->A->nnz);
    const auto all_nnz = comm.allgather(c, my_nnz);
    const std::vector<int64_t>& b = L[0]->bounds;
    std::vector<size_t> bytes;
    for (size_t i = 0; i < np; ++i) bytes.push_back(suitor_block(L[i]->A->nrows, L[i]->A->nnz).bytes);
    const auto blocks = comm.shared_blocks(c, bytes);
    SuitorView g;
    g.world = W;
    for (int r = 0; r <= W; ++r) g.bounds[r] = static_cast<int>(b[r]);
    for (int r = 0; r < W; ++r) {
        const SuitorBlock sb = suitor_block(b[r + 1] - b[r], all_nnz[r]);
        char* base = static_cast<char*>(blocks[r]);
        g.S[r] = base + sb.s_off;
        g.cand[r] = base + sb.cand_off;
        g.rp[r] = reinterpret_cast<const int32_t*>(base + sb.rp_off);
        g.ncand[r] = reinterpret_cast<const int32_t*>(base + sb.ncand_off);
    }
    for (size_t i = 0; i < np; ++i) {
        const int me = d.parts[i].rank;
        const DevCsr& A = *L[i]->A;
        d2d(c, const_cast<int32_t*>(g.rp[me]), A.rp.get(), sizeof(int32_t) * (A.nrows + 1));
        candidates_into(c, A.nrows, A.nnz, A.rp.get(), L[i]->cg.get(), wt[i].get(),
                        const_cast<void*>(g.cand[me]), const_cast<int32_t*>(g.ncand[me]));
    }
    const bool sys = comm.peer_memory();
    comm.barrier(c); // no rank still reads the previous step's words
    for (size_t i = 0; i < np; ++i) {
        const int me = d.parts[i].rank;
        suitor_global_init(c, g.S[me], b[me + 1] - b[me]);
    }
    comm.barrier(c);
    gmark("suitor start");
    for (size_t i = 0; i < np; ++i) suitor_global(c, g, d.parts[i].rank, sys);
    gmark("suitor done");
    comm.barrier(c);
    std::vector<DBuf<int32_t>> mate(np);
    for (size_t i = 0; i < np; ++i) {
        mate[i].alloc(L[i]->A->nrows, c.stream);
        mate_global(c, g, d.parts[i].rank, sys, mate[i].get());
    }
    gmark("6. aggregates");
    // ---- 6. aggregates: leaders own them, ids follow the leaders globally
    std::vector<DBuf<int32_t>> ids(np);
    std::vector<int64_t> ncs;
    for (size_t i = 0; i < np; ++i) {
        const int64_t n = L[i]->A->nrows;
        ids[i].alloc(n + 1, c.stream);
        if (n) {
            k_leaders_g<<<blocks_for(n, kBlock), kBlock, 0, c.stream>>>(
                n, static_cast<int>(L[i]->g0), mate[i].get(), ids[i].get());
            c.count();
        }
        exclusive_scan_i32(c, ids[i].get(), ids[i].get(), n);
        ncs.push_back(read_i32(c, ids[i].get() + n));
    }
    on_all_ranks(c, comm, [&] { sync_checked(c); }); // diagonal / weight checks; zero edges
    zero_edges = total_of(comm.allgather(c, zs));
    cb = prefix_of(comm.allgather(c, ncs));
    const int64_t nc_glob = cb.back();
    std::vector<DBuf<int32_t>> aggx(np), mslot(np);
    std::vector<DBuf<double>> pvx(np);
    for (size_t i = 0; i < np; ++i) {
        PLevel& lv = *L[i];
        const int me = d.parts[i].rank;
        const int64_t n = lv.A->nrows, ext = n + lv.halo.nghost;
        out[i].nc_own = ncs[i];
        aggx[i].alloc(ext, c.stream);
        mslot[i].alloc(n, c.stream);
        pvx[i].alloc(ext, c.stream);
        if (n) {
            k_agg_first<<<blocks_for(n, kBlock), kBlock, 0, c.stream>>>(
                n, static_cast<int>(lv.g0), lv.A->rp.get(), lv.A->ci.get(), lv.cg.get(),
                mate[i].get(), ids[i].get(), static_cast<int>(cb[me]), aggx[i].get(),
                mslot[i].get());
            c.count();
        }
    }
    comm.halo_i32(c, lh, ptrs(aggx)); // leaders' ids reach their remote followers
    for (size_t i = 0; i < np; ++i) {
        const int64_t n = L[i]->A->nrows;
        if (n) {
            k_agg_remote<<<blocks_for(n, kBlock), kBlock, 0, c.stream>>>(n, mslot[i].get(),
                                                                         aggx[i].get());
            c.count();
        }
    }
    comm.halo_i32(c, lh, ptrs(aggx)); // every ghost column's aggregate
    for (size_t i = 0; i < np; ++i) {
        const int64_t n = L[i]->A->nrows;
        int32_t* vanish = defer_flags(c, 1, [](int, int32_t a) {
            invalid("build_prolongator: smooth vector vanishes on aggregate " + std::to_string(a), a);
        });
        if (n) {
            k_pvals_g<<<blocks_for(n, kBlock), kBlock, 0, c.stream>>>(
                n, static_cast<int>(L[i]->g0), mate[i].get(), mslot[i].get(), wx[i].get(),
                aggx[i].get(), pvx[i].get(), vanish);
            c.count();
        }
    }
    comm.halo_f64(c, lh, ptrs(pvx)); // every ghost column's p
    gmark("7. followers");
    // ---- 7. followers with a remote (always lower) leader -> leader's part
    std::vector<std::vector<int64_t>> fsend(np);
    std::vector<DBuf<int32_t>> flist(np);
    for (size_t i = 0; i < np; ++i) {
        const int me = d.parts[i].rank;
        flist[i] = group_by_owner(c, L[i]->A->nrows, mate[i].get(), L[i]->bounds, me, 0, me, fsend[i]);
    }
    const auto frecv = exchange_counts(c, comm, fsend);
    std::vector<Halo> fw(np);
    std::vector<DBuf<int32_t>> gidx(np), lenx(np);
    std::vector<DBuf<double>> pvaug(np), waug(np);
    for (size_t i = 0; i < np; ++i) {
        PLevel& lv = *L[i];
        const int64_t n = lv.A->nrows;
        const int64_t nexp = total_of(fsend[i]);
        out[i].exp_pos.alloc(n, c.stream);
        if (n) {
            k_fill_i32<<<blocks_for(n, kBlock), kBlock, 0, c.stream>>>(n, out[i].exp_pos.get(), -1);
            c.count();
        }
        if (nexp) {
            k_scatter_pos<<<blocks_for(nexp, kBlock), kBlock, 0, c.stream>>>(
                nexp, flist[i].get(), out[i].exp_pos.get());
            c.count();
        }
        fw[i] = make_halo(c, n, std::move(flist[i]), fsend[i], frecv[i]);
        const int64_t ext = n + fw[i].nghost;
        gidx[i].alloc(ext, c.stream);
        lenx[i].alloc(ext + 1, c.stream);
        pvaug[i].alloc(ext, c.stream);
        waug[i].alloc(ext, c.stream);
        if (n) {
            k_iota<<<blocks_for(n, kBlock), kBlock, 0, c.stream>>>(n, static_cast<int32_t>(lv.g0),
                                                                   gidx[i].get());
            k_rowlen<<<blocks_for(n, kBlock), kBlock, 0, c.stream>>>(n, lv.A->rp.get(),
                                                                     lenx[i].get());
            c.count(2);
        }
        d2d(c, pvaug[i].get(), pvx[i].get(), sizeof(double) * n);
        d2d(c, waug[i].get(), w[i], sizeof(double) * n);
    }
    {
        auto fwp = hptrs(fw);
        comm.halo_i32(c, fwp, ptrs(gidx));
        comm.halo_i32(c, fwp, ptrs(lenx));
        comm.halo_f64(c, fwp, ptrs(pvaug));
        comm.halo_f64(c, fwp, ptrs(waug));
    }
    // payload: the exported rows' contributions, concatenated in send order;
    // both sides derive the segment sizes from the exchanged row lengths
    std::vector<Halo> pl(np);
    std::vector<DBuf<int32_t>> PJ(np), ioff(np);
    std::vector<DBuf<double>> PV(np);
    std::vector<int64_t> psend_tot(np);
    for (size_t i = 0; i < np; ++i) {
        PLevel& lv = *L[i];
        const int64_t n = lv.A->nrows;
        const Halo& f = fw[i];
        const int64_t nexp = f.send_off.back(), nimp = f.nghost;
        DBuf<int32_t> soff(nexp + 1, c.stream);
        if (nexp) {
            k_gather_i32<<<blocks_for(nexp, kBlock), kBlock, 0, c.stream>>>(
                nexp, f.send_idx.get(), lenx[i].get(), soff.get());
            c.count();
        }
        exclusive_scan_i32(c, soff.get(), soff.get(), nexp);
        ioff[i].alloc(nimp + 1, c.stream);
        d2d(c, ioff[i].get(), lenx[i].get() + n, sizeof(int32_t) * nimp);
        exclusive_scan_i32(c, ioff[i].get(), ioff[i].get(), nimp);
        std::vector<int32_t> hs(nexp + 1), hr(nimp + 1);
        MAMG_CU(cudaMemcpyAsync(hs.data(), soff.get(), sizeof(int32_t) * (nexp + 1),
                                cudaMemcpyDeviceToHost, c.stream));
        MAMG_CU(cudaMemcpyAsync(hr.data(), ioff[i].get(), sizeof(int32_t) * (nimp + 1),
                                cudaMemcpyDeviceToHost, c.stream));
        c.sync();
        std::vector<int64_t> ps(W), pr(W);
        for (int q = 0; q < W; ++q) {
            ps[q] = hs[f.send_off[q + 1]] - hs[f.send_off[q]];
            pr[q] = hr[f.recv_off[q + 1]] - hr[f.recv_off[q]];
        }
        const int64_t stot = hs[nexp], rtot = hr[nimp];
        psend_tot[i] = stot;
        PJ[i].alloc(stot + rtot, c.stream);
        PV[i].alloc(stot + rtot, c.stream);
        if (nexp) {
            k_payload<<<blocks_for(nexp, kBlock), kBlock, 0, c.stream>>>(
                nexp, f.send_idx.get(), soff.get(), lv.A->rp.get(), lv.A->ci.get(), lv.A->v.get(),
                aggx[i].get(), pvx[i].get(), PJ[i].get(), PV[i].get());
            c.count();
        }
        DBuf<int32_t> ident(stot, c.stream);
        if (stot) {
            k_iota<<<blocks_for(stot, kBlock), kBlock, 0, c.stream>>>(stot, 0, ident.get());
            c.count();
        }
        pl[i] = make_halo(c, stot, std::move(ident), ps, pr);
    }
    comm.halo_i32(c, hptrs(pl), ptrs(PJ));
    comm.halo_f64(c, hptrs(pl), ptrs(PV));
    // ---- 8. own aggregates over the augmented rows (owned + imported)
    for (size_t i = 0; i < np; ++i) {
        PLevel& lv = *L[i];
        GStep& o = out[i];
        const int64_t n = lv.A->nrows, nimp = fw[i].nghost, nc = o.nc_own;
        DevAgg ga;
        ga.n = n;
        ga.nc = nc;
        ga.mptr.alloc(nc + 1, c.stream);
        ga.members.alloc(n + nimp, c.stream);
        MAMG_CU(cudaMemsetAsync(ga.mptr.get(), 0, sizeof(int32_t) * (nc + 1), c.stream));
        o.imp_agg.alloc(nimp, c.stream);
        int32_t* bad = defer_flags(c, 1, [](int, int32_t row) {
            throw Error(MAMG_RUNTIME,
                        "global matching: remote follower missing for row " + std::to_string(row),
                        row);
        });
        if (n) {
            k_agg_size_g<<<blocks_for(n, kBlock), kBlock, 0, c.stream>>>(
                n, static_cast<int>(lv.g0), mate[i].get(), ids[i].get(), ga.mptr.get());
            c.count();
        }
        exclusive_scan_i32(c, ga.mptr.get(), ga.mptr.get(), nc);
        if (n) {
            k_members_g<<<blocks_for(n, kBlock), kBlock, 0, c.stream>>>(
                n, static_cast<int>(lv.g0), mate[i].get(), ids[i].get(), ga.mptr.get(),
                gidx[i].get() + n, static_cast<int>(nimp), ga.members.get(), o.imp_agg.get(), bad);
            c.count();
        }
        DBuf<int32_t> ub(nc + 1, c.stream);
        if (nc) {
            k_gal_ub_g<<<blocks_for(nc, kBlock), kBlock, 0, c.stream>>>(
                nc, ga.mptr.get(), ga.members.get(), lv.A->rp.get(), n, ioff[i].get(), ub.get());
            c.count();
        }
        MAMG_LAUNCH_CHECK();
        GalerkinG pb{ga.mptr.get(), ga.members.get(), lv.A->rp.get(), lv.A->ci.get(),
                     lv.A->v.get(),  aggx[i].get(),    pvx[i].get(),    static_cast<int>(n),
                     ioff[i].get(),  PJ[i].get() + psend_tot[i],       PV[i].get() + psend_tot[i]};
        o.Ac = rowprod_run(c, pb, nc, nc_glob, ub);
        o.wc.alloc(nc, c.stream);
        restrict_members(c, ga, pvaug[i].get(), waug[i].get(), o.wc.get());
        o.pc.alloc(n, c.stream);
        o.pv.alloc(n, c.stream);
        d2d(c, o.pc.get(), aggx[i].get(), sizeof(int32_t) * n);
        d2d(c, o.pv.get(), pvx[i].get(), sizeof(double) * n);
        o.fw = std::move(fw[i]);
    }
    on_all_ranks(c, comm, [&] { sync_checked(c); });
}

// P = P1 * P2 over the parts: a row whose coarse-1 aggregate is remote gets
// that aggregate's (P2 column, P2 value) through step 1's plan reversed
void compose_global(Ctx& c, DistHier& d, std::vector<PLevel*>& L, std::vector<GStep>& s1,
                    const std::vector<int64_t>& cb1, std::vector<GStep>& s2,
                    std::vector<DBuf<int32_t>>& pc, std::vector<DBuf<double>>& pv) {
    Comm& comm = *d.comm;
    const size_t np = L.size();
    std::vector<Halo> rev(np);
    std::vector<DBuf<int32_t>> x2c(np);
    std::vector<DBuf<double>> x2v(np);
    for (size_t i = 0; i < np; ++i) {
        const Halo& f = s1[i].fw;
        const int64_t nc1 = s1[i].nc_own, nexp = f.send_off.back(), nimp = f.nghost;
        DBuf<int32_t> sidx(nimp, c.stream);
        d2d(c, sidx.get(), s1[i].imp_agg.get(), sizeof(int32_t) * nimp);
        rev[i] = make_halo(c, nc1, std::move(sidx), counts_of(f.recv_off), counts_of(f.send_off));
        x2c[i].alloc(nc1 + nexp, c.stream);
        x2v[i].alloc(nc1 + nexp, c.stream);
        d2d(c, x2c[i].get(), s2[i].pc.get(), sizeof(int32_t) * nc1);
        d2d(c, x2v[i].get(), s2[i].pv.get(), sizeof(double) * nc1);
    }
    comm.halo_i32(c, hptrs(rev), ptrs(x2c));
    comm.halo_f64(c, hptrs(rev), ptrs(x2v));
    pc.clear();
    pv.clear();
    pc.resize(np);
    pv.resize(np);
    for (size_t i = 0; i < np; ++i) {
        const int64_t n = L[i]->A->nrows;
        const int me = d.parts[i].rank;
        pc[i].alloc(n, c.stream);
        pv[i].alloc(n, c.stream);
        if (n) {
            k_compose_g<<<blocks_for(n, kBlock), kBlock, 0, c.stream>>>(
                n, s1[i].pc.get(), s1[i].pv.get(), s1[i].exp_pos.get(), static_cast<int>(cb1[me]),
                static_cast<int>(s1[i].nc_own), x2c[i].get(), x2v[i].get(), pc[i].get(), pv[i].get());
            c.count();
        }
    }
    MAMG_LAUNCH_CHECK();
}

// The level's P and R from the final (global) aggregate map, with the halo
// plans of the cycle: rhalo (fine values of remote members -> the
// aggregate's part) and phalo (its reverse, coarse values back).
void finalize_global(Ctx& c, DistHier& d, std::vector<PLevel*>& L, std::vector<DBuf<int32_t>>& pc,
                     std::vector<DBuf<double>>& pv, const std::vector<int64_t>& cb) {
    Comm& comm = *d.comm;
    const int W = comm.world;
    const size_t np = L.size();
    std::vector<std::vector<int64_t>> scnt(np);
    std::vector<DBuf<int32_t>> rem(np);
    for (size_t i = 0; i < np; ++i)
        rem[i] = group_by_owner(c, L[i]->A->nrows, pc[i].get(), cb, d.parts[i].rank, 0, W, scnt[i]);
    const auto rcnt = exchange_counts(c, comm, scnt);
    std::vector<Halo> rh(np);
    std::vector<DBuf<int32_t>> rem_pos(np), gidx(np), pcx(np);
    std::vector<DBuf<double>> pvx(np);
    for (size_t i = 0; i < np; ++i) {
        PLevel& lv = *L[i];
        const int64_t n = lv.A->nrows, nrem = total_of(scnt[i]);
        rem_pos[i].alloc(n, c.stream);
        if (n) {
            k_fill_i32<<<blocks_for(n, kBlock), kBlock, 0, c.stream>>>(n, rem_pos[i].get(), -1);
            c.count();
        }
        if (nrem) {
            k_scatter_pos<<<blocks_for(nrem, kBlock), kBlock, 0, c.stream>>>(nrem, rem[i].get(),
                                                                             rem_pos[i].get());
            c.count();
        }
        rh[i] = make_halo(c, n, std::move(rem[i]), scnt[i], rcnt[i]);
        const int64_t ext = n + rh[i].nghost;
        gidx[i].alloc(ext, c.stream);
        pcx[i].alloc(ext, c.stream);
        pvx[i].alloc(ext, c.stream);
        if (n) {
            k_iota<<<blocks_for(n, kBlock), kBlock, 0, c.stream>>>(n, static_cast<int32_t>(lv.g0),
                                                                   gidx[i].get());
            c.count();
        }
        d2d(c, pcx[i].get(), pc[i].get(), sizeof(int32_t) * n);
        d2d(c, pvx[i].get(), pv[i].get(), sizeof(double) * n);
    }
    comm.halo_i32(c, hptrs(rh), ptrs(gidx));
    comm.halo_i32(c, hptrs(rh), ptrs(pcx));
    comm.halo_f64(c, hptrs(rh), ptrs(pvx));
    for (size_t i = 0; i < np; ++i) {
        PLevel& lv = *L[i];
        const int me = d.parts[i].rank;
        const int64_t n = lv.A->nrows, nrecv = rh[i].nghost, nrem = rh[i].send_off.back();
        const int cbme = static_cast<int>(cb[me]);
        const int64_t ncown = cb[me + 1] - cb[me];
        // R: own aggregates, members ascending by global id
        auto R = std::make_unique<DevCsr>();
        R->nrows = ncown;
        R->ncols = n + nrecv;
        R->rp.alloc(ncown + 1, c.stream);
        MAMG_CU(cudaMemsetAsync(R->rp.get(), 0, sizeof(int32_t) * (ncown + 1), c.stream));
        const int64_t aug = n + nrecv;
        if (aug) {
            k_r_count<<<blocks_for(aug, kBlock), kBlock, 0, c.stream>>>(
                n, nrecv, pc[i].get(), pcx[i].get() + n, cbme, static_cast<int>(ncown), R->rp.get());
            c.count();
        }
        exclusive_scan_i32(c, R->rp.get(), R->rp.get(), ncown);
        R->nnz = read_i32(c, R->rp.get() + ncown);
        R->ci.alloc(R->nnz, c.stream);
        R->v.alloc(R->nnz, c.stream);
        lv.Rg.alloc(R->nnz, c.stream);
        if (aug && R->nnz) {
            DBuf<int32_t> cursor(ncown + 1, c.stream);
            d2d(c, cursor.get(), R->rp.get(), sizeof(int32_t) * (ncown + 1));
            k_r_fill<<<blocks_for(aug, kBlock), kBlock, 0, c.stream>>>(
                n, nrecv, pc[i].get(), pcx[i].get() + n, cbme, static_cast<int>(ncown), cursor.get(),
                R->ci.get());
            k_r_sort<<<blocks_for(ncown, kBlock), kBlock, 0, c.stream>>>(
                ncown, R->rp.get(), n, static_cast<int>(lv.g0), gidx[i].get() + n, pv[i].get(),
                pvx[i].get() + n, R->ci.get(), R->v.get(), lv.Rg.get());
            c.count(2);
        }
        MAMG_LAUNCH_CHECK();
        csr_finalize(c, *R);
        set_policy(*R, cb.back(), d.level_n.back(), false);
        // P: own rows; a remote aggregate is read from its phalo slot
        auto P = std::make_unique<DevCsr>();
        P->nrows = n;
        P->ncols = ncown + nrem;
        P->nnz = n;
        P->rp.alloc(n + 1, c.stream);
        P->ci.alloc(n, c.stream);
        P->v.alloc(n, c.stream);
        k_p_local<<<blocks_for(n + 1, kBlock), kBlock, 0, c.stream>>>(
            n, pc[i].get(), pv[i].get(), rem_pos[i].get(), cbme, static_cast<int>(ncown),
            P->rp.get(), P->ci.get(), P->v.get());
        c.count();
        P->max_tile = 256;
        set_policy(*P, d.level_n.back(), d.level_n.back(), true);
        // phalo: for every received member, its aggregate's coarse value back
        DBuf<int32_t> sidx(nrecv, c.stream);
        if (nrecv) {
            k_sub_i32<<<blocks_for(nrecv, kBlock), kBlock, 0, c.stream>>>(nrecv, pcx[i].get() + n,
                                                                          cbme, sidx.get());
            c.count();
        }
        lv.phalo = make_halo(c, ncown, std::move(sidx), counts_of(rh[i].recv_off),
                             counts_of(rh[i].send_off));
        lv.rhalo = std::move(rh[i]);
        lv.Pg = std::move(pc[i]);
        lv.P = std::move(P);
        lv.R = std::move(R);
    }
    MAMG_LAUNCH_CHECK();
}

} // namespace

bool dist_step_global(Ctx& c, DistHier& d, int k, int aggregation, std::vector<PLevel>& coarse,
                      int64_t& zero_edges) {
    const size_t np = d.parts.size();
    const int W = d.comm->world;
    std::vector<PLevel*> L;
    std::vector<const double*> w;
    for (auto& p : d.parts) {
        L.push_back(&p.lv[k]);
        w.push_back(p.lv[k].w.get());
    }
    std::vector<GStep> s1, s2;
    std::vector<int64_t> cb1, cb2;
    int64_t z1 = 0, z2 = 0;
    gstep(c, d, L, w, s1, cb1, z1);
    zero_edges = z1;
    std::vector<DBuf<int32_t>> pc(np);
    std::vector<DBuf<double>> pv(np);
    std::vector<GStep>* fin = &s1;
    std::vector<int64_t> cbf = cb1;
    std::vector<PLevel> tmp(np);
    if (aggregation != 1) {
        std::vector<int64_t> nnzs;
        for (auto& s : s1) nnzs.push_back(s.Ac->nnz);
        const int64_t nnz1 = sum_all(d.comm->allgather(c, nnzs));
        std::vector<PLevel*> T;
        std::vector<const double*> tw;
        for (size_t i = 0; i < np; ++i) {
            tmp[i].bounds = cb1;
            tmp[i].nglob = cb1.back();
            tmp[i].nnzglob = nnz1;
            tmp[i].A = std::move(s1[i].Ac);
            localize(c, W, d.parts[i].rank, tmp[i]);
            set_policy(*tmp[i].A, cb1.back(), nnz1, false);
            T.push_back(&tmp[i]);
            tw.push_back(s1[i].wc.get());
        }
        gstep(c, d, T, tw, s2, cb2, z2);
        zero_edges += z2;
        compose_global(c, d, L, s1, cb1, s2, pc, pv);
        fin = &s2;
        cbf = cb2;
    } else {
        for (size_t i = 0; i < np; ++i) {
            pc[i] = std::move(s1[i].pc);
            pv[i] = std::move(s1[i].pv);
        }
    }
    if (cbf.back() == d.level_n[k]) return false; // stall (coarsening.cpp:224-227)
    finalize_global(c, d, L, pc, pv, cbf);
    std::vector<int64_t> nnzs;
    for (auto& s : *fin) nnzs.push_back(s.Ac->nnz);
    const int64_t nnz_c = sum_all(d.comm->allgather(c, nnzs));
    coarse.clear();
    coarse.resize(np);
    for (size_t i = 0; i < np; ++i) {
        PLevel& C = coarse[i];
        C.bounds = cbf;
        C.nglob = cbf.back();
        C.nnzglob = nnz_c;
        C.A = std::move((*fin)[i].Ac);
        C.A->ncols = cbf.back();
        C.w = std::move((*fin)[i].wc);
    }
    return true;
}

} // namespace mamg
