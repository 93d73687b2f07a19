// matching.cu — edge weights C(A, w) and the parallel Suitor matching on
// sm_100a (proj/src/matching.cpp).
//
// Weights (matching.cpp:28-101) are computed in place over A's pattern: the
// graph is A's off-diagonal pattern, so the weight array is aligned with A's
// entries and the diagonal slots hold -1 (a negative weight is never proposed
// along, matching.cpp:130, which is the same as the edge being absent). Each
// weight is evaluated from the upper-triangle entry A(min, max) with the
// reference's exact operation order, so both directions carry the identical
// double (the total edge order below needs that).
//
// Suitor (matching.cpp:117-154) runs one thread per start vertex. A suitor
// slot is one 64-bit word: (proposer index << 32) | (position of the edge in
// the proposer's adjacency row); the proposal's weight is read from that
// position, so a plain 64-bit atomicCAS installs a proposal exactly — no
// weight rounding — and the order "heavier wins, equal weight -> smaller
// opposite endpoint" (edge_beats, matching.cpp:108-113, specialised to a
// shared endpoint) is evaluated on the full doubles. A dislodged vertex is
// re-proposed by the same thread inside the same kernel (matching.cpp:139-143),
// so the long dislodgement chains of constant-coefficient grids cost no extra
// launches. Under a strict total edge order the Suitor fixed point is unique
// (= greedy matching, matching.hpp:51-57), hence the mate array equals the
// sequential reference's for any interleaving.
#include <cstdlib>

#include "ops.cuh"

namespace mamg {
namespace {

constexpr int kBlock = 256;
constexpr unsigned long long kEmpty = ~0ull;
constexpr int kSuitorCap = 16; // proposals before a chain is parked (k_suitor_resume)

__device__ __forceinline__ int find_in_row(const int32_t* __restrict__ ci, int lo, int hi, int j) {
    while (lo < hi) {
        const int mid = lo + ((hi - lo) >> 1); // no int32 overflow past 2^30 entries
        if (ci[mid] < j)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}

// diagonal(A) (csr.cpp:99-104) + the positivity check (matching.cpp:35-40)
// cg: global (sorted) column ids used for lookups; g0: global id of local row 0
__global__ void k_diag(int64_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ cg,
                       const double* __restrict__ v, int g0, double* dg, int32_t* bad) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int lo = rp[i], hi = rp[i + 1];
    const int gi = g0 + static_cast<int>(i);
    const int p = find_in_row(cg, lo, hi, gi);
    const double d = (p < hi && cg[p] == gi) ? v[p] : 0.0;
    dg[i] = d;
    if (!(d > 0.0)) atomicMin(bad, static_cast<int32_t>(i));
}

// flags: [0] lowest asymmetric row, [1] lowest non-finite-weight row
// Partitioned matrices: ci holds local ids (owned rows < n, ghosts >= n),
// cg the global ids; an edge to a ghost column is masked (weight -1, matching
// on local graph blocks only). Unpartitioned: cg == ci, g0 == 0.
// An S-lane group per row (S >= the mean row length, like the lane policy):
// lane l evaluates entries lo+l, lo+l+S, ... so the row's loads coalesce and
// the per-entry lookups of A(j, i) run in parallel.
template <int S>
__global__ void __launch_bounds__(kBlock)
k_weights(int64_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
          const int32_t* __restrict__ cg, int g0, const double* __restrict__ v,
          const double* __restrict__ dg, const double* __restrict__ w, double* wt, int32_t* flags,
          unsigned long long* zero_edges) {
    const int64_t row = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / S;
    if (row >= n) return;
    const int i = static_cast<int>(row);
    const int lane = threadIdx.x & (S - 1);
    unsigned zeros = 0;
    for (int k = rp[i] + lane; k < rp[i + 1]; k += S) {
        const int j = ci[k];
        if (j == i || j >= n) {
            wt[k] = -1.0;
            continue;
        }
        const int jlo = rp[j], jhi = rp[j + 1];
        const int m = find_in_row(cg, jlo, jhi, g0 + i);
        if (m >= jhi || cg[m] != g0 + i) {
            atomicMin(&flags[0], i);
            wt[k] = -1.0;
            continue;
        }
        const int p = i < j ? i : j, q = i < j ? j : i;
        const double apq = i < j ? v[k] : v[m];
        // den = d_p*w_p*w_p + d_q*w_q*w_q   (left to right, no contraction)
        const double den = rn_add(rn_mul(rn_mul(dg[p], w[p]), w[p]), rn_mul(rn_mul(dg[q], w[q]), w[q]));
        double c;
        if (den == 0.0) {
            c = 0.0;
            if (i < j) ++zeros;
        } else {
            // c = 1 - 2*a_pq*w_p*w_q/den
            c = rn_sub(1.0, rn_div(rn_mul(rn_mul(rn_mul(2.0, apq), w[p]), w[q]), den));
        }
        if (!isfinite(c)) atomicMin(&flags[1], i);
        wt[k] = c;
    }
    if (zeros) atomicAdd(zero_edges, static_cast<unsigned long long>(zeros));
}

__device__ __forceinline__ bool beats(double c1, int u1, double c2, int u2) {
    return c1 > c2 || (c1 == c2 && u1 < u2);
}

// One candidate of a vertex: opposite endpoint + edge weight (16 B, one load).
struct __align__(16) Cand {
    int32_t v;
    int32_t pad;
    double w;
};


// Per vertex: its admissible edges (c >= 0, matching.cpp:130) sorted by the
// proposal order of matching.cpp:134-136 — weight descending, then opposite
// endpoint ascending — stored in the vertex's own slice [rp[i], rp[i+1]).
// An S-lane group per vertex ranks every candidate against all others of the
// row (a strict total order: endpoints are distinct) with group shuffles and
// scatters it to its rank: no data-dependent loops, coalesced loads.
template <int S>
__global__ void __launch_bounds__(kBlock)
k_candidates(int64_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
             const double* __restrict__ wt, Cand* cand, int32_t* ncand) {
    const int64_t row = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / S;
    const int lane = threadIdx.x & (S - 1);
    const unsigned gmask =
        S == 32 ? 0xffffffffu : (((1u << S) - 1u) << (threadIdx.x & 31 & ~(S - 1)));
    int lo = 0, hi = 0; // rows past n stay in the loop with no entries (shuffle partners)
    if (row < n) {
        lo = rp[row];
        hi = rp[row + 1];
    }
    int total = 0;
    for (int base = lo; base < hi; base += S) {
        const int k = base + lane;
        double wk = -1.0;
        int vk = 0;
        if (k < hi) {
            wk = wt[k];
            vk = ci[k];
        }
        int rank = 0;
        for (int b2 = lo; b2 < hi; b2 += S) {
            const int k2 = b2 + lane;
            double w2 = -1.0;
            int v2 = 0;
            if (k2 < hi) {
                w2 = wt[k2];
                v2 = ci[k2];
            }
#pragma unroll
            for (int l = 0; l < S; ++l) {
                const double wl = __shfl_sync(gmask, w2, l, S);
                const int vl = __shfl_sync(gmask, v2, l, S);
                rank += (wl >= 0.0) & beats(wl, vl, wk, vk);
            }
        }
        const bool ok = wk >= 0.0;
        if (ok) cand[lo + rank] = Cand{vk, 0, wk};
        total += __popc(__ballot_sync(gmask, ok) & gmask);
    }
    // the slice's unused slots (non-admissible entries) get a sentinel: the
    // Suitor's speculative next-candidate prefetch may read them
    for (int k = lo + total + lane; k < hi; k += S) cand[k] = Cand{-1, 0, -1.0};
    if (lane == 0 && row < n) ncand[row] = total;
}

// Bitonic sort of a full warp's candidate pairs, Q per lane (Q <= 4 of the
// caller's 4-slot arrays; sorted position Q lane + q), into the proposal
// order (beats first). Every lane of the warp takes part.
struct WV {
    double w;
    int v;
};
template <int Q>
__device__ __forceinline__ void sort_cands(double (&w)[4], int (&v)[4], int lane) {
    WV x[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) x[q] = WV{w[q], v[q]};
    warp_bitonic<Q>(
        x, lane, [](const WV& a, const WV& b) { return beats(a.w, a.v, b.w, b.v); },
        [](const WV& a, int m) {
            return WV{__shfl_xor_sync(0xffffffffu, a.w, m), __shfl_xor_sync(0xffffffffu, a.v, m)};
        });
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        w[q] = x[q].w;
        v[q] = x[q].v;
    }
}

// The edge weight of entry k of row i (matching.cpp:60-79), -1 for the
// diagonal, masked ghost columns and asymmetric entries (flagged).
__device__ __forceinline__ double edge_weight(int i, int k, int lo_i, int n,
                                              const int32_t* __restrict__ rp,
                                              const int32_t* __restrict__ ci,
                                              const int32_t* __restrict__ cg, int g0,
                                              const double* __restrict__ v,
                                              const double* __restrict__ dg,
                                              const double* __restrict__ w, int32_t* flags,
                                              unsigned& zeros, bool check_upper = true,
                                              int32_t* asym = nullptr) {
    const int j = ci[k];
    if (j == i || j >= n) return -1.0;
    // the mirror entry A(j, i): needed for the value of a lower entry, and
    // for the pattern check (matching.cpp:64) — which levels that are
    // symmetric by construction (Galerkin products) skip for upper entries
    int m = k;
    if (i > j || check_upper) {
        const int jlo = rp[j], jhi = rp[j + 1];
        // stencil-symmetric rows (interior rows of a stencil, and rows of
        // the same shape): j at position p of row i puts i at position
        // len_j - 1 - p of row j. Taken when it holds (the first entry with
        // column i); otherwise the bisection. Scalar stencils only (rows of
        // up to 32 entries): in block stencils (3 dofs per node) the guess
        // misses two times in three and costs more than it saves (measured).
        const int m0 = jhi - 1 - (k - lo_i);
        const int key = g0 + i;
        if (jhi - jlo <= 32 && m0 >= jlo && __ldg(cg + m0) == key &&
            (m0 == jlo || __ldg(cg + m0 - 1) != key)) {
            m = m0;
        } else {
            m = find_in_row(cg, jlo, jhi, key);
            if (m >= jhi || cg[m] != key) {
                atomicMin(asym ? asym : &flags[0], i);
                return -1.0;
            }
        }
    }
    const int p = i < j ? i : j, q = i < j ? j : i;
    const double apq = i < j ? v[k] : v[m];
    const double den = rn_add(rn_mul(rn_mul(dg[p], w[p]), w[p]), rn_mul(rn_mul(dg[q], w[q]), w[q]));
    double c;
    if (den == 0.0) {
        c = 0.0;
        if (i < j) ++zeros;
    } else {
        c = rn_sub(1.0, rn_div(rn_mul(rn_mul(rn_mul(2.0, apq), w[p]), w[q]), den));
    }
    if (!isfinite(c)) atomicMin(&flags[1], i);
    return c;
}

// build_weights + candidate ranking fused (the setup's pairwise step never
// needs the weights themselves, only the sorted candidates): an S-lane group
// per row computes the row's weights into registers (up to 4 chunks of S),
// ranks them with group shuffles and scatters the admissible ones. Longer
// rows spill their weights to `wt` and rank from there. flags: the three
// build_weights check slots [diag, asymmetric, non-finite] (k_diag writes [0]).
#ifndef MAMG_WCAND_MINB
#define MAMG_WCAND_MINB 6
#endif
template <int S>
__global__ void __launch_bounds__(kBlock, MAMG_WCAND_MINB)
k_weights_cand(int64_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
               const int32_t* __restrict__ cg, int g0, const double* __restrict__ v,
               const double* __restrict__ dg,
               const double* __restrict__ w, double* wt, Cand* cand, int32_t* ncand,
               int32_t* flags, unsigned long long* zero_edges, int check_upper, int32_t* asym) {
    constexpr int kCh = 4;
    const int64_t row = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / S;
    const int lane = threadIdx.x & (S - 1);
    const unsigned gmask =
        S == 32 ? 0xffffffffu : (((1u << S) - 1u) << (threadIdx.x & 31 & ~(S - 1)));
    int lo = 0, hi = 0;
    if (row < n) {
        lo = rp[row];
        hi = rp[row + 1];
    }
    const int i = static_cast<int>(row);
    const int nch = (hi - lo + S - 1) / S;
    unsigned zeros = 0;
    int total = 0;
    if (nch <= kCh) {
        double wk[kCh];
        int vk[kCh];
#pragma unroll
        for (int q = 0; q < kCh; ++q) {
            const int k = lo + q * S + lane;
            wk[q] = -1.0;
            vk[q] = 0;
            if (q < nch && k < hi) {
                vk[q] = ci[k];
                wk[q] = edge_weight(i, k, lo, static_cast<int>(n), rp, ci, cg, g0, v, dg, w, flags + 1, zeros, check_upper != 0, asym);
            }
        }
        if (S == 32 && nch >= 1) {
            // rows of a whole warp: bitonic sort of the (weight, vertex) pairs
            // in registers (position Q lane + q) under the proposal order
            // (beats; non-admissible w = -1 sort last) — the sorted position
            // is the candidate's rank, without the all-pairs ranking (for one
            // chunk: 15 exchange stages instead of 32 shuffle rounds)
            const int Q = nch <= 1 ? 1 : (nch <= 2 ? 2 : 4);
#pragma unroll
            for (int q = 0; q < kCh; ++q) total += __popc(__ballot_sync(gmask, wk[q] >= 0.0));
            if (nch <= 1)
                sort_cands<1>(wk, vk, lane);
            else if (nch <= 2)
                sort_cands<2>(wk, vk, lane);
            else
                sort_cands<4>(wk, vk, lane);
#pragma unroll
            for (int q = 0; q < kCh; ++q) {
                const int pos = Q * lane + q;
                if (q < Q && pos < total) cand[lo + pos] = Cand{vk[q], 0, wk[q]};
            }
        } else {
#pragma unroll
        for (int q = 0; q < kCh; ++q) {
            if (q >= nch) break;
            int rank = 0;
#pragma unroll
            for (int q2 = 0; q2 < kCh; ++q2) {
                if (q2 >= nch) break;
#pragma unroll
                for (int l = 0; l < S; ++l) {
                    const double wl = __shfl_sync(gmask, wk[q2], l, S);
                    const int vl = __shfl_sync(gmask, vk[q2], l, S);
                    rank += (wl >= 0.0) & beats(wl, vl, wk[q], vk[q]);
                }
            }
            const bool ok = wk[q] >= 0.0;
            if (ok) cand[lo + rank] = Cand{vk[q], 0, wk[q]};
            total += __popc(__ballot_sync(gmask, ok) & gmask);
        }
        }
    } else {
        for (int k = lo + lane; k < hi; k += S)
            wt[k] = edge_weight(i, k, lo, static_cast<int>(n), rp, ci, cg, g0, v, dg, w, flags + 1, zeros, check_upper != 0, asym);
        __syncwarp(gmask);
        for (int base = lo; base < hi; base += S) {
            const int k = base + lane;
            double wkk = -1.0;
            int vkk = 0;
            if (k < hi) {
                wkk = wt[k];
                vkk = ci[k];
            }
            int rank = 0;
            for (int b2 = lo; b2 < hi; b2 += S) {
                const int k2 = b2 + lane;
                double w2 = -1.0;
                int v2 = 0;
                if (k2 < hi) {
                    w2 = wt[k2];
                    v2 = ci[k2];
                }
#pragma unroll
                for (int l = 0; l < S; ++l) {
                    const double wl = __shfl_sync(gmask, w2, l, S);
                    const int vl = __shfl_sync(gmask, v2, l, S);
                    rank += (wl >= 0.0) & beats(wl, vl, wkk, vkk);
                }
            }
            const bool ok = wkk >= 0.0;
            if (ok) cand[lo + rank] = Cand{vkk, 0, wkk};
            total += __popc(__ballot_sync(gmask, ok) & gmask);
        }
    }
    if (zeros) atomicAdd(zero_edges, static_cast<unsigned long long>(zeros));
    for (int k = lo + total + lane; k < hi; k += S) cand[k] = Cand{-1, 0, -1.0}; // (see k_candidates)
    if (lane == 0 && row < n) ncand[row] = total;
}

// Suitor with per-vertex cursors. A vertex u walks its sorted candidates;
// the first v whose current suitor u beats is the reference's `best`
// (every earlier candidate is either better-suited already — and suitors
// only improve, so it stays that way — or was taken from u by a better
// proposer); a dislodged proposer resumes right after the slot it lost, so
// each vertex scans its list once overall.
// The suitor word is 16 bytes {weight, (proposer << 32) | slot}:
// the current suitor's weight travels with it, so deciding whether a
// proposal wins needs no dependent load of the holder's candidate slot — one
// memory round trip less per link of a dislodgement chain. The word is read
// with one single-copy-atomic 128-bit load (LDG.E.128.STRONG.GPU) and
// replaced with a 128-bit CAS (ATOMG.E.CAS.128), so the comparison always
// sees a consistent (weight, proposer) pair.
struct __align__(16) Suit {
    double w;
    unsigned long long u; // (proposer << 32) | slot, kEmpty if none
};

__device__ __forceinline__ Suit ld_suit(const Suit* p) {
    unsigned long long lo, hi;
    asm volatile("{ .reg .b128 r; ld.relaxed.gpu.global.b128 r, [%2]; mov.b128 {%0, %1}, r; }"
                 : "=l"(lo), "=l"(hi)
                 : "l"(p)
                 : "memory");
    Suit x;
    x.w = __longlong_as_double(static_cast<long long>(lo));
    x.u = hi;
    return x;
}

__global__ void k_suit_init(int n, Suit* S) {
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v < n) S[v] = Suit{0.0, kEmpty};
}

// Per link of a dislodgement chain three dependent round trips remain: the
// dislodged vertex's next candidate, the target's suitor word, the CAS. The
// first overlaps the previous CAS: the word read before a CAS already names
// the vertex the CAS would dislodge, so its next candidate (and list end) is
// loaded alongside the CAS and is in registers when the chain continues.
#ifdef MAMG_SUITOR_PROF
__device__ unsigned long long g_prof_t0 = ~0ull;
__device__ unsigned long long g_prof_st[1 << 23];
__device__ unsigned long long g_prof_fin[1 << 23];
__device__ int g_prof_np[1 << 23];
__device__ unsigned long long g_cyc_ld[1 << 23], g_cyc_cas[1 << 23], g_cyc_pf[1 << 23];
__global__ void k_suitor_prof_report(int n) {
    // one thread: finish-time percentiles (us after the first start) and proposals
    if (threadIdx.x || blockIdx.x) return;
    unsigned long long tmax = 0;
    long long tot = 0;
    int npmax = 0, imax = 0;
    for (int i = 0; i < n; ++i) g_prof_t0 = g_prof_st[i] < g_prof_t0 ? g_prof_st[i] : g_prof_t0;
    for (int i = 0; i < n; ++i) {
        if (g_prof_np[i] > npmax) imax = i;
        const unsigned long long d = g_prof_fin[i] - g_prof_t0;
        tmax = d > tmax ? d : tmax;
        tot += g_prof_np[i];
        npmax = g_prof_np[i] > npmax ? g_prof_np[i] : npmax;
    }
    int hist[20] = {0};
    for (int i = 0; i < n; ++i) {
        int b = static_cast<int>((g_prof_fin[i] - g_prof_t0) * 20 / (tmax + 1));
        hist[b]++;
    }
    printf("suitor n=%d span=%.1f us proposals=%lld max/thread=%d | finish hist (20 bins):", n,
           tmax / 1e3, tot, npmax);
    for (int b = 0; b < 20; ++b) printf(" %d", hist[b]);
    unsigned long long lastst = 0;
    for (int i = 0; i < n; ++i) lastst = g_prof_st[i] - g_prof_t0 > lastst ? g_prof_st[i] - g_prof_t0 : lastst;
    printf(" | longest chain thread %d: start %.1f us finish %.1f us; last thread start %.1f us; "
           "per proposal ns: cand+ld_suit %.0f cas %.0f; CAS attempts %.2f per proposal\n", imax,
           (g_prof_st[imax] - g_prof_t0) / 1e3, (g_prof_fin[imax] - g_prof_t0) / 1e3, lastst / 1e3,
           (double)g_cyc_ld[imax] / npmax, (double)g_cyc_cas[imax] / npmax, (double)g_cyc_pf[imax] / npmax);
    for (int i = 0; i < n; ++i) g_cyc_ld[i] = g_cyc_cas[i] = g_cyc_pf[i] = 0;
    g_prof_t0 = ~0ull;
}
#endif

// One chain of proposals starting with vertex `start` at candidate slot rk
// (rk < 0: its first candidate). cap > 0: after `cap` proposals the chain is
// parked (current vertex, candidate slot) in park[] and the thread leaves;
// the parked chains continue in k_suitor_resume — a later interleaving of the
// same proposals, so the fixed point is unchanged.
__device__ __forceinline__ void suitor_chain(int start, int rk, int64_t ncand_total,
                                             const int32_t* __restrict__ rp,
                                             const Cand* __restrict__ cand,
                                             const int32_t* __restrict__ ncand, Suit* S, int cap,
                                             int2* park, int* npark) {
    int nprop_cap = 0;
#ifdef MAMG_SUITOR_PROF
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    if (rk < 0) g_prof_st[start] = t0;
    int nprop = 0;
    struct Fin {
        int& np;
        int st;
        __device__ ~Fin() {
            unsigned long long t1;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
            g_prof_fin[st] = t1;
            g_prof_np[st] = np;
        }
    } fin{nprop, start};
#endif
    int cur = start;
    int k = __ldg(rp + cur);
    int end = k + __ldg(ncand + cur);
    if (rk >= 0) k = rk;
    Cand pref{};
    bool have = false;
    for (;;) {
        unsigned long long won = kEmpty;
        bool placed = false;
        Cand nxt{};
        int w_rp = 0, w_nc = 0; // list start / length of the would-be dislodged vertex
        for (; k < end; ++k) {
            if (cap > 0 && ++nprop_cap > cap) {
                park[atomicAdd(npark, 1)] = make_int2(cur, k);
                return;
            }
            const Cand e = have ? pref : cand[k];
            have = false;
#ifdef MAMG_SUITOR_PROF
            unsigned long long c_a, c_b;
            if (e.v == -12345) nprop += 7;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(c_a));
#endif
            Suit s = ld_suit(&S[e.v]);
            const Suit mine{e.w, (static_cast<unsigned long long>(static_cast<uint32_t>(cur)) << 32) |
                                     static_cast<uint32_t>(k)};
#ifdef MAMG_SUITOR_PROF
            if (s.u == 0x123456789ull) nprop += 7;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(c_b));
            g_cyc_ld[start] += c_b - c_a;
            ++nprop;
#endif
            for (;;) {
                if (s.u != kEmpty && !beats(e.w, cur, s.w, static_cast<int>(s.u >> 32))) break;
                if (s.u != kEmpty) { // prefetch the would-be dislodged vertex's next candidate
                    const int w = static_cast<int>(s.u >> 32);
                    const int64_t ws = static_cast<int64_t>(static_cast<uint32_t>(s.u)) + 1;
                    nxt = cand[ws < ncand_total ? ws : ncand_total - 1];
                    // consumed only after the CAS: combining them here made the
                    // CAS wait for these loads (ncu: a third round trip per link)
                    w_rp = __ldg(rp + w);
                    w_nc = __ldg(ncand + w);
                }
#ifdef MAMG_SUITOR_PROF
                unsigned long long c_c, c_d;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(c_c));
#endif
                const Suit old = atomicCAS(&S[e.v], s, mine);
#ifdef MAMG_SUITOR_PROF
                if (old.u == 0x123456789ull) nprop += 7;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(c_d));
                g_cyc_cas[start] += c_d - c_c;
                g_cyc_pf[start] += 1; // CAS attempts
#endif
                if (old.u == s.u && __double_as_longlong(old.w) == __double_as_longlong(s.w)) {
                    placed = true;
                    break;
                }
                s = old;
            }
            if (placed) {
                won = s.u;
                break;
            }
        }
        if (!placed || won == kEmpty) return;
#ifdef MAMG_SUITOR_PROF
#endif
        cur = static_cast<int>(won >> 32);
        k = static_cast<int>(static_cast<uint32_t>(won)) + 1;
        end = w_rp + w_nc;
        pref = nxt;
        have = k < end;
    }
}

__global__ void __launch_bounds__(kBlock)
k_suitor128(int n, int64_t ncand_total, const int32_t* __restrict__ rp,
            const Cand* __restrict__ cand, const int32_t* __restrict__ ncand, Suit* S, int cap,
            int2* park, int* npark) {
    const int start = blockIdx.x * kBlock + threadIdx.x;
    if (start >= n) return;
    suitor_chain(start, -1, ncand_total, rp, cand, ncand, S, cap, park, npark);
}

// The parked chains, one per warp while they fit in the grid (more lanes per
// warp when many were parked), grid-strided. Measured: the long dislodgement
// chains of constant-coefficient grids advance faster here than among the
// first launch's millions of short ones (cfg 2 setup 10.2 -> 8.7 ms); where
// most chains are long anyway (cfg 4: 3% of the vertices parked) the extra
// phase costs ~0.5 ms of a 14 ms setup.
__global__ void __launch_bounds__(kBlock)
k_suitor_resume(int64_t ncand_total, const int32_t* __restrict__ rp, const Cand* __restrict__ cand,
                const int32_t* __restrict__ ncand, Suit* S, const int* __restrict__ nparked,
                const int2* __restrict__ parked) {
    const int gt = blockIdx.x * kBlock + threadIdx.x;
    const int np = *nparked;
    const int warps = gridDim.x * (kBlock / 32);
    // chains per warp: one while they fit, more lanes when many were parked
    const int per = min(32, max(1, (np + warps - 1) / warps));
    const int lane = gt & 31;
    if (lane >= per) return;
    for (int q = (gt >> 5) * per + lane; q < np; q += warps * per)
        suitor_chain(parked[q].x, parked[q].y, ncand_total, rp, cand, ncand, S, 0, nullptr, nullptr);
}

__global__ void k_mate128(int n, const Suit* __restrict__ S, int32_t* mate) {
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    const unsigned long long s = S[v].u;
    int m = -1;
    if (s != kEmpty) {
        const int u = static_cast<int>(s >> 32);
        const unsigned long long su = S[u].u;
        if (su != kEmpty && static_cast<int>(su >> 32) == v) m = u;
    }
    mate[v] = m;
}

__global__ void k_offdiag_count(int64_t n, const int32_t* __restrict__ rp,
                                const int32_t* __restrict__ ci, int32_t* deg) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int d = 0;
    for (int k = rp[i]; k < rp[i + 1]; ++k) d += ci[k] != i;
    deg[i] = d;
}

__global__ void k_offdiag_copy(int64_t n, const int32_t* __restrict__ rp,
                               const int32_t* __restrict__ ci, const double* __restrict__ wt,
                               const int32_t* __restrict__ xadj, int32_t* adj, double* gw) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int pos = xadj[i];
    for (int k = rp[i]; k < rp[i + 1]; ++k) {
        if (ci[k] == i) continue;
        adj[pos] = ci[k];
        gw[pos] = wt[k];
        ++pos;
    }
}

// ------------------------------------------------- global (cross-part) --
// Same Suitor walk over a partitioned graph: vertex
// ids are global, a vertex's candidates / suitor word live in its owner
// part's block, reached through the view's pointer table. The proposer id
// in a suitor word is global and its slot indexes the proposer's part's
// candidate array. Sys = system-scope loads / CAS (the words of other GPUs
// are NVLink peer memory); otherwise device scope (all parts on one GPU).
template <bool Sys>
__device__ __forceinline__ Suit ld_suit_s(const Suit* p) {
    unsigned long long lo, hi;
    if constexpr (Sys)
        asm volatile("{ .reg .b128 r; ld.relaxed.sys.global.b128 r, [%2]; mov.b128 {%0, %1}, r; }"
                     : "=l"(lo), "=l"(hi)
                     : "l"(p)
                     : "memory");
    else
        asm volatile("{ .reg .b128 r; ld.relaxed.gpu.global.b128 r, [%2]; mov.b128 {%0, %1}, r; }"
                     : "=l"(lo), "=l"(hi)
                     : "l"(p)
                     : "memory");
    Suit x;
    x.w = __longlong_as_double(static_cast<long long>(lo));
    x.u = hi;
    return x;
}

template <bool Sys>
__device__ __forceinline__ Suit cas_suit_s(Suit* p, Suit cmp, Suit val) {
    const unsigned long long cw = static_cast<unsigned long long>(__double_as_longlong(cmp.w));
    const unsigned long long vw = static_cast<unsigned long long>(__double_as_longlong(val.w));
    unsigned long long lo, hi;
    if constexpr (Sys)
        asm volatile(
            "{ .reg .b128 d, c, s; mov.b128 c, {%2, %3}; mov.b128 s, {%4, %5};"
            " atom.relaxed.sys.global.cas.b128 d, [%6], c, s; mov.b128 {%0, %1}, d; }"
            : "=l"(lo), "=l"(hi)
            : "l"(cw), "l"(cmp.u), "l"(vw), "l"(val.u), "l"(p)
            : "memory");
    else
        asm volatile(
            "{ .reg .b128 d, c, s; mov.b128 c, {%2, %3}; mov.b128 s, {%4, %5};"
            " atom.relaxed.gpu.global.cas.b128 d, [%6], c, s; mov.b128 {%0, %1}, d; }"
            : "=l"(lo), "=l"(hi)
            : "l"(cw), "l"(cmp.u), "l"(vw), "l"(val.u), "l"(p)
            : "memory");
    Suit x;
    x.w = __longlong_as_double(static_cast<long long>(lo));
    x.u = hi;
    return x;
}

__device__ __forceinline__ int owner_of(const SuitorView& g, int v) {
    int r = 0;
    while (r + 1 < g.world && v >= g.bounds[r + 1]) ++r;
    return r;
}

// One chain of the cross-part Suitor from global vertex cur at slot k of
// its part's list; with cap > 0 it is parked after cap proposals (as in the
// single-device Suitor: a later interleaving of the same proposals)
template <bool Sys>
__device__ __forceinline__ void suitor_glob_chain(const SuitorView& g, int cur, int k, int cap,
                                                  int2* park, int* npark) {
    int rc = owner_of(g, cur);
    int end = g.rp[rc][cur - g.bounds[rc]] + g.ncand[rc][cur - g.bounds[rc]];
    int nprop = 0;
    for (;;) {
        const Cand* cl = static_cast<const Cand*>(g.cand[rc]);
        unsigned long long won = kEmpty;
        bool placed = false;
        for (; k < end; ++k) {
            if (cap > 0 && ++nprop > cap) {
                park[atomicAdd(npark, 1)] = make_int2(cur, k);
                return;
            }
            const Cand e = cl[k];
            const int re = owner_of(g, e.v);
            Suit* tgt = static_cast<Suit*>(g.S[re]) + (e.v - g.bounds[re]);
            Suit s = ld_suit_s<Sys>(tgt);
            const Suit mine{e.w, (static_cast<unsigned long long>(static_cast<uint32_t>(cur)) << 32) |
                                     static_cast<uint32_t>(k)};
            for (;;) {
                if (s.u != kEmpty && !beats(e.w, cur, s.w, static_cast<int>(s.u >> 32))) break;
                const Suit old = cas_suit_s<Sys>(tgt, s, mine);
                if (old.u == s.u && __double_as_longlong(old.w) == __double_as_longlong(s.w)) {
                    placed = true;
                    break;
                }
                s = old;
            }
            if (placed) {
                won = s.u;
                break;
            }
        }
        if (!placed || won == kEmpty) return;
        // the dislodged vertex (any part) resumes after its lost slot
        cur = static_cast<int>(won >> 32);
        rc = owner_of(g, cur);
        k = static_cast<int>(static_cast<uint32_t>(won)) + 1;
        const int lc = cur - g.bounds[rc];
        end = g.rp[rc][lc] + g.ncand[rc][lc];
    }
}

template <bool Sys>
__global__ void __launch_bounds__(kBlock)
k_suitor_glob(const SuitorView g, int me, int cap, int2* park, int* npark) {
    const int t = blockIdx.x * kBlock + threadIdx.x;
    if (t >= g.bounds[me + 1] - g.bounds[me]) return;
    suitor_glob_chain<Sys>(g, g.bounds[me] + t, g.rp[me][t], cap, park, npark);
}

// the parked chains, spread over the warps (k_suitor_resume)
template <bool Sys>
__global__ void __launch_bounds__(kBlock)
k_suitor_glob_resume(const SuitorView g, const int* __restrict__ nparked,
                     const int2* __restrict__ parked) {
    const int gt = blockIdx.x * kBlock + threadIdx.x;
    const int np = *nparked;
    const int warps = gridDim.x * (kBlock / 32);
    const int per = min(32, max(1, (np + warps - 1) / warps));
    const int lane = gt & 31;
    if (lane >= per) return;
    for (int q = (gt >> 5) * per + lane; q < np; q += warps * per)
        suitor_glob_chain<Sys>(g, parked[q].x, parked[q].y, 0, nullptr, nullptr);
}

template <bool Sys>
__global__ void k_mate_glob(const SuitorView g, int me, int32_t* mate) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= g.bounds[me + 1] - g.bounds[me]) return;
    const int v = g.bounds[me] + t;
    const unsigned long long s = ld_suit_s<Sys>(static_cast<const Suit*>(g.S[me]) + t).u;
    int m = -1;
    if (s != kEmpty) {
        const int u = static_cast<int>(s >> 32);
        const int ru = owner_of(g, u);
        const unsigned long long su =
            ld_suit_s<Sys>(static_cast<const Suit*>(g.S[ru]) + (u - g.bounds[ru])).u;
        if (su != kEmpty && static_cast<int>(su >> 32) == v) m = u;
    }
    mate[t] = m;
}

// Weights of the owned rows of a partitioned level (see weights_global).
template <int S>
__global__ void __launch_bounds__(kBlock)
k_weights_glob(int64_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
               const int32_t* __restrict__ cg, int g0, const double* __restrict__ v,
               const double* __restrict__ dg, const double* __restrict__ w, double* wt,
               int32_t* flags, unsigned long long* zero_edges) {
    const int64_t row = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / S;
    if (row >= n) return;
    const int i = static_cast<int>(row);
    const int I = g0 + i;
    const int lane = threadIdx.x & (S - 1);
    unsigned zeros = 0;
    for (int k = rp[i] + lane; k < rp[i + 1]; k += S) {
        const int J = cg[k];
        if (J == I) {
            wt[k] = -1.0;
            continue;
        }
        if (J < g0) continue; // lower part: its owner evaluates A(J, I)
        const int j = ci[k];
        int p, q;
        double apq;
        if (j < n) {
            const int m = find_in_row(cg, rp[j], rp[j + 1], I);
            if (m >= rp[j + 1] || cg[m] != I) {
                atomicMin(&flags[0], i);
                wt[k] = -1.0;
                continue;
            }
            p = i < j ? i : j;
            q = i < j ? j : i;
            apq = i < j ? v[k] : v[m];
        } else { // ghost of a higher part: this row holds the upper entry
            p = i;
            q = j;
            apq = v[k];
        }
        const double den = rn_add(rn_mul(rn_mul(dg[p], w[p]), w[p]), rn_mul(rn_mul(dg[q], w[q]), w[q]));
        double c;
        if (den == 0.0) {
            c = 0.0;
            if (I < J) ++zeros;
        } else {
            c = rn_sub(1.0, rn_div(rn_mul(rn_mul(rn_mul(2.0, apq), w[p]), w[q]), den));
        }
        if (!isfinite(c)) atomicMin(&flags[1], i);
        wt[k] = c;
    }
    if (zeros) atomicAdd(zero_edges, static_cast<unsigned long long>(zeros));
}

// lanes per row group for the setup's row kernels: the lane policy's rule
// (smallest power of two >= the mean row length), at least 4, at most 32
int group_lanes(int64_t n, int64_t nnz) {
    const double mean = n > 0 ? static_cast<double>(nnz) / static_cast<double>(n) : 0.0;
    int S = 4;
    while (S < 32 && S < mean) S *= 2;
    return S;
}

} // namespace

void build_weights_aligned(Ctx& c, const DevCsr& A, const double* w, DBuf<double>& wt,
                           int64_t& zero_edges, const int32_t* cg, int64_t g0) {
    wt.alloc(A.nnz, c.stream);
    build_weights_into(c, A, w, wt.get(), zero_edges, cg, g0);
}

void build_weights_into(Ctx& c, const DevCsr& A, const double* w, double* wt_out,
                        int64_t& zero_edges, const int32_t* cg, int64_t g0) {
    if (!cg && A.nrows != A.ncols) invalid("build_weights: matrix is not square");
    if (!cg) cg = A.ci.get();
    const int64_t n = A.nrows;
    zero_edges = 0;
    if (n == 0) return;
    DBuf<double> dg(n, c.stream);
    // scratch: [0] bad diag, [1] bad pattern, [2] bad weight (int32), then u64 zero count
    int32_t* flags = reinterpret_cast<int32_t*>(c.d_small.get());
    unsigned long long* zc = reinterpret_cast<unsigned long long*>(c.d_small.get() + 2);
    const int32_t init[4] = {INT32_MAX, INT32_MAX, INT32_MAX, 0};
    MAMG_CU(cudaMemcpyAsync(flags, init, sizeof(init), cudaMemcpyHostToDevice, c.stream));
    MAMG_CU(cudaMemsetAsync(zc, 0, sizeof(unsigned long long), c.stream));
    k_diag<<<blocks_for(n, kBlock), kBlock, 0, c.stream>>>(n, A.rp.get(), cg, A.v.get(),
                                                           static_cast<int>(g0), dg.get(), flags);
    {
        const int S = group_lanes(A.nrows, A.nnz);
        auto go = [&](auto kern) {
            kern<<<blocks_for(n * S, kBlock), kBlock, 0, c.stream>>>(
                n, A.rp.get(), A.ci.get(), cg, static_cast<int>(g0), A.v.get(), dg.get(), w,
                wt_out, flags + 1, zc);
        };
        switch (S) {
            case 4: go(k_weights<4>); break;
            case 8: go(k_weights<8>); break;
            case 16: go(k_weights<16>); break;
            default: go(k_weights<32>); break;
        }
    }
    c.count(2);
    MAMG_LAUNCH_CHECK();
    int64_t h[3];
    MAMG_CU(cudaMemcpyAsync(h, c.d_small.get(), sizeof(h), cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    const int32_t* hf = reinterpret_cast<const int32_t*>(h);
    if (hf[0] != INT32_MAX)
        invalid("build_weights: non-positive diagonal in row " + std::to_string(hf[0]), hf[0]);
    if (hf[1] != INT32_MAX)
        invalid("build_weights: pattern not symmetric, offending row " + std::to_string(hf[1]),
                hf[1]);
    if (hf[2] != INT32_MAX)
        invalid("build_weights: non-finite weight produced in row " + std::to_string(hf[2]),
                hf[2]);
    zero_edges = h[2];
}

// Suitor over candidate lists already built (cand/ncand in the context's
// scratch slots): 16-byte suitor words, then the mutual test.
static void suitor_from_candidates(Ctx& c, int64_t n, int64_t cand_total, const int32_t* rp,
                                   const Cand* cand, const int32_t* ncand, int32_t* mate) {
    Suit* S2 = c.scratch<Suit>(Ctx::kScrSuitor, n);
    k_suit_init<<<blocks_for(n, kBlock), kBlock, 0, c.stream>>>(static_cast<int>(n), S2);
    // chains still running after kSuitorCap proposals are parked and resumed
    // by k_suitor_resume (cfg 2 setup: 10.2 -> 8.7 ms; MAMG_SUITOR_CAP=0 runs
    // every chain to its end in the first launch)
    static const int cap = [] {
        const char* e = std::getenv("MAMG_SUITOR_CAP");
        return e ? std::atoi(e) : kSuitorCap;
    }();
    if (cap > 0 && n > 4096) {
        int2* park = c.scratch<int2>(Ctx::kScrPark, n);
        int* np = reinterpret_cast<int*>(c.d_small.get() + 24);
        MAMG_CU(cudaMemsetAsync(np, 0, sizeof(int), c.stream));
        k_suitor128<<<blocks_for(n, kBlock), kBlock, 0, c.stream>>>(
            static_cast<int>(n), cand_total, rp, cand, ncand, S2, cap, park, np);
        k_suitor_resume<<<c.num_sms * 8, kBlock, 0, c.stream>>>(cand_total, rp, cand, ncand, S2, np,
                                                                park);
        c.count();
    } else {
        k_suitor128<<<blocks_for(n, kBlock), kBlock, 0, c.stream>>>(
            static_cast<int>(n), cand_total, rp, cand, ncand, S2, 0, nullptr, nullptr);
    }
#ifdef MAMG_SUITOR_PROF
    k_suitor_prof_report<<<1, 1, 0, c.stream>>>(static_cast<int>(n));
    c.sync();
#endif
    k_mate128<<<blocks_for(n, kBlock), kBlock, 0, c.stream>>>(static_cast<int>(n), S2, mate);
    c.count(3);
    MAMG_LAUNCH_CHECK();
}

void suitor(Ctx& c, int64_t n, int64_t nnz, const int32_t* rp, const int32_t* ci,
            const double* wt, int32_t* mate) {
    if (n == 0) return;
    Cand* cand = c.scratch<Cand>(Ctx::kScrCand, nnz > 0 ? nnz : 1);
    int32_t* ncand = c.scratch<int32_t>(Ctx::kScrCandN, n);
    {
        const int S = group_lanes(n, nnz);
        auto go = [&](auto kern) {
            kern<<<blocks_for(n * S, kBlock), kBlock, 0, c.stream>>>(n, rp, ci, wt, cand, ncand);
        };
        switch (S) {
            case 4: go(k_candidates<4>); break;
            case 8: go(k_candidates<8>); break;
            case 16: go(k_candidates<16>); break;
            default: go(k_candidates<32>); break;
        }
        c.count();
    }
    suitor_from_candidates(c, n, nnz > 0 ? nnz : 1, rp, cand, ncand, mate);
}

static void wtrace(Ctx& c, const char* what, int64_t n) {
    static const bool on = std::getenv("MAMG_TRACE_W") != nullptr;
    if (!on) return;
    c.sync();
    std::fprintf(stderr, "[weights_suitor n=%lld] %s done\n", static_cast<long long>(n), what);
}

void weights_suitor(Ctx& c, const DevCsr& A, const double* w, int32_t* mate, int64_t& zero_edges,
                    const int32_t* cg, int64_t g0, const WeightsCheck& chk) {
    if (!cg && A.nrows != A.ncols) invalid("build_weights: matrix is not square");
    if (!cg) cg = A.ci.get();
    const int64_t n = A.nrows;
    zero_edges = 0;
    if (n == 0) return;
    DBuf<double> dg(n, c.stream);
    // the checks of build_weights (matching.cpp:35-99) are deferred to the
    // next readback (aggregate_from_mate's); zero_edges is filled then too
    int32_t* flags = defer_flags(c, 3, [](int j, int32_t row) {
        if (j == 0) invalid("build_weights: non-positive diagonal in row " + std::to_string(row), row);
        if (j == 1)
            invalid("build_weights: pattern not symmetric, offending row " + std::to_string(row), row);
        invalid("build_weights: non-finite weight produced in row " + std::to_string(row), row);
    });
    int64_t* zdst = &zero_edges;
    unsigned long long* zc = defer_counter(c, [zdst](int64_t v) { *zdst = v; });
    k_diag<<<blocks_for(n, kBlock), kBlock, 0, c.stream>>>(n, A.rp.get(), cg, A.v.get(),
                                                           static_cast<int>(g0), dg.get(), flags);
    wtrace(c, "diag", n);
    Cand* cand = c.scratch<Cand>(Ctx::kScrCand, A.nnz > 0 ? A.nnz : 1);
    int32_t* ncand = c.scratch<int32_t>(Ctx::kScrCandN, n);
    double* wt = c.scratch<double>(Ctx::kScrWeights, A.nnz > 0 ? A.nnz : 1);
    wtrace(c, "scratch", n);
    {
        const int S = group_lanes(A.nrows, A.nnz);
        auto go = [&](auto kern) {
            kern<<<blocks_for(n * S, kBlock), kBlock, 0, c.stream>>>(
                n, A.rp.get(), A.ci.get(), cg, static_cast<int>(g0), A.v.get(), dg.get(), w, wt, cand,
                ncand, flags, zc, chk.check_upper ? 1 : 0, chk.sym_flag);
        };
        switch (S) {
            case 4: go(k_weights_cand<4>); break;
            case 8: go(k_weights_cand<8>); break;
            case 16: go(k_weights_cand<16>); break;
            default: go(k_weights_cand<32>); break;
        }
    }
    c.count(2);
    MAMG_LAUNCH_CHECK();
    wtrace(c, "weights_cand", n);
    suitor_from_candidates(c, n, A.nnz > 0 ? A.nnz : 1, A.rp.get(), cand, ncand, mate);
    wtrace(c, "suitor", n);
}

// ------------------------------------------------ global matching (host) --
SuitorBlock suitor_block(int64_t n, int64_t nnz) {
    auto up = [](size_t x) { return (x + 255) & ~static_cast<size_t>(255); };
    SuitorBlock b;
    b.s_off = 0;
    b.cand_off = up(sizeof(Suit) * static_cast<size_t>(n > 0 ? n : 1));
    b.rp_off = b.cand_off + up(sizeof(Cand) * static_cast<size_t>(nnz > 0 ? nnz : 1));
    b.ncand_off = b.rp_off + up(sizeof(int32_t) * static_cast<size_t>(n + 1));
    b.bytes = b.ncand_off + up(sizeof(int32_t) * static_cast<size_t>(n > 0 ? n : 1));
    return b;
}

void diag_owned(Ctx& c, const DevCsr& A, const int32_t* cg, int64_t g0, double* dg, int32_t* flag) {
    if (A.nrows == 0) return;
    k_diag<<<blocks_for(A.nrows, kBlock), kBlock, 0, c.stream>>>(A.nrows, A.rp.get(), cg, A.v.get(),
                                                                 static_cast<int>(g0), dg, flag);
    c.count();
    MAMG_LAUNCH_CHECK();
}

void weights_global(Ctx& c, const DevCsr& A, const int32_t* cg, int64_t g0, const double* dg,
                    const double* w, double* wt, int32_t* flags, unsigned long long* zeros) {
    const int64_t n = A.nrows;
    if (n == 0) return;
    const int S = group_lanes(A.nrows, A.nnz);
    auto go = [&](auto kern) {
        kern<<<blocks_for(n * S, kBlock), kBlock, 0, c.stream>>>(n, A.rp.get(), A.ci.get(), cg,
                                                                 static_cast<int>(g0), A.v.get(),
                                                                 dg, w, wt, flags, zeros);
    };
    switch (S) {
        case 4: go(k_weights_glob<4>); break;
        case 8: go(k_weights_glob<8>); break;
        case 16: go(k_weights_glob<16>); break;
        default: go(k_weights_glob<32>); break;
    }
    c.count();
    MAMG_LAUNCH_CHECK();
}

void candidates_into(Ctx& c, int64_t n, int64_t nnz, const int32_t* rp, const int32_t* ids,
                     const double* wt, void* cand, int32_t* ncand) {
    if (n == 0) return;
    const int S = group_lanes(n, nnz);
    Cand* cd = static_cast<Cand*>(cand);
    auto go = [&](auto kern) {
        kern<<<blocks_for(n * S, kBlock), kBlock, 0, c.stream>>>(n, rp, ids, wt, cd, ncand);
    };
    switch (S) {
        case 4: go(k_candidates<4>); break;
        case 8: go(k_candidates<8>); break;
        case 16: go(k_candidates<16>); break;
        default: go(k_candidates<32>); break;
    }
    c.count();
    MAMG_LAUNCH_CHECK();
}

void suitor_global_init(Ctx& c, void* S, int64_t n) {
    if (n == 0) return;
    k_suit_init<<<blocks_for(n, kBlock), kBlock, 0, c.stream>>>(static_cast<int>(n),
                                                               static_cast<Suit*>(S));
    c.count();
    MAMG_LAUNCH_CHECK();
}

void suitor_global(Ctx& c, const SuitorView& g, int me, bool sys) {
    const int64_t n = g.bounds[me + 1] - g.bounds[me];
    if (n == 0) return;
    static const int cap = [] {
        const char* e = std::getenv("MAMG_SUITOR_CAP");
        return e ? std::atoi(e) : kSuitorCap;
    }();
    const bool parking = cap > 0 && n > 4096;
    int2* park = parking ? c.scratch<int2>(Ctx::kScrPark, n) : nullptr;
    int* np = reinterpret_cast<int*>(c.d_small.get() + 24);
    if (parking) MAMG_CU(cudaMemsetAsync(np, 0, sizeof(int), c.stream));
    const int cp = parking ? cap : 0;
    if (sys)
        k_suitor_glob<true><<<blocks_for(n, kBlock), kBlock, 0, c.stream>>>(g, me, cp, park, np);
    else
        k_suitor_glob<false><<<blocks_for(n, kBlock), kBlock, 0, c.stream>>>(g, me, cp, park, np);
    if (parking) {
        if (sys)
            k_suitor_glob_resume<true><<<c.num_sms * 8, kBlock, 0, c.stream>>>(g, np, park);
        else
            k_suitor_glob_resume<false><<<c.num_sms * 8, kBlock, 0, c.stream>>>(g, np, park);
        c.count();
    }
    c.count();
    MAMG_LAUNCH_CHECK();
}

void mate_global(Ctx& c, const SuitorView& g, int me, bool sys, int32_t* mate) {
    const int64_t n = g.bounds[me + 1] - g.bounds[me];
    if (n == 0) return;
    if (sys)
        k_mate_glob<true><<<blocks_for(n, kBlock), kBlock, 0, c.stream>>>(g, me, mate);
    else
        k_mate_glob<false><<<blocks_for(n, kBlock), kBlock, 0, c.stream>>>(g, me, mate);
    c.count();
    MAMG_LAUNCH_CHECK();
}

std::unique_ptr<DevGraph> graph_from_aligned(Ctx& c, const DevCsr& A, const double* wt,
                                             int64_t zero_edges) {
    auto G = std::make_unique<DevGraph>();
    const int64_t n = A.nrows;
    G->n = n;
    G->zero_edges = zero_edges;
    G->xadj.alloc(n + 1, c.stream);
    if (n > 0) {
        k_offdiag_count<<<blocks_for(n, kBlock), kBlock, 0, c.stream>>>(n, A.rp.get(), A.ci.get(),
                                                                        G->xadj.get());
        c.count();
    }
    exclusive_scan_i32(c, G->xadj.get(), G->xadj.get(), n);
    G->nedges = read_i32(c, G->xadj.get() + n);
    G->adj.alloc(G->nedges, c.stream);
    G->wt.alloc(G->nedges, c.stream);
    if (n > 0) {
        k_offdiag_copy<<<blocks_for(n, kBlock), kBlock, 0, c.stream>>>(
            n, A.rp.get(), A.ci.get(), wt, G->xadj.get(), G->adj.get(), G->wt.get());
        c.count();
    }
    MAMG_LAUNCH_CHECK();
    return G;
}

} // namespace mamg
