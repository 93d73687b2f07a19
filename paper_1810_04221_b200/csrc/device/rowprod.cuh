// rowprod.cuh — ordered sparse row accumulation shared by the Galerkin
// product (proj/src/coarsening.cpp:115-146) and the general SpGEMM
// (proj/src/kernels.cpp:237-285).
//
// An output row is the concatenation, in order, of "outer" items, each of
// which contributes the entries of one inner CSR row. The reference adds the
// contributions for one output column in ENCOUNTER order, the first one
// assigning (not 0.0 + v), and emits the columns sorted. A warp (or, for
// rows with more than kWarpCap contributions, a whole CTA) stages the row's
// contributions in shared memory and, for every distinct column, one lane
// replays that column's contributions in encounter order — so the FP sum is
// bit-identical to the reference's sequential accumulator while different
// columns are summed in parallel. No sort is needed: a column's output slot
// is the number of distinct smaller columns.
#pragma once

#include <functional>
#include <memory>

#include "ops.cuh"

namespace mamg {

constexpr int kWarpCap = 512;      // contributions per warp-handled row
constexpr int kRowprodWarps = 4;   // warps per CTA in the warp kernel

// Processes output row `r` with GT cooperating threads (tid in [0, GT)); used
// by the CTA-per-row kernel for rows above kWarpCap contributions.
// cols/vals/head are shared scratch of capacity >= m.
template <int GT, class Prob>
__device__ void rowprod_one(const Prob& pb, int r, int m, int64_t off, int tid, int32_t* cols,
                            double* vals, unsigned char* head, int32_t* out_ci, double* out_v,
                            int32_t* cnt, int* red) {
    auto gsync = [] {
        if constexpr (GT == 32) __syncwarp(); else __syncthreads();
    };
    // 1. stage contributions in encounter order
    int base = 0;
    const int nout = pb.outer_count(r);
    for (int o = 0; o < nout; ++o) {
        int lo, hi;
        typename Prob::Outer ou = pb.outer(r, o, lo, hi);
        for (int e = lo + tid; e < hi; e += GT) {
            int32_t col;
            double val;
            pb.contrib(ou, e, col, val);
            cols[base + (e - lo)] = col;
            vals[base + (e - lo)] = val;
        }
        base += hi - lo;
    }
    gsync();
    // 2. head = first occurrence of its column
    for (int t = tid; t < m; t += GT) {
        const int32_t J = cols[t];
        unsigned char h = 1;
        for (int s = 0; s < t; ++s)
            if (cols[s] == J) {
                h = 0;
                break;
            }
        head[t] = h;
    }
    gsync();
    // 3. each head replays its column in encounter order; slot = rank of J
    int nheads = 0;
    for (int t = tid; t < m; t += GT) {
        if (!head[t]) continue;
        ++nheads;
        const int32_t J = cols[t];
        double acc = vals[t];
        int slot = 0;
        for (int s = 0; s < m; ++s) {
            const int32_t c = cols[s];
            if (s > t && c == J) acc = rn_add(acc, vals[s]);
            if (head[s] && c < J) ++slot;
        }
        out_ci[off + slot] = J;
        out_v[off + slot] = acc;
    }
    // 4. distinct-column count
    if constexpr (GT == 32) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) nheads += __shfl_down_sync(0xffffffffu, nheads, o);
        if (tid == 0) cnt[r] = nheads;
    } else {
        if (tid == 0) *red = 0;
        __syncthreads();
        atomicAdd(red, nheads);
        __syncthreads();
        if (tid == 0) cnt[r] = *red;
    }
    gsync();
}

// Rows with at most 32 contributions: lane t holds contribution t; lanes
// with the same column are grouped by __match_any_sync; the lowest lane of a
// group (the column's first contribution) replays the group's values in lane
// (= encounter) order, and its output slot is the number of group leaders
// with a smaller column.
template <class Prob>
__device__ void rowprod_small(const Prob& pb, int r, int m, int64_t off, int lane, int32_t* cols,
                              double* vals, int32_t* out_ci, double* out_v, int32_t* cnt) {
    int32_t col = INT32_MAX;
    double val = 0.0;
    {
        int base = 0;
        const int nout = pb.outer_count(r);
        for (int o = 0; o < nout; ++o) {
            int lo, hi;
            typename Prob::Outer ou = pb.outer(r, o, lo, hi);
            const int t = lane - base;
            if (t >= 0 && t < hi - lo) pb.contrib(ou, lo + t, col, val);
            base += hi - lo;
        }
    }
    cols[lane] = col;
    vals[lane] = val;
    __syncwarp();
    const unsigned active = (m >= 32) ? 0xffffffffu : ((1u << m) - 1u);
    const unsigned grp = __match_any_sync(0xffffffffu, col);
    const unsigned g = grp & active;
    const bool head = lane < m && (__ffs(g) - 1) == lane;
    const unsigned heads = __ballot_sync(0xffffffffu, head);
    if (head) {
        double acc = val;
        for (unsigned rest = g & ~(1u << lane); rest; rest &= rest - 1)
            acc = rn_add(acc, vals[__ffs(rest) - 1]);
        int slot = 0;
        for (unsigned h = heads; h; h &= h - 1) slot += cols[__ffs(h) - 1] < col;
        out_ci[off + slot] = col;
        out_v[off + slot] = acc;
    }
    if (lane == 0) cnt[r] = __popc(heads);
    __syncwarp();
}

// Two rows of <= 16 contributions per warp (lanes 0-15 / 16-31): the
// same grouping as rowprod_small with the half index in the match key, so
// the two rows never share a group. Doubles the rows in flight per warp for
// the common case (7-point Galerkin rows: ~14 contributions).
template <class Prob>
__device__ void rowprod_half(const Prob& pb, int r, int m, int64_t off, int lane, int32_t* cols,
                             double* vals, int32_t* out_ci, double* out_v, int32_t* cnt) {
    const int half = lane >> 4, hl = lane & 15;
    int32_t col = INT32_MAX;
    double val = 0.0;
    if (r >= 0) {
        int base = 0;
        const int nout = pb.outer_count(r);
        for (int o = 0; o < nout; ++o) {
            int lo, hi;
            typename Prob::Outer ou = pb.outer(r, o, lo, hi);
            const int t = hl - base;
            if (t >= 0 && t < hi - lo) pb.contrib(ou, lo + t, col, val);
            base += hi - lo;
        }
    }
    cols[lane] = col;
    vals[lane] = val;
    __syncwarp();
    const unsigned hmask = 0xffffu << (16 * half);
    const unsigned active = (r < 0 ? 0u : (m >= 16 ? 0xffffu : ((1u << m) - 1u))) << (16 * half);
    const unsigned long long key =
        (static_cast<unsigned long long>(half) << 32) | static_cast<uint32_t>(col);
    const unsigned g = __match_any_sync(0xffffffffu, key) & active;
    const bool head = ((active >> lane) & 1u) && (__ffs(g) - 1) == lane;
    const unsigned heads = __ballot_sync(0xffffffffu, head) & hmask;
    if (head) {
        double acc = val;
        for (unsigned rest = g & ~(1u << lane); rest; rest &= rest - 1)
            acc = rn_add(acc, vals[__ffs(rest) - 1]);
        int slot = 0;
        for (unsigned h = heads; h; h &= h - 1) slot += cols[__ffs(h) - 1] < col;
        out_ci[off + slot] = col;
        out_v[off + slot] = acc;
    }
    if (hl == 0 && r >= 0) cnt[r] = __popc(heads);
    __syncwarp();
}

// Rows with 32 < m <= kWarpCap contributions, one warp: the (column,
// encounter index) pairs are bitonic-sorted in shared memory, so each
// column's contributions end up adjacent AND in encounter order; the first
// position of a run (its head) replays the run sequentially — the
// reference's first-assigns-then-adds accumulation — and its output slot is
// the number of heads before it. O(m log^2 m) instead of O(m^2).
// bitonic sort of the first m (column, encounter index) pairs of cols /
// idx (encounter index = position on entry) with Q keys per lane in
// registers (m <= 32 Q); writes the sorted pairs back
template <int Q>
__device__ __forceinline__ void reg_sort(int m, int lane, int32_t* cols, uint16_t* idx) {
    unsigned long long kv[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        const int t = lane + 32 * q; // any placement: the key carries its encounter index
        kv[q] = t < m ? ((static_cast<unsigned long long>(static_cast<uint32_t>(cols[t])) << 16) |
                         static_cast<unsigned long long>(t))
                      : ~0ull;
    }
    warp_bitonic<Q>(
        kv, lane, [](unsigned long long a, unsigned long long b) { return a < b; },
        [](unsigned long long v, int m) { return __shfl_xor_sync(0xffffffffu, v, m); });
    __syncwarp(); // every lane has read its keys before any writes back (racecheck: explicit)
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        const int pos = Q * lane + q;
        if (pos < m) {
            cols[pos] = static_cast<int32_t>(kv[q] >> 16);
            idx[pos] = static_cast<uint16_t>(kv[q] & 0xffffu);
        }
    }
}

template <class Prob>
__device__ void rowprod_sorted(const Prob& pb, int r, int m, int64_t off, int lane, int32_t* cols,
                               double* vals, uint16_t* idx, int32_t* out_ci, double* out_v,
                               int32_t* cnt) {
    {
        int base = 0;
        const int nout = pb.outer_count(r);
        for (int o = 0; o < nout; ++o) {
            int lo, hi;
            typename Prob::Outer ou = pb.outer(r, o, lo, hi);
            for (int e = lo + lane; e < hi; e += 32) {
                int32_t col;
                double val;
                pb.contrib(ou, e, col, val);
                cols[base + (e - lo)] = col;
                vals[base + (e - lo)] = val;
                idx[base + (e - lo)] = static_cast<uint16_t>(base + (e - lo));
            }
            base += hi - lo;
        }
    }
    if (m <= 256) {
        // <= 256 contributions: bitonic sort of (column, encounter index) keys
        // held in registers (Q per lane, position Q lane + q); partners in
        // the same lane are swapped in registers, the others exchanged by
        // shuffles — no shared-memory stage or warp barrier per step
        __syncwarp();
        if (m <= 64)
            reg_sort<2>(m, lane, cols, idx);
        else if (m <= 128)
            reg_sort<4>(m, lane, cols, idx);
        else
            reg_sort<8>(m, lane, cols, idx);
        __syncwarp();
    } else {
    int P = 64;
    while (P < m) P <<= 1;
    for (int t = m + lane; t < P; t += 32) {
        cols[t] = INT32_MAX;
        idx[t] = 0xffff;
    }
    __syncwarp();
    for (int k = 2; k <= P; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int t = lane; t < P; t += 32) {
                const int u = t ^ j;
                if (u > t) {
                    const int32_t ca = cols[t], cb = cols[u];
                    const uint16_t ia = idx[t], ib = idx[u];
                    const bool gt = ca > cb || (ca == cb && ia > ib);
                    if (gt == ((t & k) == 0)) {
                        cols[t] = cb;
                        cols[u] = ca;
                        idx[t] = ib;
                        idx[u] = ia;
                    }
                }
            }
            __syncwarp();
        }
    }
    }
    int heads = 0;
    for (int base = 0; base < m; base += 32) {
        const int t = base + lane;
        const int32_t col = t < m ? cols[t] : INT32_MAX;
        const bool head = t < m && (t == 0 || cols[t - 1] != col);
        const unsigned hb = __ballot_sync(0xffffffffu, head);
        if (head) {
            double acc = vals[idx[t]];
            for (int s2 = t + 1; s2 < m && cols[s2] == col; ++s2) acc = rn_add(acc, vals[idx[s2]]);
            const int slot = heads + __popc(hb & ((1u << lane) - 1u));
            out_ci[off + slot] = col;
            out_v[off + slot] = acc;
        }
        heads += __popc(hb);
    }
    if (lane == 0) cnt[r] = heads;
    __syncwarp();
}

// Rows with <= 32 contributions, one warp each, 8 warps per CTA with 3 KB of
// shared memory (high occupancy: these are almost all rows of a Galerkin
// product). Rows above kWarpCap are appended to the long list (counts[1] =
// its length, counts[2] = longest); mid rows are left to k_rowprod_mid.
constexpr int kSmallWarps = 8;
#ifndef MAMG_ROWPROD_MINB
#define MAMG_ROWPROD_MINB 8
#endif
template <class Prob>
__global__ void __launch_bounds__(32 * kSmallWarps, MAMG_ROWPROD_MINB)
k_rowprod_warp(Prob pb, int nrows, const int32_t* __restrict__ ub_off, int32_t* out_ci,
               double* out_v, int32_t* cnt, int32_t* long_rows, int32_t* counts) {
    __shared__ int32_t s_cols[kSmallWarps][32];
    __shared__ double s_vals[kSmallWarps][32];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int r0 = 2 * (blockIdx.x * kSmallWarps + wid); // this warp's two rows
    if (r0 >= nrows) return;
    const bool two = r0 + 1 < nrows;
    const int m0 = ub_off[r0 + 1] - ub_off[r0];
    const int m1 = two ? ub_off[r0 + 2] - ub_off[r0 + 1] : 0;
    if (m0 <= 16 && m1 <= 16) {
        const int half = lane >> 4;
        const int r = half == 0 ? r0 : (two ? r0 + 1 : -1);
        rowprod_half(pb, r, half == 0 ? m0 : m1, r >= 0 ? ub_off[r] : 0, lane, s_cols[wid],
                     s_vals[wid], out_ci, out_v, cnt);
        return;
    }
    for (int q = 0; q < (two ? 2 : 1); ++q) {
        const int r = r0 + q;
        const int m = q == 0 ? m0 : m1;
        if (m > 32) {
            if (lane == 0 && m > kWarpCap) {
                long_rows[atomicAdd(&counts[1], 1)] = r;
                atomicMax(&counts[2], m);
            }
            continue; // mid rows: k_rowprod_mid
        }
        rowprod_small(pb, r, m, ub_off[r], lane, s_cols[wid], s_vals[wid], out_ci, out_v, cnt);
    }
}

// Mid rows (33..kWarpCap contributions): a persistent grid of warps strides
// over ALL rows and takes those in range (no list, no atomics: a Galerkin
// product of 27-point or elasticity rows has every coarse row here).
template <class Prob>
__global__ void __launch_bounds__(32 * kRowprodWarps)
k_rowprod_mid(Prob pb, int nrows, const int32_t* __restrict__ ub_off, int32_t* out_ci,
              double* out_v, int32_t* cnt) {
    __shared__ int32_t s_cols[kRowprodWarps][kWarpCap];
    __shared__ double s_vals[kRowprodWarps][kWarpCap];
    __shared__ uint16_t s_idx[kRowprodWarps][kWarpCap];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // each warp scans `per` rows at a time (one per lane) and processes the
    // mid rows among them one after the other: 32 on large levels, fewer
    // when the level has fewer rows than 32 per warp (small coarse levels
    // of long rows: one warp per row instead of a few warps doing them all)
    const int nwarps = static_cast<int>(gridDim.x) * kRowprodWarps;
    const int per = max(1, min(32, (nrows + nwarps - 1) / nwarps));
    for (int base = (blockIdx.x * kRowprodWarps + wid) * per; base < nrows; base += nwarps * per) {
        const int rl = base + lane;
        const int ml = (lane < per && rl < nrows) ? ub_off[rl + 1] - ub_off[rl] : 0;
        unsigned todo = __ballot_sync(0xffffffffu, ml > 32 && ml <= kWarpCap);
        while (todo) {
            const int t = __ffs(todo) - 1;
            todo &= todo - 1;
            const int r = base + t;
            const int m = __shfl_sync(0xffffffffu, ml, t);
            rowprod_sorted(pb, r, m, ub_off[r], lane, s_cols[wid], s_vals[wid], s_idx[wid], out_ci,
                           out_v, cnt);
        }
    }
}

// Long rows: one CTA (256 threads) per row, CTA-strided over the list, with a
// fixed dynamic shared memory of kBlockSmem (m <= (kBlockSmem - 16) / 13);
// longer rows raise counts[3] and go to the global-memory path
// (rowprod_global_row) after this kernel.
constexpr int kBlockSmem = 200 * 1024;
// the CTA path is O(m^2) per row: rows above this go to the sort-based
// global-memory path even when they would fit in shared memory
constexpr int kBlockMaxRow = 4096;
__host__ __device__ constexpr bool block_row_fits(int64_t m) {
    return m <= kBlockMaxRow && m * 13 + 16 <= kBlockSmem;
}
template <class Prob>
__global__ void __launch_bounds__(256)
k_rowprod_block(Prob pb, const int32_t* __restrict__ ub_off, const int32_t* long_rows,
                int32_t* counts, int32_t* out_ci, double* out_v, int32_t* cnt) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ int red;
    const int nlong = counts[1];
    for (int q = blockIdx.x; q < nlong; q += gridDim.x) {
        const int r = long_rows[q];
        const int64_t off = ub_off[r];
        const int m = ub_off[r + 1] - ub_off[r];
        if (!block_row_fits(m)) {
            if (threadIdx.x == 0) atomicMax(&counts[3], m);
            continue;
        }
        double* vals = reinterpret_cast<double*>(smem);
        int32_t* cols = reinterpret_cast<int32_t*>(vals + m);
        unsigned char* head = reinterpret_cast<unsigned char*>(cols + m);
        rowprod_one<256>(pb, r, m, off, threadIdx.x, cols, vals, head, out_ci, out_v, cnt, &red);
        __syncthreads();
    }
}

// Rows above the CTA kernel's shared-memory capacity (no limit in the
// reference: coarsening.cpp:115-146, kernels.cpp:237-285): one row at a
// time in global memory — the (column, encounter index) keys of its
// contributions are bitonic-sorted by a grid-wide kernel per step, then every
// run head replays its run in encounter order (first assigns, later add) and
// takes the slot = number of heads before it.
template <class Prob>
__global__ void __launch_bounds__(1024)
k_rowprod_stage_g(Prob pb, int r, int64_t m, int64_t P, unsigned long long* keys, double* vals) {
    int64_t base = 0;
    const int nout = pb.outer_count(r);
    for (int o = 0; o < nout; ++o) {
        int lo, hi;
        typename Prob::Outer ou = pb.outer(r, o, lo, hi);
        for (int e = lo + static_cast<int>(threadIdx.x); e < hi; e += blockDim.x) {
            int32_t col;
            double val;
            pb.contrib(ou, e, col, val);
            const int64_t t = base + (e - lo);
            keys[t] = (static_cast<unsigned long long>(static_cast<uint32_t>(col)) << 32) |
                      static_cast<unsigned long long>(t);
            vals[t] = val;
        }
        base += hi - lo;
    }
    for (int64_t t = m + threadIdx.x; t < P; t += blockDim.x) keys[t] = ~0ull;
}

static __global__ void k_bitonic_step_g(unsigned long long* keys, int64_t P, int64_t k, int64_t j) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= P) return;
    const int64_t u = t ^ j;
    if (u <= t) return;
    const unsigned long long a = keys[t], b = keys[u];
    if ((a > b) == ((t & k) == 0)) {
        keys[t] = b;
        keys[u] = a;
    }
}

static __global__ void k_run_heads_g(const unsigned long long* __restrict__ keys, int64_t m, int32_t* flag) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= m) return;
    flag[t] = (t == 0 || (keys[t] >> 32) != (keys[t - 1] >> 32)) ? 1 : 0;
}

static __global__ void k_run_replay_g(const unsigned long long* __restrict__ keys,
                               const double* __restrict__ vals, int64_t m,
                               const int32_t* __restrict__ pos, int64_t off, int r, int32_t* out_ci,
                               double* out_v, int32_t* cnt) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t == 0) cnt[r] = pos[m];
    if (t >= m || pos[t + 1] == pos[t]) return; // not a run head
    const uint32_t col = static_cast<uint32_t>(keys[t] >> 32);
    double acc = vals[keys[t] & 0xffffffffull];
    for (int64_t s = t + 1; s < m && static_cast<uint32_t>(keys[s] >> 32) == col; ++s)
        acc = rn_add(acc, vals[keys[s] & 0xffffffffull]);
    out_ci[off + pos[t]] = static_cast<int32_t>(col);
    out_v[off + pos[t]] = acc;
}

template <class Prob>
void rowprod_global_row(Ctx& c, const Prob& pb, int r, int64_t m, int64_t off, int32_t* out_ci,
                        double* out_v, int32_t* cnt) {
    int64_t P = 1;
    while (P < m) P <<= 1;
    DBuf<unsigned long long> keys(P, c.stream);
    DBuf<double> vals(m, c.stream);
    DBuf<int32_t> pos(m + 1, c.stream);
    k_rowprod_stage_g<Prob><<<1, 1024, 0, c.stream>>>(pb, r, m, P, keys.get(), vals.get());
    c.count();
    for (int64_t k = 2; k <= P; k <<= 1)
        for (int64_t j = k >> 1; j > 0; j >>= 1) {
            k_bitonic_step_g<<<blocks_for(P, 256), 256, 0, c.stream>>>(keys.get(), P, k, j);
            c.count();
        }
    k_run_heads_g<<<blocks_for(m, 256), 256, 0, c.stream>>>(keys.get(), m, pos.get());
    c.count();
    exclusive_scan_i32(c, pos.get(), pos.get(), m);
    k_run_replay_g<<<blocks_for(m, 256), 256, 0, c.stream>>>(keys.get(), vals.get(), m, pos.get(),
                                                             off, r, out_ci, out_v, cnt);
    c.count();
    MAMG_LAUNCH_CHECK();
}

// Copies each row's cnt[r] leading entries from the scratch (at ub_off) to
// the final CSR (at rp); S lanes per row (S from the mean row length).
template <int S>
__global__ void k_rowprod_compact(int nrows, const int32_t* __restrict__ ub_off,
                                  const int32_t* __restrict__ rp, const int32_t* __restrict__ tci,
                                  const double* __restrict__ tv, int32_t* ci, double* v) {
    const int r = static_cast<int>((static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / S);
    const int lane = threadIdx.x & (S - 1);
    if (r >= nrows) return;
    const int src = ub_off[r], dst = rp[r], len = rp[r + 1] - rp[r];
#pragma unroll 2
    for (int t = lane; t < len; t += S) {
        ci[dst + t] = tci[src + t];
        v[dst + t] = tv[src + t];
    }
}

// Host driver: ub[0..nrows) = contribution count per output row (device,
// capacity nrows + 1; overwritten by its exclusive scan). known_total: the
// total contribution count when the caller knows it (Galerkin: nnz(A)), which
// saves a readback. Host syncs: the nnz readback (exact allocation of the
// output) and csr_finalize's flags (or none: defer_finalize); `between` is
// independent stream work run while the host waits for the nnz.
template <class Prob>
std::unique_ptr<DevCsr> rowprod_run(Ctx& c, const Prob& pb, int64_t nrows, int64_t ncols,
                                    DBuf<int32_t>& ub, int64_t known_total = -1,
                                    bool defer_finalize = false,
                                    const std::function<void()>& between = {}) {
    exclusive_scan_i32(c, ub.get(), ub.get(), nrows);
    const int64_t total = known_total >= 0 ? known_total : read_i32(c, ub.get() + nrows);
    // contribution scratch: persistent per context (no per-step GB allocations)
    int32_t* tci = c.scratch<int32_t>(Ctx::kScrProdCol, total > 0 ? total : 1);
    double* tv = c.scratch<double>(Ctx::kScrProdVal, total > 0 ? total : 1);
    DBuf<int32_t> cnt(nrows + 1, c.stream);
    DBuf<int32_t> longs(nrows > 0 ? nrows : 1, c.stream);
    DBuf<int32_t> counts(4, c.stream);
    MAMG_CU(cudaMemsetAsync(counts.get(), 0, 4 * sizeof(int32_t), c.stream));
    if (nrows > 0) {
        k_rowprod_warp<Prob><<<blocks_for((nrows + 1) / 2, kSmallWarps), 32 * kSmallWarps, 0,
                               c.stream>>>(
            pb, static_cast<int>(nrows), ub.get(), tci, tv, cnt.get(), longs.get(),
            counts.get());
        k_rowprod_mid<Prob><<<8 * c.num_sms, 32 * kRowprodWarps, 0, c.stream>>>(
            pb, static_cast<int>(nrows), ub.get(), tci, tv, cnt.get());
        ensure_dyn_smem(k_rowprod_block<Prob>, kBlockSmem);
        k_rowprod_block<Prob><<<c.num_sms, 256, kBlockSmem, c.stream>>>(
            pb, ub.get(), longs.get(), counts.get(), tci, tv, cnt.get());
        c.count(3);
        MAMG_LAUNCH_CHECK();
    }
    auto C = std::make_unique<DevCsr>();
    C->nrows = nrows;
    C->ncols = ncols;
    C->rp.alloc(nrows + 1, c.stream);
    exclusive_scan_i32(c, cnt.get(), C->rp.get(), nrows);
    // one readback: nnz and the long-row overflow flag
    int32_t* hs = reinterpret_cast<int32_t*>(c.h_small);
    MAMG_CU(cudaMemcpyAsync(hs, C->rp.get() + nrows, sizeof(int32_t), cudaMemcpyDeviceToHost,
                            c.stream));
    MAMG_CU(cudaMemcpyAsync(hs + 1, counts.get() + 3, sizeof(int32_t), cudaMemcpyDeviceToHost,
                            c.stream));
    sync_checked(c, between); // also raises deferred checks (the prolongator's)
    if (hs[1] > 0) {
        // rows above the CTA kernel's capacity: the global-memory path, row
        // by row (rare: hub rows), then the row pointers again
        int32_t nlong = 0;
        MAMG_CU(cudaMemcpy(&nlong, counts.get() + 1, sizeof(int32_t), cudaMemcpyDeviceToHost));
        std::vector<int32_t> rows(nlong);
        MAMG_CU(cudaMemcpy(rows.data(), longs.get(), sizeof(int32_t) * nlong, cudaMemcpyDeviceToHost));
        for (int32_t r : rows) {
            int32_t lohi[2];
            MAMG_CU(cudaMemcpy(lohi, ub.get() + r, 2 * sizeof(int32_t), cudaMemcpyDeviceToHost));
            const int64_t m = lohi[1] - lohi[0];
            if (!block_row_fits(m))
                rowprod_global_row(c, pb, r, m, lohi[0], tci, tv, cnt.get());
        }
        exclusive_scan_i32(c, cnt.get(), C->rp.get(), nrows);
        MAMG_CU(cudaMemcpyAsync(hs, C->rp.get() + nrows, sizeof(int32_t), cudaMemcpyDeviceToHost,
                                c.stream));
        c.sync();
    }
    C->nnz = hs[0];
    C->ci.alloc(C->nnz, c.stream);
    C->v.alloc(C->nnz, c.stream);
    if (nrows > 0) {
        if (C->nnz > 24 * nrows)
            k_rowprod_compact<32><<<blocks_for(nrows * 32, 256), 256, 0, c.stream>>>(
                static_cast<int>(nrows), ub.get(), C->rp.get(), tci, tv, C->ci.get(),
                C->v.get());
        else
            k_rowprod_compact<8><<<blocks_for(nrows * 8, 256), 256, 0, c.stream>>>(
                static_cast<int>(nrows), ub.get(), C->rp.get(), tci, tv, C->ci.get(),
                C->v.get());
        c.count();
        MAMG_LAUNCH_CHECK();
    }
    if (defer_finalize)
        csr_finalize_deferred(c, *C);
    else
        csr_finalize(c, *C);
    return C;
}

} // namespace mamg
