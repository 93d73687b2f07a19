// spmv_tile.cuh — the TMA-fed SpMV tile machinery shared by the SpMV family
// (sparse.cu) and the fused SpMV + PCG triple dot (solve.cu): staging of a
// tile's entry range with cp.async.bulk + mbarriers, the reference's G-lane
// tree evaluated by T-thread row groups, and the launch plan.
#pragma once

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"

namespace mamg {
namespace {

// Persistent, TMA-fed CSR SpMV for every lane policy G, with T threads per
// row (T | G, T <= 16). A tile is R = 256/T consecutive rows; their entries
// form ONE contiguous range of values / col_idx. Each CTA walks tiles
// t = blockIdx.x, +gridDim.x, ... with two shared-memory buffers: while the
// CTA computes tile i from buffer i&1, one elected thread has already issued
// cp.async.bulk (TMA 1D bulk) copies of tile i+1's range into the other
// buffer, completion tracked by an mbarrier transaction count. The only
// scattered traffic left is the x gather (L2-resident). Tiles whose range
// exceeds the buffer are read straight from global memory.
//
// Exact arithmetic: the reference's G-lane tree (kernels.cpp:42-58) — lane l
// sums entries lo+l, lo+l+G, ... sequentially from 0.0, then
// acc[l] += acc[l+off] for off = G/2 .. 1. Thread t of a row's T-group holds
// the G/T lanes l = t + T*m in registers, i.e. it reads entries lo+t, lo+t+T,
// ... (coalesced across the group); the folds with off >= T stay in
// registers, off < T go through __shfl_down within the group. Same
// expression tree for every T, so y is bit-identical to spmv_lanes<G>.
constexpr int kTileThreads = 256;
// Two launch configurations of the 2-stage ring (the x gathers of a row want
// resident warps more than a deeper TMA ring: 3-4 stages at 2 CTAs/SM ran
// the cfg 2 smoother in 127 us, 2 stages at 3 CTAs/SM in 95 us). Measured:
//   config 0: 5 CTAs/SM, 1800-entry stages -> 81.9 us (91% of HBM), used
//             when every 256-row tile fits (7-point level 0: 1792 entries)
//   config 1: 4 CTAs/SM, 2200-entry stages -> 85.7 us, the general case
template <int CFG>
struct SpmvCfg;
template <>
struct SpmvCfg<0> {
    static constexpr int ctas = 5, stage = 1800;
};
template <>
struct SpmvCfg<1> {
    static constexpr int ctas = 4, stage = 2200;
};
constexpr int kStagePad = 8;     // alignment slack (ranges are rounded to 16 B)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(phase)
            : "memory");
    }
}

template <int S>
struct TileStage {
    double v[S + kStagePad];
    int32_t c[S + kStagePad];
};

template <int G, int T>
__device__ __forceinline__ double group_tree(int lo, int hi, int t, const int32_t* c,
                                             const double* a, const double* __restrict__ x) {
    constexpr int L = G / T;
    double s[L];
#pragma unroll
    for (int m = 0; m < L; ++m) s[m] = 0.0;
#pragma unroll 1
    for (int base = lo + t; base < hi; base += G) {
#pragma unroll
        for (int m = 0; m < L; ++m) {
            const int k = base + T * m;
            if (k < hi) s[m] = rn_add(s[m], rn_mul(a[k], __ldg(x + c[k])));
        }
    }
#pragma unroll
    for (int off = G / 2; off >= T; off >>= 1) {
#pragma unroll
        for (int m = 0; m < off / T; ++m) s[m] = rn_add(s[m], s[m + off / T]);
    }
    if constexpr (T > 1) {
#pragma unroll
        for (int off = T / 2; off > 0; off >>= 1)
            s[0] = rn_add(s[0], __shfl_down_sync(0xffffffffu, s[0], off, T));
    }
    return s[0];
}

// thread 0: issue the bulk copies of tile t's entry range into `st`;
// returns the aligned start offsets (or -1 when the range does not fit)
template <int R, int S>
__device__ __forceinline__ void stage_tile(int t, int n, const int32_t* __restrict__ rp,
                                           const int32_t* __restrict__ ci,
                                           const double* __restrict__ v, TileStage<S>* st,
                                           uint64_t* bar, int* ev0, int* ec0) {
    const int r0 = t * R;
    const int r1 = min(r0 + R, n);
    const int e0 = rp[r0], e1 = rp[r1];
    const int v0 = e0 & ~1, v1 = (e1 + 1) & ~1;  // doubles: 16 B = 2 entries
    const int c0 = e0 & ~3, c1 = (e1 + 3) & ~3;  // ints: 16 B = 4 entries
    if (v1 - v0 > S + kStagePad || c1 - c0 > S + kStagePad || e1 == e0) {
        *ev0 = -1;
        mbar_expect_tx(bar, 0); // complete the phase without a transfer
        return;
    }
    *ev0 = v0;
    *ec0 = c0;
    const uint32_t bv = static_cast<uint32_t>(v1 - v0) * 8u;
    const uint32_t bc = static_cast<uint32_t>(c1 - c0) * 4u;
    mbar_expect_tx(bar, bv + bc);
    tma_load_1d(st->v, v + v0, bv, bar);
    tma_load_1d(st->c, ci + c0, bc, bar);
}


// Launch plan: T threads per row and the configuration. T = 1 whenever the
// longest 256-row tile (DevCsr::max_tile, from csr_finalize) fits a stage;
// otherwise the smallest T (<= G, <= 16) whose 256/T-row tiles fit
// configuration 0's stage at 97% of the mean row length (a tile that still
// overflows is read straight from global memory).
struct SpmvPlan {
    int T, cfg;
};
inline SpmvPlan spmv_plan_(const DevCsr& A, int G);
inline SpmvPlan spmv_plan(const DevCsr& A, int G) {
    const SpmvPlan p = spmv_plan_(A, G);
    static const bool debug = std::getenv("MAMG_SPMV_DEBUG") != nullptr;
    if (debug)
        std::fprintf(stderr, "[spmv plan] n=%lld nnz=%lld G=%d max_tile=%d -> T=%d cfg=%d\n",
                     static_cast<long long>(A.nrows), static_cast<long long>(A.nnz), G, A.max_tile, p.T, p.cfg);
    return p;
}
inline SpmvPlan spmv_plan_(const DevCsr& A, int G) {
    const double mean = A.nrows > 0 ? static_cast<double>(A.nnz) / static_cast<double>(A.nrows) : 0.0;
    auto pick = [&](int stage, double fill) {
        int T = G == 32 ? 2 : 1; // no 32-register-lane instance for G = 32
        while (T < G && T < 16 && (kTileThreads / T) * mean > fill * stage) T *= 2;
        return T;
    };
    // small, latency-bound levels (fewer than ~2 tiles per SM): configuration
    // 1's larger register budget shortens the per-row chain (measured: the
    // 4k-row coarsest sweep 5.0 us vs 6.0 us under configuration 0)
    if (A.nrows < 2 * 148 * kTileThreads) {
        if (G < 32 && A.max_tile >= 0 && A.max_tile <= SpmvCfg<1>::stage) return {1, 1};
        // a 256-row tile just over the stage (coarse 7-point levels: 2,386 and
        // 2,557 entries): 128-row tiles of two threads per row fit instead of
        // spilling to the global-memory path (cfg 2 V-cycle 374.6 -> ~370 us)
        if (G < 32 && G >= 2 && A.max_tile >= 0 && A.max_tile <= 2 * SpmvCfg<1>::stage) return {2, 1};
        return {pick(SpmvCfg<1>::stage, 0.9), 1};
    }
    // configuration 0 caps registers at 51: at most 8 register lanes (G / T)
    if (G < 32 && A.max_tile >= 0) {
        if (A.max_tile <= SpmvCfg<0>::stage && G <= 8) return {1, 0};
        if (A.max_tile <= SpmvCfg<1>::stage) return {1, 1};
    }
    const int T0 = pick(SpmvCfg<0>::stage, 0.97);
    if (G / T0 <= 8) return {T0, 0};
    return {pick(SpmvCfg<1>::stage, 0.97), 1};
}


} // namespace
} // namespace mamg
