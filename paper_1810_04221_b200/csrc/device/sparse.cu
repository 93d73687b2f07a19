// sparse.cu — device CSR plumbing and the sparse kernels of
// proj/src/kernels.cpp + proj/src/csr.cpp on sm_100a:
//  * lane-group CSR SpMV (kernels.cpp:36-61): a G-lane sub-warp per row, lane l
//    sums entries lo+l, lo+l+G, ... sequentially from 0.0, then the lanes fold
//    with a __shfl_down tree (off = G/2 .. 1) — the reference's exact
//    expression tree, so y is bit-identical. Epilogues fuse the consumers that
//    follow a SpMV in the V-cycle: the residual (multigrid.cpp:93-95) and the
//    l1-Jacobi update (multigrid.cpp:55-60).
//  * l1 diagonal (kernels.cpp:295-324), pattern symmetry (csr.cpp:106-112),
//    transpose (kernels.cpp:116-134), SpGEMM (kernels.cpp:237-285).
#include <algorithm>
#include <mutex>
#include <type_traits>
#include <unordered_set>

#include "ops.cuh"
#include "rowprod.cuh"
#include "spmv_tile.cuh"

namespace mamg {
namespace {

constexpr int kBlock = 256;

// ---------------------------------------------------------------- upload --
__global__ void k_widen(int64_t n, const int32_t* __restrict__ src, int64_t* dst) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) dst[i] = src[i];
}

// flags[2] = max over 256-row tiles of the tile's entry count
__global__ void k_max_tile(int64_t n, const int32_t* __restrict__ rp, int32_t* flags) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t r0 = t * 256;
    if (r0 >= n) return;
    const int64_t r1 = r0 + 256 < n ? r0 + 256 : n;
    atomicMax(&flags[2], rp[r1] - rp[r0]);
}

// flags[0] = 1 if every row holds exactly one entry; flags[1] = 1 if all finite
// (thread t: row t and values [4t, 4t + 4), 16-byte loads when v is aligned)
__global__ void k_flags(int64_t n, int64_t nnz, const int32_t* __restrict__ rp,
                        const double* __restrict__ v, int32_t* flags) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n && rp[i] != i) flags[0] = 0;
    const int64_t k = 4 * i;
    bool bad = false;
    if (k + 4 <= nnz && (reinterpret_cast<uintptr_t>(v) & 15) == 0) {
        const double2 a = __ldcs(reinterpret_cast<const double2*>(v + k));
        const double2 b = __ldcs(reinterpret_cast<const double2*>(v + k + 2));
        bad = !isfinite(a.x) || !isfinite(a.y) || !isfinite(b.x) || !isfinite(b.y);
    } else {
        for (int64_t e = k; e < k + 4 && e < nnz; ++e) bad |= !isfinite(v[e]);
    }
    if (bad) flags[1] = 0;
}

// ---------------------------------------------------------------- SpMV --
// Epilogues: prefetch() loads the row's epilogue operands before the tile's
// entries arrive; finish() consumes them (operator() is the one-shot form
// used by the lane-group kernel).
struct EpiStore {
    double* y;
    struct Pre {};
    __device__ Pre prefetch(int) const { return {}; }
    __device__ void finish(int i, double s, const Pre&) const { y[i] = s; }
    __device__ void operator()(int i, double s) const { y[i] = s; }
};
struct EpiResidual {
    const double* __restrict__ b;
    double* r;
    struct Pre {
        double b;
    };
    __device__ Pre prefetch(int i) const { return {b[i]}; }
    __device__ void finish(int i, double s, const Pre& p) const { r[i] = rn_sub(p.b, s); }
    __device__ void operator()(int i, double s) const { r[i] = rn_sub(b[i], s); }
};
struct EpiSmooth {
    const double* __restrict__ b;
    const double* __restrict__ d;
    const double* __restrict__ xi;
    double* xo;
    struct Pre {
        double b, d, x;
    };
    __device__ Pre prefetch(int i) const { return {b[i], d[i], xi[i]}; }
    __device__ void finish(int i, double s, const Pre& p) const {
        xo[i] = rn_add(p.x, rn_div(rn_sub(p.b, s), p.d));
    }
    __device__ void operator()(int i, double s) const {
        xo[i] = rn_add(xi[i], rn_div(rn_sub(b[i], s), d[i]));
    }
};

// tile staging, group trees and launch plans: spmv_tile.cuh
constexpr int kNS = 2; // ring depth (tiles in flight per CTA = kNS - 1)

template <int G, int T, int CFG, class Epi>
__global__ void __launch_bounds__(kTileThreads, SpmvCfg<CFG>::ctas)
k_spmv_rows(int n, int ntiles, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
            const double* __restrict__ v, const double* __restrict__ x, Epi epi,
            const int* __restrict__ gate, int row0) {
    constexpr int R = kTileThreads / T;
    constexpr int S = SpmvCfg<CFG>::stage;
    pdl_wait();
    if (gate && *gate) return;
    extern __shared__ __align__(128) unsigned char dyn_smem[];
    TileStage<S>* stage = reinterpret_cast<TileStage<S>*>(dyn_smem);
    __shared__ __align__(8) uint64_t bar[kNS];
    __shared__ int ev0[kNS], ec0[kNS];
    if (threadIdx.x == 0) {
#pragma unroll
        for (int b = 0; b < kNS; ++b) mbar_init(&bar[b], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    int t = blockIdx.x;
    if (t >= ntiles) return;
    // prologue: tiles i = 0 .. kNS-2 of this CTA in flight
    if (threadIdx.x == 0) {
        for (int j = 0; j < kNS - 1; ++j) {
            const int tj = t + j * static_cast<int>(gridDim.x);
            if (tj < ntiles) stage_tile<R, S>(tj, n, rp, ci, v, &stage[j], &bar[j], &ev0[j], &ec0[j]);
        }
    }
    const int sub = threadIdx.x % T;
    for (int i = 0; t < ntiles; ++i, t += gridDim.x) {
        const int b = i % kNS;
        // refill the buffer consumed in iteration i - 1 with tile i + kNS - 1
        const int tn = t + (kNS - 1) * static_cast<int>(gridDim.x);
        if (threadIdx.x == 0 && tn < ntiles) {
            const int bn = (i + kNS - 1) % kNS;
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            stage_tile<R, S>(tn, n, rp, ci, v, &stage[bn], &bar[bn], &ev0[bn], &ec0[bn]);
        }
        const int row = t * R + static_cast<int>(threadIdx.x) / T;
        int lo = 0, hi = 0;
        typename Epi::Pre pre{};
        if (row < n) {
            lo = rp[row];
            hi = rp[row + 1];
            if (sub == 0) pre = epi.prefetch(row0 + row);
        }
        mbar_wait(&bar[b], static_cast<uint32_t>(i / kNS) & 1u);
        // every thread of the warp takes part in the group shuffles
        const double s = ev0[b] >= 0
                             ? group_tree<G, T>(lo, hi, sub, stage[b].c - ec0[b], stage[b].v - ev0[b], x)
                             : group_tree<G, T>(lo, hi, sub, ci, v, x);
        if (row < n && sub == 0) epi.finish(row0 + row, s, pre);
        __syncthreads(); // buffer b is refilled in iteration i + 1
    }
    pdl_trigger();
}

// rows [r0, r1) of A (default: all); the kernel sees the shifted row
// pointers (entry offsets stay absolute) and shifts the epilogue's row index
template <class Epi>
void launch_spmv(Ctx& c, const DevCsr& A, int G, const double* x, Epi epi, const int* gate,
                 int64_t r0 = 0, int64_t r1 = -1) {
    if (r1 < 0) r1 = A.nrows;
    if (r1 <= r0) return;
    const int n = static_cast<int>(r1 - r0);
    const int row0 = static_cast<int>(r0);
    const auto rp = A.rp.get() + r0;
    const auto ci = A.ci.get();
    const auto v = A.v.get();
    if (G != 1 && G != 2 && G != 4 && G != 8 && G != 16 && G != 32)
        invalid("spmv: invalid lane group size " + std::to_string(G));
    const SpmvPlan plan = spmv_plan(A, G);
    const int T = plan.T;
    const int R = kTileThreads / T;
    const int ntiles = static_cast<int>((n + R - 1) / R);
    auto go2 = [&](auto k0, auto k1) {
        const bool c0 = plan.cfg == 0;
        const void* kernel = c0 ? reinterpret_cast<const void*>(k0) : reinterpret_cast<const void*>(k1);
        const int smem = c0 ? static_cast<int>(kNS * sizeof(TileStage<SpmvCfg<0>::stage>))
                            : static_cast<int>(kNS * sizeof(TileStage<SpmvCfg<1>::stage>));
        const int per_sm = c0 ? SpmvCfg<0>::ctas : SpmvCfg<1>::ctas;
        const unsigned grid = static_cast<unsigned>(std::min(ntiles, per_sm * c.num_sms));
        set_kernel_attr(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (c0)
            launch_pdl(c.stream, k0, dim3(grid), dim3(kTileThreads), smem, n, ntiles, rp, ci, v, x,
                       epi, gate, row0);
        else
            launch_pdl(c.stream, k1, dim3(grid), dim3(kTileThreads), smem, n, ntiles, rp, ci, v, x,
                       epi, gate, row0);
    };
#define MAMG_GO(GG, TT)                                                              \
    do {                                                                              \
        if constexpr ((GG) / (TT) > 8)                                                \
            go2(k_spmv_rows<GG, TT, 1, Epi>, k_spmv_rows<GG, TT, 1, Epi>);            \
        else                                                                          \
            go2(k_spmv_rows<GG, TT, 0, Epi>, k_spmv_rows<GG, TT, 1, Epi>);            \
    } while (0)
#define MAMG_SPMV_T(GG)                                                                  \
    switch (T) {                                                                          \
        case 1: if constexpr (GG < 32) MAMG_GO(GG, (GG < 32 ? 1 : 2)); break;             \
        case 2: if constexpr (GG >= 2) MAMG_GO(GG, (GG >= 2 ? 2 : 1)); break;             \
        case 4: if constexpr (GG >= 4) MAMG_GO(GG, (GG >= 4 ? 4 : 1)); break;             \
        case 8: if constexpr (GG >= 8) MAMG_GO(GG, (GG >= 8 ? 8 : 1)); break;             \
        default: if constexpr (GG >= 16) MAMG_GO(GG, (GG >= 16 ? 16 : 1)); break;         \
    }
    switch (G) {
        case 1: MAMG_SPMV_T(1) break;
        case 2: MAMG_SPMV_T(2) break;
        case 4: MAMG_SPMV_T(4) break;
        case 8: MAMG_SPMV_T(8) break;
        case 16: MAMG_SPMV_T(16) break;
        default: MAMG_SPMV_T(32) break;
    }
#undef MAMG_GO
#undef MAMG_SPMV_T
    c.count();
    MAMG_LAUNCH_CHECK();
}

__global__ void k_smooth_zero(int64_t n, const double* __restrict__ d,
                              const double* __restrict__ b, double* x,
                              const int* __restrict__ gate) {
    pdl_wait();
    if (gate && *gate) return;
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    // A*0 == +0 exactly for finite A, so the sweep from x = 0 reduces to this
    if (i < n) x[i] = rn_add(0.0, rn_div(b[i], d[i]));
}

// 4 consecutive elements per thread with 16-byte loads/stores (the scalar
// kernels reached ~3.7 TB/s DRAM; more bytes in flight per thread)
__host__ __device__ inline bool aligned16(const void* p) {
    return (reinterpret_cast<uintptr_t>(p) & 15u) == 0;
}
__global__ void k_smooth_zero4(int64_t n, const double* __restrict__ d,
                               const double* __restrict__ b, double* x,
                               const int* __restrict__ gate) {
    pdl_wait();
    if (gate && *gate) return;
    const int64_t i = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 4;
    if (i + 4 <= n) {
        const double2 b0 = *reinterpret_cast<const double2*>(b + i);
        const double2 b1 = *reinterpret_cast<const double2*>(b + i + 2);
        const double2 d0 = *reinterpret_cast<const double2*>(d + i);
        const double2 d1 = *reinterpret_cast<const double2*>(d + i + 2);
        *reinterpret_cast<double2*>(x + i) =
            make_double2(rn_add(0.0, rn_div(b0.x, d0.x)), rn_add(0.0, rn_div(b0.y, d0.y)));
        *reinterpret_cast<double2*>(x + i + 2) =
            make_double2(rn_add(0.0, rn_div(b1.x, d1.x)), rn_add(0.0, rn_div(b1.y, d1.y)));
    } else {
        for (int64_t j = i; j < n; ++j) x[j] = rn_add(0.0, rn_div(b[j], d[j]));
    }
}
// x += 1.0 * (0.0 + p_i * xc[agg_i])   (spmv with G=1, then axpy 1.0)
__global__ void k_prolong_correct(int64_t n, const int32_t* __restrict__ agg,
                                  const double* __restrict__ p, const double* __restrict__ xc,
                                  double* x, const int* __restrict__ gate) {
    pdl_wait();
    if (gate && *gate) return;
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) x[i] = rn_add(x[i], rn_mul(1.0, rn_add(0.0, rn_mul(p[i], xc[agg[i]]))));
}
__global__ void k_prolong_correct4(int64_t n, const int32_t* __restrict__ agg,
                                   const double* __restrict__ p, const double* __restrict__ xc,
                                   double* x, const int* __restrict__ gate) {
    pdl_wait();
    if (gate && *gate) return;
    const int64_t i = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 4;
    auto one = [&](double xi, double pi, int a) {
        return rn_add(xi, rn_mul(1.0, rn_add(0.0, rn_mul(pi, __ldg(xc + a)))));
    };
    if (i + 4 <= n) {
        const int4 a = *reinterpret_cast<const int4*>(agg + i);
        const double2 p0 = *reinterpret_cast<const double2*>(p + i);
        const double2 p1 = *reinterpret_cast<const double2*>(p + i + 2);
        const double2 x0 = *reinterpret_cast<const double2*>(x + i);
        const double2 x1 = *reinterpret_cast<const double2*>(x + i + 2);
        *reinterpret_cast<double2*>(x + i) = make_double2(one(x0.x, p0.x, a.x), one(x0.y, p0.y, a.y));
        *reinterpret_cast<double2*>(x + i + 2) = make_double2(one(x1.x, p1.x, a.z), one(x1.y, p1.y, a.w));
    } else {
        for (int64_t j = i; j < n; ++j) x[j] = one(x[j], p[j], agg[j]);
    }
}

// ------------------------------------------------------------ l1 / pattern --
__global__ void k_l1(int64_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                     const double* __restrict__ v, double* d, int32_t* bad) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double diag = 0.0, off = 0.0;
    bool seen = false;
    for (int k = rp[i]; k < rp[i + 1]; ++k) {
        if (ci[k] == i) {
            diag = v[k];
            seen = true;
        } else {
            off = rn_add(off, fabs(v[k]));
        }
    }
    const double r = (!seen || diag == 0.0) ? __longlong_as_double(0x7ff8000000000000LL)
                                            : rn_add(diag, off);
    d[i] = r;
    if (isnan(r)) atomicMin(bad, static_cast<int32_t>(i));
}

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

// S lanes per row, each searching row j of one entry (i, j) for (j, i): the
// searches of a row are independent, so S of them are in flight at once
template <int S>
__global__ void k_sym_pattern(int64_t n, const int32_t* __restrict__ rp,
                              const int32_t* __restrict__ ci, int32_t* ok) {
    const int64_t i = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / S;
    if (i >= n) return;
    const int lane = threadIdx.x & (S - 1);
    for (int k = rp[i] + lane; k < rp[i + 1]; k += S) {
        const int j = ci[k];
        const int lo = rp[j], hi = rp[j + 1];
        const int p = find_in_row(ci, lo, hi, static_cast<int>(i));
        if (p >= hi || ci[p] != i) {
            *ok = 0;
            return;
        }
    }
}

// --------------------------------------------------------------- transpose --
__global__ void k_count_cols(int64_t n, const int32_t* __restrict__ rp,
                             const int32_t* __restrict__ ci, int32_t* cnt) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    for (int k = rp[i]; k < rp[i + 1]; ++k) atomicAdd(&cnt[ci[k]], 1);
}

__global__ void k_scatter_t(int64_t n, const int32_t* __restrict__ rp,
                            const int32_t* __restrict__ ci, const double* __restrict__ v,
                            int32_t* cursor, int32_t* tci, double* tv) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    for (int k = rp[i]; k < rp[i + 1]; ++k) {
        const int pos = atomicAdd(&cursor[ci[k]], 1);
        tci[pos] = static_cast<int32_t>(i);
        tv[pos] = v[k];
    }
}

// rows of the transpose list source rows in ascending order (the reference
// scatters in ascending source-row order, kernels.cpp:125-132)
__global__ void k_sort_rows(int64_t n, const int32_t* __restrict__ rp, int32_t* ci, double* v) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int lo = rp[i], hi = rp[i + 1];
    for (int a = lo + 1; a < hi; ++a) {
        const int32_t key = ci[a];
        const double val = v[a];
        int b = a - 1;
        while (b >= lo && ci[b] > key) {
            ci[b + 1] = ci[b];
            v[b + 1] = v[b];
            --b;
        }
        ci[b + 1] = key;
        v[b + 1] = val;
    }
}

// ------------------------------------------------------------------ SpGEMM --
struct SpgemmProb {
    const int32_t* __restrict__ arp;
    const int32_t* __restrict__ aci;
    const double* __restrict__ av;
    const int32_t* __restrict__ brp;
    const int32_t* __restrict__ bci;
    const double* __restrict__ bv;
    struct Outer {
        double a;
    };
    __device__ int outer_count(int r) const { return arp[r + 1] - arp[r]; }
    __device__ Outer outer(int r, int o, int& lo, int& hi) const {
        const int k = arp[r] + o;
        const int j = aci[k];
        lo = brp[j];
        hi = brp[j + 1];
        return Outer{av[k]};
    }
    __device__ void contrib(const Outer& ou, int e, int32_t& col, double& val) const {
        col = bci[e];
        val = rn_mul(ou.a, bv[e]);
    }
};

// contributions of each row of A B (counted in int64: the total may pass
// 2^31 even when A, B and C fit int32) and their int64 total (warp-summed)
__global__ void k_spgemm_ub(int64_t n, const int32_t* __restrict__ arp,
                            const int32_t* __restrict__ aci, const int32_t* __restrict__ brp,
                            int32_t* ub, unsigned long long* total) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    int64_t s = 0;
    if (i < n) {
        for (int k = arp[i]; k < arp[i + 1]; ++k) s += brp[aci[k] + 1] - brp[aci[k]];
        ub[i] = static_cast<int32_t>(s < INT32_MAX ? s : INT32_MAX);
    }
    unsigned long long w = static_cast<unsigned long long>(s);
    for (int o = 16; o > 0; o >>= 1) w += __shfl_down_sync(0xffffffffu, w, o);
    if ((threadIdx.x & 31) == 0 && w) atomicAdd(total, w);
}

} // namespace

// ================================================================= host API ==
std::unique_ptr<DevCsr> csr_upload(Ctx& c, int64_t nrows, int64_t ncols, const int64_t* rp,
                                   const int64_t* ci, const double* v, std::vector<UpSeg> extra) {
    if (nrows < 0 || ncols < 0) invalid("CsrMatrix: negative dimension");
    const int64_t nnz = rp[nrows];
    if (nrows >= INT32_MAX || ncols >= INT32_MAX || nnz >= INT32_MAX || nnz < 0)
        invalid("CsrMatrix: dimensions exceed the device's int32 index range");
    auto A = std::make_unique<DevCsr>();
    A->nrows = nrows;
    A->ncols = ncols;
    A->nnz = nnz;
    A->rp.alloc(nrows + 1, c.stream);
    A->ci.alloc(nnz, c.stream);
    A->v.alloc(nnz, c.stream);
    c.sync(); // allocations are stream-ordered; the staging threads use other streams
    std::vector<UpSeg> segs{
        UpSeg{UpSeg::ROW_PTR, A->rp.get(), rp, static_cast<size_t>(nrows + 1), 0, nnz},
        UpSeg{UpSeg::INDEX, A->ci.get(), ci, static_cast<size_t>(nnz), 0, ncols},
        UpSeg{UpSeg::F64, A->v.get(), v, static_cast<size_t>(nnz), 0, 0}};
    segs.insert(segs.end(), extra.begin(), extra.end());
    const std::vector<bool> ok = upload_many(c, segs);
    if (!ok[0]) invalid("CsrMatrix: row_ptr is not a valid CSR row pointer array");
    if (!ok[1]) invalid("CsrMatrix: column index out of range");
    csr_finalize(c, *A);
    return A;
}

void csr_finalize(Ctx& c, DevCsr& A) {
    DBuf<int32_t> flags(3, c.stream);
    const int32_t init[3] = {1, 1, 0};
    MAMG_CU(cudaMemcpyAsync(flags.get(), init, sizeof(init), cudaMemcpyHostToDevice, c.stream));
    const int64_t work = std::max(A.nrows, (A.nnz + 3) / 4);
    if (work > 0) {
        k_flags<<<blocks_for(work, kBlock), kBlock, 0, c.stream>>>(
            A.nnz == A.nrows ? A.nrows : 0, A.nnz, A.rp.get(), A.v.get(), flags.get());
        c.count();
        MAMG_LAUNCH_CHECK();
    }
    if (A.nrows > 0) {
        const int64_t ntiles = (A.nrows + 255) / 256;
        k_max_tile<<<blocks_for(ntiles, kBlock), kBlock, 0, c.stream>>>(A.nrows, A.rp.get(),
                                                                        flags.get());
        c.count();
        MAMG_LAUNCH_CHECK();
    }
    int32_t h[3];
    MAMG_CU(cudaMemcpyAsync(h, flags.get(), sizeof(h), cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    A.single = A.nrows > 0 && A.nnz == A.nrows && h[0] == 1;
    A.finite = h[1] == 1;
    A.max_tile = h[2];
    A.group = lane_policy_from(A.nrows, A.nnz, A.single);
}

void csr_finalize_deferred(Ctx& c, DevCsr& A) {
    if (A.nrows == 0 || A.nnz == A.nrows) {
        csr_finalize(c, A);
        return;
    }
    A.single = false;
    A.group = lane_policy_from(A.nrows, A.nnz, false);
    const int32_t init[3] = {1, 1, 0};
    DevCsr* a = &A;
    int32_t* flags = defer_values(c, 3, init, [a](int j, int32_t v) {
        if (j == 1) a->finite = v == 1;
        if (j == 2) a->max_tile = v;
    });
    k_flags<<<blocks_for(std::max(A.nrows, (A.nnz + 3) / 4), kBlock), kBlock, 0, c.stream>>>(
        0, A.nnz, A.rp.get(), A.v.get(), flags);
    k_max_tile<<<blocks_for((A.nrows + 255) / 256, kBlock), kBlock, 0, c.stream>>>(A.nrows,
                                                                                  A.rp.get(), flags);
    c.count(2);
    MAMG_LAUNCH_CHECK();
}

void csr_download(Ctx& c, const DevCsr& A, int64_t* rp, int64_t* ci, double* v) {
    DBuf<int64_t> wide(std::max<int64_t>(A.nrows + 1, A.nnz), c.stream);
    k_widen<<<blocks_for(A.nrows + 1, kBlock), kBlock, 0, c.stream>>>(A.nrows + 1, A.rp.get(),
                                                                      wide.get());
    c.count();
    MAMG_CU(cudaMemcpyAsync(rp, wide.get(), sizeof(int64_t) * (A.nrows + 1),
                            cudaMemcpyDeviceToHost, c.stream));
    if (A.nnz > 0) {
        // the copy above is ordered before the widen below on the same stream
        c.sync();
        k_widen<<<blocks_for(A.nnz, kBlock), kBlock, 0, c.stream>>>(A.nnz, A.ci.get(), wide.get());
        c.count();
        MAMG_CU(cudaMemcpyAsync(ci, wide.get(), sizeof(int64_t) * A.nnz, cudaMemcpyDeviceToHost,
                                c.stream));
        MAMG_CU(cudaMemcpyAsync(v, A.v.get(), sizeof(double) * A.nnz, cudaMemcpyDeviceToHost,
                                c.stream));
    }
    MAMG_LAUNCH_CHECK();
    c.sync();
}

std::unique_ptr<DevCsr> csr_clone(Ctx& c, const DevCsr& A) {
    auto B = std::make_unique<DevCsr>();
    B->nrows = A.nrows;
    B->ncols = A.ncols;
    B->nnz = A.nnz;
    B->group = A.group;
    B->single = A.single;
    B->finite = A.finite;
    B->max_tile = A.max_tile;
    B->rp.alloc(A.nrows + 1, c.stream);
    B->ci.alloc(A.nnz, c.stream);
    B->v.alloc(A.nnz, c.stream);
    MAMG_CU(cudaMemcpyAsync(B->rp.get(), A.rp.get(), sizeof(int32_t) * (A.nrows + 1),
                            cudaMemcpyDeviceToDevice, c.stream));
    if (A.nnz) {
        MAMG_CU(cudaMemcpyAsync(B->ci.get(), A.ci.get(), sizeof(int32_t) * A.nnz,
                                cudaMemcpyDeviceToDevice, c.stream));
        MAMG_CU(cudaMemcpyAsync(B->v.get(), A.v.get(), sizeof(double) * A.nnz,
                                cudaMemcpyDeviceToDevice, c.stream));
    }
    return B;
}

void spmv(Ctx& c, const DevCsr& A, int G, const double* x, double* y, const int* gate) {
    launch_spmv(c, A, G, x, EpiStore{y}, gate);
}

void residual(Ctx& c, const DevCsr& A, const double* b, const double* x, double* r,
              const int* gate) {
    launch_spmv(c, A, A.group, x, EpiResidual{b, r}, gate);
}

void smooth_sweep(Ctx& c, const DevCsr& A, const double* d, const double* b, const double* xi,
                  double* xo, const int* gate) {
    launch_spmv(c, A, A.group, xi, EpiSmooth{b, d, xi, xo}, gate);
}

void spmv_rows(Ctx& c, const DevCsr& A, int G, const double* x, double* y, const int* gate,
               int64_t r0, int64_t r1) {
    launch_spmv(c, A, G, x, EpiStore{y}, gate, r0, r1);
}

void residual_rows(Ctx& c, const DevCsr& A, const double* b, const double* x, double* r,
                   const int* gate, int64_t r0, int64_t r1) {
    launch_spmv(c, A, A.group, x, EpiResidual{b, r}, gate, r0, r1);
}

void smooth_sweep_rows(Ctx& c, const DevCsr& A, const double* d, const double* b, const double* xi,
                       double* xo, const int* gate, int64_t r0, int64_t r1) {
    launch_spmv(c, A, A.group, xi, EpiSmooth{b, d, xi, xo}, gate, r0, r1);
}

void smooth_from_zero(Ctx& c, int64_t n, const double* d, const double* b, double* x,
                      const int* gate) {
    if (n == 0) return;
    if (aligned16(d) && aligned16(b) && aligned16(x))
        launch_pdl(c.stream, k_smooth_zero4, dim3(blocks_for((n + 3) / 4, kBlock)), dim3(kBlock), 0, n,
                   d, b, x, gate);
    else
        launch_pdl(c.stream, k_smooth_zero, dim3(blocks_for(n, kBlock)), dim3(kBlock), 0, n, d, b, x,
                   gate);
    c.count();
    MAMG_LAUNCH_CHECK();
}

void prolong_correct(Ctx& c, const DevCsr& P, const double* xc, double* x, const int* gate) {
    if (P.nrows == 0) return;
    const bool vec = aligned16(P.ci.get()) && aligned16(P.v.get()) && aligned16(x);
    launch_pdl(c.stream, vec ? k_prolong_correct4 : k_prolong_correct,
               dim3(blocks_for(vec ? (P.nrows + 3) / 4 : P.nrows, kBlock)), dim3(kBlock), 0,
               static_cast<int64_t>(P.nrows), static_cast<const int32_t*>(P.ci.get()),
               static_cast<const double*>(P.v.get()), xc, x, gate);
    c.count();
    MAMG_LAUNCH_CHECK();
}

void l1_diagonal(Ctx& c, const DevCsr& A, double* d) {
    if (A.nrows != A.ncols) invalid("l1_diagonal: matrix is not square");
    l1_diagonal_local(c, A, d);
}

void l1_diagonal_local(Ctx& c, const DevCsr& A, double* d, bool defer) {
    if (A.nrows == 0) return;
    auto missing = [](int, int32_t row) {
        invalid("l1_diagonal: zero or missing diagonal entry in row " + std::to_string(row), row);
    };
    int32_t* bad;
    if (defer) {
        bad = defer_flags(c, 1, missing);
    } else {
        bad = reinterpret_cast<int32_t*>(c.d_small.get());
        const int32_t init = INT32_MAX;
        MAMG_CU(cudaMemcpyAsync(bad, &init, sizeof(init), cudaMemcpyHostToDevice, c.stream));
    }
    k_l1<<<blocks_for(A.nrows, kBlock), kBlock, 0, c.stream>>>(A.nrows, A.rp.get(), A.ci.get(),
                                                               A.v.get(), d, bad);
    c.count();
    MAMG_LAUNCH_CHECK();
    if (!defer) {
        const int64_t b = read_i32(c, bad);
        if (b != INT32_MAX) missing(0, static_cast<int32_t>(b));
    }
}

bool has_symmetric_pattern(Ctx& c, const DevCsr& A) {
    if (A.nrows != A.ncols) return false;
    if (A.nrows == 0) return true;
    int32_t* ok = reinterpret_cast<int32_t*>(c.d_small.get());
    const int32_t one = 1;
    MAMG_CU(cudaMemcpyAsync(ok, &one, sizeof(one), cudaMemcpyHostToDevice, c.stream));
    const int64_t avg = A.nnz / A.nrows;
    auto launch = [&](auto s_) {
        constexpr int S = decltype(s_)::value;
        k_sym_pattern<S><<<blocks_for(A.nrows * S, kBlock), kBlock, 0, c.stream>>>(
            A.nrows, A.rp.get(), A.ci.get(), ok);
    };
    if (avg <= 4)
        launch(std::integral_constant<int, 4>{});
    else if (avg <= 8)
        launch(std::integral_constant<int, 8>{});
    else if (avg <= 16)
        launch(std::integral_constant<int, 16>{});
    else
        launch(std::integral_constant<int, 32>{});
    c.count();
    MAMG_LAUNCH_CHECK();
    return read_i32(c, ok) == 1;
}

static std::unique_ptr<DevCsr> transpose_impl(Ctx& c, const DevCsr& A, int max_members);

std::unique_ptr<DevCsr> transpose(Ctx& c, const DevCsr& A) { return transpose_impl(c, A, 0); }

std::unique_ptr<DevCsr> transpose_agg(Ctx& c, const DevCsr& P, int max_members) {
    return transpose_impl(c, P, max_members);
}

static std::unique_ptr<DevCsr> transpose_impl(Ctx& c, const DevCsr& A, int max_members) {
    auto T = std::make_unique<DevCsr>();
    T->nrows = A.ncols;
    T->ncols = A.nrows;
    T->nnz = A.nnz;
    T->rp.alloc(A.ncols + 1, c.stream);
    T->ci.alloc(A.nnz, c.stream);
    T->v.alloc(A.nnz, c.stream);
    MAMG_CU(cudaMemsetAsync(T->rp.get(), 0, sizeof(int32_t) * (A.ncols + 1), c.stream));
    if (A.nrows > 0) {
        k_count_cols<<<blocks_for(A.nrows, kBlock), kBlock, 0, c.stream>>>(A.nrows, A.rp.get(),
                                                                           A.ci.get(), T->rp.get());
        c.count();
    }
    exclusive_scan_i32(c, T->rp.get(), T->rp.get(), A.ncols);
    if (A.nrows > 0) {
        DBuf<int32_t> cursor(A.ncols + 1, c.stream);
        MAMG_CU(cudaMemcpyAsync(cursor.get(), T->rp.get(), sizeof(int32_t) * (A.ncols + 1),
                                cudaMemcpyDeviceToDevice, c.stream));
        k_scatter_t<<<blocks_for(A.nrows, kBlock), kBlock, 0, c.stream>>>(
            A.nrows, A.rp.get(), A.ci.get(), A.v.get(), cursor.get(), T->ci.get(), T->v.get());
        c.count();
        k_sort_rows<<<blocks_for(T->nrows, kBlock), kBlock, 0, c.stream>>>(
            T->nrows, T->rp.get(), T->ci.get(), T->v.get());
        c.count();
    }
    MAMG_LAUNCH_CHECK();
    if (max_members > 0) {
        // R = P^T of a one-entry-per-row P: rows = aggregates (<= max_members
        // entries each, several per row as n_c < n), values copied from P
        T->single = T->nrows > 0 && T->nnz == T->nrows;
        T->finite = A.finite;
        T->max_tile = static_cast<int>(std::min<int64_t>(T->nnz, 256LL * max_members));
        T->group = lane_policy_from(T->nrows, T->nnz, T->single);
    } else {
        csr_finalize(c, *T);
    }
    return T;
}

std::unique_ptr<DevCsr> spgemm(Ctx& c, const DevCsr& A, const DevCsr& B) {
    if (A.ncols != B.nrows)
        invalid("spgemm: inner dimensions " + std::to_string(A.ncols) + " and " +
                std::to_string(B.nrows) + " differ");
    DBuf<int32_t> ub(A.nrows + 1, c.stream);
    int64_t total = 0;
    if (A.nrows > 0) {
        DBuf<unsigned long long> tot(1, c.stream);
        MAMG_CU(cudaMemsetAsync(tot.get(), 0, sizeof(unsigned long long), c.stream));
        k_spgemm_ub<<<blocks_for(A.nrows, kBlock), kBlock, 0, c.stream>>>(
            A.nrows, A.rp.get(), A.ci.get(), B.rp.get(), ub.get(), tot.get());
        c.count();
        MAMG_LAUNCH_CHECK();
        unsigned long long h = 0;
        MAMG_CU(cudaMemcpyAsync(&h, tot.get(), sizeof(h), cudaMemcpyDeviceToHost, c.stream));
        c.sync();
        // the contribution scratch and its scan are int32-indexed
        if (h >= static_cast<unsigned long long>(INT32_MAX))
            throw Error(MAMG_RUNTIME,
                        "spgemm: " + std::to_string(h) +
                            " intermediate products exceed the device's int32 index range",
                        -1);
        total = static_cast<int64_t>(h);
    }
    SpgemmProb pb{A.rp.get(), A.ci.get(), A.v.get(), B.rp.get(), B.ci.get(), B.v.get()};
    auto C = rowprod_run(c, pb, A.nrows, B.ncols, ub, total);
    return C;
}

} // namespace mamg
