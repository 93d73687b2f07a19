// tail.cu — the coarse end of the V/W cycle in ONE launch.
//
// Below a few tens of thousands of rows every level of the cycle is a string
// of tiny, latency-bound kernels (the coarsest level alone is 20 dependent
// sweeps). Here one thread-block cluster (16 CTAs x 512 threads, hardware
// cluster barriers) walks levels t..L of multigrid.cpp:65-109 directly: each
// dependent phase (sweep, residual, restriction, prolongation) is a
// grid-stride loop over the level's rows followed by a cluster barrier
// (barrier.cluster release/acquire orders the global-memory writes between
// the 16 SMs). Every row is evaluated with the same expression trees as the
// per-level kernels, so the cycle stays bit-identical.
#include <cooperative_groups.h>

#include "ops.cuh"
#include "tail.cuh"

namespace cg = cooperative_groups;

namespace mamg {
namespace {

constexpr int kTailThreads = 512;

// the reference's G-lane tree for one row (kernels.cpp:48-58), thread-local
template <int G>
__device__ __forceinline__ double row_tree_g(int lo, int hi, const int32_t* __restrict__ ci,
                                             const double* __restrict__ v,
                                             const double* x) {
    double s[G];
#pragma unroll
    for (int l = 0; l < G; ++l) s[l] = 0.0;
#pragma unroll 1
    for (int base = lo; base < hi; base += G) {
#pragma unroll
        for (int l = 0; l < G; ++l) {
            const int k = base + l;
            if (k < hi) s[l] = rn_add(s[l], rn_mul(v[k], __ldcg(x + ci[k])));
        }
    }
#pragma unroll
    for (int off = G / 2; off > 0; off >>= 1) {
#pragma unroll
        for (int l = 0; l < off; ++l) s[l] = rn_add(s[l], s[l + off]);
    }
    return s[0];
}

__device__ double row_sum(int G, int i, const int32_t* __restrict__ rp,
                          const int32_t* __restrict__ ci, const double* __restrict__ v,
                          const double* x) {
    const int lo = rp[i], hi = rp[i + 1];
    switch (G) {
        case 1: return row_tree_g<1>(lo, hi, ci, v, x);
        case 2: return row_tree_g<2>(lo, hi, ci, v, x);
        case 4: return row_tree_g<4>(lo, hi, ci, v, x);
        case 8: return row_tree_g<8>(lo, hi, ci, v, x);
        case 16: return row_tree_g<16>(lo, hi, ci, v, x);
        default:
            // G = 32: tail levels with G = 32 have rows of <= 32 entries
            // (alloc_workspace), whose tree is the same under G = 16
            // (nnz <= 2G' => V(G) = V(G'))
            return row_tree_g<16>(lo, hi, ci, v, x);
    }
}

struct Ctx1 {
    int gt, nt; // global thread index / count within the cluster
};

__device__ __forceinline__ void csync() { cg::this_cluster().sync(); }

// k sweeps from `src` (nullptr = zero) into dst, intermediates in xw/scratch
// (same buffer plan as the host-driven path in solve.cu)
__device__ void t_sweeps(const Ctx1& t, const TailLevel& L, const double* b, const double* src,
                         double* dst, int k) {
    double* xa = L.xw;
    double* xb = L.scratch;
    if (k == 0) {
        for (int i = t.gt; i < L.n; i += t.nt) dst[i] = src ? __ldcg(src + i) : 0.0;
        csync();
        return;
    }
    // backward plan: out[k-1] = dst, then alternate within {xa, xb}
    double* before_last = dst == xa ? xb : (dst == xb ? xa : xb);
    // out[j] for j = k-2 .. 0: alternate starting from before_last
    auto out_of = [&](int j, double* bl) -> double* {
        if (j == k - 1) return dst;
        const int dist = (k - 2) - j; // 0 for j = k-2
        return (dist & 1) ? (bl == xa ? xb : xa) : bl;
    };
    if (k >= 2 && src != nullptr && out_of(0, before_last) == src) before_last = xa;
    const double* cur = src;
    for (int j = 0; j < k; ++j) {
        double* o = out_of(j, before_last);
        for (int i = t.gt; i < L.n; i += t.nt) {
            if (cur == nullptr) {
                o[i] = rn_add(0.0, rn_div(__ldcg(b + i), L.l1[i]));
            } else {
                const double s = row_sum(L.G, i, L.rp, L.ci, L.v, cur);
                o[i] = rn_add(__ldcg(cur + i), rn_div(rn_sub(__ldcg(b + i), s), L.l1[i]));
            }
        }
        csync();
        cur = o;
    }
}

// G-lane tree over a row cached in registers (m <= 16 entries): lane
// j % G accumulates entries j in increasing order, then the halving fold.
template <int G>
__device__ __forceinline__ double cached_tree(const int (&cc)[16], const double (&vv)[16], int m,
                                              const double* x) {
    double lane[G];
#pragma unroll
    for (int l = 0; l < G; ++l) lane[l] = 0.0;
#pragma unroll
    for (int j = 0; j < 16; ++j)
        if (j < m) lane[j % G] = rn_add(lane[j % G], rn_mul(vv[j], __ldcg(x + cc[j])));
#pragma unroll
    for (int off = G / 2; off > 0; off >>= 1) {
#pragma unroll
        for (int l = 0; l < off; ++l) lane[l] = rn_add(lane[l], lane[l + off]);
    }
    return lane[0];
}

// Coarsest level with one row per thread: the row (<= 16 entries), b_i and
// d_i stay in registers for all sweeps; each sweep is one x gather + update.
// Same buffer plan as t_sweeps (from zero, last sweep into x_out).
__device__ void t_coarsest_cached(const Ctx1& t, const TailLevel& L, const double* b,
                                  double* x_out, int k) {
    const int i = t.gt;
    int cc[16];
    double vv[16];
    int lo = 0, m = 0;
    double bi = 0.0, di = 1.0;
    const bool mine = i < L.n;
    if (mine) {
        lo = L.rp[i];
        m = L.rp[i + 1] - lo;
        bi = __ldcg(b + i);
        di = L.l1[i];
    }
    const bool fits = m <= 16;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        cc[j] = (j < m && fits) ? L.ci[lo + j] : 0;
        vv[j] = (j < m && fits) ? L.v[lo + j] : 0.0;
    }
    double* xa = L.xw;
    double* xb = L.scratch;
    // out[k-1] = x_out; out[k-2] = xb, then alternate (src is zero -> no clash)
    const double* cur = nullptr;
    for (int s = 0; s < k; ++s) {
        const int dist = (k - 2) - s;
        double* o = (s == k - 1) ? x_out : ((dist & 1) ? xa : xb);
        if (mine) {
            double val;
            if (cur == nullptr) {
                val = rn_add(0.0, rn_div(bi, di));
            } else if (fits) {
                double sum;
                switch (L.G) {
                    case 1: sum = cached_tree<1>(cc, vv, m, cur); break;
                    case 2: sum = cached_tree<2>(cc, vv, m, cur); break;
                    case 4: sum = cached_tree<4>(cc, vv, m, cur); break;
                    case 8: sum = cached_tree<8>(cc, vv, m, cur); break;
                    default: sum = cached_tree<16>(cc, vv, m, cur); break; // m <= 16: G=32 tree too
                }
                val = rn_add(__ldcg(cur + i), rn_div(rn_sub(bi, sum), di));
            } else {
                const double sum = row_sum(L.G, i, L.rp, L.ci, L.v, cur);
                val = rn_add(__ldcg(cur + i), rn_div(rn_sub(bi, sum), di));
            }
            o[i] = val;
        }
        csync();
        cur = o;
    }
}

// The V/W recursion of multigrid.cpp:65-109 as an explicit walk over the
// tail levels (no device recursion, no spills): `up` marks returning to
// level k after a visit of level k + 1.
__device__ void t_cycle(const Ctx1& t, const TailParams& P) {
    const int last = P.nlev - 1;
    const int visits = P.cycle == 1 ? 2 : 1;
    int cnt[kMaxTail];
    for (int j = 0; j < kMaxTail; ++j) cnt[j] = 0;
    int k = 0;
    bool zero = P.zero != 0, up = false;
    for (;;) {
        const TailLevel& L = P.lv[k];
        const double* b = k == 0 ? P.b : P.lv[k - 1].cb;
        double* x_out = k == 0 ? P.x_out : P.lv[k - 1].cx;
        if (!up) {
            if (k == last) {
                if (P.cache_coarsest && L.n <= t.nt && P.coarsest >= 2)
                    t_coarsest_cached(t, L, b, x_out, P.coarsest);
                else
                    t_sweeps(t, L, b, nullptr, x_out, P.coarsest);
                if (k == 0) return;
                --k;
                up = true;
                continue;
            }
            if (P.pre == 0) {
                for (int i = t.gt; i < L.n; i += t.nt) L.xw[i] = zero ? 0.0 : __ldcg(x_out + i);
                csync();
            } else {
                t_sweeps(t, L, b, zero ? nullptr : x_out, L.xw, P.pre);
            }
            for (int i = t.gt; i < L.n; i += t.nt)
                L.scratch[i] = rn_sub(__ldcg(b + i), row_sum(L.G, i, L.rp, L.ci, L.v, L.xw));
            csync();
            for (int I = t.gt; I < L.nc; I += t.nt)
                L.cb[I] = row_sum(L.GR, I, L.Rrp, L.Rci, L.Rv, L.scratch);
            csync();
            cnt[k] = 1;
            ++k;
            zero = true;
            continue;
        }
        // back at level k after a coarse visit
        if (cnt[k] < visits) { // W-cycle: second visit from the current coarse x
            ++cnt[k];
            ++k;
            zero = false;
            up = false;
            continue;
        }
        for (int i = t.gt; i < L.n; i += t.nt)
            L.xw[i] = rn_add(__ldcg(L.xw + i),
                             rn_mul(1.0, rn_add(0.0, rn_mul(L.Pv[i], __ldcg(L.cx + L.Pci[i])))));
        csync();
        if (P.post == 0) {
            for (int i = t.gt; i < L.n; i += t.nt) x_out[i] = __ldcg(L.xw + i);
            csync();
        } else {
            t_sweeps(t, L, b, L.xw, x_out, P.post);
        }
        if (k == 0) return;
        --k; // up stays true
    }
}

__global__ void __launch_bounds__(kTailThreads, 1) k_tail(TailParams P) {
    if (P.gate && *P.gate) return;
    cg::cluster_group cl = cg::this_cluster();
    Ctx1 t;
    t.gt = static_cast<int>(cl.block_rank()) * kTailThreads + threadIdx.x;
    t.nt = static_cast<int>(cl.num_blocks()) * kTailThreads;
    t_cycle(t, P);
}

int g_cluster = 0; // chosen cluster size (16 if the device allows, else 8)

} // namespace

bool tail_supported(Ctx& c) {
    if (g_cluster == 0) {
        int cs = 16;
        if (cudaFuncSetAttribute(k_tail, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) !=
            cudaSuccess) {
            cudaGetLastError();
            cs = 8;
        }
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(cs);
        cfg.blockDim = dim3(kTailThreads);
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cs;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int nclusters = 0;
        if (cudaOccupancyMaxActiveClusters(&nclusters, k_tail, &cfg) != cudaSuccess ||
            nclusters < 1) {
            cudaGetLastError();
            cs = 8;
            at[0].val.clusterDim.x = cs;
            cfg.gridDim = dim3(cs);
            if (cudaOccupancyMaxActiveClusters(&nclusters, k_tail, &cfg) != cudaSuccess ||
                nclusters < 1) {
                cudaGetLastError();
                cs = -1;
            }
        }
        g_cluster = cs;
    }
    (void)c;
    return g_cluster > 0;
}

int cluster_size_limit() { return g_cluster > 0 ? g_cluster : 8; }

void tail_launch(Ctx& c, const TailParams& P) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(g_cluster);
    cfg.blockDim = dim3(kTailThreads);
    cfg.stream = c.stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = g_cluster;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    MAMG_CU(cudaLaunchKernelEx(&cfg, k_tail, P));
    c.count();
}

} // namespace mamg
