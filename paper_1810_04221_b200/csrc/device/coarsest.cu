// coarsest.cu — the coarsest-level solve of the V/W/K cycle (multigrid.cpp:
// 82-88: x = 0, then `coarsest_sweeps` l1-Jacobi sweeps) in ONE launch.
//
// The coarsest level is small (<= 40 cbrt(n_0) rows by the stop rule) but its
// 20 dependent sweeps are each a latency-bound kernel. Here a thread-block
// cluster of CS CTAs x 512 threads owns the level, one row per thread: a row
// of <= 16 entries (and b_i, d_i) is loaded into registers once and kept for
// all sweeps; the iterate lives in the CTAs' shared memory (each CTA its own
// rows, two buffers) and x_j is gathered from the owning CTA — a local shared
// load or a DSMEM load through the cluster window; one cluster barrier
// (release/acquire) per sweep. Each row uses the reference's G-lane tree
// (thread-local), so the result is bit-identical. The last sweep writes x_out
// in global memory.
#include <cooperative_groups.h>

#include <algorithm>
#include <vector>

#include "ops.cuh"
#include "tail.cuh"

namespace cg = cooperative_groups;

namespace mamg {
namespace {

constexpr int kCoThreads = 512;

// x value of global column j from the cluster: the owning CTA's shared copy
// (a local shared load or a DSMEM load through the cluster window)
__device__ __forceinline__ double xget(cg::cluster_group& cl, const double* xloc, int j, int rpc,
                                       int me) {
    const int q = j / rpc;
    const double* p = xloc + (j - q * rpc);
    return q == me ? *p : *cl.map_shared_rank(p, q);
}

// G-lane tree over a row cached in registers (m <= 16), x gathered from the
// cluster; lane j % G accumulates entry j in order, then the halving fold
template <int G>
__device__ __forceinline__ double ctree(const int (&cc)[16], const double (&vv)[16], int m,
                                        cg::cluster_group& cl, const double* xin, int rpc, int me) {
    double lane[G];
#pragma unroll
    for (int l = 0; l < G; ++l) lane[l] = 0.0;
#pragma unroll
    for (int j = 0; j < 16; ++j)
        if (j < m) lane[j % G] = rn_add(lane[j % G], rn_mul(vv[j], xget(cl, xin, cc[j], rpc, me)));
#pragma unroll
    for (int off = G / 2; off > 0; off >>= 1) {
#pragma unroll
        for (int l = 0; l < off; ++l) lane[l] = rn_add(lane[l], lane[l + off]);
    }
    return lane[0];
}

// general row (any length) read from global memory each sweep
template <int G>
__device__ __forceinline__ double gtree(int lo, int hi, const int32_t* __restrict__ ci,
                                        const double* __restrict__ v, cg::cluster_group& cl,
                                        const double* xin, int rpc, int me) {
    double s[G];
#pragma unroll
    for (int l = 0; l < G; ++l) s[l] = 0.0;
#pragma unroll 1
    for (int base = lo; base < hi; base += G) {
#pragma unroll
        for (int l = 0; l < G; ++l) {
            const int k = base + l;
            if (k < hi) s[l] = rn_add(s[l], rn_mul(v[k], xget(cl, xin, ci[k], rpc, me)));
        }
    }
#pragma unroll
    for (int off = G / 2; off > 0; off >>= 1) {
#pragma unroll
        for (int l = 0; l < off; ++l) s[l] = rn_add(s[l], s[l + off]);
    }
    return s[0];
}

// One row per thread: rows [r*rpc, (r+1)*rpc) belong to CTA r, whose shared
// memory holds their x values (two buffers). Rows of <= 16 entries stay in
// registers for all sweeps; x is gathered from the owning CTA (local or
// DSMEM load); one cluster barrier per sweep.
__global__ void __launch_bounds__(kCoThreads, 1)
k_coarsest(int n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
           const double* __restrict__ v, const double* __restrict__ l1, const double* b,
           double* x_out, int k, int G, int rpc, const int* __restrict__ gate) {
    pdl_wait();
    if (gate && *gate) return;
    cg::cluster_group cl = cg::this_cluster();
    const int me = static_cast<int>(cl.block_rank());
    __shared__ double X[2][kCoThreads];
    const int i = me * rpc + static_cast<int>(threadIdx.x);
    const bool mine = static_cast<int>(threadIdx.x) < rpc && i < n;
    int lo = 0, m = 0;
    double bi = 0.0, di = 1.0;
    int cc[16];
    double vv[16];
    if (mine) {
        lo = rp[i];
        m = rp[i + 1] - lo;
        bi = b[i];
        di = l1[i];
    }
    const bool cached = m <= 16;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        cc[j] = (mine && cached && j < m) ? ci[lo + j] : 0;
        vv[j] = (mine && cached && j < m) ? v[lo + j] : 0.0;
    }
    const int Gc = G >= 16 ? 16 : G; // rows <= 16 = 2*8: G and min(G, 16) give the same tree
    for (int s = 0; s < k; ++s) {
        const double* xin = X[(s + 1) & 1];
        double* xo = X[s & 1];
        double val = 0.0;
        if (mine) {
            if (s == 0) {
                val = rn_add(0.0, rn_div(bi, di)); // A * 0 == +0 (finite A)
            } else {
                double y;
                if (cached) {
                    switch (Gc) {
                        case 1: y = ctree<1>(cc, vv, m, cl, xin, rpc, me); break;
                        case 2: y = ctree<2>(cc, vv, m, cl, xin, rpc, me); break;
                        case 4: y = ctree<4>(cc, vv, m, cl, xin, rpc, me); break;
                        case 8: y = ctree<8>(cc, vv, m, cl, xin, rpc, me); break;
                        default: y = ctree<16>(cc, vv, m, cl, xin, rpc, me); break;
                    }
                } else {
                    switch (G) {
                        case 1: y = gtree<1>(lo, lo + m, ci, v, cl, xin, rpc, me); break;
                        case 2: y = gtree<2>(lo, lo + m, ci, v, cl, xin, rpc, me); break;
                        case 4: y = gtree<4>(lo, lo + m, ci, v, cl, xin, rpc, me); break;
                        case 8: y = gtree<8>(lo, lo + m, ci, v, cl, xin, rpc, me); break;
                        case 16: y = gtree<16>(lo, lo + m, ci, v, cl, xin, rpc, me); break;
                        default: y = gtree<32>(lo, lo + m, ci, v, cl, xin, rpc, me); break;
                    }
                }
                val = rn_add(xin[threadIdx.x], rn_div(rn_sub(bi, y), di));
            }
            if (s == k - 1)
                x_out[i] = val;
            else
                xo[threadIdx.x] = val;
        }
        if (s < k - 1) cl.sync();
    }
    // peers may still be reading this CTA's shared x (DSMEM) in the last sweep
    cl.sync();
}

} // namespace

// Plan for a level: CS = smallest power-of-two cluster with at most
// kCoThreads rows per CTA (one row per thread), CS <= the cluster limit.
bool coarsest_plan(Ctx& c, const DevCsr& A, CoarsestPlan& p) {
    p.cs = 0;
    const int64_t n = A.nrows;
    if (n == 0 || !A.finite || !tail_supported(c)) return false;
    const int max_cs = cluster_size_limit();
    int cs = 1;
    while (cs < max_cs && static_cast<int64_t>(cs) * kCoThreads < n) cs *= 2;
    if (static_cast<int64_t>(cs) * kCoThreads < n) return false;
    p.cs = cs;
    p.smem = static_cast<int>((n + cs - 1) / cs); // rows per CTA
    return true;
}

void coarsest_launch(Ctx& c, const DevCsr& A, const double* l1, const CoarsestPlan& p,
                     const double* b, double* x_out, int k, const int* gate) {
    static bool attr = false;
    if (!attr) {
        MAMG_CU(cudaFuncSetAttribute(k_coarsest, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        attr = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(p.cs);
    cfg.blockDim = dim3(kCoThreads);
    cfg.stream = c.stream;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = p.cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    MAMG_CU(cudaLaunchKernelEx(&cfg, k_coarsest, static_cast<int>(A.nrows), A.rp.get(), A.ci.get(),
                               A.v.get(), l1, b, x_out, k, A.group, p.smem, gate));
    c.count();
}

} // namespace mamg
