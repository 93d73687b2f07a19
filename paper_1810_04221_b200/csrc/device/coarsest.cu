// coarsest.cu — the coarsest-level solve of the V/W/K cycle (multigrid.cpp:
// 82-88: x = 0, then `coarsest_sweeps` l1-Jacobi sweeps) in ONE launch.
//
// The coarsest level is small (<= 40 cbrt(n_0) rows by the stop rule) but its
// 20 dependent sweeps are each a latency-bound kernel (~5 us). Here a thread-
// block cluster of CS CTAs (CS in {2, 4, 8, 16}) keeps the whole level in
// distributed shared memory: CTA r stages its contiguous block of rows
// (entries, b, l1) once, and every CTA holds a full copy of the iterate x in
// two buffers. A sweep reads x from the local copy, computes its rows with
// the reference's G-lane tree (thread-local, same expression as the per-level
// kernels, so bit-identical), and broadcasts the new values into every CTA's
// other buffer with DSMEM stores; one cluster barrier (release/acquire) per
// sweep orders them. The last sweep writes x_out in global memory.
#include <cooperative_groups.h>

#include <algorithm>
#include <vector>

#include "ops.cuh"
#include "tail.cuh"

namespace cg = cooperative_groups;

namespace mamg {
namespace {

constexpr int kCoThreads = 512;
constexpr size_t kCoSmemMax = 200 * 1024;

// the reference's G-lane tree over a row, thread-local (kernels.cpp:42-58)
template <int G>
__device__ __forceinline__ double tree(int lo, int hi, const int32_t* c, const double* a,
                                       const double* x) {
    double s[G];
#pragma unroll
    for (int l = 0; l < G; ++l) s[l] = 0.0;
#pragma unroll 1
    for (int base = lo; base < hi; base += G) {
#pragma unroll
        for (int l = 0; l < G; ++l) {
            const int k = base + l;
            if (k < hi) s[l] = rn_add(s[l], rn_mul(a[k], x[c[k]]));
        }
    }
#pragma unroll
    for (int off = G / 2; off > 0; off >>= 1) {
#pragma unroll
        for (int l = 0; l < off; ++l) s[l] = rn_add(s[l], s[l + off]);
    }
    return s[0];
}

// G = 32 rows longer than 32 entries with 16 live accumulators: lanes l and
// l + 16 summed side by side, folded at once (the tree's off = 16 step)
__device__ __forceinline__ double tree32(int lo, int hi, const int32_t* c, const double* a,
                                         const double* x) {
    double u[16];
#pragma unroll
    for (int l = 0; l < 16; ++l) {
        double p = 0.0, q = 0.0;
#pragma unroll 1
        for (int k = lo + l; k < hi; k += 32) p = rn_add(p, rn_mul(a[k], x[c[k]]));
#pragma unroll 1
        for (int k = lo + l + 16; k < hi; k += 32) q = rn_add(q, rn_mul(a[k], x[c[k]]));
        u[l] = rn_add(p, q);
    }
#pragma unroll
    for (int off = 8; off > 0; off >>= 1) {
#pragma unroll
        for (int l = 0; l < off; ++l) u[l] = rn_add(u[l], u[l + off]);
    }
    return u[0];
}

__device__ __forceinline__ double row_sum(int G, int lo, int hi, const int32_t* c, const double* a,
                                          const double* x) {
    switch (G) {
        case 1: return tree<1>(lo, hi, c, a, x);
        case 2: return tree<2>(lo, hi, c, a, x);
        case 4: return tree<4>(lo, hi, c, a, x);
        case 8: return tree<8>(lo, hi, c, a, x);
        case 16: return tree<16>(lo, hi, c, a, x);
        default:
            // a row of <= 32 entries has the same tree under G = 16
            // (nnz <= 2G' => V(G) = V(G'))
            return hi - lo <= 32 ? tree<16>(lo, hi, c, a, x) : tree32(lo, hi, c, a, x);
    }
}

__global__ void __launch_bounds__(kCoThreads, 1)
k_coarsest(int n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
           const double* __restrict__ v, const double* __restrict__ l1, const double* b,
           double* x_out, int k, int G, const int32_t* __restrict__ split,
           const int* __restrict__ gate) {
    if (gate && *gate) return;
    cg::cluster_group cl = cg::this_cluster();
    const int r = static_cast<int>(cl.block_rank());
    const int CS = static_cast<int>(cl.num_blocks());
    const int r0 = split[r], r1 = split[r + 1];
    const int nr = r1 - r0;
    const int e0 = rp[r0], ne = rp[r1] - e0;
    extern __shared__ __align__(16) double sm[];
    double* X0 = sm;
    double* X1 = X0 + n;
    double* sv = X1 + n;
    double* sb = sv + ne;
    double* sd = sb + nr;
    int32_t* sc = reinterpret_cast<int32_t*>(sd + nr);
    int32_t* srp = sc + ne;
    for (int e = threadIdx.x; e < ne; e += kCoThreads) {
        sv[e] = v[e0 + e];
        sc[e] = ci[e0 + e];
    }
    for (int i = threadIdx.x; i < nr; i += kCoThreads) {
        sb[i] = b[r0 + i];
        sd[i] = l1[r0 + i];
    }
    for (int i = threadIdx.x; i <= nr; i += kCoThreads) srp[i] = rp[r0 + i] - e0;
    cl.sync(); // staged, and every CTA of the cluster is running
    for (int s = 0; s < k; ++s) {
        const double* xin = (s & 1) ? X0 : X1; // iterate s - 1
        double* xo = (s & 1) ? X1 : X0;
        const bool last = s == k - 1;
        for (int i = threadIdx.x; i < nr; i += kCoThreads) {
            double val;
            if (s == 0) {
                val = rn_add(0.0, rn_div(sb[i], sd[i])); // A * 0 == +0 (finite A)
            } else {
                const double y = row_sum(G, srp[i], srp[i + 1], sc, sv, xin);
                val = rn_add(xin[r0 + i], rn_div(rn_sub(sb[i], y), sd[i]));
            }
            if (last) {
                x_out[r0 + i] = val;
            } else {
                for (int q = 0; q < CS; ++q) *cl.map_shared_rank(xo + r0 + i, q) = val;
            }
        }
        if (!last) cl.sync();
    }
}

} // namespace

// Plan for a level: balanced row split over CS CTAs (by entries); CS is the
// smallest cluster whose largest CTA share fits kCoSmemMax and that gives
// every thread at most two rows per sweep. Reads the row pointers back once
// (setup time).
bool coarsest_plan(Ctx& c, const DevCsr& A, CoarsestPlan& p) {
    p.cs = 0;
    const int64_t n = A.nrows;
    if (n == 0 || n > 20000 || !A.finite || !tail_supported(c)) return false;
    std::vector<int32_t> rp(static_cast<size_t>(n + 1));
    MAMG_CU(cudaMemcpyAsync(rp.data(), A.rp.get(), sizeof(int32_t) * (n + 1),
                            cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    const int max_cs = cluster_size_limit();
    int cs0 = 2;
    while (cs0 < max_cs && static_cast<int64_t>(cs0) * 2 * kCoThreads < n) cs0 *= 2;
    for (int cs = cs0; cs <= max_cs; cs *= 2) {
        std::vector<int32_t> split(static_cast<size_t>(cs + 1), 0);
        const int64_t nnz = rp[n];
        int64_t row = 0;
        for (int q = 1; q < cs; ++q) {
            const int64_t target = nnz * q / cs;
            while (row < n && rp[row] < target) ++row;
            split[q] = static_cast<int32_t>(row);
        }
        split[cs] = static_cast<int32_t>(n);
        size_t worst = 0;
        for (int q = 0; q < cs; ++q) {
            const int64_t nr = split[q + 1] - split[q];
            const int64_t ne = rp[split[q + 1]] - rp[split[q]];
            const size_t bytes = sizeof(double) * (2 * n + ne + 2 * nr) + sizeof(int32_t) * (ne + nr + 1);
            worst = std::max(worst, bytes);
        }
        if (worst <= kCoSmemMax) {
            p.cs = cs;
            p.smem = static_cast<int>(worst);
            p.split.alloc(cs + 1, c.stream);
            MAMG_CU(cudaMemcpyAsync(p.split.get(), split.data(), sizeof(int32_t) * (cs + 1),
                                    cudaMemcpyHostToDevice, c.stream));
            c.sync();
            return true;
        }
    }
    return false;
}

void coarsest_launch(Ctx& c, const DevCsr& A, const double* l1, const CoarsestPlan& p,
                     const double* b, double* x_out, int k, const int* gate) {
    static bool attr = false;
    if (!attr) {
        MAMG_CU(cudaFuncSetAttribute(k_coarsest, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        MAMG_CU(cudaFuncSetAttribute(k_coarsest, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(kCoSmemMax)));
        attr = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(p.cs);
    cfg.blockDim = dim3(kCoThreads);
    cfg.dynamicSmemBytes = static_cast<size_t>(p.smem);
    cfg.stream = c.stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = p.cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    MAMG_CU(cudaLaunchKernelEx(&cfg, k_coarsest, static_cast<int>(A.nrows), A.rp.get(), A.ci.get(),
                               A.v.get(), l1, b, x_out, k, A.group, p.split.get(), gate));
    c.count();
}

} // namespace mamg
