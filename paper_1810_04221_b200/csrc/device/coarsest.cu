// coarsest.cu — the coarsest-level solve of the V/W/K cycle (multigrid.cpp:
// 82-88: x = 0, then `coarsest_sweeps` l1-Jacobi sweeps) in ONE launch.
//
// The coarsest level is small (<= 40 cbrt(n_0) rows by the stop rule) but its
// 20 dependent sweeps are each a latency-bound kernel (~3 us per launch in
// the replayed graph). Here a thread-block cluster of CS CTAs x 512 threads
// owns the level, one row per thread: the CTA's rows are staged once in
// shared memory (transposed ELL, conflict-free) with b_i, d_i in registers,
// and kept for all sweeps (a row re-read from L2 each sweep would put an L2
// round trip per 8 entries on every sweep's critical path). Every CTA keeps its
// own copy of the iterate in shared memory (two buffers, all n entries
// addressable) and reads x only from it: no remote loads. A sweep's new value
// x_i is stored into the own copy and PUSHED (st.shared::cluster, fire and
// forget) into the copies of exactly the CTAs that read it — those owning a
// row with column i (a bitmask per row, built once per setup). One cluster barrier
// (release / acquire) per sweep makes the pushes visible; the two buffers
// alternate, so a sweep never overwrites values a slower CTA still reads.
// Each row uses the reference's G-lane tree (thread-local), so the result is
// bit-identical. The last sweep writes x_out in global memory.
//
// Cost model per sweep: ~3m local shared loads + the row tree, ~|halo|
// remote 8-byte stores per CTA (DSMEM ~21 B/clk per SM), one cluster barrier
// (~380 clk) — vs a kernel launch + an L2 round trip per sweep.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>
#include <vector>

#include "ops.cuh"

namespace cg = cooperative_groups;

namespace mamg {
namespace {

constexpr int kCoThreads = 512;
constexpr int kCoMaxCluster = 16;
constexpr size_t kCoSmemMax = 227 * 1024; // dynamic shared memory per CTA (B200 opt-in max)

__device__ __forceinline__ void push_remote(double* local_addr, int rank, double val) {
    const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(local_addr));
    uint32_t ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
    asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(ra), "d"(val) : "memory");
}

__device__ __forceinline__ void cluster_barrier() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                     : "memory");
}

// G-lane tree of row entries staged in shared memory (entry j of the CTA's
// row t at [j * rpc + t]: conflict-free across the warp; padded to the
// warp's longest row with v = 0, column = the row itself), x from the own
// copy. Lane j % G accumulates entry j in order, then the halving fold. The
// loop runs to the warp's longest row `mw` (uniform: no divergent branches,
// so the G loads of a round are all in flight together); entries past the
// row's own length m are dropped by a select, never added — the sum is the
// reference's expression exactly.
template <int G>
__device__ __forceinline__ double stree(int m, int mw, const int32_t* sci, const double* sv,
                                        int rpc, const double* xin) {
    double s[G];
#pragma unroll
    for (int l = 0; l < G; ++l) s[l] = 0.0;
#pragma unroll 1
    for (int base = 0; base < mw; base += G) {
        double p[G];
#pragma unroll
        for (int l = 0; l < G; ++l) {
            const int j = base + l;
            p[l] = rn_mul(sv[j * rpc], xin[sci[j * rpc]]);
        }
#pragma unroll
        for (int l = 0; l < G; ++l) s[l] = base + l < m ? rn_add(s[l], p[l]) : s[l];
    }
#pragma unroll
    for (int off = G / 2; off > 0; off >>= 1) {
#pragma unroll
        for (int l = 0; l < off; ++l) s[l] = rn_add(s[l], s[l + off]);
    }
    return s[0];
}

// One row per thread: rows [r*rpc, (r+1)*rpc) belong to CTA r. Dynamic
// shared memory: two full-length copies of x (2 n doubles), the CTA's rows
// in the transposed ELL layout (rpc x Wp values, rpc x Wp column ids; Wp =
// the longest row rounded up to a multiple of G), its row pointers.
__global__ void __launch_bounds__(kCoThreads, 1)
k_coarsest(int n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
           const double* __restrict__ v, const double* __restrict__ l1, const double* b,
           const uint32_t* __restrict__ readers_of, double* x_out, int k, int G, int rpc, int Wp,
           const int* __restrict__ gate) {
    extern __shared__ __align__(16) double X[]; // [2][n], values, column ids, row pointers
    double* sv = X + 2 * static_cast<size_t>(n);
    int32_t* sci = reinterpret_cast<int32_t*>(sv + static_cast<size_t>(rpc) * Wp);
    int32_t* srp = sci + static_cast<size_t>(rpc) * Wp;
    const int me = static_cast<int>(cg::this_cluster().block_rank());
    const int t = static_cast<int>(threadIdx.x);
    const int r0 = me * rpc;
    const int nr = max(0, min(rpc, n - r0)); // rows of this CTA
    const int i = r0 + t;
    const bool mine = t < nr;
    // stage the CTA's rows: row pointers, then every entry with coalesced
    // loads (the row of entry e by binary search over the row pointers)
    for (int u = t; u <= nr; u += kCoThreads) srp[u] = rp[r0 + u];
    __syncthreads();
    const int e0 = srp[0], ne = srp[nr] - e0;
    for (int e = t; e < ne; e += kCoThreads) {
        int lo = 0, hi = nr - 1;
        while (lo < hi) {
            const int mid = lo + ((hi - lo + 1) >> 1);
            if (srp[mid] - e0 <= e) lo = mid; else hi = mid - 1;
        }
        const int j = e - (srp[lo] - e0);
        sci[j * rpc + lo] = ci[e0 + e];
        sv[j * rpc + lo] = v[e0 + e];
    }
    int m = 0;
    double di = 1.0;
    unsigned readers = 0u;
    if (mine) {
        m = srp[t + 1] - srp[t];
        di = l1[i];
        readers = readers_of[i];
        for (int j = m; j < Wp; ++j) { // padding: never added (select), always a valid column
            sci[j * rpc + t] = i;
            sv[j * rpc + t] = 0.0;
        }
    }
    // the warp's longest row: the uniform trip count of the row trees
    const int mw = __reduce_max_sync(0xffffffffu, m);
    // everything above is setup data; b is the predecessor's output
    pdl_wait();
    if (gate && *gate) return; // uniform: every CTA of the cluster leaves here
    const double bi = mine ? b[i] : 0.0;
    // every CTA of the cluster runs (and has staged its rows) before the
    // first remote store
    cluster_barrier();
    const int32_t* rci = sci + t;
    const double* rv = sv + t;
    for (int s = 0; s < k; ++s) {
        const double* xin = X + static_cast<size_t>((s + 1) & 1) * n;
        double* xo = X + static_cast<size_t>(s & 1) * n;
        if (mine) {
            double val;
            if (s == 0) {
                val = rn_add(0.0, rn_div(bi, di)); // A * 0 == +0 (finite A)
            } else {
                double y;
                switch (G) {
                    case 1: y = stree<1>(m, mw, rci, rv, rpc, xin); break;
                    case 2: y = stree<2>(m, mw, rci, rv, rpc, xin); break;
                    case 4: y = stree<4>(m, mw, rci, rv, rpc, xin); break;
                    case 8: y = stree<8>(m, mw, rci, rv, rpc, xin); break;
                    case 16: y = stree<16>(m, mw, rci, rv, rpc, xin); break;
                    default: y = stree<32>(m, mw, rci, rv, rpc, xin); break;
                }
                val = rn_add(xin[i], rn_div(rn_sub(bi, y), di));
            }
            if (s == k - 1) {
                x_out[i] = val;
            } else {
                xo[i] = val;
                for (unsigned r = readers; r; r &= r - 1) push_remote(xo + i, __ffs(r) - 1, val);
            }
        }
        if (s < k - 1) cluster_barrier();
    }
    // the last sweep pushes nothing: every remote store into this CTA's
    // shared memory completed before the last barrier
}

// readers[j] |= bit of the CTA owning row i, for every column j of row i
// owned by another CTA (global atomics, once per setup)
__global__ void k_coarsest_readers(int n, const int32_t* __restrict__ rp,
                                   const int32_t* __restrict__ ci, int rpc, uint32_t* readers) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int q = i / rpc;
    for (int e = rp[i]; e < rp[i + 1]; ++e) {
        const int j = ci[e];
        if (j / rpc != q) atomicOr(readers + j, 1u << q);
    }
}

int g_cluster = 0; // usable cluster size (16 when non-portable sizes work, else 8; -1 none)

int cluster_limit(size_t smem) {
    if (g_cluster == 0) {
        int cs = kCoMaxCluster;
        if (cudaFuncSetAttribute(k_coarsest, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) !=
            cudaSuccess) {
            cudaGetLastError();
            cs = 8;
        }
        cudaFuncSetAttribute(k_coarsest, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem));
        cudaGetLastError();
        for (; cs >= 8; cs /= 2) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(cs);
            cfg.blockDim = dim3(kCoThreads);
            cfg.dynamicSmemBytes = smem;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = cs;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            int nclusters = 0;
            if (cudaOccupancyMaxActiveClusters(&nclusters, k_coarsest, &cfg) == cudaSuccess &&
                nclusters >= 1)
                break;
            cudaGetLastError();
        }
        g_cluster = cs >= 8 ? cs : -1;
    }
    return g_cluster;
}

} // namespace

// Plan for a level: CS = smallest power-of-two cluster with at most
// kCoThreads rows per CTA (one row per thread), CS <= the cluster limit; two
// copies of x plus the CTA's rows (ELL, width = the longest row) must fit in
// shared memory. MAMG_COARSEST=0 disables it.
bool coarsest_plan(Ctx& c, const DevCsr& A, CoarsestPlan& p) {
    p.cs = 0;
    static const bool off = [] {
        const char* e = std::getenv("MAMG_COARSEST");
        return e && e[0] == '0';
    }();
    const int64_t n = A.nrows;
    if (off || n == 0 || !A.finite) return false;
    const int max_cs = cluster_limit(kCoSmemMax);
    if (max_cs < 1) return false;
    int cs = 1;
    while (cs < max_cs && static_cast<int64_t>(cs) * kCoThreads < n) cs *= 2;
    if (static_cast<int64_t>(cs) * kCoThreads < n) return false;
    const int rpc = static_cast<int>((n + cs - 1) / cs);
    // ELL width: the longest row rounded up to the tree's lane count (the
    // uniform loop reads whole rounds of G entries)
    const int G = A.group > 0 ? A.group : 1;
    const int W = static_cast<int>((max_row_nnz(c, A) + G - 1) / G * G);
    const size_t smem = sizeof(double) * 2 * static_cast<size_t>(n) +
                        (sizeof(double) + sizeof(int32_t)) * static_cast<size_t>(rpc) * W +
                        sizeof(int32_t) * (rpc + 1);
    if (smem > kCoSmemMax) return false;
    p.cs = cs;
    p.rpc = rpc;
    p.width = W;
    p.smem = smem;
    p.readers.alloc(n, c.stream);
    MAMG_CU(cudaMemsetAsync(p.readers.get(), 0, sizeof(uint32_t) * n, c.stream));
    k_coarsest_readers<<<blocks_for(n, 256), 256, 0, c.stream>>>(static_cast<int>(n), A.rp.get(),
                                                                  A.ci.get(), rpc, p.readers.get());
    c.count();
    MAMG_LAUNCH_CHECK();
    return true;
}

void coarsest_launch(Ctx& c, const DevCsr& A, const double* l1, const CoarsestPlan& p,
                     const double* b, double* x_out, int k, const int* gate) {
    set_kernel_attr(reinterpret_cast<const void*>(k_coarsest),
                    cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    ensure_dyn_smem(k_coarsest, kCoSmemMax);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(p.cs);
    cfg.blockDim = dim3(kCoThreads);
    cfg.dynamicSmemBytes = p.smem;
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
                               A.v.get(), l1, b, static_cast<const uint32_t*>(p.readers.get()),
                               x_out, k, A.group, p.rpc, p.width, gate));
    c.count();
}

} // namespace mamg
