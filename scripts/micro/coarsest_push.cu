// Micro-benchmark for the one-launch coarsest solve (coarsest.cu): where does
// a sweep's time go? A 16-CTA cluster x 512 threads, one row per thread, rows
// staged in shared memory (transposed ELL), K sweeps per launch. The matrix is
// /tmp/coarsest.bin (scripts/micro/dump_coarsest.py: the cfg-2 coarsest level
// of the reference hierarchy) or, without it, a 7-point 16x16x17 grid.
//   mode 0: compute + per-thread pushes (st.shared::cluster) + cluster barrier
//   mode 1: compute + cluster barrier (no pushes)
//   mode 2: per-thread pushes + cluster barrier (no compute)
//   mode 3: cluster barrier only
//   mode 4: compute + __syncthreads + coalesced block pushes to neighbours + barrier
//   mode 5: compute only (no barrier, no pushes)
#include <cooperative_groups.h>
#include <algorithm>
#include <cstdio>
#include <vector>
namespace cg = cooperative_groups;

constexpr int T = 512;

__device__ __forceinline__ void push_remote(double* p, int rank, double val) {
    uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(p)), ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
    asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(ra), "d"(val) : "memory");
}
__device__ __forceinline__ void cbar() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__global__ void __launch_bounds__(T, 1) k(int n, const int* rp, const int* ci, const double* v,
                                         const double* d, double* out, int K, int rpc, int W,
                                         int mode, int* stats) {
    extern __shared__ double X[];
    double* sv = X + 2 * n;
    int* sci = reinterpret_cast<int*>(sv + rpc * W);
    __shared__ unsigned rmask[T];
    __shared__ unsigned nbr;
    cg::cluster_group cl = cg::this_cluster();
    const int me = cl.block_rank();
    const int t = threadIdx.x;
    const int i = me * rpc + t;
    const bool mine = t < rpc && i < n;
    int* srp = sci + rpc * W;
    const int r0 = me * rpc, nr = max(0, min(rpc, n - r0));
    for (int u = t; u <= nr; u += T) srp[u] = rp[r0 + u];
    __syncthreads();
    const int e0 = srp[0], ne = srp[nr] - e0;
    for (int e = t; e < ne; e += T) {
        int lo = 0, hi = nr - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (srp[mid] - e0 <= e) lo = mid; else hi = mid - 1;
        }
        const int j = e - (srp[lo] - e0);
        sci[j * rpc + lo] = ci[e0 + e];
        sv[j * rpc + lo] = v[e0 + e];
    }
    int m = 0;
    double bi = 1.0, di = 1;
    if (mine) {
        m = srp[t + 1] - srp[t];
        for (int j = m; j < W; ++j) { sci[j * rpc + t] = i; sv[j * rpc + t] = 0.0; }
        di = d[i];
    }
    const int mw = __reduce_max_sync(0xffffffffu, m);
    rmask[t] = 0;
    if (t == 0) nbr = 0;
    cbar();
    if (mine)
        for (int j = 0; j < m; ++j) {
            int c = sci[j * rpc + t];
            int q = c / rpc;
            if (q != me) {
                atomicOr(cl.map_shared_rank(rmask + (c - q * rpc), q), 1u << me);
                atomicOr(&nbr, 1u << q);
            }
        }
    cbar();
    const unsigned readers = mine ? rmask[t] : 0;
    const unsigned nb = nbr;
    if (stats && mine) {
        atomicAdd(stats, __popc(readers));
        if (t == 0) atomicAdd(stats + 1, __popc(nb));
    }
    double val = 0;
    for (int s = 0; s < K; ++s) {
        const double* xin = X + ((s + 1) & 1) * n;
        double* xo = X + (s & 1) * n;
        if (mine) {
            if (mode == 2 || mode == 3) {
                val = bi;
            } else {
                double l[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) l[j] = 0.0;
                for (int base = 0; base < mw; base += 8) {
                    double p[8];
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        p[j] = __dmul_rn(sv[(base + j) * rpc + t], xin[sci[(base + j) * rpc + t]]);
#pragma unroll
                    for (int j = 0; j < 8; ++j) l[j] = base + j < m ? __dadd_rn(l[j], p[j]) : l[j];
                }
#pragma unroll
                for (int o = 4; o > 0; o >>= 1)
#pragma unroll
                    for (int j = 0; j < o; ++j) l[j] = __dadd_rn(l[j], l[j + o]);
                val = s == 0 ? __ddiv_rn(bi, di) : __dadd_rn(xin[i], __ddiv_rn(__dsub_rn(bi, l[0]), di));
            }
            xo[i] = val;
            if ((mode == 0 || mode == 2) && s < K - 1)
                for (unsigned r = readers; r; r &= r - 1) push_remote(xo + i, __ffs(r) - 1, val);
        }
        if (mode == 4 && s < K - 1) {
            __syncthreads();
            const int lo = me * rpc, cnt = min(rpc, n - lo);
            for (unsigned r = nb; r; r &= r - 1) {
                const int q = __ffs(r) - 1;
                double* dst = cl.map_shared_rank(xo, q);
                for (int u = t; u < cnt; u += T) dst[lo + u] = xo[lo + u];
            }
        }
        if (s < K - 1 && mode != 5) cbar();
    }
    if (mine) out[i] = val;
}

int main() {
    setvbuf(stdout, nullptr, _IONBF, 0);
    int n;
    std::vector<int> rp{0}, ci;
    std::vector<double> v, dg;
    if (FILE* f = fopen("/tmp/coarsest.bin", "rb")) {
        long long hdr[2];
        if (fread(hdr, 8, 2, f) != 2) return 1;
        n = static_cast<int>(hdr[0]);
        rp.resize(n + 1);
        ci.resize(hdr[1]);
        v.resize(hdr[1]);
        dg.resize(n);
        size_t got = fread(rp.data(), 4, n + 1, f) + fread(ci.data(), 4, hdr[1], f) +
                     fread(v.data(), 8, hdr[1], f) + fread(dg.data(), 8, n, f);
        fclose(f);
        printf("matrix: /tmp/coarsest.bin n=%d nnz=%lld (read %zu)\n", n, hdr[1], got);
    } else {
        const int nx = 16, ny = 16, nz = 17;
        n = nx * ny * nz;
        for (int z = 0; z < nz; ++z)
            for (int y = 0; y < ny; ++y)
                for (int x = 0; x < nx; ++x) {
                    int i = (z * ny + y) * nx + x;
                    int nb[7] = {i - nx * ny, i - nx, i - 1, i, i + 1, i + nx, i + nx * ny};
                    bool ok[7] = {z > 0, y > 0, x > 0, true, x < nx - 1, y < ny - 1, z < nz - 1};
                    for (int j = 0; j < 7; ++j)
                        if (ok[j]) {
                            ci.push_back(nb[j]);
                            v.push_back(nb[j] == i ? 6.0 : -1.0);
                        }
                    rp.push_back(ci.size());
                }
        dg.assign(n, 12.0);
        printf("matrix: 7-point 16x16x17 n=%d\n", n);
    }
    int W = 0;
    for (int i = 0; i < n; ++i) W = std::max(W, rp[i + 1] - rp[i]);
    W = (W + 7) / 8 * 8;
    int *drp, *dci, *dstats;
    double *dv, *dd, *dout;
    cudaMalloc(&drp, rp.size() * 4);
    cudaMalloc(&dci, ci.size() * 4);
    cudaMalloc(&dv, v.size() * 8);
    cudaMalloc(&dd, n * 8);
    cudaMalloc(&dout, n * 8);
    cudaMalloc(&dstats, 8);
    cudaMemset(dstats, 0, 8);
    cudaMemcpy(drp, rp.data(), rp.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dci, ci.data(), ci.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dv, v.data(), v.size() * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dd, dg.data(), n * 8, cudaMemcpyHostToDevice);
    const int cs = 16, rpc = (n + cs - 1) / cs;
    const size_t smem = 2 * n * 8 + (size_t)rpc * W * 12 + 4 * (rpc + 1);
    printf("rpc=%d W=%d smem=%zu\n", rpc, W, smem);
    cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int mode : {0, 1, 2, 3, 4, 5}) {
        for (int K : {1, 20}) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(cs);
            cfg.blockDim = dim3(T);
            cfg.dynamicSmemBytes = smem;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = cs;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            int* st = (mode == 0 && K == 1) ? dstats : nullptr;
            cudaError_t e = cudaLaunchKernelEx(&cfg, k, n, (const int*)drp, (const int*)dci,
                                               (const double*)dv, (const double*)dd, dout, K, rpc,
                                               W, mode, st);
            if (e != cudaSuccess || (e = cudaDeviceSynchronize()) != cudaSuccess) {
                printf("mode %d: %s\n", mode, cudaGetErrorString(e));
                return 1;
            }
            if (st) {
                int h[2];
                cudaMemcpy(h, dstats, 8, cudaMemcpyDeviceToHost);
                printf("pushes per sweep (all CTAs): %d, neighbour CTAs: %d\n", h[0], h[1]);
            }
            for (int w = 0; w < 5; ++w)
                cudaLaunchKernelEx(&cfg, k, n, (const int*)drp, (const int*)dci, (const double*)dv,
                                   (const double*)dd, dout, K, rpc, W, mode, (int*)nullptr);
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0);
            const int R = 200;
            for (int r = 0; r < R; ++r)
                cudaLaunchKernelEx(&cfg, k, n, (const int*)drp, (const int*)dci, (const double*)dv,
                                   (const double*)dd, dout, K, rpc, W, mode, (int*)nullptr);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            printf("mode %d K %2d: %.2f us/launch  err=%s\n", mode, K, ms * 1e3 / R,
                   cudaGetErrorString(cudaGetLastError()));
        }
    }
}
