// Cost of one cluster barrier (cg::cluster_group::sync) per iteration, and of
// a barrier + one DSMEM load round, for cluster sizes 2..16 and 256..1024
// threads per CTA. Timed with CUDA events over K iterations in one launch.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

template <bool Load>
__global__ void k(int iters, double* out) {
    cg::cluster_group cl = cg::this_cluster();
    __shared__ double x[1024];
    x[threadIdx.x] = threadIdx.x;
    cl.sync();
    const int me = cl.block_rank();
    const int peer = (me + 1) % cl.num_blocks();
    double* px = cl.map_shared_rank(x, peer);
    double acc = 0;
    for (int i = 0; i < iters; ++i) {
        if (Load) acc += px[(threadIdx.x + i) & 1023];
        cl.sync();
    }
    if (threadIdx.x == 0) out[blockIdx.x] = acc;
}

int main() {
    double* out;
    cudaMalloc(&out, 1 << 20);
    cudaFuncSetAttribute(k<false>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(k<true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int threads : {256, 512, 1024})
        for (int cs : {1, 2, 4, 8, 16}) {
            for (int ld = 0; ld < 2; ++ld) {
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(cs);
                cfg.blockDim = dim3(threads);
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeClusterDimension;
                at[0].val.clusterDim.x = cs;
                at[0].val.clusterDim.y = 1;
                at[0].val.clusterDim.z = 1;
                cfg.attrs = at;
                cfg.numAttrs = 1;
                const int iters = 2000;
                cudaEvent_t a, b;
                cudaEventCreate(&a);
                cudaEventCreate(&b);
                auto kern = ld ? k<true> : k<false>;
                cudaLaunchKernelEx(&cfg, kern, 10, out);
                cudaEventRecord(a);
                cudaError_t e = cudaLaunchKernelEx(&cfg, kern, iters, out);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms = 0;
                cudaEventElapsedTime(&ms, a, b);
                printf("threads %4d cluster %2d %s: %7.3f us/iter (%s)\n", threads, cs,
                       ld ? "sync+dsmem" : "sync      ", ms * 1e3 / iters, cudaGetErrorString(e));
            }
        }
    return 0;
}
