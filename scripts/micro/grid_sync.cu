// Cost of a grid-wide barrier per iteration in one cooperative launch
// (cg::grid_group::sync) and of a hand-rolled barrier (one global arrival
// counter + generation word, release/acquire), for 148..592 CTAs.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_cg(int iters, double* out) {
    cg::grid_group g = cg::this_grid();
    double acc = 0;
    for (int i = 0; i < iters; ++i) {
        acc += out[(blockIdx.x + i) & 1023];
        g.sync();
    }
    if (threadIdx.x == 0) out[2048 + blockIdx.x] = acc;
}

__device__ __forceinline__ void my_sync(unsigned* count, volatile unsigned* gen, unsigned& mygen) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned g0 = mygen;
        __threadfence();
        if (atomicAdd(count, 1u) == gridDim.x - 1) {
            *count = 0;
            __threadfence();
            atomicExch(const_cast<unsigned*>(gen), g0 + 1);
        } else {
            while (*gen == g0) { }
        }
        __threadfence();
        mygen = g0 + 1;
    }
    __syncthreads();
}

__global__ void k_my(int iters, double* out, unsigned* count, unsigned* gen) {
    __shared__ unsigned mygen;
    if (threadIdx.x == 0) mygen = *gen;
    __syncthreads();
    unsigned mg = mygen;
    double acc = 0;
    for (int i = 0; i < iters; ++i) {
        acc += out[(blockIdx.x + i) & 1023];
        my_sync(count, gen, mg);
    }
    if (threadIdx.x == 0) out[2048 + blockIdx.x] = acc;
}

int main() {
    double* out;
    cudaMalloc(&out, 1 << 20);
    cudaMemset(out, 0, 1 << 20);
    unsigned* ctr;
    cudaMalloc(&ctr, 64);
    cudaMemset(ctr, 0, 64);
    for (int threads : {256, 512, 1024})
        for (int mult : {1, 2}) {
            const int grid = 148 * mult;
            int per_sm = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_cg, threads, 0);
            if (per_sm < mult) continue;
            const int iters = 2000;
            cudaEvent_t a, b;
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            int it0 = 10;
            void* args0[] = {&it0, &out};
            cudaLaunchCooperativeKernel((void*)k_cg, grid, threads, args0);
            int it = iters;
            void* args[] = {&it, &out};
            cudaEventRecord(a);
            cudaError_t e = cudaLaunchCooperativeKernel((void*)k_cg, grid, threads, args);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            printf("grid %3d x %4d  cg::grid.sync : %6.3f us/iter (%s)\n", grid, threads, ms * 1e3 / iters,
                   cudaGetErrorString(e));
            unsigned* gen = ctr + 8;
            void* args2[] = {&it, &out, &ctr, &gen};
            cudaEventRecord(a);
            e = cudaLaunchCooperativeKernel((void*)k_my, grid, threads, args2);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b);
            printf("grid %3d x %4d  counter+gen   : %6.3f us/iter (%s)\n", grid, threads, ms * 1e3 / iters,
                   cudaGetErrorString(e));
        }
    return 0;
}
