// Micro-benchmark: HBM bandwidth of many concurrent sequential streams, the
// access pattern of the blocked reductions (each 2048-element block is a
// stream consumed in order). One CTA per SM; each CTA owns NB consecutive
// blocks of each of R vectors and reads them piece by piece (PIECE doubles
// per block per step) with cp.async into a 3-stage ring, 2 pieces ahead, one
// __syncthreads per step; the consumer just sums (no dependent chain).
// Prints GB/s for several (R, NB, PIECE).
#include <cstdio>
#include <vector>

__device__ __forceinline__ void cp16(void* s, const void* g, int bytes) {
    unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(s));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(a), "l"(g), "r"(bytes) : "memory");
}

template <int R, int NB, int PIECE>
__global__ void __launch_bounds__(288, 1) k(const double* const* vec, long n, double* out) {
    extern __shared__ double ring[];
    constexpr int STRIDE = PIECE + 2, STAGE = R * NB * STRIDE, P = 2048 / PIECE;
    const int tid = threadIdx.x;
    const long b0 = static_cast<long>(blockIdx.x) * NB;
    auto issue = [&](int p) {
        double* st = ring + (p % 3) * STAGE;
        constexpr int U = R * NB * (PIECE / 2);
        for (int u = tid - 32; u < U; u += 256) {
            const int kk = u % (PIECE / 2), b = (u / (PIECE / 2)) % NB, j = u / ((PIECE / 2) * NB);
            const long i = (b0 + b) * 2048 + static_cast<long>(p) * PIECE + 2 * kk;
            cp16(st + (j * NB + b) * STRIDE + 2 * kk, vec[j] + (i < n ? i : 0), i < n ? 16 : 0);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0}; // independent sums: no dependent chain
    if (tid >= 32) { issue(0); issue(1); }
    for (int p = 0; p < P; ++p) {
        if (tid >= 32) asm volatile("cp.async.wait_group 1;" ::: "memory");
        __syncthreads();
        if (tid >= 32) {
            if (p + 2 < P) issue(p + 2);
            else asm volatile("cp.async.commit_group;" ::: "memory");
        } else if (tid < NB) {
            const double* st = ring + (p % 3) * STAGE + tid * STRIDE;
            for (int kk = 0; kk < PIECE; kk += 8)
#pragma unroll
                for (int q = 0; q < 8; ++q)
#pragma unroll
                    for (int j = 0; j < R; ++j) acc[q] += st[j * NB * STRIDE + kk + q];
        }
    }
    if (tid < NB) out[b0 + tid] = acc[0] + acc[1] + acc[2] + acc[3] + acc[4] + acc[5] + acc[6] + acc[7];
}

// plain coalesced streaming read of the same bytes (reference point)
__global__ void kplain(const double* const* vec, int R, long n, double* out) {
    double acc = 0.0;
    for (long i = blockIdx.x * 256L + threadIdx.x; i < n; i += gridDim.x * 256L)
        for (int j = 0; j < R; ++j) acc += vec[j][i];
    if (acc == 1.2345) out[0] = acc;
}

template <int R, int NB, int PIECE>
void run(const double* const* dvec, long n, double* dout) {
    const long nb = (n + 2047) / 2048;
    const int grid = static_cast<int>((nb + NB - 1) / NB);
    const size_t smem = 3ul * R * NB * (PIECE + 2) * 8;
    cudaFuncSetAttribute(k<R, NB, PIECE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int w = 0; w < 3; ++w) k<R, NB, PIECE><<<grid, 288, smem>>>(dvec, n, dout);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int r = 0; r < 20; ++r) k<R, NB, PIECE><<<grid, 288, smem>>>(dvec, n, dout);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double us = ms * 1e3 / 20;
    printf("R=%d NB=%2d PIECE=%4d grid=%4d smem=%6zu: %7.2f us  %7.1f GB/s  err=%s\n", R, NB, PIECE,
           grid, smem, us, R * n * 8.0 / us / 1e3, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    const long n = 4096000;
    std::vector<double*> v(4);
    for (auto& p : v) {
        cudaMalloc(&p, n * 8);
        cudaMemset(p, 0, n * 8);
    }
    const double** dvec;
    cudaMalloc(&dvec, 4 * sizeof(double*));
    cudaMemcpy(dvec, v.data(), 4 * sizeof(double*), cudaMemcpyHostToDevice);
    double* dout;
    cudaMalloc(&dout, 1 << 20);
    {
        for (int w = 0; w < 3; ++w) kplain<<<148 * 8, 256>>>(dvec, 4, n, dout);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a);
        for (int r = 0; r < 20; ++r) kplain<<<148 * 8, 256>>>(dvec, 4, n, dout);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("plain coalesced R=4: %.2f us %.1f GB/s\n", ms * 1e3 / 20, 4 * n * 8.0 / (ms * 1e3 / 20) / 1e3);
    }
    run<4, 14, 128>(dvec, n, dout);
    run<4, 7, 256>(dvec, n, dout);
    run<4, 4, 512>(dvec, n, dout);
    run<4, 2, 1024>(dvec, n, dout);
    run<2, 14, 128>(dvec, n, dout);
    run<2, 14, 256>(dvec, n, dout);
    run<2, 7, 512>(dvec, n, dout);
    run<1, 14, 512>(dvec, n, dout);
    run<4, 7, 128>(dvec, n, dout);
    run<4, 28, 64>(dvec, n, dout);
}
