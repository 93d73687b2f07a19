// microbenchmark: latency of a dependent __dadd_rn chain (cycles per add)
#include <cstdio>
__global__ void k(double* out, long long* cyc, double seed, int n) {
    double a = seed, b = seed * 0.5, c = seed * 0.25;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        a = __dadd_rn(a, b);
    }
    long long t1 = clock64();
    out[threadIdx.x] = a + c;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k3(double* out, long long* cyc, double seed, int n) {
    double a = seed, a2 = seed + 1, a3 = seed + 2, b = seed * 0.5;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        a = __dadd_rn(a, b); a2 = __dadd_rn(a2, b); a3 = __dadd_rn(a3, b);
    }
    long long t1 = clock64();
    out[threadIdx.x] = a + a2 + a3;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
    double* o; long long* c; cudaMalloc(&o, 1024 * 8); cudaMalloc(&c, 8);
    long long h;
    for (int rep = 0; rep < 2; ++rep) {
        k<<<1, 32>>>(o, c, 1.0, 2048); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("1 chain: %.2f cycles/add\n", h / 2048.0);
        k3<<<1, 32>>>(o, c, 1.0, 2048); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("3 chains: %.2f cycles/step\n", h / 2048.0);
    }
}
