// micro: host->device of a 228 MB pageable array: cudaHostRegister + DMA vs plain pageable memcpy
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
int main() {
    const size_t n = 28518400, bytes = n * 8;
    std::vector<double> h(n);
    for (size_t i = 0; i < n; ++i) h[i] = (double)i;
    double* d; cudaMalloc(&d, bytes);
    cudaStream_t s; cudaStreamCreate(&s);
    for (int rep = 0; rep < 3; ++rep) {
        auto t0 = std::chrono::steady_clock::now();
        cudaHostRegister(h.data(), bytes, cudaHostRegisterDefault);
        auto t1 = std::chrono::steady_clock::now();
        cudaMemcpyAsync(d, h.data(), bytes, cudaMemcpyHostToDevice, s);
        cudaStreamSynchronize(s);
        auto t2 = std::chrono::steady_clock::now();
        cudaHostUnregister(h.data());
        auto t3 = std::chrono::steady_clock::now();
        cudaMemcpy(d, h.data(), bytes, cudaMemcpyHostToDevice);
        auto t4 = std::chrono::steady_clock::now();
        auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
        printf("register %.2f ms  dma %.2f ms (%.1f GB/s)  unregister %.2f ms | pageable memcpy %.2f ms\n",
               ms(t0, t1), ms(t1, t2), bytes / ms(t1, t2) / 1e6, ms(t2, t3), ms(t3, t4));
    }
}
