// Raw host->device bandwidth from pinned memory: one 512 MB copy, and the
// same split into 4 MB chunks on 1, 4 and 16 streams (the staging pool's shape).
#include <cstdio>
#include <vector>
int main() {
    const size_t bytes = size_t{512} << 20, chunk = size_t{4} << 20;
    char *h, *d;
    cudaHostAlloc(&h, bytes, cudaHostAllocDefault);
    cudaMalloc(&d, bytes);
    for (size_t i = 0; i < bytes; i += 4096) h[i] = 1;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("one copy           : %.1f GB/s\n", bytes / ms / 1e6);
        for (int ns : {1, 4, 16}) {
            std::vector<cudaStream_t> s(ns);
            for (auto& x : s) cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking);
            cudaDeviceSynchronize();
            cudaEventRecord(a);
            for (size_t off = 0, k = 0; off < bytes; off += chunk, ++k)
                cudaMemcpyAsync(d + off, h + off, chunk, cudaMemcpyHostToDevice, s[k % ns]);
            for (auto& x : s) cudaStreamSynchronize(x);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b);
            printf("4 MB chunks, %2d str: %.1f GB/s\n", ns, bytes / ms / 1e6);
        }
    }
    return 0;
}
