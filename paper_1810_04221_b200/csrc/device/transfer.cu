// transfer.cu — host<->device staging for the end-to-end C-ABI calls.
//
// The reference API hands over pageable std::vector storage with int64
// indices. Pageable cudaMemcpy runs at ~10 GB/s; instead, T host threads each
// own a slice of the array and two pinned chunks: a thread narrows/validates
// (int64 -> int32) or copies its next chunk into one pinned buffer while the
// DMA of the previous chunk (its own stream) drains the other. Narrowing on
// the host also halves the index bytes that cross PCIe.
#include <algorithm>
#include <atomic>
#include <cstring>
#include <thread>
#include <vector>

#include "ops.cuh"

namespace mamg {

struct StagingPool {
    int threads = 0;
    size_t chunk = 0; // bytes per pinned buffer
    std::vector<void*> bufs;       // 2 per thread
    std::vector<cudaStream_t> streams;
    std::vector<cudaEvent_t> events; // 2 per thread
    ~StagingPool() {
        for (void* p : bufs) cudaFreeHost(p);
        for (auto s : streams) cudaStreamDestroy(s);
        for (auto e : events) cudaEventDestroy(e);
    }
};

static StagingPool& pool_for(Ctx& c) {
    if (!c.staging) {
        auto* p = new StagingPool;
        const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
        p->threads = static_cast<int>(std::min(12u, hw));
        p->chunk = size_t{4} << 20;
        for (int t = 0; t < p->threads; ++t) {
            cudaStream_t s;
            MAMG_CU(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
            p->streams.push_back(s);
            for (int k = 0; k < 2; ++k) {
                void* b = nullptr;
                MAMG_CU(cudaHostAlloc(&b, p->chunk, cudaHostAllocDefault));
                p->bufs.push_back(b);
                cudaEvent_t e;
                MAMG_CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
                p->events.push_back(e);
            }
        }
        c.staging = p;
        c.staging_free = [](void* q) { delete static_cast<StagingPool*>(q); };
    }
    return *static_cast<StagingPool*>(c.staging);
}

// Generic staged upload: conv(src_index_begin, count, dst_chunk, thread) fills
// a pinned chunk of D; returns false to flag invalid input.
template <class D, class Conv>
static bool staged_upload(Ctx& c, D* dst, size_t n, Conv conv) {
    if (n == 0) return true;
    StagingPool& P = pool_for(c);
    const size_t per_chunk = P.chunk / sizeof(D);
    const int T = static_cast<int>(std::min<size_t>(P.threads, (n + per_chunk - 1) / per_chunk));
    std::atomic<bool> ok{true};
    std::atomic<int> cuda_err{0};
    auto work = [&](int t) {
        if (cudaSetDevice(c.device) != cudaSuccess) {
            cuda_err = 1;
            return;
        }
        const size_t lo = n * t / T, hi = n * (t + 1) / T;
        int j = 0;
        for (size_t at = lo; at < hi; at += per_chunk, ++j) {
            const size_t cnt = std::min(per_chunk, hi - at);
            const int b = 2 * t + (j & 1);
            if (j >= 2 && cudaEventSynchronize(P.events[b]) != cudaSuccess) cuda_err = 1;
            if (!conv(at, cnt, static_cast<D*>(P.bufs[b]))) ok = false;
            if (cudaMemcpyAsync(dst + at, P.bufs[b], cnt * sizeof(D), cudaMemcpyHostToDevice,
                                P.streams[t]) != cudaSuccess ||
                cudaEventRecord(P.events[b], P.streams[t]) != cudaSuccess)
                cuda_err = 1;
        }
        if (cudaStreamSynchronize(P.streams[t]) != cudaSuccess) cuda_err = 1;
    };
    std::vector<std::thread> th;
    for (int t = 1; t < T; ++t) th.emplace_back(work, t);
    work(0);
    for (auto& x : th) x.join();
    if (cuda_err) throw Error(MAMG_CUDA, "staged host-to-device copy failed");
    return ok;
}

void upload_f64(Ctx& c, double* dst, const double* src, size_t n) {
    staged_upload<double>(c, dst, n, [&](size_t at, size_t cnt, double* out) {
        std::memcpy(out, src + at, cnt * sizeof(double));
        return true;
    });
}

bool upload_index(Ctx& c, int32_t* dst, const int64_t* src, size_t n, int64_t lo, int64_t hi) {
    return staged_upload<int32_t>(c, dst, n, [&](size_t at, size_t cnt, int32_t* out) {
        bool good = true;
        for (size_t i = 0; i < cnt; ++i) {
            const int64_t a = src[at + i];
            good &= (a >= lo) & (a < hi);
            out[i] = static_cast<int32_t>(a);
        }
        return good;
    });
}

bool upload_row_ptr(Ctx& c, int32_t* dst, const int64_t* src, size_t n_plus_1, int64_t nnz) {
    return staged_upload<int32_t>(c, dst, n_plus_1, [&](size_t at, size_t cnt, int32_t* out) {
        bool good = true;
        int64_t prev = at == 0 ? 0 : src[at - 1];
        for (size_t i = 0; i < cnt; ++i) {
            const int64_t a = src[at + i];
            good &= (a >= prev) & (a <= nnz);
            prev = a;
            out[i] = static_cast<int32_t>(a);
        }
        if (at == 0 && src[0] != 0) good = false;
        if (at + cnt == n_plus_1 && src[n_plus_1 - 1] != nnz) good = false;
        return good;
    });
}

void download_f64(Ctx& c, double* dst, const double* src, size_t n) {
    if (n == 0) return;
    StagingPool& P = pool_for(c);
    const size_t per_chunk = P.chunk / sizeof(double);
    const int T = static_cast<int>(std::min<size_t>(P.threads, (n + per_chunk - 1) / per_chunk));
    std::atomic<int> cuda_err{0};
    c.sync(); // results produced on the context stream
    auto work = [&](int t) {
        if (cudaSetDevice(c.device) != cudaSuccess) {
            cuda_err = 1;
            return;
        }
        const size_t lo = n * t / T, hi = n * (t + 1) / T;
        for (size_t at = lo; at < hi; at += per_chunk) {
            const size_t cnt = std::min(per_chunk, hi - at);
            void* buf = P.bufs[2 * t];
            if (cudaMemcpyAsync(buf, src + at, cnt * sizeof(double), cudaMemcpyDeviceToHost,
                                P.streams[t]) != cudaSuccess ||
                cudaStreamSynchronize(P.streams[t]) != cudaSuccess)
                cuda_err = 1;
            std::memcpy(dst + at, buf, cnt * sizeof(double));
        }
    };
    std::vector<std::thread> th;
    for (int t = 1; t < T; ++t) th.emplace_back(work, t);
    work(0);
    for (auto& x : th) x.join();
    if (cuda_err) throw Error(MAMG_CUDA, "staged device-to-host copy failed");
}

} // namespace mamg
