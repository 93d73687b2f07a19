// transfer.cu — host<->device staging for the end-to-end C-ABI calls.
//
// The reference API hands over pageable std::vector storage with int64
// indices. Pageable cudaMemcpy runs at ~10 GB/s; instead, T host threads each
// own two pinned chunks: a thread narrows/validates (int64 -> int32) or copies
// its next piece into one pinned buffer while the DMA of the previous piece
// (its own stream) drains the other. All arrays of a call (row_ptr, col_idx,
// values, b, w) go through ONE pass (upload_many), so the DMA queue never
// drains between arrays. Narrowing on the host also halves the index bytes
// that cross PCIe.
#include <algorithm>
#include <nmmintrin.h> // SSE4.2: streaming stores, 64-bit compares
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
        p->threads = static_cast<int>(std::min(16u, hw));
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

// One staged pass over a batch of host arrays (UpSeg list): every array is cut
// into pinned-chunk-sized pieces, the T threads pull pieces from one shared
// counter and alternate between their two pinned buffers, so the DMA queue
// never drains between arrays. Returns one validity flag per segment.
namespace {
struct Piece {
    int seg;
    size_t at, cnt;
};

// Pinned chunks are written with non-temporal (streaming) stores: no
// read-for-ownership of the destination lines and no cache pollution, which
// matters because the staging is bound by host memory bandwidth.
inline void stream_copy_f64(double* out, const double* src, size_t cnt) {
    size_t i = 0;
    if ((reinterpret_cast<uintptr_t>(out) & 15u) == 0) {
        for (; i + 2 <= cnt; i += 2)
            _mm_stream_pd(out + i, _mm_loadu_pd(src + i));
    }
    for (; i < cnt; ++i) out[i] = src[i];
}

bool convert(const UpSeg& s, size_t at, size_t cnt, void* out) {
    switch (s.kind) {
    case UpSeg::F64:
        stream_copy_f64(static_cast<double*>(out), static_cast<const double*>(s.src) + at, cnt);
        _mm_sfence();
        return true;
    case UpSeg::INDEX: {
        const int64_t* src = static_cast<const int64_t*>(s.src) + at;
        int32_t* o = static_cast<int32_t*>(out);
        const __m128i lo = _mm_set1_epi64x(s.lo), hi = _mm_set1_epi64x(s.hi);
        __m128i bad = _mm_setzero_si128();
        size_t i = 0;
        if ((reinterpret_cast<uintptr_t>(o) & 15u) == 0) {
            for (; i + 4 <= cnt; i += 4) {
                const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i));
                const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 2));
                // a < lo or a >= hi (signed 64-bit compares, SSE4.2)
                bad = _mm_or_si128(bad, _mm_or_si128(_mm_cmpgt_epi64(lo, a), _mm_cmpgt_epi64(lo, b)));
                bad = _mm_or_si128(bad, _mm_or_si128(_mm_cmpgt_epi64(hi, a) ^ _mm_set1_epi64x(-1),
                                                     _mm_cmpgt_epi64(hi, b) ^ _mm_set1_epi64x(-1)));
                // low 32-bit halves of the four int64 -> one 16-byte store
                const __m128 pa = _mm_castsi128_ps(a), pb = _mm_castsi128_ps(b);
                const __m128i packed = _mm_castps_si128(_mm_shuffle_ps(pa, pb, _MM_SHUFFLE(2, 0, 2, 0)));
                _mm_stream_si128(reinterpret_cast<__m128i*>(o + i), packed);
            }
        }
        bool good = _mm_movemask_epi8(bad) == 0;
        for (; i < cnt; ++i) {
            const int64_t a = src[i];
            good &= (a >= s.lo) & (a < s.hi);
            o[i] = static_cast<int32_t>(a);
        }
        _mm_sfence();
        return good;
    }
    case UpSeg::ROW_PTR: {
        const int64_t* src = static_cast<const int64_t*>(s.src);
        int32_t* o = static_cast<int32_t*>(out);
        bool good = true;
        int64_t prev = at == 0 ? 0 : src[at - 1];
        for (size_t i = 0; i < cnt; ++i) {
            const int64_t a = src[at + i];
            good &= (a >= prev) & (a <= s.hi);
            prev = a;
            o[i] = static_cast<int32_t>(a);
        }
        if (at == 0 && src[0] != 0) good = false;
        if (at + cnt == s.n && src[s.n - 1] != s.hi) good = false;
        return good;
    }
    }
    return false;
}

size_t out_size(const UpSeg& s) { return s.kind == UpSeg::F64 ? sizeof(double) : sizeof(int32_t); }
} // namespace

std::vector<bool> upload_many(Ctx& c, const std::vector<UpSeg>& segs) {
    std::vector<bool> result(segs.size(), true);
    StagingPool& P = pool_for(c);
    std::vector<Piece> pieces;
    for (size_t k = 0; k < segs.size(); ++k) {
        const size_t per = P.chunk / out_size(segs[k]);
        for (size_t at = 0; at < segs[k].n; at += per)
            pieces.push_back({static_cast<int>(k), at, std::min(per, segs[k].n - at)});
    }
    if (pieces.empty()) return result;
    const int T = static_cast<int>(std::min<size_t>(P.threads, pieces.size()));
    std::atomic<size_t> next{0};
    std::atomic<int> cuda_err{0};
    std::vector<std::atomic<bool>> ok(segs.size());
    for (auto& o : ok) o = true;
    auto work = [&](int t) {
        if (cudaSetDevice(c.device) != cudaSuccess) {
            cuda_err = 1;
            return;
        }
        for (int j = 0;; ++j) {
            const size_t q = next.fetch_add(1);
            if (q >= pieces.size()) break;
            const Piece& pc = pieces[q];
            const UpSeg& s = segs[pc.seg];
            const int b = 2 * t + (j & 1);
            if (j >= 2 && cudaEventSynchronize(P.events[b]) != cudaSuccess) cuda_err = 1;
            if (!convert(s, pc.at, pc.cnt, P.bufs[b])) ok[pc.seg] = false;
            const size_t es = out_size(s);
            if (cudaMemcpyAsync(static_cast<char*>(s.dst) + pc.at * es, P.bufs[b], pc.cnt * es,
                                cudaMemcpyHostToDevice, P.streams[t]) != cudaSuccess ||
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
    for (size_t k = 0; k < segs.size(); ++k) result[k] = ok[k];
    return result;
}

void upload_f64(Ctx& c, double* dst, const double* src, size_t n) {
    upload_many(c, {UpSeg{UpSeg::F64, dst, src, n, 0, 0}});
}

bool upload_index(Ctx& c, int32_t* dst, const int64_t* src, size_t n, int64_t lo, int64_t hi) {
    return upload_many(c, {UpSeg{UpSeg::INDEX, dst, src, n, lo, hi}})[0];
}

bool upload_row_ptr(Ctx& c, int32_t* dst, const int64_t* src, size_t n_plus_1, int64_t nnz) {
    return upload_many(c, {UpSeg{UpSeg::ROW_PTR, dst, src, n_plus_1, 0, nnz}})[0];
}

void download_f64(Ctx& c, double* dst, const double* src, size_t n) {
    if (n == 0) return;
    StagingPool& P = pool_for(c);
    const size_t per_chunk = P.chunk / sizeof(double);
    const size_t nchunks = (n + per_chunk - 1) / per_chunk;
    const int T = static_cast<int>(std::min<size_t>(P.threads, nchunks));
    std::atomic<int> cuda_err{0};
    c.sync(); // results produced on the context stream
    // thread t handles chunks t, t+T, ...: the DMA of its next chunk runs while
    // it copies the previous one out of the other pinned buffer
    auto work = [&](int t) {
        if (cudaSetDevice(c.device) != cudaSuccess) {
            cuda_err = 1;
            return;
        }
        size_t prev = SIZE_MAX;
        int j = 0;
        auto drain = [&](size_t q, int slot) {
            if (cudaEventSynchronize(P.events[2 * t + slot]) != cudaSuccess) cuda_err = 1;
            const size_t at = q * per_chunk, cnt = std::min(per_chunk, n - at);
            std::memcpy(dst + at, P.bufs[2 * t + slot], cnt * sizeof(double));
        };
        for (size_t q = static_cast<size_t>(t); q < nchunks; q += T, ++j) {
            const size_t at = q * per_chunk, cnt = std::min(per_chunk, n - at);
            const int slot = j & 1;
            if (cudaMemcpyAsync(P.bufs[2 * t + slot], src + at, cnt * sizeof(double),
                                cudaMemcpyDeviceToHost, P.streams[t]) != cudaSuccess ||
                cudaEventRecord(P.events[2 * t + slot], P.streams[t]) != cudaSuccess)
                cuda_err = 1;
            if (prev != SIZE_MAX) drain(prev, slot ^ 1);
            prev = q;
        }
        if (prev != SIZE_MAX) drain(prev, (j - 1) & 1);
    };
    std::vector<std::thread> th;
    for (int t = 1; t < T; ++t) th.emplace_back(work, t);
    work(0);
    for (auto& x : th) x.join();
    if (cuda_err) throw Error(MAMG_CUDA, "staged device-to-host copy failed");
}

} // namespace mamg
