// common.cuh — shared infrastructure of the sm_100a AMG library: error
// handling, stream-ordered device buffers, the device CSR type and the
// IEEE-exact arithmetic helpers every parity-critical kernel uses.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <functional>
#include <utility>
#include <vector>
#include <vector>

#include "mamg_capi.h"

namespace mamg {

// Internal error carrying the C-ABI status and the offending index.
struct Error : std::runtime_error {
    int status;
    int64_t index;
    Error(int s, const std::string& m, int64_t idx = -1)
        : std::runtime_error(m), status(s), index(idx) {}
};

[[noreturn]] inline void throw_cuda(cudaError_t e, const char* what, const char* file,
                                    int line) {
    throw Error(MAMG_CUDA, std::string("CUDA error ") + cudaGetErrorString(e) + " in " +
                               what + " at " + file + ":" + std::to_string(line));
}

#define MAMG_CU(x)                                                          \
    do {                                                                    \
        cudaError_t e_ = (x);                                               \
        if (e_ != cudaSuccess) ::mamg::throw_cuda(e_, #x, __FILE__, __LINE__); \
    } while (0)

inline void invalid(const std::string& msg, int64_t idx = -1) {
    throw Error(MAMG_INVALID_ARGUMENT, msg, idx);
}

// Large blocks (>= kBigBlock bytes) are recycled per stream (bigblock.cu):
// big_alloc takes a cached block that fits or allocates from the pool,
// big_put keeps a freed one (false: too large for the cache, free it),
// big_flush frees the cached blocks of a stream (or, all = true, of every
// stream on the same device).
constexpr size_t kBigBlock = size_t{32} << 20;
void* big_alloc(cudaStream_t s, size_t bytes, size_t* cap);
bool big_put(cudaStream_t s, void* p, size_t cap);
void big_flush(cudaStream_t s, bool all = false);
// a context's stream starts / stops caching (stop: its cached blocks are freed)
void big_stream_live(cudaStream_t s, bool live);

// Stream-ordered device buffer (cudaMallocAsync / cudaFreeAsync on the
// owning stream; the device pool keeps freed blocks cached between setups).
template <class T>
class DBuf {
public:
    DBuf() = default;
    DBuf(size_t n, cudaStream_t s) { alloc(n, s); }
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    DBuf(DBuf&& o) noexcept { *this = std::move(o); }
    DBuf& operator=(DBuf&& o) noexcept {
        if (this != &o) {
            release();
            p_ = o.p_;
            n_ = o.n_;
            s_ = o.s_;
            cap_ = o.cap_;
            o.p_ = nullptr;
            o.n_ = 0;
            o.cap_ = 0;
        }
        return *this;
    }
    ~DBuf() { release(); }

    void alloc(size_t n, cudaStream_t s) {
        release();
        s_ = s;
        n_ = n;
        // +32 bytes of tail padding: TMA bulk copies round ranges up to 16 B
        const size_t bytes = n * sizeof(T) + 32;
        cap_ = 0;
        if (n == 0) return;
        if (bytes >= kBigBlock)
            p_ = static_cast<T*>(big_alloc(s, bytes, &cap_));
        else
            MAMG_CU(cudaMallocAsync(reinterpret_cast<void**>(&p_), bytes, s));
    }
    void release() {
        if (p_ && !(cap_ >= kBigBlock && big_put(s_, p_, cap_))) cudaFreeAsync(p_, s_);
        p_ = nullptr;
        n_ = 0;
        cap_ = 0;
    }
    T* get() const { return p_; }
    size_t size() const { return n_; }
    // the caller frees the block with cudaFreeAsync (never cached)
    T* release_ownership() {
        T* p = p_;
        p_ = nullptr;
        n_ = 0;
        cap_ = 0;
        return p;
    }

private:
    T* p_ = nullptr;
    size_t n_ = 0;
    cudaStream_t s_ = nullptr;
    size_t cap_ = 0; // bytes of the block (large blocks go back to the cache)
};

// Device CSR: int32 row pointers and columns, fp64 values. `group` caches
// LaneGroupPolicy::for_matrix (proj/src/kernels.cpp:11-24), which fixes the
// SpMV summation order; `single` marks one entry per row (prolongators).
struct DevCsr {
    int64_t nrows = 0, ncols = 0, nnz = 0;
    DBuf<int32_t> rp, ci;
    DBuf<double> v;
    int group = 2;
    bool single = false;
    bool finite = true; // every value finite (enables the x=0 sweep shortcut)
    int max_tile = -1;  // entries of the longest 256-row tile (SpMV staging plan; -1 unknown)
};

// Lane policy from the shape (the `single` flag must already be known).
inline int lane_policy_from(int64_t nrows, int64_t nnz, bool single) {
    if (nrows > 0 && nnz == nrows && single) return 1;
    const double mean = nrows > 0 ? static_cast<double>(nnz) / static_cast<double>(nrows) : 0.0;
    for (int g = 2; g <= 32; g *= 2)
        if (static_cast<double>(g) >= mean) return g;
    return 32;
}

struct Ctx {
    int device = 0;
    int num_sms = 148;
    cudaStream_t stream = nullptr;
    std::string err;
    int64_t err_index = -1;
    int64_t launches = 0;
    // pinned host scratch for small readbacks
    int64_t* h_small = nullptr; // 64 int64 slots
    DBuf<int64_t> d_small;      // 64 int64 slots of device scratch
    // pinned staging ring for host<->device transfers (transfer.cu)
    void* staging = nullptr;
    void (*staging_free)(void*) = nullptr;

    // Persistent device scratch for the setup's big temporaries (edge
    // weights, Suitor candidates and words, Galerkin contributions): grown to
    // the high-water mark and reused across steps and setups, so a setup does
    // not allocate and free GBs per step (the stream-ordered pool then
    // occasionally had to map new memory: 0.5-0.9 s stalls measured on cfg 5).
    enum Scratch { kScrWeights, kScrCand, kScrCandN, kScrSuitor, kScrProdCol, kScrProdVal,
                   kScrScan, kScrPark, kScrSlots };
    void* scr_p[kScrSlots] = {};
    size_t scr_n[kScrSlots] = {};
    template <class T>
    T* scratch(int slot, size_t n) {
        const size_t bytes = n * sizeof(T) + 32;
        if (scr_n[slot] < bytes) {
            if (scr_p[slot]) MAMG_CU(cudaFreeAsync(scr_p[slot], stream));
            const size_t nb = bytes + bytes / 8;
            MAMG_CU(cudaMallocAsync(&scr_p[slot], nb, stream));
            scr_n[slot] = nb;
        }
        return static_cast<T*>(scr_p[slot]);
    }
    void release_scratch() {
        for (int k = 0; k < kScrSlots; ++k) {
            if (scr_p[k]) cudaFreeAsync(scr_p[k], stream);
            scr_p[k] = nullptr;
            scr_n[k] = 0;
        }
    }

    // Deferred device checks (setup): a kernel records a violation (lowest
    // row / aggregate, INT32_MAX = none) or a counter in device memory; the
    // host reads all pending values at the NEXT readback it needs anyway
    // (sync_checked) and raises the first violation in registration order —
    // the reference's order — instead of a synchronisation per check.
    struct Pending {
        const void* dev;
        int bytes; // 4 (int32 flag) or 8 (uint64 counter)
        std::function<void(int64_t)> on_value;
    };
    std::vector<Pending> pending;
    void* d_defer = nullptr; // device slots for deferred flags / counters
    int defer_used = 0;      // int32 slots handed out since the last check
    cudaEvent_t ev_read = nullptr; // marks the readback copies (sync_checked with work between)

    void count(int64_t k = 1) { launches += k; }
    void sync() { MAMG_CU(cudaStreamSynchronize(stream)); }
};

// Grid size helpers
inline unsigned blocks_for(int64_t work, int per_block) {
    return static_cast<unsigned>((work + per_block - 1) / per_block);
}

#define MAMG_LAUNCH_CHECK() MAMG_CU(cudaGetLastError())

// Programmatic dependent launch (sm_90+): a kernel launched with launch_pdl
// may start while its predecessor drains; it must call pdl_wait() before it
// touches anything the predecessor wrote (the wait returns once the
// predecessor grid has completed and its writes are visible). pdl_trigger()
// lets the successor launch early. Both are no-ops for ordinary launches.
// MAMG_NO_PDL=1 turns the attribute off (A/B).
bool pdl_enabled();

// Kernel attributes apply to the CURRENT device only: set `attr` = `value`
// on kernel `fn` once per (device, kernel, attribute), raising it when a
// larger value is asked for (thread-safe; solve.cu).
void set_kernel_attr(const void* fn, cudaFuncAttribute attr, int value);
template <class K>
inline void ensure_dyn_smem(K* kernel, size_t bytes) {
    set_kernel_attr(reinterpret_cast<const void*>(kernel), cudaFuncAttributeMaxDynamicSharedMemorySize,
                    static_cast<int>(bytes));
}

template <class... KArgs, class... Args>
inline void launch_pdl(cudaStream_t s, void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    MAMG_CU(cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...));
}

} // namespace mamg

// ---- IEEE-exact arithmetic (no contraction; the library is also built with
// -fmad=false). Every parity-critical expression uses these. -----------------
// CTA-wide barrier reached from different code paths (warp-uniform
// branches): the non-aligned form of bar.sync 0 (PTX barrier.sync), which
// unlike __syncthreads allows the threads to execute different barrier
// instructions
__device__ __forceinline__ void cta_barrier_divergent() {
    asm volatile("barrier.sync 0;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" :::); }
__device__ __forceinline__ double rn_add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double rn_sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double rn_mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double rn_div(double a, double b) { return __ddiv_rn(a, b); }
