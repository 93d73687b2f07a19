// scan.cu — hand-written device-wide exclusive prefix sum (reduce-then-scan,
// 2048-element tiles of 256 threads x 8 items). Used for aggregate numbering
// (proj/src/coarsening.cpp:20-32), CSR row pointers and graph offsets.
#include <cstdlib>

#include "ops.cuh"

namespace mamg {
namespace {

constexpr int kThreads = 256;
constexpr int kItems = 8;
constexpr int kTile = kThreads * kItems;

// Block-wide exclusive scan of one int per thread; returns the block total.
__device__ int block_exclusive(int v, int& total) {
    __shared__ int warp_tot[kThreads / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[wid] = x;
    __syncthreads();
    if (wid == 0) {
        int s = lane < kThreads / 32 ? warp_tot[lane] : 0;
#pragma unroll
        for (int o = 1; o < kThreads / 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        if (lane < kThreads / 32) warp_tot[lane] = s;
    }
    __syncthreads();
    const int before = wid ? warp_tot[wid - 1] : 0;
    total = warp_tot[kThreads / 32 - 1];
    __syncthreads();
    return before + x - v;
}

// Each thread owns kItems consecutive elements of the tile.
__global__ void k_tile_scan(const int32_t* in, int64_t n, int32_t* out,
                            const int32_t* __restrict__ offsets) {
    const int64_t base = static_cast<int64_t>(blockIdx.x) * kTile + threadIdx.x * kItems;
    int vals[kItems];
    int run = 0;
#pragma unroll
    for (int j = 0; j < kItems; ++j) {
        const int64_t i = base + j;
        vals[j] = i < n ? in[i] : 0;
        run += vals[j];
    }
    int total;
    int pre = block_exclusive(run, total);
    const int off = offsets ? offsets[blockIdx.x] : 0;
    pre += off;
#pragma unroll
    for (int j = 0; j < kItems; ++j) {
        const int64_t i = base + j;
        if (i < n) out[i] = pre;
        pre += vals[j];
    }
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) out[n] = off + total;
}

// Single-pass scan with decoupled look-back: a tile takes the next tile id
// (atomic counter: tiles are processed in acquisition order, so every
// predecessor is already running), publishes its aggregate, then warp 0 walks
// back over the predecessors' status words 32 at a time — summing aggregates
// until it meets an inclusive prefix — and publishes its own inclusive
// prefix. Status word = (flag << 32) | value; flag 1 = aggregate, 2 =
// inclusive prefix; release stores / acquire loads at device scope.
__device__ __forceinline__ void st_status(unsigned long long* p, unsigned flag, int value) {
    const unsigned long long w =
        (static_cast<unsigned long long>(flag) << 32) | static_cast<uint32_t>(value);
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(w) : "memory");
}
__device__ __forceinline__ unsigned long long ld_status(const unsigned long long* p) {
    unsigned long long w;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(w) : "l"(p) : "memory");
    return w;
}

__global__ void __launch_bounds__(kThreads)
k_scan_lookback(const int32_t* in, int64_t n, int32_t* out, unsigned long long* state) {
    __shared__ int64_t s_tile;
    __shared__ int s_prefix;
    if (threadIdx.x == 0) s_tile = static_cast<int64_t>(atomicAdd(state, 1ull));
    __syncthreads();
    const int64_t t = s_tile;
    unsigned long long* status = state + 1;
    const int64_t base = t * kTile + threadIdx.x * kItems;
    int vals[kItems];
    int run = 0;
#pragma unroll
    for (int j = 0; j < kItems; ++j) {
        const int64_t i = base + j;
        vals[j] = i < n ? in[i] : 0;
        run += vals[j];
    }
    int total;
    int pre = block_exclusive(run, total);
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        if (t == 0) {
            if (lane == 0) {
                st_status(status, 2u, total);
                s_prefix = 0;
            }
        } else {
            if (lane == 0) st_status(status + t, 1u, total);
            int prefix = 0;
            int64_t j = t - 1;
            for (;;) {
                const int64_t q = j - lane;
                unsigned long long w = q >= 0 ? ld_status(status + q) : (2ull << 32);
                while (__any_sync(0xffffffffu, (w >> 32) == 0)) {
                    if ((w >> 32) == 0) w = ld_status(status + q);
                }
                const unsigned flag = static_cast<unsigned>(w >> 32);
                const unsigned m2 = __ballot_sync(0xffffffffu, flag == 2u);
                const int stop = m2 ? __ffs(m2) - 1 : 32; // nearest inclusive prefix
                int v = lane <= stop ? static_cast<int>(static_cast<uint32_t>(w)) : 0;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                prefix += v;
                if (m2) break;
                j -= 32;
            }
            if (lane == 0) {
                st_status(status + t, 2u, prefix + total);
                s_prefix = prefix;
            }
        }
    }
    __syncthreads();
    pre += s_prefix;
#pragma unroll
    for (int j = 0; j < kItems; ++j) {
        const int64_t i = base + j;
        if (i < n) out[i] = pre;
        pre += vals[j];
    }
    if (t == (n + kTile - 1) / kTile - 1 && threadIdx.x == kThreads - 1) out[n] = s_prefix + total;
}

} // namespace

void exclusive_scan_i32(Ctx& c, const int32_t* in, int32_t* out, int64_t n) {
    const int64_t tiles = (n + kTile - 1) / kTile;
    if (tiles > 1) {
        // [tile counter | status words], zeroed per scan (persistent scratch)
        auto* state = c.scratch<unsigned long long>(Ctx::kScrScan, static_cast<size_t>(tiles + 1));
        MAMG_CU(cudaMemsetAsync(state, 0, sizeof(unsigned long long) * (tiles + 1), c.stream));
        k_scan_lookback<<<static_cast<unsigned>(tiles), kThreads, 0, c.stream>>>(in, n, out, state);
        c.count();
        MAMG_LAUNCH_CHECK();
        return;
    }
    k_tile_scan<<<1, kThreads, 0, c.stream>>>(in, n, out, nullptr);
    c.count();
    MAMG_LAUNCH_CHECK();
}

namespace {
constexpr int kDeferSlots = 128; // int32 slots; counters take two
}

static int32_t* defer_slots(Ctx& c, int k) {
    if (!c.d_defer) MAMG_CU(cudaMalloc(&c.d_defer, kDeferSlots * sizeof(int32_t)));
    if (c.defer_used + k > kDeferSlots) sync_checked(c); // drains and resets the slots
    int32_t* p = static_cast<int32_t*>(c.d_defer) + c.defer_used;
    c.defer_used += k;
    return p;
}

int32_t* defer_flags(Ctx& c, int k, std::function<void(int, int32_t)> fail) {
    int32_t* p = defer_slots(c, k);
    MAMG_CU(cudaMemsetAsync(p, 0x7f, sizeof(int32_t) * k, c.stream));
    for (int j = 0; j < k; ++j)
        c.pending.push_back({p + j, 4, [fail, j](int64_t v) {
                                 if (v != kNoViolation) fail(j, static_cast<int32_t>(v));
                             }});
    return p;
}

int32_t* defer_values(Ctx& c, int k, const int32_t* init, std::function<void(int, int32_t)> take) {
    int32_t* p = defer_slots(c, k);
    MAMG_CU(cudaMemcpyAsync(p, init, sizeof(int32_t) * k, cudaMemcpyHostToDevice, c.stream));
    for (int j = 0; j < k; ++j)
        c.pending.push_back({p + j, 4, [take, j](int64_t v) { take(j, static_cast<int32_t>(v)); }});
    return p;
}

unsigned long long* defer_counter(Ctx& c, std::function<void(int64_t)> take) {
    if (c.defer_used & 1) ++c.defer_used; // 8-byte alignment
    auto* p = reinterpret_cast<unsigned long long*>(defer_slots(c, 2));
    MAMG_CU(cudaMemsetAsync(p, 0, sizeof(unsigned long long), c.stream));
    c.pending.push_back({p, 8, std::move(take)});
    return p;
}

void sync_checked(Ctx& c, const std::function<void()>& between) {
    std::vector<Ctx::Pending> todo;
    todo.swap(c.pending);
    // pinned host slots 32..63 of h_small receive the values
    const size_t m = std::min<size_t>(todo.size(), 32);
    for (size_t j = 0; j < m; ++j)
        MAMG_CU(cudaMemcpyAsync(c.h_small + 32 + j, todo[j].dev, todo[j].bytes,
                                cudaMemcpyDeviceToHost, c.stream));
    if (between) {
        if (!c.ev_read) MAMG_CU(cudaEventCreateWithFlags(&c.ev_read, cudaEventDisableTiming));
        MAMG_CU(cudaEventRecord(c.ev_read, c.stream));
        between();
        MAMG_CU(cudaEventSynchronize(c.ev_read));
    } else {
        c.sync();
    }
    c.defer_used = 0;
    for (size_t j = 0; j < m; ++j) {
        const int64_t raw = c.h_small[32 + j];
        const int64_t v = todo[j].bytes == 4 ? static_cast<int64_t>(static_cast<int32_t>(raw & 0xffffffff))
                                             : raw;
        todo[j].on_value(v);
    }
    if (todo.size() > m) { // (more than 32 pending: the rest in a second round)
        c.pending.assign(todo.begin() + static_cast<long>(m), todo.end());
        sync_checked(c);
    }
}

int64_t read_i32(Ctx& c, const int32_t* d) {
    int32_t h = 0;
    MAMG_CU(cudaMemcpyAsync(&h, d, sizeof(int32_t), cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    return h;
}

} // namespace mamg
