// scan.cu — hand-written device-wide exclusive prefix sum (reduce-then-scan,
// 2048-element tiles of 256 threads x 8 items). Used for aggregate numbering
// (proj/src/coarsening.cpp:20-32), CSR row pointers and graph offsets.
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

__global__ void k_tile_reduce(const int32_t* __restrict__ in, int64_t n, int32_t* sums) {
    const int64_t base = static_cast<int64_t>(blockIdx.x) * kTile;
    int s = 0;
#pragma unroll
    for (int j = 0; j < kItems; ++j) {
        const int64_t i = base + j * kThreads + threadIdx.x;
        if (i < n) s += in[i];
    }
    int total;
    block_exclusive(s, total);
    if (threadIdx.x == 0) sums[blockIdx.x] = total;
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

} // namespace

void exclusive_scan_i32(Ctx& c, const int32_t* in, int32_t* out, int64_t n) {
    const int64_t tiles = (n + kTile - 1) / kTile;
    if (tiles <= 1) {
        k_tile_scan<<<1, kThreads, 0, c.stream>>>(in, n, out, nullptr);
        c.count();
        MAMG_LAUNCH_CHECK();
        return;
    }
    DBuf<int32_t> sums(tiles + 1, c.stream);
    k_tile_reduce<<<static_cast<unsigned>(tiles), kThreads, 0, c.stream>>>(in, n, sums.get());
    c.count();
    MAMG_LAUNCH_CHECK();
    exclusive_scan_i32(c, sums.get(), sums.get(), tiles);
    k_tile_scan<<<static_cast<unsigned>(tiles), kThreads, 0, c.stream>>>(in, n, out, sums.get());
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

unsigned long long* defer_counter(Ctx& c, std::function<void(int64_t)> take) {
    if (c.defer_used & 1) ++c.defer_used; // 8-byte alignment
    auto* p = reinterpret_cast<unsigned long long*>(defer_slots(c, 2));
    MAMG_CU(cudaMemsetAsync(p, 0, sizeof(unsigned long long), c.stream));
    c.pending.push_back({p, 8, std::move(take)});
    return p;
}

void sync_checked(Ctx& c) {
    std::vector<Ctx::Pending> todo;
    todo.swap(c.pending);
    // pinned host slots 32..63 of h_small receive the values
    const size_t m = std::min<size_t>(todo.size(), 32);
    for (size_t j = 0; j < m; ++j)
        MAMG_CU(cudaMemcpyAsync(c.h_small + 32 + j, todo[j].dev, todo[j].bytes,
                                cudaMemcpyDeviceToHost, c.stream));
    c.sync();
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
