// bigblock.cu — reuse of large device blocks across setups (DBuf, common.cuh).
//
// Measured on cfg 5 (elasticity 100^3): cudaMallocAsync of 0.1-0.9 GB blocks
// from the device pool took 2-700 ms of host time at irregular intervals
// (the setup then ranged 38-780 ms), although the pool kept ample free
// memory (unlimited release threshold). Freed blocks of >= kBigBlock bytes
// are therefore kept here, per stream, and handed back to a later request of
// the same stream that they fit within 25 % (stream order makes the reuse
// safe without events). The cache holds at most a fixed share of the device
// memory; it is flushed when an allocation fails and when a context's stream
// is destroyed. Only the streams of live contexts cache (big_stream_live).
#include <list>
#include <mutex>
#include <set>

#include "common.cuh"

namespace mamg {
namespace {

struct Block {
    cudaStream_t s;
    void* p;
    size_t cap;
    int dev; // device of the stream (an allocation failure frees this device's blocks)
};

struct BigCache {
    std::mutex m;
    std::list<Block> blocks; // oldest first
    size_t bytes = 0;
    size_t limit = 0;
    std::set<cudaStream_t> live; // streams whose blocks may be cached
};

BigCache& cache() {
    static BigCache c;
    return c;
}

size_t cache_limit() {
    size_t fr = 0, tot = 0;
    if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) {
        cudaGetLastError();
        return size_t{4} << 30;
    }
    return std::min<size_t>(size_t{16} << 30, tot / 8);
}

} // namespace

void* big_take(cudaStream_t s, size_t bytes, size_t* cap) {
    BigCache& c = cache();
    std::lock_guard<std::mutex> g(c.m);
    auto best = c.blocks.end();
    for (auto it = c.blocks.begin(); it != c.blocks.end(); ++it)
        if (it->s == s && it->cap >= bytes && it->cap - bytes <= bytes / 4 &&
            (best == c.blocks.end() || it->cap < best->cap))
            best = it;
    if (best == c.blocks.end()) return nullptr;
    void* p = best->p;
    *cap = best->cap;
    c.bytes -= best->cap;
    c.blocks.erase(best);
    return p;
}

bool big_put(cudaStream_t s, void* p, size_t cap) {
    BigCache& c = cache();
    std::lock_guard<std::mutex> g(c.m);
    if (c.limit == 0) c.limit = cache_limit();
    // only streams announced by big_stream_live (contexts); a block freed
    // after its stream is gone is not kept
    if (cap > c.limit || !c.live.count(s)) return false;
    int dev = -1;
    if (cudaStreamGetDevice(s, &dev) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    c.blocks.push_back({s, p, cap, dev});
    c.bytes += cap;
    while (c.bytes > c.limit) { // evict the oldest
        const Block b = c.blocks.front();
        c.blocks.pop_front();
        c.bytes -= b.cap;
        cudaFreeAsync(b.p, b.s);
    }
    return true;
}

void big_flush(cudaStream_t s, bool all) {
    BigCache& c = cache();
    std::lock_guard<std::mutex> g(c.m);
    int dev = -1;
    if (all && cudaStreamGetDevice(s, &dev) != cudaSuccess) cudaGetLastError();
    for (auto it = c.blocks.begin(); it != c.blocks.end();) {
        // all: every block of s's device (the memory an allocation there competes for)
        if (all ? it->dev == dev : it->s == s) {
            cudaFreeAsync(it->p, it->s);
            c.bytes -= it->cap;
            it = c.blocks.erase(it);
        } else {
            ++it;
        }
    }
}

void big_stream_live(cudaStream_t s, bool live) {
    if (!live) big_flush(s);
    BigCache& c = cache();
    std::lock_guard<std::mutex> g(c.m);
    if (live)
        c.live.insert(s);
    else
        c.live.erase(s);
}

void* big_alloc(cudaStream_t s, size_t bytes, size_t* cap) {
    if (void* p = big_take(s, bytes, cap)) return p;
    void* p = nullptr;
    cudaError_t e = cudaMallocAsync(&p, bytes, s);
    if (e == cudaErrorMemoryAllocation) { // cached blocks are memory too
        cudaGetLastError();
        big_flush(s, true);
        e = cudaMallocAsync(&p, bytes, s);
    }
    MAMG_CU(e);
    *cap = bytes;
    return p;
}

} // namespace mamg
