// solve.cu — the solve phase on sm_100a: blocked deterministic reductions
// (proj/src/vector_ops.cpp), the V/W multigrid cycle (proj/src/multigrid.cpp)
// and the reordered flexible PCG (proj/src/krylov.cpp), with the whole PCG
// iteration device-resident and replayed as a CUDA graph.
//
// Bit-exact reductions: the reference sums each 2048-element block
// sequentially from 0.0 and folds the block partials pairwise with the odd
// tail carried (vector_ops.cpp:12-44). Here a warp owns a block: its 32 lanes
// stream the block in coalesced 128-element chunks (loads for chunk c+1 are
// in flight while lane 0 runs the serial add chain of chunk c out of shared
// memory), and a single CTA folds the partials in shared memory in the
// reference's tree order. Consumers that produce the reduced vector (the
// second PCG axpy pair -> ||r||, the audit residual) are fused into the same
// pass.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <type_traits>
#include <mutex>
#include <tuple>
#include <unordered_map>
#include <vector>

#include "ops.cuh"
#include "dist.cuh"

namespace mamg {

void set_kernel_attr(const void* fn, cudaFuncAttribute attr, int value) {
    static std::mutex mu;
    static std::map<std::tuple<int, const void*, int>, int> set;
    int dev = 0;
    MAMG_CU(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    const auto key = std::make_tuple(dev, fn, static_cast<int>(attr));
    auto it = set.find(key);
    if (it != set.end() && it->second >= value) return;
    MAMG_CU(cudaFuncSetAttribute(fn, attr, value));
    set[key] = value;
}

bool pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("MAMG_NO_PDL");
        return !(e && e[0] == '1');
    }();
    return on;
}

struct PcgState {
    double norm_b, rho, alpha, t, step, rtol;
    double audit_max_rel, bd_rho;
    long long it, itmax, audit_checks, audit_failures, bd_it;
    int done, status, no_audit, pad;
    double* hist;
};

namespace {

constexpr int kBlock = 256;
constexpr int64_t kRedBlock = 2048; // vector_ops.cpp:12

// ------------------------------------------------------------- chain ops --
struct OpDot {
    const double* __restrict__ x;
    const double* __restrict__ y;
    struct V {
        double a, b;
    };
    __device__ void init() {}
    __device__ V load(int64_t i) const { return V{x[i], y[i]}; }
    __device__ void apply(int64_t, const V& s, double (&p)[1]) const { p[0] = rn_mul(s.a, s.b); }
};

struct OpPair { // (w.r, w.v)
    const double* __restrict__ w;
    const double* __restrict__ r;
    const double* __restrict__ v;
    struct V {
        double w, r, v;
    };
    __device__ void init() {}
    __device__ V load(int64_t i) const { return V{w[i], r[i], v[i]}; }
    __device__ void apply(int64_t, const V& s, double (&p)[2]) const {
        p[0] = rn_mul(s.w, s.r);
        p[1] = rn_mul(s.w, s.v);
    }
};

struct OpTriple { // vector_ops.cpp:69-74
    const double* __restrict__ w;
    const double* __restrict__ r;
    const double* __restrict__ v;
    const double* __restrict__ q;
    struct V {
        double w, r, v, q;
    };
    __device__ void init() {}
    __device__ V load(int64_t i) const { return V{w[i], r[i], v[i], q[i]}; }
    __device__ void apply(int64_t, const V& s, double (&p)[3]) const {
        p[0] = rn_mul(s.w, s.r);
        p[1] = rn_mul(s.w, s.v);
        p[2] = rn_mul(s.w, s.q);
    }
};

// y += a x with ||y||^2 partials (krylov.cpp:107 + :109)
struct OpAxpyNorm {
    double* y;
    const double* __restrict__ x;
    const PcgState* st; // a = -st->step when st != nullptr
    double a;
    struct V {
        double y, x;
    };
    double c = 0.0; // the coefficient, read once per thread (init)
    __device__ void init() { c = st ? -st->step : a; }
    __device__ V load(int64_t i) const { return V{y[i], x[i]}; }
    __device__ void apply(int64_t i, const V& s, double (&p)[1]) const {
        const double ny = rn_add(s.y, rn_mul(c, s.x));
        y[i] = ny;
        p[0] = rn_mul(ny, ny);
    }
};

// fused_axpy_pair(v, r, q, -t, -step) + ||r||^2 partials (krylov.cpp:129-134)
struct OpPcgPair2 {
    double* y1;
    double* y2;
    const double* __restrict__ x;
    const PcgState* st;
    struct V {
        double y1, y2, x;
    };
    // the PCG scalars, read once per thread (init): read per element they
    // were reloaded after every store (y1 / y2 may alias st)
    double mt = 0.0, ms = 0.0;
    __device__ void init() {
        mt = -st->t;
        ms = -st->step;
    }
    __device__ V load(int64_t i) const { return V{y1[i], y2[i], x[i]}; }
    __device__ void apply(int64_t i, const V& s, double (&p)[1]) const {
        const double tt = rn_add(s.y1, rn_mul(mt, s.x));
        y1[i] = tt;
        const double ny = rn_add(s.y2, rn_mul(ms, tt));
        y2[i] = ny;
        p[0] = rn_mul(ny, ny);
    }
};

// audit residual r - (b - A u) (krylov.cpp:31-35)
struct OpAudit {
    const double* __restrict__ r;
    const double* __restrict__ b;
    const double* __restrict__ au;
    struct V {
        double r, b, au;
    };
    __device__ void init() {}
    __device__ V load(int64_t i) const { return V{r[i], b[i], au[i]}; }
    __device__ void apply(int64_t, const V& s, double (&p)[1]) const {
        const double d = rn_sub(s.r, rn_sub(s.b, s.au));
        p[0] = rn_mul(d, d);
    }
};

// One CTA = 1 chain warp + 8 producer warps and owns kBPC consecutive
// 2048-element blocks. Producers stream the blocks in 256-element pieces
// (coalesced: piece e of all kBPC blocks) and write the products into a
// double-buffered shared tile; lanes 0..kBPC-1 of warp 0 each run one
// block's strictly sequential add chain (vector_ops.cpp:39-41) over the
// previous piece. Partials go to global memory; the last CTA to finish
// folds them in the reference's pairwise order (vector_ops.cpp:16-25) and
// runs the epilogue, so a reduction is a single launch.
constexpr int kBPC = 8;                  // 2048-blocks per CTA
constexpr int kPiece = 256;              // elements per block per piece
constexpr int kPieces = kRedBlock / kPiece;
constexpr int kTileStride = kPiece + 2;  // padding: chain lanes' 16 B reads hit distinct banks
constexpr int kDotThreads = 32 + kPiece; // warp 0 chains, warps 1..8 produce

template <int NV>
constexpr int dot_tile_doubles() { return 2 * NV * kBPC * kTileStride; }

// pairwise fold with the odd tail carried (vector_ops.cpp:16-25) in shared
// memory: level l reads one region and writes the other (no in-place
// hazard); buf holds m + ceil(m / 2) doubles, the input in the first m.
template <int T>
__device__ double fold_smem(double* buf, int64_t m) {
    double* src = buf;
    double* dst = buf + m;
    while (m > 1) {
        const int64_t half = m / 2, outm = (m + 1) / 2;
        for (int64_t i = threadIdx.x; i < outm; i += T)
            dst[i] = i < half ? rn_add(src[2 * i], src[2 * i + 1]) : src[m - 1];
        __syncthreads();
        double* t = src;
        src = dst;
        dst = t;
        m = outm;
    }
    return src[0];
}

// Fold of any number of partials, get(i) = partial i. The pairwise tree
// with the odd tail carried has aligned subtrees: after L levels over chunks
// of C = 2^L partials, element i is the same fold of chunk i alone (chunk
// boundaries stay even for every level below L, so the tail carry of the
// last, partial chunk is its own). So the fold of m > C partials = the fold
// of the chunks' folds: one CTA folds chunk after chunk in shared memory,
// keeps the chunk results, then folds them — no length limit short of C^2.
// buf: fold_doubles(m) doubles.
constexpr int64_t kFoldChunk = 4096;
__host__ __device__ constexpr int64_t fold_doubles(int64_t m) {
    return m <= kFoldChunk ? (m > 0 ? m : 1) * 3 / 2 + 2
                           : kFoldChunk * 3 / 2 + 2 + ((m + kFoldChunk - 1) / kFoldChunk) * 3 / 2 + 2;
}

template <int T, class Get>
__device__ double fold_any(double* buf, int64_t m, Get get) {
    if (m <= 0) return 0.0;
    if (m <= kFoldChunk) {
        for (int64_t i = threadIdx.x; i < m; i += T) buf[i] = get(i);
        __syncthreads();
        const double r = fold_smem<T>(buf, m);
        __syncthreads();
        return r;
    }
    double* res = buf + kFoldChunk * 3 / 2 + 2;
    const int64_t nch = (m + kFoldChunk - 1) / kFoldChunk;
    for (int64_t ch = 0; ch < nch; ++ch) {
        const int64_t lo = ch * kFoldChunk;
        const int64_t cnt = m - lo < kFoldChunk ? m - lo : kFoldChunk;
        for (int64_t i = threadIdx.x; i < cnt; i += T) buf[i] = get(lo + i);
        __syncthreads();
        const double r = fold_smem<T>(buf, cnt);
        __syncthreads();
        if (threadIdx.x == 0) res[ch] = r;
    }
    __syncthreads();
    const double r = fold_smem<T>(res, nch);
    __syncthreads();
    return r;
}

// Partitioned reductions with the allgather fused in (peer memory): every
// rank's gathered-partials buffer (two parities) and arrival counter are
// mapped into every rank (CUDA IPC over NVLink; the parts' own buffers for
// the loopback). world == 0: write the partials to `part` (no peer output).
struct PeerOut {
    int world = 0, me = 0;
    double* gath[kMaxWorld] = {};                // each rank's buffer base
    unsigned long long* arrive[kMaxWorld] = {}; // each rank's arrival counter
    const unsigned long long* epoch = nullptr;  // this rank's completed reductions
    int64_t rstride = 0; // a rank's segment inside one parity (NV * nbmax)
    int64_t pstride = 0; // one parity (world * 3 * nbmax)
};

template <int NV, class Op, class Epi, bool Fold = true>
__global__ void __launch_bounds__(kDotThreads, 2)
k_blockdot(int64_t n, Op op_in, Epi epi, double* part, int64_t nb, unsigned* counter,
           const int* __restrict__ gate, const PeerOut po) {
    pdl_wait();
    // a gated (finished-solve) peer reduction still signals its arrival so
    // every rank's fold stays in step; it computes and sends nothing
    const bool gated = gate && *gate;
    if (gated && po.world == 0) return;
    extern __shared__ __align__(16) double tile[]; // [2][NV][kBPC][kTileStride], reused by the fold
    __shared__ bool last;
    const int tid = threadIdx.x;
    const int64_t b0 = static_cast<int64_t>(blockIdx.x) * kBPC;
    const int nblk = static_cast<int>(nb - b0 < kBPC ? nb - b0 : kBPC);
    double acc[NV];
#pragma unroll
    for (int c = 0; c < NV; ++c) acc[c] = 0.0;
    auto T = [&](int buf, int c, int blk, int e) -> double& {
        return tile[((buf * NV + c) * kBPC + blk) * kTileStride + e];
    };
    // Warp 0 (chains) and warps 1..8 (producers) run separate loops with the
    // same barrier sequence (kPieces + 1 barriers each, the branch is
    // warp-uniform), so their register live ranges do not overlap. The two
    // loops reach the barrier from different instructions: the non-aligned
    // `barrier.sync` (not __syncthreads' aligned form, undefined there).
    if (gated) {
        // (peer reduction past the end of the solve: signal only)
    } else if (tid >= 32) {
        // producers keep the operands of the next piece in registers so their
        // loads are in flight across the barrier
        typename Op::V cur[kBPC];
        Op op = op_in;
        op.init();
        const int e = tid - 32;
        auto load_piece = [&](int p) {
#pragma unroll
            for (int blk = 0; blk < kBPC; ++blk) {
                const int64_t i = (b0 + blk) * kRedBlock + p * kPiece + e;
                if (blk < nblk && i < n) cur[blk] = op.load(i);
            }
        };
        load_piece(0);
        for (int p = 0; p <= kPieces; ++p) {
            if (p < kPieces) {
#pragma unroll
                for (int blk = 0; blk < kBPC; ++blk) {
                    const int64_t i = (b0 + blk) * kRedBlock + p * kPiece + e;
                    if (blk < nblk && i < n) {
                        double pr[NV];
                        op.apply(i, cur[blk], pr);
#pragma unroll
                        for (int c = 0; c < NV; ++c) T(p & 1, c, blk, e) = pr[c];
                    }
                }
                if (p + 1 < kPieces) load_piece(p + 1);
            }
            cta_barrier_divergent();
        }
    } else {
        for (int p = 0; p <= kPieces; ++p) {
            if (tid < nblk && p > 0) {
                const int q = p - 1;
                const int64_t lo = (b0 + tid) * kRedBlock + q * kPiece;
                const int cnt = lo >= n ? 0 : static_cast<int>(n - lo < kPiece ? n - lo : kPiece);
                if (cnt == kPiece) {
                    // full piece: 16-byte shared loads, two register batches
                    // ping-ponged so the next batch is in flight while the
                    // current one feeds the (8-cycle DADD latency) chain
                    constexpr int B = NV == 3 ? 4 : 8; // doubles per batch (register budget)
                    double2 ba[NV][B / 2], bb[NV][B / 2];
                    auto ld = [&](double2 (&dst)[NV][B / 2], int k) {
#pragma unroll
                        for (int c = 0; c < NV; ++c)
#pragma unroll
                            for (int j = 0; j < B / 2; ++j)
                                dst[c][j] = *reinterpret_cast<const double2*>(&T(q & 1, c, tid, k + 2 * j));
                    };
                    auto add = [&](const double2 (&src)[NV][B / 2]) {
#pragma unroll
                        for (int j = 0; j < B / 2; ++j) {
#pragma unroll
                            for (int c = 0; c < NV; ++c) acc[c] = rn_add(acc[c], src[c][j].x);
#pragma unroll
                            for (int c = 0; c < NV; ++c) acc[c] = rn_add(acc[c], src[c][j].y);
                        }
                    };
                    ld(ba, 0);
#pragma unroll 1
                    for (int k = 0; k < kPiece; k += 2 * B) {
                        ld(bb, k + B);
                        add(ba);
                        if (k + 2 * B < kPiece) ld(ba, k + 2 * B);
                        add(bb);
                    }
                } else {
                    for (int k = 0; k < cnt; ++k) {
#pragma unroll
                        for (int c = 0; c < NV; ++c) acc[c] = rn_add(acc[c], T(q & 1, c, tid, k));
                    }
                }
            }
            cta_barrier_divergent();
        }
    }
    if (po.world > 0) {
        // fused allgather: this rank's partials straight into every rank's
        // buffer (parity = completed reductions mod 2), then the last CTA
        // signals each rank's arrival counter (system scope)
        const int64_t base = (static_cast<int64_t>(*po.epoch & 1ull)) * po.pstride +
                             static_cast<int64_t>(po.me) * po.rstride;
        if (tid < nblk && !gated) {
            for (int r = 0; r < po.world; ++r) {
                double* dst = po.gath[r] + base;
#pragma unroll
                for (int c = 0; c < NV; ++c) dst[c * nb + b0 + tid] = acc[c];
            }
        }
        __syncthreads(); // then one cumulative system fence per CTA
        if (tid == 0) {
            __threadfence_system();
            last = atomicAdd(counter, 1u) == gridDim.x - 1;
        }
        __syncthreads();
        if (last && tid == 0) {
            __threadfence_system();
            for (int r = 0; r < po.world; ++r) atomicAdd_system(po.arrive[r], 1ull);
            *counter = 0u;
        }
        pdl_trigger();
        return;
    }
    if (tid < nblk) {
#pragma unroll
        for (int c = 0; c < NV; ++c) part[c * nb + b0 + tid] = acc[c];
    }
    pdl_trigger();
    if constexpr (!Fold) return; // partitioned runs fold after the allgather
    __threadfence();
    __syncthreads();
    if (tid == 0) last = atomicAdd(counter, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    double res[NV];
    for (int c = 0; c < NV; ++c)
        res[c] = fold_any<kDotThreads>(tile, nb, [&](int64_t i) { return __ldcg(part + c * nb + i); });
    if (tid == 0) {
        epi(res);
        *counter = 0u; // ready for the next launch (graph replay)
    }
}

// Fold of already-gathered partials (partitioned runs: every rank folds the
// rank-ordered concatenation, i.e. the unpartitioned partial array).
template <int NV, class Epi>
__global__ void __launch_bounds__(kDotThreads)
k_fold_epi(const double* __restrict__ part, int64_t nb, Epi epi, const int* __restrict__ gate) {
    if (gate && *gate) return;
    extern __shared__ __align__(16) double buf[];
    double res[NV];
    for (int c = 0; c < NV; ++c)
        res[c] = fold_any<kDotThreads>(buf, nb, [&](int64_t i) { return part[c * nb + i]; });
    if (threadIdx.x == 0) epi(res);
}

// The partitioned fold: the ranks' partial arrays arrive padded (rank r's
// NV x nb_r partials at r * rstride, component c at + c * nb_r); block i of
// the global order is rank r's block i - roff[r]. Same fold as k_fold_epi.
template <int NV, class Epi>
__global__ void __launch_bounds__(kDotThreads)
k_fold_seg(const double* __restrict__ g, const int64_t* __restrict__ roff, int world,
           int64_t rstride, int64_t nb, Epi epi, const int* __restrict__ gate) {
    if (gate && *gate) return;
    extern __shared__ __align__(16) double buf[];
    double res[NV];
    for (int c = 0; c < NV; ++c)
        res[c] = fold_any<kDotThreads>(buf, nb, [&](int64_t i) {
            int r = 0;
            while (r + 1 < world && i >= roff[r + 1]) ++r;
            const int64_t nbr = roff[r + 1] - roff[r];
            return g[r * rstride + c * nbr + (i - roff[r])];
        });
    if (threadIdx.x == 0) epi(res);
}

// The fold of a fused peer reduction: wait (bounded) until every rank has
// signalled this reduction, fold the gathered partials of the current parity
// like k_fold_seg, advance the local reduction count. A wait that exceeds the
// bound sets *err (the solve then fails loudly instead of hanging).
template <int NV, class Epi>
__global__ void __launch_bounds__(kDotThreads)
k_fold_peer(const double* __restrict__ gath, const int64_t* __restrict__ roff, int world,
            int64_t rstride, int64_t pstride, int64_t nb, unsigned long long* arrive,
            unsigned long long* epoch, unsigned long long* err, Epi epi, const int* __restrict__ gate) {
    extern __shared__ __align__(16) double buf[];
    __shared__ unsigned long long ep;
    if (threadIdx.x == 0) {
        ep = *epoch;
        const unsigned long long target = (ep + 1) * static_cast<unsigned long long>(world);
        long long spins = 0;
        for (;;) {
            unsigned long long a;
            asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(a) : "l"(arrive) : "memory");
            if (a >= target) break;
            if (++spins > (1ll << 26)) { // ~7 s
                atomicExch(err, 1ull);
                break;
            }
            __nanosleep(100);
        }
    }
    __syncthreads();
    const double* g = gath + static_cast<int64_t>(ep & 1ull) * pstride;
    if (!(gate && *gate)) {
        double res[NV];
        for (int c = 0; c < NV; ++c)
            res[c] = fold_any<kDotThreads>(buf, nb, [&](int64_t i) {
                int r = 0;
                while (r + 1 < world && i >= roff[r + 1]) ++r;
                const int64_t nbr = roff[r + 1] - roff[r];
                return __ldcg(g + r * rstride + c * nbr + (i - roff[r]));
            });
        if (threadIdx.x == 0) epi(res);
    }
    if (threadIdx.x == 0) *epoch = ep + 1;
}

// ------------------------------------------------------------- epilogues --
template <int NV>
struct EpiOut {
    double* out;
    __device__ void operator()(const double (&r)[NV]) const {
        for (int c = 0; c < NV; ++c) out[c] = r[c];
    }
};
struct EpiNormB {
    PcgState* st;
    __device__ void operator()(const double (&r)[1]) const {
        st->norm_b = sqrt(r[0]);
        if (st->norm_b == 0.0) st->done = 1;
    }
};
// first residual norm (krylov.cpp:88-93)
struct EpiHist0 {
    PcgState* st;
    __device__ void operator()(const double (&r)[1]) const {
        const double h = sqrt(r[0]);
        st->hist[0] = h;
        if (rn_div(h, st->norm_b) <= st->rtol) st->done = 1;
    }
};
// alpha, rho of the first step (krylov.cpp:100-105)
struct EpiInit {
    PcgState* st;
    __device__ void operator()(const double (&r)[2]) const {
        st->alpha = r[0];
        st->rho = r[1];
        if (!isfinite(r[0]) || !isfinite(r[1]) || r[1] <= 0.0) {
            st->status = MAMG_BREAKDOWN;
            st->bd_it = 0;
            st->bd_rho = r[1];
            st->done = 1;
            return;
        }
        st->step = rn_div(r[0], r[1]);
    }
};
// scalars of the reordered iteration (krylov.cpp:115-125)
struct EpiTriple {
    PcgState* st;
    __device__ void operator()(const double (&r)[3]) const {
        const double wr = r[0], wv = r[1], wq = r[2];
        st->alpha = wr;
        const double rho_next = rn_sub(wv, rn_div(rn_mul(wq, wq), st->rho));
        if (!isfinite(wr) || !isfinite(wv) || !isfinite(wq) || !isfinite(rho_next) ||
            rho_next <= 0.0) {
            st->status = MAMG_BREAKDOWN;
            st->bd_it = st->it;
            st->bd_rho = rho_next;
            st->done = 1;
            return;
        }
        st->t = rn_div(wq, st->rho);
        st->step = rn_div(wr, rho_next);
        st->rho = rho_next;
    }
};
// ++iterations; history; loop test (krylov.cpp:111, :133-135)
struct EpiHistNext {
    PcgState* st;
    __device__ void operator()(const double (&r)[1]) const {
        const long long it = st->it + 1;
        st->it = it;
        const double h = sqrt(r[0]);
        st->hist[it] = h;
        const double rel = rn_div(h, st->norm_b);
        if (!(rel > st->rtol) || it >= st->itmax) st->done = 1;
        st->no_audit = (it % 50 != 0);
    }
};
// residual-recurrence audit (krylov.cpp:35-38)
struct EpiAudit {
    PcgState* st;
    __device__ void operator()(const double (&r)[1]) const {
        const double rel = rn_div(sqrt(r[0]), st->norm_b);
        st->audit_checks += 1;
        if (rel > st->audit_max_rel) st->audit_max_rel = rel;
        if (rel > 1e-10) st->audit_failures += 1;
        st->no_audit = 1;
    }
};

// ------------------------------------------------------------ K-cycle --
// Scalars of one level's two-step flexible CG (Notay & Vassilevski's
// K-cycle, the north star's "K-cycle driver"; not in the reference, so this
// definition is pinned by the oracle port, oracle/matchamg_oracle.c
// orc_kcycle_coarse).
struct KState {
    double rho1, s1, gamma, a1, a2;
    int ok1, skip2, two, pad;
};
struct OpSq2 { // (x.x, y.y)
    const double* __restrict__ x;
    const double* __restrict__ y;
    struct V {
        double x, y;
    };
    __device__ void init() {}
    __device__ V load(int64_t i) const { return V{x[i], y[i]}; }
    __device__ void apply(int64_t, const V& s, double (&p)[2]) const {
        p[0] = rn_mul(s.x, s.x);
        p[1] = rn_mul(s.y, s.y);
    }
};
// (c1.v1, c1.bc) -> rho1, s1 = alpha1 / rho1
struct EpiK1 {
    KState* ks;
    __device__ void operator()(const double (&r)[2]) const {
        ks->rho1 = r[0];
        ks->ok1 = r[0] > 0.0;
        ks->s1 = ks->ok1 ? rn_div(r[1], r[0]) : 0.0;
    }
};
// (rt.rt, bc.bc): second step unless ||rt|| <= 0.25 ||bc|| (or rho1 <= 0)
struct EpiK2 {
    KState* ks;
    __device__ void operator()(const double (&r)[2]) const {
        ks->skip2 = (!ks->ok1 || sqrt(r[0]) <= rn_mul(0.25, sqrt(r[1]))) ? 1 : 0;
    }
};
// (c2.v1, c2.v2, c2.rt) -> rho2 = beta - gamma^2 / rho1, a2, a1
struct EpiK3 {
    KState* ks;
    __device__ void operator()(const double (&r)[3]) const {
        const double gamma = r[0], beta = r[1], alpha2 = r[2];
        const double rho2 = rn_sub(beta, rn_div(rn_mul(gamma, gamma), ks->rho1));
        ks->two = rho2 > 0.0;
        if (!ks->two) return;
        const double a2 = rn_div(alpha2, rho2);
        ks->gamma = gamma;
        ks->a2 = a2;
        ks->a1 = rn_sub(ks->s1, rn_div(rn_mul(gamma, a2), ks->rho1));
    }
};
// skip flag of the second branch starts as the parent's gate
__global__ void k_kgate(int* skip2, const int* __restrict__ parent) {
    pdl_wait();
    *skip2 = (parent && *parent) ? 1 : 0;
}
// rt = bc + (-s1) v1 ; xc = ok1 ? 0.0 + s1 c1 : 0.0
__global__ void k_kstep1(int64_t n, const double* __restrict__ bc, const double* __restrict__ v1,
                         const double* __restrict__ c1, double* rt, double* xc,
                         const KState* ks, const int* __restrict__ gate) {
    pdl_wait();
    if (gate && *gate) return;
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double s1 = ks->s1;
    rt[i] = rn_add(bc[i], rn_mul(-s1, v1[i]));
    xc[i] = ks->ok1 ? rn_add(0.0, rn_mul(s1, c1[i])) : 0.0;
}
// xc = (0.0 + a1 c1) + a2 c2 when the second step is taken and rho2 > 0
__global__ void k_kstep2(int64_t n, const double* __restrict__ c1, const double* __restrict__ c2,
                         double* xc, const KState* ks, const int* __restrict__ gate) {
    pdl_wait();
    if ((gate && *gate) || !ks->two) return;
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    xc[i] = rn_add(rn_add(0.0, rn_mul(ks->a1, c1[i])), rn_mul(ks->a2, c2[i]));
}

// ------------------------------------------------------ elementwise kernels --
__global__ void k_axpy(int64_t n, double* y, double a, const double* __restrict__ x,
                       const int* __restrict__ gate) {
    pdl_wait();
    if (gate && *gate) return;
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) y[i] = rn_add(y[i], rn_mul(a, x[i]));
}
// u += step d with step on the device (krylov.cpp:106)
__global__ void k_axpy_step(int64_t n, double* y, const double* __restrict__ x,
                            const PcgState* st, const int* __restrict__ gate) {
    pdl_wait();
    if (gate && *gate) return;
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) y[i] = rn_add(y[i], rn_mul(st->step, x[i]));
}
// vector_ops.cpp:86-91
__global__ void k_axpy_pair(int64_t n, double* y1, double* y2, const double* __restrict__ x,
                            double a, double b) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double t = rn_add(y1[i], rn_mul(a, x[i]));
    y1[i] = t;
    y2[i] = rn_add(y2[i], rn_mul(b, t));
}
// fused_axpy_pair(w, u, d, -t, step) (krylov.cpp:127)
__global__ void k_pcg_pair1(int64_t n, double* w, double* u, const double* __restrict__ d,
                            const PcgState* st, const int* __restrict__ gate) {
    pdl_wait();
    if (gate && *gate) return;
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double t = rn_add(w[i], rn_mul(-st->t, d[i]));
    w[i] = t;
    u[i] = rn_add(u[i], rn_mul(st->step, t));
}
__global__ void k_copy(int64_t n, double* dst, const double* __restrict__ src,
                       const int* __restrict__ gate) {
    pdl_wait();
    if (gate && *gate) return;
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) dst[i] = src[i];
}
__global__ void k_fill(int64_t n, double* dst, double v, const int* __restrict__ gate) {
    pdl_wait();
    if (gate && *gate) return;
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) dst[i] = v;
}

// ------------------------------------------------------ reduction drivers --
int64_t nblocks(int64_t n) { return (n + kRedBlock - 1) / kRedBlock; }

// Scratch of one reduction site: NV * nb partials + the completion counter.
struct RedScratch {
    DBuf<double> part;
    DBuf<unsigned> counter;
    void ensure(Ctx& c, int64_t need) {
        if (part.size() < static_cast<size_t>(need)) part.alloc(need, c.stream);
        if (!counter.get()) {
            counter.alloc(1, c.stream);
            MAMG_CU(cudaMemsetAsync(counter.get(), 0, sizeof(unsigned), c.stream));
        }
    }
};

template <int NV, class Op, class Epi>
void reduce(Ctx& c, int64_t n, const Op& op, const Epi& epi, RedScratch& s, const int* gate) {
    const int64_t nb = nblocks(n);
    s.ensure(c, NV * (nb > 0 ? nb : 1));
    const int grid = static_cast<int>(nb > 0 ? (nb + kBPC - 1) / kBPC : 1);
    const size_t smem =
        sizeof(double) * std::max<int64_t>(dot_tile_doubles<NV>(), fold_doubles(nb));
    auto kernel = k_blockdot<NV, Op, Epi>;
    ensure_dyn_smem(kernel, smem);
    launch_pdl(c.stream, kernel, dim3(grid), dim3(kDotThreads), smem, n, op, epi, s.part.get(), nb,
               s.counter.get(), gate, PeerOut{});
    c.count();
    MAMG_LAUNCH_CHECK();
}

unsigned eblocks(int64_t n) { return blocks_for(n > 0 ? n : 1, kBlock); }

} // namespace

// K-cycle workspace of level k (vectors of level k + 1)
struct KWork {
    DBuf<double> c1, c2, v1, v2, rt;
    DBuf<KState> ks;
    RedScratch red;
};


// ================================================================= vectors ==
double dot(Ctx& c, int64_t n, const double* x, const double* y) {
    RedScratch s;
    double* out = reinterpret_cast<double*>(c.d_small.get() + 16);
    reduce<1>(c, n, OpDot{x, y}, EpiOut<1>{out}, s, nullptr);
    double h = 0.0;
    MAMG_CU(cudaMemcpyAsync(&h, out, sizeof(double), cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    return h;
}

void triple_dot(Ctx& c, int64_t n, const double* w, const double* r, const double* v,
                const double* q, double* out3) {
    RedScratch s;
    double* out = reinterpret_cast<double*>(c.d_small.get() + 16);
    reduce<3>(c, n, OpTriple{w, r, v, q}, EpiOut<3>{out}, s, nullptr);
    MAMG_CU(cudaMemcpyAsync(out3, out, 3 * sizeof(double), cudaMemcpyDeviceToHost, c.stream));
    c.sync();
}

void axpy(Ctx& c, int64_t n, double* y, double a, const double* x, const int* gate) {
    if (n == 0) return;
    launch_pdl(c.stream, k_axpy, dim3(eblocks(n)), dim3(kBlock), 0, n, y, a, x, gate);
    c.count();
    MAMG_LAUNCH_CHECK();
}

void axpy_pair(Ctx& c, int64_t n, double* y1, double* y2, const double* x, double a, double b) {
    if (n == 0) return;
    k_axpy_pair<<<eblocks(n), kBlock, 0, c.stream>>>(n, y1, y2, x, a, b);
    c.count();
    MAMG_LAUNCH_CHECK();
}

// ================================================================== cycles ==
static void copy_vec(Ctx& c, int64_t n, double* dst, const double* src, const int* gate) {
    if (n == 0) return;
    launch_pdl(c.stream, k_copy, dim3(eblocks(n)), dim3(kBlock), 0, n, dst, src, gate);
    c.count();
}
static void fill_vec(Ctx& c, int64_t n, double* dst, double v, const int* gate) {
    if (n == 0) return;
    launch_pdl(c.stream, k_fill, dim3(eblocks(n)), dim3(kBlock), 0, n, dst, v, gate);
    c.count();
}

// k l1-Jacobi sweeps (multigrid.cpp:52-61). The start is `src` (or zero when
// src == nullptr) and the result lands in `dst`; intermediate iterates live
// in the level's two work buffers, assigned backwards from `dst` so that no
// sweep reads the vector it writes. A sweep from zero on a finite matrix is
// x = 0 + b/d exactly (A*0 sums to +0).
static void sweeps(Ctx& c, DevLevel& L, const double* b, const double* src, double* dst, int k,
                   const int* gate) {
    const DevCsr& A = *L.A;
    const int64_t n = A.nrows;
    double* xa = L.xw.get();
    double* xb = L.scratch.get();
    if (k == 0) {
        if (src == nullptr)
            fill_vec(c, n, dst, 0.0, gate);
        else if (src != dst)
            copy_vec(c, n, dst, src, gate);
        return;
    }
    std::vector<double*> out(static_cast<size_t>(k));
    auto plan = [&](double* before_last) {
        out[k - 1] = dst;
        double* cur = before_last;
        for (int j = k - 2; j >= 0; --j) {
            out[j] = cur;
            cur = (cur == xa) ? xb : xa;
        }
    };
    const bool dst_in_pair = (dst == xa || dst == xb);
    plan(dst == xa ? xb : (dst == xb ? xa : xb));
    if (k >= 2 && src != nullptr && out[0] == src) {
        if (dst_in_pair) throw Error(MAMG_RUNTIME, "sweeps: no buffer assignment");
        plan(xa);
    }
    const double* cur = src;
    for (int j = 0; j < k; ++j) {
        double* o = out[j];
        if (cur == nullptr) {
            if (A.finite) {
                smooth_from_zero(c, n, L.l1.get(), b, o, gate);
            } else {
                double* z = (o == xa) ? xb : xa;
                fill_vec(c, n, z, 0.0, gate);
                smooth_sweep(c, A, L.l1.get(), b, z, o, gate);
            }
        } else {
            smooth_sweep(c, A, L.l1.get(), b, cur, o, gate);
        }
        cur = o;
    }
}

static void cycle_rec(Ctx& c, DevHier& h, int k, const mamg_cycle_cfg& cfg, const double* b,
                      double* x_out, bool x_zero, const int* gate);

// K-cycle coarse correction of level k: cx solves A_{k+1} cx = cb by two
// steps of flexible CG preconditioned with the K-cycle of level k + 1
// (Notay & Vassilevski 2008). The second step is skipped on the device when
// ||rt|| <= 0.25 ||cb||: its kernels take the level's skip flag as gate.
static void kcycle_coarse(Ctx& c, DevHier& h, int k, const mamg_cycle_cfg& cfg, const int* gate) {
    DevLevel& L = h.lv[k];
    DevLevel& C = h.lv[k + 1];
    const int64_t m = C.A->nrows;
    if (!L.kw) {
        auto w = std::make_shared<KWork>();
        w->c1.alloc(m, c.stream);
        w->c2.alloc(m, c.stream);
        w->v1.alloc(m, c.stream);
        w->v2.alloc(m, c.stream);
        w->rt.alloc(m, c.stream);
        w->ks.alloc(1, c.stream);
        MAMG_CU(cudaMemsetAsync(w->ks.get(), 0, sizeof(KState), c.stream));
        w->red.ensure(c, 3 * (nblocks(m) > 0 ? nblocks(m) : 1));
        L.kw = std::move(w);
    }
    KWork& W = *L.kw;
    KState* ks = W.ks.get();
    int* skip2 = &ks->skip2;
    const double* bc = L.cb.get();
    double* xc = L.cx.get();
    // step 1: c1 = K(bc), v1 = A c1, rho1 = c1.v1, s1 = (c1.bc) / rho1
    cycle_rec(c, h, k + 1, cfg, bc, W.c1.get(), true, gate);
    spmv(c, *C.A, C.A->group, W.c1.get(), W.v1.get(), gate);
    reduce<2>(c, m, OpPair{W.c1.get(), W.v1.get(), bc}, EpiK1{ks}, W.red, gate);
    if (m) {
        launch_pdl(c.stream, k_kstep1, dim3(eblocks(m)), dim3(kBlock), 0, m, bc,
                   static_cast<const double*>(W.v1.get()), static_cast<const double*>(W.c1.get()),
                   W.rt.get(), xc, static_cast<const KState*>(ks), gate);
        c.count();
    }
    launch_pdl(c.stream, k_kgate, dim3(1), dim3(1), 0, skip2, gate);
    c.count();
    reduce<2>(c, m, OpSq2{W.rt.get(), bc}, EpiK2{ks}, W.red, gate);
    // step 2 (gated): c2 = K(rt), v2 = A c2, (gamma, beta, alpha2), combination
    cycle_rec(c, h, k + 1, cfg, W.rt.get(), W.c2.get(), true, skip2);
    spmv(c, *C.A, C.A->group, W.c2.get(), W.v2.get(), skip2);
    reduce<3>(c, m, OpTriple{W.c2.get(), W.v1.get(), W.v2.get(), W.rt.get()}, EpiK3{ks}, W.red,
              skip2);
    if (m) {
        launch_pdl(c.stream, k_kstep2, dim3(eblocks(m)), dim3(kBlock), 0, m,
                   static_cast<const double*>(W.c1.get()), static_cast<const double*>(W.c2.get()), xc,
                   static_cast<const KState*>(ks), static_cast<const int*>(skip2));
        c.count();
    }
    MAMG_LAUNCH_CHECK();
}

static void cycle_rec(Ctx& c, DevHier& h, int k, const mamg_cycle_cfg& cfg, const double* b,
                      double* x_out, bool x_zero, const int* gate) {
    DevLevel& L = h.lv[k];
    const int64_t n = L.A->nrows;
    if (k == h.nl() - 1) {
        // coarsest: x = 0, then coarsest_sweeps sweeps (multigrid.cpp:82-88);
        // x_out is written only by the last sweep so it may double as input
        if (h.coarsest.cs > 0)
            coarsest_launch(c, *L.A, L.l1.get(), h.coarsest, b, x_out, cfg.coarsest_sweeps, gate);
        else
            sweeps(c, L, b, nullptr, x_out, cfg.coarsest_sweeps, gate);
        return;
    }
    double* xw = L.xw.get();
    // pre-smoothing into the working vector
    if (cfg.pre_sweeps == 0) {
        if (x_zero)
            fill_vec(c, n, xw, 0.0, gate);
        else
            copy_vec(c, n, xw, x_out, gate);
    } else {
        // the intermediate iterates must not overwrite xw before the last
        // sweep: sweeps() only writes xw as the final destination or as a
        // buffer different from the current source.
        sweeps(c, L, b, x_zero ? nullptr : x_out, xw, cfg.pre_sweeps, gate);
    }
    // fresh residual, restricted (multigrid.cpp:93-99)
    residual(c, *L.A, b, xw, L.scratch.get(), gate);
    spmv(c, *L.R, L.R->group, L.scratch.get(), L.cb.get(), gate);
    if (cfg.cycle == 2 && k + 2 < h.nl()) {
        kcycle_coarse(c, h, k, cfg, gate);
    } else {
        const int visits = cfg.cycle == 1 ? 2 : 1;
        for (int t = 0; t < visits; ++t)
            cycle_rec(c, h, k + 1, cfg, L.cb.get(), L.cx.get(), t == 0, gate);
    }
    // prolongate and correct (multigrid.cpp:105-106)
    if (L.P->single) {
        prolong_correct(c, *L.P, L.cx.get(), xw, gate);
    } else {
        spmv(c, *L.P, L.P->group, L.cx.get(), L.scratch.get(), gate);
        axpy(c, n, xw, 1.0, L.scratch.get(), gate);
    }
    // post-smoothing from xw into x_out
    if (cfg.post_sweeps == 0) {
        copy_vec(c, n, x_out, xw, gate);
    } else {
        // sweeps() alternates between xw and scratch; with src == xw the
        // intermediates use scratch, never xw as a destination before src is read
        sweeps(c, L, b, xw, x_out, cfg.post_sweeps, gate);
    }
}

void apply_cycle(Ctx& c, DevHier& h, int level, const mamg_cycle_cfg& cfg, const double* b,
                 double* x, bool x_is_zero, const int* gate) {
    if (level < 0 || level >= h.nl())
        invalid("apply_cycle: level " + std::to_string(level) + " outside [0, " +
                std::to_string(h.nl()) + ")");
    if (cfg.pre_sweeps < 0 || cfg.post_sweeps < 0)
        invalid("CycleConfig: sweep counts must be >= 0");
    if (cfg.coarsest_sweeps < 1) invalid("CycleConfig: coarsest_sweeps must be >= 1");
    if (cfg.cycle < 0 || cfg.cycle > 2) invalid("CycleConfig: unknown cycle type");
    cycle_rec(c, h, level, cfg, b, x, x_is_zero, gate);
    MAMG_LAUNCH_CHECK();
}

void l1_jacobi(Ctx& c, const DevCsr& A, const double* d, const double* b, double* x, int k) {
    if (k <= 0 || A.nrows == 0) return;
    DBuf<double> tmp(A.nrows, c.stream);
    double* cur = x;
    double* other = tmp.get();
    for (int s = 0; s < k; ++s) {
        smooth_sweep(c, A, d, b, cur, other);
        std::swap(cur, other);
    }
    if (cur != x) copy_vec(c, A.nrows, x, cur, nullptr);
    MAMG_LAUNCH_CHECK();
}

// =================================================================== PCG ==
namespace {

struct PcgBufs {
    int64_t n;
    DBuf<double> r, w, d, v, q, hist;
    DBuf<PcgState> st;
    RedScratch red;
};

} // namespace

int pcg_solve(Ctx& c, const DevCsr& A, DevHier* h, const mamg_cycle_cfg* cyc,
              mamg_host_precond hp, void* user, const double* b, const double* u0,
              const mamg_solve_cfg& cfg, double* u, double* hist_out, mamg_report* rep) {
    using clock = std::chrono::steady_clock;
    const auto t0 = clock::now();
    if (!(cfg.rtol > 0.0)) invalid("SolveConfig: rtol must be > 0");
    if (cfg.itmax < 1) invalid("SolveConfig: itmax must be >= 1");
    if (A.nrows != A.ncols) invalid("pcg_solve: matrix is not square");
    if (h) {
        if (!cyc) invalid("pcg_solve: cycle configuration missing");
        if (h->lv[0].A->nrows != A.nrows) invalid("pcg_solve: dimension mismatch");
        if (cyc->pre_sweeps < 0 || cyc->post_sweeps < 0)
            invalid("CycleConfig: sweep counts must be >= 0");
        if (cyc->coarsest_sweeps < 1) invalid("CycleConfig: coarsest_sweeps must be >= 1");
        if (cyc->cycle < 0 || cyc->cycle > 2) invalid("CycleConfig: unknown cycle type");
    }
    const int64_t n = A.nrows;
    std::memset(rep, 0, sizeof(*rep));
    rep->breakdown_iteration = -1;

    PcgBufs B;
    B.n = n;
    B.r.alloc(n, c.stream);
    B.w.alloc(n, c.stream);
    B.d.alloc(n, c.stream);
    B.v.alloc(n, c.stream);
    B.q.alloc(n, c.stream);
    B.hist.alloc(cfg.itmax + 2, c.stream);
    B.st.alloc(1, c.stream);
    {
        // reduction scratch sized up front: nothing may allocate during capture
        const int64_t nb = nblocks(n) > 0 ? nblocks(n) : 1;
        B.red.ensure(c, 3 * nb);
    }
    PcgState hs{};
    hs.rtol = cfg.rtol;
    hs.itmax = cfg.itmax;
    hs.no_audit = 1;
    hs.hist = B.hist.get();
    PcgState* st = B.st.get();
    MAMG_CU(cudaMemcpyAsync(st, &hs, sizeof(hs), cudaMemcpyHostToDevice, c.stream));
    const int* done = &st->done;
    const int* no_audit = &st->no_audit;

    auto read_state = [&](PcgState& out) {
        MAMG_CU(cudaMemcpyAsync(&out, st, sizeof(PcgState), cudaMemcpyDeviceToHost, c.stream));
        c.sync();
    };
    auto finish = [&](int status) {
        PcgState fs;
        read_state(fs);
        rep->iterations = fs.it;
        const int64_t nh = (status == 0 && fs.norm_b == 0.0) ? 1 : fs.it + 1;
        std::vector<double> hh(static_cast<size_t>(nh));
        if (fs.norm_b == 0.0) {
            hh[0] = 0.0;
        } else {
            MAMG_CU(cudaMemcpyAsync(hh.data(), B.hist.get(), sizeof(double) * nh,
                                    cudaMemcpyDeviceToHost, c.stream));
            c.sync();
        }
        if (hist_out) std::copy(hh.begin(), hh.end(), hist_out);
        if (fs.norm_b > 0.0) rep->final_relres = hh.back() / fs.norm_b;
        rep->converged = fs.norm_b == 0.0 ? 1 : (rep->final_relres <= cfg.rtol ? 1 : 0);
        rep->audit_checks = fs.audit_checks;
        rep->audit_failures = fs.audit_failures;
        rep->audit_max_rel = fs.audit_max_rel;
        if (fs.status == MAMG_BREAKDOWN) {
            rep->breakdown_iteration = fs.bd_it;
            rep->breakdown_rho = fs.bd_rho;
            rep->converged = 0;
        }
        rep->solve_ms = std::chrono::duration<double, std::milli>(clock::now() - t0).count();
        return fs.status == MAMG_BREAKDOWN ? MAMG_BREAKDOWN : MAMG_OK;
    };

    // ||b|| (krylov.cpp:56) and the zero right-hand side (krylov.cpp:66-70)
    reduce<1>(c, n, OpDot{b, b}, EpiNormB{st}, B.red, nullptr);
    {
        PcgState s0;
        read_state(s0);
        if (s0.norm_b == 0.0) {
            if (n) fill_vec(c, n, u, 0.0, nullptr);
            return finish(MAMG_OK);
        }
    }
    // u = u0; r0 = b - A u (krylov.cpp:73-86)
    if (u0) {
        if (u0 != u) copy_vec(c, n, u, u0, nullptr);
    } else {
        fill_vec(c, n, u, 0.0, nullptr);
    }
    residual(c, A, b, u, B.r.get(), nullptr);
    reduce<1>(c, n, OpDot{B.r.get(), B.r.get()}, EpiHist0{st}, B.red, nullptr);

    std::vector<double> hbuf_r, hbuf_z;
    auto precond = [&](const double* r, double* z, const int* gate) {
        if (h) {
            cycle_rec(c, *h, 0, *cyc, r, z, true, gate);
        } else if (hp) {
            // host PrecondFn through staging copies (only when not done)
            PcgState s;
            read_state(s);
            if (s.done) return;
            hbuf_r.resize(n);
            hbuf_z.assign(n, 0.0);
            MAMG_CU(cudaMemcpyAsync(hbuf_r.data(), r, sizeof(double) * n, cudaMemcpyDeviceToHost,
                                    c.stream));
            c.sync();
            hp(user, hbuf_r.data(), hbuf_z.data(), n);
            MAMG_CU(cudaMemcpyAsync(z, hbuf_z.data(), sizeof(double) * n, cudaMemcpyHostToDevice,
                                    c.stream));
        } else {
            copy_vec(c, n, z, r, gate);
        }
    };

    // first step (krylov.cpp:95-109)
    precond(B.r.get(), B.w.get(), done);
    copy_vec(c, n, B.d.get(), B.w.get(), done);
    spmv(c, A, A.group, B.w.get(), B.v.get(), done);
    copy_vec(c, n, B.q.get(), B.v.get(), done);
    reduce<2>(c, n, OpPair{B.w.get(), B.r.get(), B.v.get()}, EpiInit{st}, B.red, done);
    if (n) {
        launch_pdl(c.stream, k_axpy_step, dim3(eblocks(n)), dim3(kBlock), 0, n, u,
                   static_cast<const double*>(B.d.get()), static_cast<const PcgState*>(st), done);
        c.count();
    }
    reduce<1>(c, n, OpAxpyNorm{B.r.get(), B.q.get(), st, 0.0}, EpiHistNext{st}, B.red, done);

    double* w = B.w.get();
    double* d = B.d.get();
    double* v = B.v.get();
    double* q = B.q.get();
    double* r = B.r.get();

    // the loop body for one buffer parity (krylov.cpp:111-137)
    auto body = [&](double* w_, double* d_, double* v_, double* q_) {
        precond(r, w_, done);
        spmv(c, A, A.group, w_, v_, done);
        reduce<3>(c, n, OpTriple{w_, r, v_, q_}, EpiTriple{st}, B.red, done);
        if (n) {
            launch_pdl(c.stream, k_pcg_pair1, dim3(eblocks(n)), dim3(kBlock), 0, n, w_, u,
                       static_cast<const double*>(d_), static_cast<const PcgState*>(st), done);
            c.count();
        }
        reduce<1>(c, n, OpPcgPair2{v_, r, q_, st}, EpiHistNext{st}, B.red, done);
    };
    auto audit = [&](double* scratch) {
        spmv(c, A, A.group, u, scratch, no_audit);
        reduce<1>(c, n, OpAudit{r, b, scratch}, EpiAudit{st}, B.red, no_audit);
    };

    // Graph per parity when the preconditioner is device-resident.
    const bool use_graph = (h != nullptr || hp == nullptr);
    cudaGraphExec_t exec[2] = {nullptr, nullptr};
    int64_t nodes[2] = {0, 0};
    if (use_graph) {
        for (int p = 0; p < 2; ++p) {
            cudaGraph_t g;
            const int64_t before = c.launches;
            MAMG_CU(cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeThreadLocal));
            if (p == 0)
                body(w, d, v, q);
            else
                body(d, w, q, v);
            MAMG_CU(cudaStreamEndCapture(c.stream, &g));
            nodes[p] = c.launches - before;
            c.launches = before;
            MAMG_CU(cudaGraphInstantiate(&exec[p], g, 0));
            MAMG_CU(cudaGraphDestroy(g));
        }
    }

    // Host loop with one iteration of lookahead: the stop flag of iteration
    // i is read (pinned, async) while iteration i+1 is already queued; every
    // kernel of a finished solve returns immediately (device-side gate), so
    // at most one no-op iteration is ever issued.
    int parity = 0;
    int64_t it = 1;
    int* h_flags = reinterpret_cast<int*>(c.h_small); // [slot] = done flag copies
    cudaEvent_t ev[2];
    MAMG_CU(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
    MAMG_CU(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
    MAMG_CU(cudaMemcpyAsync(&h_flags[0], done, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    MAMG_CU(cudaEventRecord(ev[0], c.stream));
    int slot = 0;
    for (;;) {
        // is the state before this iteration already final?
        MAMG_CU(cudaEventSynchronize(ev[slot]));
        if (h_flags[slot]) break;
        if (use_graph) {
            MAMG_CU(cudaGraphLaunch(exec[parity], c.stream));
            c.count(nodes[parity]);
        } else if (parity == 0) {
            body(w, d, v, q);
        } else {
            body(d, w, q, v);
        }
        // after the body the roles swap: the new d lives in the old w buffer
        parity ^= 1;
        ++it;
        if (it % 50 == 0) audit(parity == 0 ? w : d); // the free buffer (old d)
        slot ^= 1;
        MAMG_CU(cudaMemcpyAsync(&h_flags[slot], done, sizeof(int), cudaMemcpyDeviceToHost,
                                c.stream));
        MAMG_CU(cudaEventRecord(ev[slot], c.stream));
        // lookahead: check the iteration before this one without waiting
        // for the one just queued
        if (cudaEventQuery(ev[slot ^ 1]) == cudaSuccess && h_flags[slot ^ 1]) break;
    }
    cudaEventDestroy(ev[0]);
    cudaEventDestroy(ev[1]);
    for (auto& e : exec)
        if (e) cudaGraphExecDestroy(e);
    return finish(0);
}

// ================================================= partitioned (dist) solve ==
namespace {

// buffer plan of `sweeps` (out[j] for sweep j; see there)
std::vector<double*> sweep_plan(double* xa, double* xb, const double* src, double* dst, int k) {
    std::vector<double*> out(static_cast<size_t>(k));
    auto plan = [&](double* before_last) {
        out[k - 1] = dst;
        double* cur = before_last;
        for (int j = k - 2; j >= 0; --j) {
            out[j] = cur;
            cur = (cur == xa) ? xb : xa;
        }
    };
    plan(dst == xa ? xb : (dst == xb ? xa : xb));
    if (k >= 2 && src != nullptr && out[0] == src) plan(xa);
    return out;
}

struct DistRun {
    Ctx& c;
    DistHier& D;
    std::vector<const int*> gate; // per part (PCG stop flag) or null
    // halo / interior overlap (peer halos only): the halo of a source vector
    // runs on s2 while every part's interior rows [ia, ib) — no ghost column
    // — compute on the main stream; the boundary rows follow the join
    cudaStream_t s2 = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;

    size_t np() const { return D.parts.size(); }
    PLevel& L(size_t i, int k) { return D.parts[i].lv[k]; }

    void halo(int k, const std::vector<double*>& x) {
        if (D.peer.on) { // NVLink stores into the receivers' mailboxes
            peer_halo_exchange(c, D, k, x);
            return;
        }
        std::vector<Halo*> h;
        for (size_t i = 0; i < np(); ++i) h.push_back(&L(i, k).halo);
        D.comm->halo_f64(c, h, x);
    }

    // halo of x at level k, then rows(i, r0, r1) for every part over all its
    // rows — with the halo overlapped by the interior rows when possible
    template <class F>
    void halo_rows(int k, const std::vector<double*>& x, F&& rows) {
        bool ov = s2 != nullptr && D.peer.on;
        for (size_t i = 0; ov && i < np(); ++i) {
            const PLevel& lv = L(i, k);
            ov = lv.interior_gen == D.gen;
        }
        if (!ov) {
            halo(k, x);
            for (size_t i = 0; i < np(); ++i) rows(i, int64_t{0}, L(i, k).A->nrows);
            return;
        }
        MAMG_CU(cudaEventRecord(ev_fork, c.stream));
        MAMG_CU(cudaStreamWaitEvent(s2, ev_fork, 0));
        {
            const cudaStream_t main = c.stream;
            c.stream = s2;
            peer_halo_exchange(c, D, k, x);
            c.stream = main;
        }
        for (size_t i = 0; i < np(); ++i) rows(i, L(i, k).ia, L(i, k).ib);
        MAMG_CU(cudaEventRecord(ev_join, s2));
        MAMG_CU(cudaStreamWaitEvent(c.stream, ev_join, 0));
        for (size_t i = 0; i < np(); ++i) {
            rows(i, int64_t{0}, L(i, k).ia);
            rows(i, L(i, k).ib, L(i, k).A->nrows);
        }
    }

    // k sweeps per part with halo exchanges of every source iterate
    void sweeps(int k, const std::vector<const double*>& b, const std::vector<const double*>& src,
                const std::vector<double*>& dst, int nsweeps) {
        if (nsweeps == 0) {
            for (size_t i = 0; i < np(); ++i) {
                const int64_t n = L(i, k).A->nrows;
                if (src[i] == nullptr)
                    fill_vec(c, n, dst[i], 0.0, gate[i]);
                else if (src[i] != dst[i])
                    copy_vec(c, n, dst[i], src[i], gate[i]);
            }
            return;
        }
        std::vector<std::vector<double*>> plan(np());
        for (size_t i = 0; i < np(); ++i)
            plan[i] = sweep_plan(L(i, k).xw.get(), L(i, k).scratch.get(), src[i], dst[i], nsweeps);
        std::vector<const double*> cur = src;
        // zero start <=> no part was given a source (an EMPTY part has null
        // buffers either way, so no single part's pointer decides it)
        bool start_zero = true;
        for (auto* p : src) start_zero = start_zero && p == nullptr;
        for (int j = 0; j < nsweeps; ++j) {
            if (j > 0 || !start_zero) {
                std::vector<double*> xs;
                for (auto* p : cur) xs.push_back(const_cast<double*>(p));
                halo_rows(k, xs, [&](size_t i, int64_t r0, int64_t r1) {
                    PLevel& lv = L(i, k);
                    if (cur[i] != nullptr)
                        smooth_sweep_rows(c, *lv.A, lv.l1.get(), b[i], cur[i], plan[i][j], gate[i], r0, r1);
                });
            }
            for (size_t i = 0; i < np(); ++i) {
                PLevel& lv = L(i, k);
                if (cur[i] == nullptr) {
                    if (!lv.A->finite) {
                        double* z = plan[i][j] == lv.xw.get() ? lv.scratch.get() : lv.xw.get();
                        fill_vec(c, lv.A->nrows + lv.halo.nghost, z, 0.0, gate[i]);
                        smooth_sweep(c, *lv.A, lv.l1.get(), b[i], z, plan[i][j], gate[i]);
                    } else {
                        smooth_from_zero(c, lv.A->nrows, lv.l1.get(), b[i], plan[i][j], gate[i]);
                    }
                }
            }
            for (size_t i = 0; i < np(); ++i) cur[i] = plan[i][j];
        }
    }

    // multigrid.cpp:65-109 over the parts (no tail kernel: halos between phases)
    void cycle(int k, const mamg_cycle_cfg& cfg, const std::vector<const double*>& b,
               const std::vector<double*>& x_out, bool zero) {
        const size_t n_p = np();
        std::vector<const double*> none(n_p, nullptr);
        if (k == D.nl - 1) {
            sweeps(k, b, none, x_out, cfg.coarsest_sweeps);
            return;
        }
        std::vector<double*> xw(n_p), scr(n_p), cb(n_p), cx(n_p);
        std::vector<const double*> xin(n_p), cbc(n_p);
        for (size_t i = 0; i < n_p; ++i) {
            xw[i] = L(i, k).xw.get();
            scr[i] = L(i, k).scratch.get();
            cb[i] = L(i, k).cb.get();
            cx[i] = L(i, k).cx.get();
            cbc[i] = cb[i];
            xin[i] = zero ? nullptr : x_out[i];
        }
        if (cfg.pre_sweeps == 0) {
            for (size_t i = 0; i < n_p; ++i) {
                if (zero)
                    fill_vec(c, L(i, k).A->nrows, xw[i], 0.0, gate[i]);
                else
                    copy_vec(c, L(i, k).A->nrows, xw[i], x_out[i], gate[i]);
            }
        } else {
            sweeps(k, b, xin, xw, cfg.pre_sweeps);
        }
        // global matching: aggregates straddle parts -> the restriction reads
        // remote members' residuals (rhalo), the prolongation remote
        // aggregates' corrections (phalo)
        const bool straddle = D.matching == 1;
        halo_rows(k, xw, [&](size_t i, int64_t r0, int64_t r1) {
            residual_rows(c, *L(i, k).A, b[i], xw[i], scr[i], gate[i], r0, r1);
        });
        if (!straddle)
            for (size_t i = 0; i < n_p; ++i)
                spmv(c, *L(i, k).R, L(i, k).R->group, scr[i], cb[i], gate[i]);
        if (straddle) {
            std::vector<Halo*> h;
            for (size_t i = 0; i < n_p; ++i) h.push_back(&L(i, k).rhalo);
            D.comm->halo_f64(c, h, scr);
            for (size_t i = 0; i < n_p; ++i)
                spmv(c, *L(i, k).R, L(i, k).R->group, scr[i], cb[i], gate[i]);
        }
        const int visits = cfg.cycle == 1 ? 2 : 1;
        if (k + 1 == D.agg_level) {
            // agglomerated coarse levels: gather the restricted residual on
            // every process, cycle the replicated levels with the
            // single-device code, prolongate from the full iterate
            const std::vector<int64_t>& cbnd = L(0, k + 1).bounds;
            std::vector<int64_t> cnt(cbnd.size() - 1);
            for (size_t q = 0; q + 1 < cbnd.size(); ++q) cnt[q] = cbnd[q + 1] - cbnd[q];
            if (D.peer.on && !D.peer.ag.empty())
                peer_agg_gather(c, D, cbc, D.rep_b.get()); // NVLink stores, no NCCL
            else
                D.comm->allgather_f64(c, cbc, cnt, std::vector<double*>(n_p, D.rep_b.get()));
            for (int t = 0; t < visits; ++t)
                apply_cycle(c, *D.rep, 0, cfg, D.rep_b.get(), D.rep_x.get(), t == 0, gate[0]);
            for (size_t i = 0; i < n_p; ++i)
                prolong_correct(c, *L(i, k).P, D.rep_x.get(), xw[i], gate[i]);
            std::vector<const double*> xwa(xw.begin(), xw.end());
            if (cfg.post_sweeps == 0) {
                for (size_t i = 0; i < n_p; ++i)
                    copy_vec(c, L(i, k).A->nrows, x_out[i], xw[i], gate[i]);
            } else {
                sweeps(k, b, xwa, x_out, cfg.post_sweeps);
            }
            return;
        }
        for (int t = 0; t < visits; ++t) cycle(k + 1, cfg, cbc, cx, t == 0);
        if (straddle) {
            std::vector<Halo*> h;
            for (size_t i = 0; i < n_p; ++i) h.push_back(&L(i, k).phalo);
            D.comm->halo_f64(c, h, cx);
        }
        for (size_t i = 0; i < n_p; ++i) prolong_correct(c, *L(i, k).P, cx[i], xw[i], gate[i]);
        std::vector<const double*> xwc(xw.begin(), xw.end());
        if (cfg.post_sweeps == 0) {
            for (size_t i = 0; i < n_p; ++i)
                copy_vec(c, L(i, k).A->nrows, x_out[i], xw[i], gate[i]);
        } else {
            sweeps(k, b, xwc, x_out, cfg.post_sweeps);
        }
    }
};

struct DPcg {
    DBuf<double> b, u, r, w, d, v, q, hist, plocal, pglob, scratch;
    DBuf<int64_t> roff; // world + 1 prefix of the ranks' block counts
    DBuf<PcgState> st;
    DBuf<unsigned> counter;
    int64_t n = 0, ext = 0, nb = 0;
};

template <class K>
void ensure_smem(K kernel, size_t bytes) {
    ensure_dyn_smem(kernel, bytes);
}

} // namespace

int dist_pcg(Ctx& c, DistHier& D, const mamg_cycle_cfg& cyc, const double* h_b,
             const mamg_solve_cfg& cfg, double* h_u, double* hist_out, mamg_report* rep,
             const double* h_u0) {
    using clock = std::chrono::steady_clock;
    const auto t0 = clock::now();
    if (!(cfg.rtol > 0.0)) invalid("SolveConfig: rtol must be > 0");
    if (cfg.itmax < 1) invalid("SolveConfig: itmax must be >= 1");
    if (cyc.pre_sweeps < 0 || cyc.post_sweeps < 0) invalid("CycleConfig: sweep counts must be >= 0");
    if (cyc.coarsest_sweeps < 1) invalid("CycleConfig: coarsest_sweeps must be >= 1");
    if (cyc.cycle != 0 && cyc.cycle != 1)
        invalid("CycleConfig: the partitioned solve supports V and W cycles");
    std::memset(rep, 0, sizeof(*rep));
    rep->breakdown_iteration = -1;
    const size_t np = D.parts.size();
    std::vector<DPcg> P(np);
    std::vector<int64_t> nbs;
    for (size_t i = 0; i < np; ++i) {
        PLevel& L = D.parts[i].lv[0];
        DPcg& x = P[i];
        x.n = L.A->nrows;
        x.ext = x.n + L.halo.nghost;
        x.nb = nblocks(x.n);
        nbs.push_back(x.nb);
        for (auto* buf : {&x.u, &x.w, &x.d, &x.scratch}) buf->alloc(x.ext, c.stream);
        for (auto* buf : {&x.b, &x.r, &x.v, &x.q}) buf->alloc(x.n, c.stream);
        x.hist.alloc(cfg.itmax + 2, c.stream);
        x.st.alloc(1, c.stream);
        x.plocal.alloc(3 * (x.nb > 0 ? x.nb : 1), c.stream);
    }
    const auto all_nb = D.comm->allgather(c, nbs);
    const int W = D.comm->world;
    int64_t nb_tot = 0, nbmax = 1;
    std::vector<int64_t> roff_h{0};
    for (auto v : all_nb) {
        nb_tot += v;
        nbmax = std::max(nbmax, v);
        roff_h.push_back(nb_tot);
    }
    // every rank's partials padded to 3 * nbmax: one equal-count allgather
    // per reduction (all components at once); in-process parts share one
    // gathered buffer
    for (auto& x : P) {
        x.plocal.alloc(3 * nbmax, c.stream);
    }
    c.sync();
    for (size_t i = 0; i < np; ++i) {
        DPcg& x = P[i];
        if (i == 0 || np == 1) x.pglob.alloc(static_cast<size_t>(W) * 3 * nbmax, c.stream);
        x.roff.alloc(W + 1, c.stream);
        MAMG_CU(cudaMemcpyAsync(x.roff.get(), roff_h.data(), sizeof(int64_t) * (W + 1),
                                cudaMemcpyHostToDevice, c.stream));
        PcgState hs{};
        hs.rtol = cfg.rtol;
        hs.itmax = cfg.itmax;
        hs.no_audit = 1;
        hs.hist = x.hist.get();
        MAMG_CU(cudaMemcpyAsync(x.st.get(), &hs, sizeof(hs), cudaMemcpyHostToDevice, c.stream));
        const int64_t g0 = D.parts[i].lv[0].bounds[D.parts[i].rank];
        c.sync();
        if (h_b) {
            if (x.n) upload_f64(c, x.b.get(), h_b + g0, static_cast<size_t>(x.n));
        } else if (x.n) {
            fill_vec(c, x.n, x.b.get(), 1.0, nullptr);
        }
        fill_vec(c, x.ext, x.u.get(), 0.0, nullptr);
        if (h_u0 && x.n) upload_f64(c, x.u.get(), h_u0 + g0, static_cast<size_t>(x.n));
    }
    double* gath = P[0].pglob.get(); // shared by the in-process parts
    // Fused peer reductions (default): the block-dot kernels write their
    // partials straight into every rank's gathered buffer (slot-1 shared
    // blocks: IPC/NVLink for NCCL, the parts' own for the loopback) and signal
    // arrival counters; MAMG_DIST_NCCL_REDUCE=1 uses the NCCL allgather.
    // (world = 1 has nothing to exchange: the Comm's self-copy is cheaper;
    // MAMG_DIST_PEER=1 forces the peer paths there, to test their plumbing)
    const bool nccl_reduce = std::getenv("MAMG_DIST_NCCL_REDUCE") != nullptr;
    const bool force_peer = std::getenv("MAMG_DIST_PEER") != nullptr;
    bool peer = !nccl_reduce && W <= kMaxWorld && (W > 1 || force_peer);
    const int64_t pstride = static_cast<int64_t>(W) * 3 * nbmax;
    const size_t gbytes = (sizeof(double) * 2 * static_cast<size_t>(pstride) + 255) & ~size_t{255};
    std::vector<PeerOut> po(np);
    std::vector<char*> pblk(np);
    std::vector<void*> blocks;
    if (peer) {
        // a rank that cannot map its peers' blocks (no IPC / peer access)
        // makes every rank use the NCCL allgather instead
        int64_t ok = 1;
        try {
            blocks = D.comm->shared_blocks(c, std::vector<size_t>(np, gbytes + 256), 1);
        } catch (const Error&) {
            ok = 0;
        }
        for (auto v : D.comm->allgather(c, std::vector<int64_t>(np, ok))) peer = peer && v != 0;
    }
    if (peer) {
        for (size_t i = 0; i < np; ++i) {
            const int me = D.parts[i].rank;
            pblk[i] = static_cast<char*>(blocks[me]);
            MAMG_CU(cudaMemsetAsync(pblk[i] + gbytes, 0, 256, c.stream)); // arrive, epoch, err
            P[i].counter.alloc(1, c.stream);
            MAMG_CU(cudaMemsetAsync(P[i].counter.get(), 0, sizeof(unsigned), c.stream));
            po[i].world = W;
            po[i].me = me;
            for (int r = 0; r < W; ++r) {
                po[i].gath[r] = static_cast<double*>(blocks[r]);
                po[i].arrive[r] =
                    reinterpret_cast<unsigned long long*>(static_cast<char*>(blocks[r]) + gbytes);
            }
            po[i].epoch = reinterpret_cast<const unsigned long long*>(pblk[i] + gbytes) + 1;
            po[i].pstride = pstride;
        }
        D.comm->barrier(c); // every rank's counters are zero before anyone signals
    }
    std::vector<const int*> done(np), no_audit(np);
    for (size_t i = 0; i < np; ++i) {
        done[i] = &P[i].st.get()->done;
        no_audit[i] = &P[i].st.get()->no_audit;
    }
    DistRun run{c, D, done};
    // halo exchanges of the partitioned levels over peer memory (default),
    // overlapped with the interior rows on a second stream
    const int npl = D.agg_level >= 0 ? D.agg_level : D.nl;
    // (on by default only where halos cross GPUs: NCCL, world > 1; the
    // loopback's parts share one GPU, nothing to hide — MAMG_DIST_OVERLAP=1
    // forces it there for testing)
    const bool want_overlap = std::getenv("MAMG_DIST_NO_OVERLAP") == nullptr &&
                              (D.comm->peer_memory() || std::getenv("MAMG_DIST_OVERLAP") != nullptr);
    if (peer_halo_prepare(c, D, npl) && want_overlap) {
        interior_ranges(c, D, npl);
        MAMG_CU(cudaStreamCreateWithFlags(&run.s2, cudaStreamNonBlocking));
        MAMG_CU(cudaEventCreateWithFlags(&run.ev_fork, cudaEventDisableTiming));
        MAMG_CU(cudaEventCreateWithFlags(&run.ev_join, cudaEventDisableTiming));
    }
    struct RunCleanup {
        DistRun& r;
        ~RunCleanup() {
            if (r.s2) {
                cudaStreamSynchronize(r.s2);
                cudaStreamDestroy(r.s2);
            }
            if (r.ev_fork) cudaEventDestroy(r.ev_fork);
            if (r.ev_join) cudaEventDestroy(r.ev_join);
        }
    } run_cleanup{run};
    D.last_solve[0] = peer ? 1 : 0;
    D.last_solve[1] = D.peer.on ? 1 : 0;
    D.last_solve[2] = run.s2 != nullptr ? 1 : 0;
    D.last_solve[3] = 0;
    const size_t fold_smem = sizeof(double) * static_cast<size_t>(fold_doubles(nb_tot));

    // reduction: local block chains -> one allgather of the padded partials
    // -> segmented fold + epilogue (bit-identical to the unpartitioned dot)
    auto reduce_d = [&](auto nvtag, auto make_op, auto make_epi, const std::vector<const int*>& g) {
        constexpr int NV = decltype(nvtag)::value;
        if (peer) {
            for (size_t i = 0; i < np; ++i) {
                auto op = make_op(i);
                auto epi = make_epi(i);
                auto kernel = k_blockdot<NV, decltype(op), decltype(epi), false>;
                const size_t smem = sizeof(double) * dot_tile_doubles<NV>();
                ensure_smem(kernel, smem);
                PeerOut p = po[i];
                p.rstride = NV * nbmax;
                // an empty part still signals (one CTA with no blocks)
                const int grid = static_cast<int>(P[i].nb > 0 ? (P[i].nb + kBPC - 1) / kBPC : 1);
                kernel<<<grid, kDotThreads, smem, c.stream>>>(P[i].n, op, epi, P[i].plocal.get(),
                                                              P[i].nb, P[i].counter.get(), g[i], p);
                c.count();
            }
            for (size_t i = 0; i < np; ++i) {
                auto epi = make_epi(i);
                auto kernel = k_fold_peer<NV, decltype(epi)>;
                ensure_smem(kernel, fold_smem);
                auto* ctr = reinterpret_cast<unsigned long long*>(pblk[i] + gbytes);
                kernel<<<1, kDotThreads, fold_smem, c.stream>>>(
                    reinterpret_cast<const double*>(pblk[i]), P[i].roff.get(), W, NV * nbmax, pstride,
                    nb_tot, ctr, ctr + 1, ctr + 2, epi, g[i]);
                c.count();
            }
            MAMG_LAUNCH_CHECK();
            return;
        }
        for (size_t i = 0; i < np; ++i) {
            auto op = make_op(i);
            auto epi = make_epi(i);
            auto kernel = k_blockdot<NV, decltype(op), decltype(epi), false>;
            const size_t smem = sizeof(double) * dot_tile_doubles<NV>();
            ensure_smem(kernel, smem);
            const int grid = static_cast<int>(P[i].nb > 0 ? (P[i].nb + kBPC - 1) / kBPC : 0);
            if (grid) {
                kernel<<<grid, kDotThreads, smem, c.stream>>>(P[i].n, op, epi, P[i].plocal.get(),
                                                              P[i].nb, nullptr, g[i], PeerOut{});
                c.count();
            }
        }
        {
            std::vector<const double*> src;
            std::vector<double*> dst;
            for (size_t i = 0; i < np; ++i) {
                src.push_back(P[i].plocal.get());
                dst.push_back(np == 1 ? P[i].pglob.get() : gath);
            }
            D.comm->allgather_equal_f64(c, src, NV * nbmax, dst);
        }
        for (size_t i = 0; i < np; ++i) {
            auto epi = make_epi(i);
            auto kernel = k_fold_seg<NV, decltype(epi)>;
            ensure_smem(kernel, fold_smem);
            kernel<<<1, kDotThreads, fold_smem, c.stream>>>(np == 1 ? P[i].pglob.get() : gath,
                                                            P[i].roff.get(), W, NV * nbmax, nb_tot,
                                                            epi, g[i]);
            c.count();
        }
        MAMG_LAUNCH_CHECK();
    };
    using One = std::integral_constant<int, 1>;
    using Two = std::integral_constant<int, 2>;
    using Three = std::integral_constant<int, 3>;
    std::vector<const int*> nogate(np, nullptr);
    auto state = [&](PcgState& out) {
        MAMG_CU(cudaMemcpyAsync(&out, P[0].st.get(), sizeof(PcgState), cudaMemcpyDeviceToHost,
                                c.stream));
        c.sync();
    };
    auto halo0 = [&](std::vector<double*> xs) { run.halo(0, xs); };
    auto vecs = [&](DBuf<double> DPcg::*m) {
        std::vector<double*> v;
        for (auto& x : P) v.push_back((x.*m).get());
        return v;
    };

    reduce_d(One{}, [&](size_t i) { return OpDot{P[i].b.get(), P[i].b.get()}; },
             [&](size_t i) { return EpiNormB{P[i].st.get()}; }, nogate);
    PcgState s0;
    state(s0);
    bool zero_rhs = s0.norm_b == 0.0;
    if (!zero_rhs) {
        halo0(vecs(&DPcg::u));
        for (size_t i = 0; i < np; ++i)
            residual(c, *D.parts[i].lv[0].A, P[i].b.get(), P[i].u.get(), P[i].r.get(), nullptr);
        reduce_d(One{}, [&](size_t i) { return OpDot{P[i].r.get(), P[i].r.get()}; },
                 [&](size_t i) { return EpiHist0{P[i].st.get()}; }, nogate);
        // first step (krylov.cpp:95-109)
        std::vector<const double*> rr;
        for (auto& x : P) rr.push_back(x.r.get());
        run.cycle(0, cyc, rr, vecs(&DPcg::w), true);
        // owned rows only: d's ghost region is filled by its halo before use
        for (size_t i = 0; i < np; ++i) copy_vec(c, P[i].n, P[i].d.get(), P[i].w.get(), done[i]);
        halo0(vecs(&DPcg::w));
        for (size_t i = 0; i < np; ++i) {
            const DevCsr& A = *D.parts[i].lv[0].A;
            spmv(c, A, A.group, P[i].w.get(), P[i].v.get(), done[i]);
            copy_vec(c, P[i].n, P[i].q.get(), P[i].v.get(), done[i]);
        }
        reduce_d(Two{}, [&](size_t i) { return OpPair{P[i].w.get(), P[i].r.get(), P[i].v.get()}; },
                 [&](size_t i) { return EpiInit{P[i].st.get()}; }, done);
        for (size_t i = 0; i < np; ++i)
            if (P[i].n) {
                k_axpy_step<<<eblocks(P[i].n), kBlock, 0, c.stream>>>(P[i].n, P[i].u.get(),
                                                                      P[i].d.get(),
                                                                      P[i].st.get(), done[i]);
                c.count();
            }
        reduce_d(One{},
                 [&](size_t i) { return OpAxpyNorm{P[i].r.get(), P[i].q.get(), P[i].st.get(), 0.0}; },
                 [&](size_t i) { return EpiHistNext{P[i].st.get()}; }, done);
        // one PCG iteration (krylov.cpp:111-139) of the given buffer parity
        auto body = [&](int par) {
            std::vector<double*> w_(np), d_(np), v_(np), q_(np);
            for (size_t i = 0; i < np; ++i) {
                w_[i] = par == 0 ? P[i].w.get() : P[i].d.get();
                d_[i] = par == 0 ? P[i].d.get() : P[i].w.get();
                v_[i] = par == 0 ? P[i].v.get() : P[i].q.get();
                q_[i] = par == 0 ? P[i].q.get() : P[i].v.get();
            }
            run.cycle(0, cyc, rr, w_, true);
            run.halo_rows(0, w_, [&](size_t i, int64_t r0, int64_t r1) {
                const DevCsr& A = *D.parts[i].lv[0].A;
                spmv_rows(c, A, A.group, w_[i], v_[i], done[i], r0, r1);
            });
            reduce_d(Three{}, [&](size_t i) { return OpTriple{w_[i], P[i].r.get(), v_[i], q_[i]}; },
                     [&](size_t i) { return EpiTriple{P[i].st.get()}; }, done);
            for (size_t i = 0; i < np; ++i)
                if (P[i].n) {
                    k_pcg_pair1<<<eblocks(P[i].n), kBlock, 0, c.stream>>>(
                        P[i].n, w_[i], P[i].u.get(), d_[i], P[i].st.get(), done[i]);
                    c.count();
                }
            reduce_d(One{}, [&](size_t i) { return OpPcgPair2{v_[i], P[i].r.get(), q_[i], P[i].st.get()}; },
                     [&](size_t i) { return EpiHistNext{P[i].st.get()}; }, done);
        };
        // Each parity's iteration is captured once as a CUDA graph (kernels,
        // halo / allgather collectives and copies) and replayed; the host runs
        // one iteration ahead: iteration j+1 is queued before the stop flag
        // after iteration j is read (a gated, no-op iteration past the end).
        static const bool no_graph_env = std::getenv("MAMG_DIST_NO_GRAPH") != nullptr;
        // a transport whose collectives wait on the host cannot be captured
        const bool no_graph = no_graph_env || !D.comm->capturable();
        D.last_solve[3] = no_graph ? 0 : 1;
        cudaGraphExec_t exec[2] = {nullptr, nullptr};
        int64_t nodes[2] = {0, 0};
        auto run_iter = [&](int par, bool eager) {
            if (no_graph || eager) {
                body(par);
                return;
            }
            if (!exec[par]) {
                const int64_t l0 = c.launches;
                cudaGraph_t g = nullptr;
                MAMG_CU(cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeRelaxed));
                try {
                    body(par);
                } catch (...) {
                    cudaStreamEndCapture(c.stream, &g);
                    if (g) cudaGraphDestroy(g);
                    throw;
                }
                MAMG_CU(cudaStreamEndCapture(c.stream, &g));
                const cudaError_t e = cudaGraphInstantiate(&exec[par], g, 0);
                cudaGraphDestroy(g);
                MAMG_CU(e);
                nodes[par] = c.launches - l0;
                c.launches = l0;
            }
            MAMG_CU(cudaGraphLaunch(exec[par], c.stream));
            c.count(nodes[par]);
        };
        int* hdone = nullptr;
        MAMG_CU(cudaHostAlloc(reinterpret_cast<void**>(&hdone), 2 * sizeof(int), cudaHostAllocDefault));
        cudaEvent_t ev[2];
        MAMG_CU(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
        MAMG_CU(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
        auto cleanup = [&] {
            for (auto& e : exec)
                if (e) cudaGraphExecDestroy(e);
            cudaEventDestroy(ev[0]);
            cudaEventDestroy(ev[1]);
            cudaFreeHost(hdone);
        };
        auto snapshot = [&](int slot) {
            MAMG_CU(cudaMemcpyAsync(&hdone[slot], done[0], sizeof(int), cudaMemcpyDeviceToHost,
                                    c.stream));
            MAMG_CU(cudaEventRecord(ev[slot], c.stream));
        };
        try {
            int64_t it = 1;
            int parity = 0;
            int cur = 0;
            snapshot(cur); // stop flag after the first step
            for (;;) {
                run_iter(parity, it == 1); // first iteration eager (kernel attributes set)
                parity ^= 1;
                ++it;
                if (it % 50 == 0) {
                    halo0(vecs(&DPcg::u));
                    for (size_t i = 0; i < np; ++i) {
                        const DevCsr& A = *D.parts[i].lv[0].A;
                        spmv(c, A, A.group, P[i].u.get(), P[i].scratch.get(), no_audit[i]);
                    }
                    reduce_d(One{},
                             [&](size_t i) { return OpAudit{P[i].r.get(), P[i].b.get(), P[i].scratch.get()}; },
                             [&](size_t i) { return EpiAudit{P[i].st.get()}; }, no_audit);
                }
                MAMG_CU(cudaEventSynchronize(ev[cur]));
                if (hdone[cur]) break; // the iteration just queued is gated
                cur ^= 1;
                snapshot(cur);
            }
        } catch (...) {
            c.sync();
            cleanup();
            throw;
        }
        c.sync();
        cleanup();
    }
    if (peer_halo_failed(c, D)) {
        D.peer.on = false;
        throw Error(MAMG_RUNTIME, "partitioned pcg: a peer halo exchange timed out waiting for a peer");
    }
    D.peer.on = false; // setup halos (dist_build) use the Comm transport
    if (peer) {
        c.sync();
        for (size_t i = 0; i < np; ++i) {
            unsigned long long e = 0;
            MAMG_CU(cudaMemcpy(&e, pblk[i] + gbytes + 2 * sizeof(unsigned long long), sizeof(e),
                               cudaMemcpyDeviceToHost));
            if (e)
                throw Error(MAMG_RUNTIME,
                            "partitioned pcg: a peer reduction timed out waiting for the other ranks");
        }
    }
    // results
    PcgState fs;
    state(fs);
    for (size_t i = 0; i < np; ++i) {
        const int64_t g0 = D.parts[i].lv[0].bounds[D.parts[i].rank];
        if (h_u && P[i].n) {
            if (zero_rhs)
                std::fill(h_u + g0, h_u + g0 + P[i].n, 0.0);
            else
                download_f64(c, h_u + g0, P[i].u.get(), static_cast<size_t>(P[i].n));
        }
    }
    rep->iterations = fs.it;
    const int64_t nh = zero_rhs ? 1 : fs.it + 1;
    std::vector<double> hh(static_cast<size_t>(nh), 0.0);
    if (!zero_rhs) {
        MAMG_CU(cudaMemcpyAsync(hh.data(), P[0].hist.get(), sizeof(double) * nh,
                                cudaMemcpyDeviceToHost, c.stream));
        c.sync();
    }
    if (hist_out) std::copy(hh.begin(), hh.end(), hist_out);
    if (fs.norm_b > 0.0) rep->final_relres = hh.back() / fs.norm_b;
    rep->converged = zero_rhs ? 1 : (rep->final_relres <= cfg.rtol ? 1 : 0);
    rep->audit_checks = fs.audit_checks;
    rep->audit_failures = fs.audit_failures;
    rep->audit_max_rel = fs.audit_max_rel;
    int status = MAMG_OK;
    if (fs.status == MAMG_BREAKDOWN) {
        rep->breakdown_iteration = fs.bd_it;
        rep->breakdown_rho = fs.bd_rho;
        rep->converged = 0;
        status = MAMG_BREAKDOWN;
    }
    rep->solve_ms = std::chrono::duration<double, std::milli>(clock::now() - t0).count();
    return status;
}

} // namespace mamg

namespace mamg {

// Device time of one partitioned operation of this process's parts, averaged
// over `reps` launches on the context stream (CUDA events; every rank calls
// it together — the cycle's halos are collective):
//   what 0: the level-0 fused l1-Jacobi sweep of the local rows (the kernel
//           alone, no halo) — the partitioned roofline kernel;
//   what 1: one preconditioner application (cycle from zero on b = ones)
//           with the solve's halo transport (peer mailboxes at world > 1).
double dist_time(Ctx& c, DistHier& D, int what, const mamg_cycle_cfg& cyc, int reps) {
    if (D.parts.empty() || D.nl == 0) invalid("mamg_dist_time: no hierarchy built");
    if (reps < 1) invalid("mamg_dist_time: reps must be >= 1");
    const size_t np = D.parts.size();
    std::vector<DBuf<double>> b(np), x0(np), x1(np);
    for (size_t i = 0; i < np; ++i) {
        const PLevel& L = D.parts[i].lv[0];
        const int64_t n = L.A->nrows, ext = n + L.halo.nghost;
        b[i].alloc(n > 0 ? n : 1, c.stream);
        x0[i].alloc(ext > 0 ? ext : 1, c.stream);
        x1[i].alloc(ext > 0 ? ext : 1, c.stream);
        if (n) fill_vec(c, n, b[i].get(), 1.0, nullptr);
        MAMG_CU(cudaMemsetAsync(x0[i].get(), 0, sizeof(double) * (ext > 0 ? ext : 1), c.stream));
        MAMG_CU(cudaMemsetAsync(x1[i].get(), 0, sizeof(double) * (ext > 0 ? ext : 1), c.stream));
    }
    std::vector<const int*> nogate(np, nullptr);
    DistRun run{c, D, nogate};
    struct Cleanup {
        DistRun& r;
        DistHier& D;
        ~Cleanup() {
            D.peer.on = false;
            if (r.s2) {
                cudaStreamSynchronize(r.s2);
                cudaStreamDestroy(r.s2);
            }
            if (r.ev_fork) cudaEventDestroy(r.ev_fork);
            if (r.ev_join) cudaEventDestroy(r.ev_join);
        }
    } cleanup{run, D};
    if (what == 1) {
        const int npl = D.agg_level >= 0 ? D.agg_level : D.nl;
        const bool want_overlap = std::getenv("MAMG_DIST_NO_OVERLAP") == nullptr &&
                                  (D.comm->peer_memory() || std::getenv("MAMG_DIST_OVERLAP") != nullptr);
        if (peer_halo_prepare(c, D, npl) && want_overlap) {
            interior_ranges(c, D, npl);
            MAMG_CU(cudaStreamCreateWithFlags(&run.s2, cudaStreamNonBlocking));
            MAMG_CU(cudaEventCreateWithFlags(&run.ev_fork, cudaEventDisableTiming));
            MAMG_CU(cudaEventCreateWithFlags(&run.ev_join, cudaEventDisableTiming));
        }
    } else if (what != 0) {
        invalid("mamg_dist_time: what must be 0 (level-0 sweep) or 1 (preconditioner)");
    }
    int flip = 0;
    auto once = [&] {
        std::vector<const double*> bb;
        std::vector<double*> xs;
        for (size_t i = 0; i < np; ++i) {
            bb.push_back(b[i].get());
            xs.push_back(flip ? x1[i].get() : x0[i].get());
        }
        if (what == 0) {
            for (size_t i = 0; i < np; ++i) {
                const PLevel& L = D.parts[i].lv[0];
                if (L.A->nrows)
                    smooth_sweep(c, *L.A, L.l1.get(), b[i].get(), flip ? x1[i].get() : x0[i].get(),
                                 flip ? x0[i].get() : x1[i].get(), nullptr);
            }
        } else {
            run.cycle(0, cyc, bb, xs, true);
        }
        flip ^= 1;
    };
    once(); // warm-up (kernel attributes, first-touch)
    D.comm->barrier(c);
    cudaEvent_t e0, e1;
    MAMG_CU(cudaEventCreate(&e0));
    MAMG_CU(cudaEventCreate(&e1));
    MAMG_CU(cudaEventRecord(e0, c.stream));
    for (int r = 0; r < reps; ++r) once();
    MAMG_CU(cudaEventRecord(e1, c.stream));
    MAMG_CU(cudaEventSynchronize(e1));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (peer_halo_failed(c, D)) throw Error(MAMG_RUNTIME, "mamg_dist_time: a peer halo exchange timed out");
    c.sync();
    return static_cast<double>(ms) / reps;
}

} // namespace mamg
