// Micro-benchmark: latency of one dependent link of a Suitor dislodgement
// chain, measured by a single thread walking a random permutation:
//   mode 0: plain 8-byte load of the next index (pointer chase)
//   mode 1: + 16-byte strong load (ld.relaxed.gpu.v2) of the slot
//   mode 2: + 128-bit atomicCAS on the slot
//   mode 3: 64-bit atomicCAS instead of the 128-bit one
//   mode 4: 128-bit CAS only (the CAS result supplies the next index)
//   mode 5: pointer chase through a 512 MB array, random jumps (TLB reach)
//   mode 6: the same with short forward jumps (+224..+1024 B, chain-like)
//   mode 7: the Suitor link exactly: .nc candidate load, 128-bit strong load,
//           .nc prefetch of the next candidate + list bounds, 128-bit CAS
// working set: 4M slots x 16 B (the cfg-2 suitor words) -> L2 / DRAM mix
#include <cstdio>
#include <vector>
#include <random>
#include <algorithm>

struct __align__(16) Suit {
    double w;
    unsigned long long u;
};

struct __align__(16) Cand {
    int v, pad;
    double w;
};
__global__ void klink(const Cand* __restrict__ cand, const int* __restrict__ rp,
                      const int* __restrict__ ncand, Suit* S, int steps, unsigned long long* out) {
    unsigned long long t0, t1;
    int k = 0;
    Cand e = cand[0];
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (int s = 0; s < steps; ++s) {
        unsigned long long a, b;
        asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(&S[e.v]) : "memory");
        const int w = static_cast<int>(b & 0xfffff);
        const Cand nxt = cand[(k + w) & 0xfffff];
        const int wr = __ldg(rp + w), wn = __ldg(ncand + w);
        Suit exp{__longlong_as_double(static_cast<long long>(a)), b};
        Suit des{1.0, b + 7};
        Suit old = atomicCAS(&S[e.v], exp, des);
        k = static_cast<int>(old.u & 0xff) + wr + wn;
        e = nxt;
        e.v = (e.v + k) & 0xfffff;
    }
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    out[0] = t1 - t0;
    out[1] = k;
}

__global__ void kbig(const long long* big, long long nbig, int steps, unsigned long long* out) {
    long long i = 0;
    unsigned long long t0, t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (int s = 0; s < steps; ++s) i = __ldcg(big + i);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    out[0] = t1 - t0;
    out[1] = i;
}

__global__ void k(const int* nxt, Suit* S, unsigned long long* S64, int steps, int mode,
                  unsigned long long* out) {
    int i = 0;
    unsigned long long t0, t1, acc = 0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (int s = 0; s < steps; ++s) {
        if (mode == 4) {
            Suit exp{0.0, 0ull}, des{1.0, static_cast<unsigned long long>(s)};
            Suit old = atomicCAS(&S[i], exp, des);
            i = static_cast<int>(old.u & 0x3fffff) ^ nxt[i & 1023];
            continue;
        }
        const int j = __ldcg(nxt + i);
        if (mode >= 1 && mode != 3) {
            unsigned long long a, b;
            asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(&S[j]) : "memory");
            acc += a ^ b;
            if (mode == 2) {
                Suit exp{__longlong_as_double(static_cast<long long>(a)), b};
                Suit des{1.0, b + 1};
                Suit old = atomicCAS(&S[j], exp, des);
                acc += old.u;
            }
        }
        if (mode == 3) {
            unsigned long long v = S64[j];
            acc += atomicCAS(&S64[j], v, v + 1);
        }
        i = j ^ static_cast<int>(acc & 0);
    }
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    out[0] = t1 - t0;
    out[1] = acc + i;
}

int main() {
    const int n = 4 << 20, steps = 20000;
    std::vector<int> perm(n);
    for (int i = 0; i < n; ++i) perm[i] = i;
    std::mt19937 rng(1);
    std::shuffle(perm.begin(), perm.end(), rng);
    std::vector<int> nxt(n);
    for (int i = 0; i < n; ++i) nxt[perm[i]] = perm[(i + 1) % n];
    int* dn;
    Suit* dS;
    unsigned long long *dS64, *dout;
    cudaMalloc(&dn, 4ll * n);
    cudaMalloc(&dS, 16ll * n);
    cudaMalloc(&dS64, 8ll * n);
    cudaMalloc(&dout, 16);
    cudaMemcpy(dn, nxt.data(), 4ll * n, cudaMemcpyHostToDevice);
    cudaMemset(dS, 0, 16ll * n);
    cudaMemset(dS64, 0, 8ll * n);
    for (int mode = 0; mode <= 4; ++mode) {
        k<<<1, 1>>>(dn, dS, dS64, 100, mode, dout);
        k<<<1, 1>>>(dn, dS, dS64, steps, mode, dout);
        unsigned long long h[2];
        cudaMemcpy(h, dout, 16, cudaMemcpyDeviceToHost);
        printf("mode %d: %.1f ns per link (%s)\n", mode, static_cast<double>(h[0]) / steps,
               cudaGetErrorString(cudaGetLastError()));
    }
    {
        const int nc = 1 << 20;
        std::vector<int> hv(2 * nc);
        std::uniform_int_distribution<int> U(0, nc - 1);
        std::vector<Cand> hc(nc);
        for (int t = 0; t < nc; ++t) hc[t] = Cand{U(rng), 0, 1.0};
        for (int t = 0; t < 2 * nc; ++t) hv[t] = U(rng) & 7;
        Cand* dc;
        int* di;
        Suit* dS2;
        cudaMalloc(&dc, sizeof(Cand) * nc);
        cudaMalloc(&di, 8ll * nc);
        cudaMalloc(&dS2, sizeof(Suit) * nc);
        cudaMemcpy(dc, hc.data(), sizeof(Cand) * nc, cudaMemcpyHostToDevice);
        cudaMemcpy(di, hv.data(), 8ll * nc, cudaMemcpyHostToDevice);
        std::vector<Suit> hs(nc);
        for (int t = 0; t < nc; ++t) hs[t] = Suit{1.0, static_cast<unsigned long long>(U(rng))};
        cudaMemcpy(dS2, hs.data(), sizeof(Suit) * nc, cudaMemcpyHostToDevice);
        klink<<<1, 1>>>(dc, di, di + nc, dS2, 100, dout);
        klink<<<1, 1>>>(dc, di, di + nc, dS2, steps, dout);
        unsigned long long h[2];
        cudaMemcpy(h, dout, 16, cudaMemcpyDeviceToHost);
        printf("mode 7: %.1f ns per link (%s)\n", static_cast<double>(h[0]) / steps,
               cudaGetErrorString(cudaGetLastError()));
    }
    const long long nbig = 64ll << 20; // 512 MB of int64
    long long* dbig;
    cudaMalloc(&dbig, 8 * nbig);
    for (int mode = 5; mode <= 6; ++mode) {
        std::vector<long long> hb(nbig);
        if (mode == 5) {
            std::uniform_int_distribution<long long> U(0, nbig - 1);
            for (long long t = 0; t < nbig; ++t) hb[t] = U(rng);
        } else {
            std::uniform_int_distribution<long long> J(28, 128); // 224 .. 1024 bytes forward
            for (long long t = 0; t < nbig; ++t) hb[t] = (t + J(rng)) % nbig;
        }
        cudaMemcpy(dbig, hb.data(), 8 * nbig, cudaMemcpyHostToDevice);
        kbig<<<1, 1>>>(dbig, nbig, 100, dout);
        kbig<<<1, 1>>>(dbig, nbig, steps, dout);
        unsigned long long h[2];
        cudaMemcpy(h, dout, 16, cudaMemcpyDeviceToHost);
        printf("mode %d: %.1f ns per link (%s)\n", mode, static_cast<double>(h[0]) / steps,
               cudaGetErrorString(cudaGetLastError()));
    }
}
