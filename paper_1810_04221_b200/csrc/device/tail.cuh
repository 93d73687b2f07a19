// tail.cuh — parameters of the single-launch coarse-level cycle (tail.cu).
#pragma once

#include "common.cuh"

namespace mamg {

constexpr int kMaxTail = 16; // levels the tail kernel may own

struct TailLevel {
    int n = 0, nc = 0;     // rows of this level / of the next coarser one
    int G = 2, GR = 2;     // lane policies of A and R
    const int32_t* rp = nullptr;
    const int32_t* ci = nullptr;
    const double* v = nullptr;
    const double* l1 = nullptr;
    const int32_t* Rrp = nullptr; // R = P^T (rows = aggregates)
    const int32_t* Rci = nullptr;
    const double* Rv = nullptr;
    const int32_t* Pci = nullptr; // P: one entry per row
    const double* Pv = nullptr;
    double* xw = nullptr;
    double* scratch = nullptr;
    double* cb = nullptr;
    double* cx = nullptr;
};

struct TailParams {
    TailLevel lv[kMaxTail];
    int nlev = 0;
    int cycle = 0, pre = 1, post = 1, coarsest = 20;
    int zero = 1;
    int cache_coarsest = 0;
    const double* b = nullptr;
    double* x_out = nullptr;
    const int* gate = nullptr;
};

bool tail_supported(Ctx& c);
// largest usable thread-block cluster size (16 when non-portable sizes work)
int cluster_size_limit();
void tail_launch(Ctx& c, const TailParams& P);

} // namespace mamg
