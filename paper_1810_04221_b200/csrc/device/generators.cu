// generators.cu — the BASELINE problem generators evaluated on the device
// (the input side of the path at large sizes). The
// matrix is assembled directly in HBM, one thread per row, with the host
// generators' exact arithmetic and entry order (csrc/host/problems.cpp: cfg 1
// nine_point, cfg 2 / cfg 4 fv7 — proj/src/problems.cpp:150-190 evaluation
// order —, cfg 3 Q1 27-point, cfg 5 Q1 elasticity): bit-identical matrices
// without a host CSR or an upload (cfg 5: 150 M entries). The few small
// tables (the 27-point stencil, the 24x24 element matrix, the lognormal
// permeability field for sigma > 0) are computed on the host exactly as
// there. Count pass -> scan -> fill pass.
#include <cmath>
#include <stdexcept>
#include <vector>

#include "ops.cuh"

namespace mamg {
namespace {

constexpr int kBlock = 256;
// std::numbers::pi (the double nearest pi)
constexpr double kPi = 3.141592653589793238462643383279502884;

// ---- cfg 1 (2D nine-point, gen_poisson_2d / gen_anisotropic_2d) ----------
struct GenNine {
    int64_t nx, ny;
    double w[9];
    __device__ int row(int64_t r, int32_t* col, double* val) const {
        const int64_t x = r % nx, y = r / nx;
        int m = 0;
#pragma unroll
        for (int s = 0; s < 9; ++s) {
            const int64_t xx = x + (s % 3) - 1, yy = y + (s / 3) - 1;
            if (w[s] == 0.0 || xx < 0 || xx >= nx || yy < 0 || yy >= ny) continue;
            if (col) {
                col[m] = static_cast<int32_t>(yy * nx + xx);
                val[m] = w[s];
            }
            ++m;
        }
        return m;
    }
};

// ---- cfg 2 / cfg 4 (7-point cell-centred FV, harmonic face means) --------
struct GenFv7 {
    int64_t nx, ny, nz;
    double h[3];
    const double* perm;
    __device__ int row(int64_t r, int32_t* col, double* val) const {
        const int64_t plane = nx * ny;
        const int64_t i = r % nx, j = (r / nx) % ny, k = r / plane;
        const double kc = perm[r];
        const bool inside[6] = {k > 0, j > 0, i > 0, i + 1 < nx, j + 1 < ny, k + 1 < nz};
        const int64_t nbr[6] = {r - plane, r - nx, r - 1, r + 1, r + nx, r + plane};
        const int axis[6] = {2, 1, 0, 0, 1, 2};
        double diag = 0.0, off[6];
        int64_t cc[6];
        int m = 0, below = 0;
#pragma unroll
        for (int f = 0; f < 6; ++f) {
            const double hh = h[axis[f]];
            if (inside[f]) {
                const double kn = perm[nbr[f]];
                const double t = 2.0 / (1.0 / kc + 1.0 / kn) / (hh * hh);
                off[m] = -t;
                cc[m] = nbr[f];
                ++m;
                diag += t;
            } else {
                diag += 2.0 * kc / (hh * hh); // boundary face at h/2
            }
            if (f == 2) below = m;
        }
        if (col) {
            int at = 0;
            for (int t = 0; t < below; ++t, ++at) {
                col[at] = static_cast<int32_t>(cc[t]);
                val[at] = off[t];
            }
            col[at] = static_cast<int32_t>(r);
            val[at] = diag;
            ++at;
            for (int t = below; t < m; ++t, ++at) {
                col[at] = static_cast<int32_t>(cc[t]);
                val[at] = off[t];
            }
        }
        return m + 1;
    }
};

// ---- cfg 3 (Q1 27-point anisotropic) --------------------------------------
struct GenQ27 {
    int64_t nx, ny, nz;
    double S[27];
    __device__ int row(int64_t r, int32_t* col, double* val) const {
        const int64_t plane = nx * ny;
        const int64_t i = r % nx, j = (r / nx) % ny, k = r / plane;
        int m = 0;
        for (int dz = -1; dz <= 1; ++dz)
            for (int dy = -1; dy <= 1; ++dy)
                for (int dx = -1; dx <= 1; ++dx) {
                    const int64_t ii = i + dx, jj = j + dy, kk = k + dz;
                    if (ii < 0 || ii >= nx || jj < 0 || jj >= ny || kk < 0 || kk >= nz) continue;
                    const double s = S[(dz + 1) * 9 + (dy + 1) * 3 + (dx + 1)];
                    const bool diag = dx == 0 && dy == 0 && dz == 0;
                    if (s == 0.0 && !diag) continue;
                    if (col) {
                        col[m] = static_cast<int32_t>((kk * ny + jj) * nx + ii);
                        val[m] = s;
                    }
                    ++m;
                }
        return m;
    }
};

// ---- cfg 5 (Q1 elasticity, 3 interleaved dofs per node) ------------------
struct GenElast {
    int64_t nx, ny, nz;
    const double* Ke; // 24 x 24 element matrix
    __device__ int row(int64_t row, int32_t* col, double* val) const {
        const int r = static_cast<int>(row % 3);
        const int64_t node = row / 3;
        const int64_t plane = nx * ny;
        const int64_t i = node % nx, j = (node / nx) % ny, k = node / plane;
        int m = 0;
        for (int dz = -1; dz <= 1; ++dz)
            for (int dy = -1; dy <= 1; ++dy)
                for (int dx = -1; dx <= 1; ++dx) {
                    const int64_t ii = i + dx, jj = j + dy, kk = k + dz;
                    if (ii < 0 || ii >= nx || jj < 0 || jj >= ny || kk < 0 || kk >= nz) continue;
                    for (int c = 0; c < 3; ++c) {
                        // elements (lower corners ex, ey, ez) holding both nodes, ascending
                        double s = 0.0;
                        bool first = true;
                        for (int64_t ez = (k > kk ? k : kk) - 1; ez <= (k < kk ? k : kk); ++ez) {
                            if (ez < 0 || ez > nz - 2) continue;
                            for (int64_t ey = (j > jj ? j : jj) - 1; ey <= (j < jj ? j : jj); ++ey) {
                                if (ey < 0 || ey > ny - 2) continue;
                                for (int64_t ex = (i > ii ? i : ii) - 1; ex <= (i < ii ? i : ii); ++ex) {
                                    if (ex < -1 || ex > nx - 2) continue;
                                    const int a = static_cast<int>((i - ex) | ((j - ey) << 1) | ((k - ez) << 2));
                                    const int b = static_cast<int>((ii - ex) | ((jj - ey) << 1) | ((kk - ez) << 2));
                                    const double e = Ke[(a * 3 + r) * 24 + b * 3 + c];
                                    s = first ? e : s + e;
                                    first = false;
                                }
                            }
                        }
                        const bool diag = dx == 0 && dy == 0 && dz == 0 && c == r;
                        if (first || (s == 0.0 && !diag)) continue;
                        if (col) {
                            col[m] = static_cast<int32_t>(3 * ((kk * ny + jj) * nx + ii) + c);
                            val[m] = s;
                        }
                        ++m;
                    }
                }
        return m;
    }
};

template <class Gen>
__global__ void k_gen_count(int64_t n, const Gen g, int32_t* cnt) {
    const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r < n) cnt[r] = g.row(r, nullptr, nullptr);
}

template <class Gen>
__global__ void k_gen_fill(int64_t n, const Gen g, const int32_t* __restrict__ rp, int32_t* ci,
                           double* v) {
    const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r < n) g.row(r, ci + rp[r], v + rp[r]);
}

__device__ __forceinline__ uint64_t splitmix64_d(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

// cfg 4 permeability: seeded piecewise-constant sub-cubes (gen_jump_3d)
__global__ void k_jump_perm(int64_t nx, int64_t ny, int64_t nz, int64_t block, uint64_t seed,
                            double lo, double hi, double* perm) {
    const int64_t c = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (c >= nx * ny * nz) return;
    const int64_t i = c % nx, j = (c / nx) % ny, k = c / (nx * ny);
    const int64_t bx = (nx + block - 1) / block, by = (ny + block - 1) / block;
    const int64_t cube = ((k / block) * by + j / block) * bx + i / block;
    const uint64_t h = splitmix64_d(seed * 0x100000001B3ULL ^ static_cast<uint64_t>(cube));
    const double K[3] = {lo, 1.0, hi};
    perm[c] = K[h % 3];
}

__global__ void k_fill_const(int64_t n, double* x, double v) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) x[i] = v;
}

template <class Gen>
std::unique_ptr<DevCsr> assemble(Ctx& c, int64_t n, const Gen& g) {
    if (n >= (int64_t{1} << 31) - 1) invalid("generator: matrix too large for int32 indices");
    auto A = std::make_unique<DevCsr>();
    A->nrows = A->ncols = n;
    A->rp.alloc(n + 1, c.stream);
    if (n) {
        k_gen_count<<<blocks_for(n, kBlock), kBlock, 0, c.stream>>>(n, g, A->rp.get());
        c.count();
    }
    exclusive_scan_i32(c, A->rp.get(), A->rp.get(), n);
    A->nnz = read_i32(c, A->rp.get() + n);
    A->ci.alloc(A->nnz, c.stream);
    A->v.alloc(A->nnz, c.stream);
    if (n) {
        k_gen_fill<<<blocks_for(n, kBlock), kBlock, 0, c.stream>>>(n, g, A->rp.get(), A->ci.get(),
                                                                   A->v.get());
        c.count();
    }
    MAMG_LAUNCH_CHECK();
    csr_finalize(c, *A);
    return A;
}

// splitmix64 stream -> 53-bit uniforms -> Box-Muller pairs (cached spare):
// the host generator's Gaussian, evaluated on the host (same libm)
class HostGaussian {
public:
    explicit HostGaussian(uint64_t seed) : s_(seed) {}
    double operator()() {
        if (cached_) {
            cached_ = false;
            return spare_;
        }
        double u1;
        do {
            u1 = unit();
        } while (u1 == 0.0);
        const double u2 = unit();
        const double r = std::sqrt(-2.0 * std::log(u1));
        const double phi = 2.0 * kPi * u2;
        spare_ = r * std::sin(phi);
        cached_ = true;
        return r * std::cos(phi);
    }

private:
    uint64_t bits() {
        uint64_t z = (s_ += 0x9E3779B97F4A7C15ULL);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
        return z ^ (z >> 31);
    }
    double unit() { return static_cast<double>(bits() >> 11) * 0x1.0p-53; }
    uint64_t s_;
    bool cached_ = false;
    double spare_ = 0.0;
};

} // namespace

std::unique_ptr<DevCsr> gen_nine_point_dev(Ctx& c, int64_t nx, int64_t ny, double a, double b,
                                           double cc) {
    if (nx < 2 || ny < 2) invalid("grid must be at least 2x2");
    const double hx = 1.0 / static_cast<double>(nx + 1);
    const double hy = 1.0 / static_cast<double>(ny + 1);
    const double east_west = -a / (hx * hx);
    const double north_south = -b / (hy * hy);
    const double corner = -2.0 * cc / (4.0 * hx * hy);
    const double centre = 2.0 * a / (hx * hx) + 2.0 * b / (hy * hy);
    GenNine g{nx, ny, {corner, north_south, -corner, east_west, centre, east_west, -corner,
                       north_south, corner}};
    return assemble(c, nx * ny, g);
}

std::unique_ptr<DevCsr> gen_randk3d_dev(Ctx& c, int64_t nx, int64_t ny, int64_t nz, double sigma,
                                        uint64_t seed) {
    if (nx < 2 || ny < 2 || nz < 2) invalid("gen_poisson_3d_randk: grid must be >= 2^3");
    if (sigma < 0.0) invalid("gen_poisson_3d_randk: sigma must be >= 0");
    const int64_t n = nx * ny * nz;
    DBuf<double> perm(n, c.stream);
    if (sigma == 0.0) {
        // exp(mu + sd * g) with sd = 0, mu = -0: every K is exactly 1.0
        k_fill_const<<<blocks_for(n, kBlock), kBlock, 0, c.stream>>>(n, perm.get(), 1.0);
        c.count();
    } else {
        const double var = std::log1p(sigma * sigma);
        const double sd = std::sqrt(var);
        const double mu = -0.5 * var;
        std::vector<double> hp(n);
        HostGaussian g(seed);
        for (int64_t i = 0; i < n; ++i) hp[i] = std::exp(mu + sd * g());
        upload_f64(c, perm.get(), hp.data(), static_cast<size_t>(n));
    }
    GenFv7 gen{nx, ny, nz, {1.0 / static_cast<double>(nx), 1.0 / static_cast<double>(ny),
                            1.0 / static_cast<double>(nz)}, perm.get()};
    auto A = assemble(c, n, gen);
    c.sync(); // perm is released below
    return A;
}

std::unique_ptr<DevCsr> gen_jump3d_dev(Ctx& c, int64_t nx, int64_t ny, int64_t nz, int64_t block,
                                       uint64_t seed, double lo, double hi) {
    if (nx < 2 || ny < 2 || nz < 2) invalid("gen_jump_3d: grid must be >= 2^3");
    if (block < 1) invalid("gen_jump_3d: block must be >= 1");
    if (!(lo > 0.0) || !(hi > 0.0)) invalid("gen_jump_3d: coefficients must be > 0");
    const int64_t n = nx * ny * nz;
    DBuf<double> perm(n, c.stream);
    k_jump_perm<<<blocks_for(n, kBlock), kBlock, 0, c.stream>>>(nx, ny, nz, block, seed, lo, hi,
                                                                perm.get());
    c.count();
    GenFv7 gen{nx, ny, nz, {1.0 / static_cast<double>(nx), 1.0 / static_cast<double>(ny),
                            1.0 / static_cast<double>(nz)}, perm.get()};
    auto A = assemble(c, n, gen);
    c.sync();
    return A;
}

std::unique_ptr<DevCsr> gen_aniso27_dev(Ctx& c, int64_t nx, int64_t ny, int64_t nz, double kx,
                                        double ky, double kz) {
    if (nx < 2 || ny < 2 || nz < 2) invalid("gen_anisotropic_3d_q1: grid must be >= 2^3");
    if (!(kx > 0.0) || !(ky > 0.0) || !(kz > 0.0))
        invalid("gen_anisotropic_3d_q1: coefficients must be > 0");
    const double hx = 1.0 / static_cast<double>(nx + 1), hy = 1.0 / static_cast<double>(ny + 1),
                 hz = 1.0 / static_cast<double>(nz + 1);
    const double K1[3] = {-1.0, 2.0, -1.0};
    const double M1[3] = {1.0 / 6.0, 2.0 / 3.0, 1.0 / 6.0};
    const double sx = kx * ((hy * hz) / hx), sy = ky * ((hx * hz) / hy), sz = kz * ((hx * hy) / hz);
    GenQ27 g{nx, ny, nz, {}};
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b)
            for (int cidx = 0; cidx < 3; ++cidx)
                g.S[a * 9 + b * 3 + cidx] = (sx * ((K1[cidx] * M1[b]) * M1[a]) +
                                             sy * ((M1[cidx] * K1[b]) * M1[a])) +
                                            sz * ((M1[cidx] * M1[b]) * K1[a]);
    return assemble(c, nx * ny * nz, g);
}

std::unique_ptr<DevCsr> gen_elast3d_dev(Ctx& c, int64_t nx, int64_t ny, int64_t nz, double mu,
                                        double lambda) {
    if (nx < 1 || ny < 2 || nz < 2) invalid("gen_elasticity_3d: need nx >= 1, ny >= 2, nz >= 2");
    if (!(mu > 0.0) || !(lambda >= 0.0)) invalid("gen_elasticity_3d: need mu > 0, lambda >= 0");
    const double h = 1.0 / static_cast<double>(nx);
    auto F = [&](int d, int p, int q, int ad, int bd) -> double {
        if (d == p && d == q) return (ad == bd ? 1.0 : -1.0) / h;
        if (d == p) return ad ? 0.5 : -0.5;
        if (d == q) return bd ? 0.5 : -0.5;
        return h * (ad == bd ? 1.0 / 3.0 : 1.0 / 6.0);
    };
    auto J = [&](int a, int b, int p, int q) {
        return (F(0, p, q, a & 1, b & 1) * F(1, p, q, (a >> 1) & 1, (b >> 1) & 1)) *
               F(2, p, q, a >> 2, b >> 2);
    };
    std::vector<double> Ke(24 * 24);
    for (int a = 0; a < 8; ++a)
        for (int i = 0; i < 3; ++i)
            for (int b = 0; b < 8; ++b)
                for (int j = 0; j < 3; ++j) {
                    const double lap = i == j ? (J(a, b, 0, 0) + J(a, b, 1, 1)) + J(a, b, 2, 2) : 0.0;
                    Ke[(a * 3 + i) * 24 + b * 3 + j] = lambda * J(a, b, i, j) + mu * (lap + J(a, b, j, i));
                }
    DBuf<double> dKe(Ke.size(), c.stream);
    MAMG_CU(cudaMemcpyAsync(dKe.get(), Ke.data(), sizeof(double) * Ke.size(), cudaMemcpyHostToDevice,
                            c.stream));
    GenElast g{nx, ny, nz, dKe.get()};
    auto A = assemble(c, 3 * nx * ny * nz, g);
    c.sync(); // Ke (pageable source, device copy) released below
    return A;
}

} // namespace mamg
