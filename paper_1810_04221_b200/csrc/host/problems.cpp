// problems.cpp — model-problem generators of the matchamg API, written to
// reproduce the reference's matrices bit for bit (same formulas, same
// left-to-right evaluation, glibc libm for exp/log/sin/cos):
//   * gen_anisotropic_2d / gen_poisson_2d: proj/src/problems.cpp:13-69
//   * gen_poisson_3d_randk:                proj/src/problems.cpp:73-193
// plus new generators for BASELINE configs 3-5 (aniso Q1 27-point, jump
// coefficient FV, Q1 elasticity), which the reference does not ship.
// These are host input producers for the B200 path.
#include "matchamg/problems.hpp"

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <numbers>
#include <stdexcept>
#include <string>
#include <thread>
#include <algorithm>
#include <vector>

#include "mamg_host.h"
#include "matchamg/matrix_market.hpp"

namespace matchamg {
namespace {

// Row-by-row CSR builder with column order supplied by the caller.
struct RowBuilder {
    CsrMatrix M;
    explicit RowBuilder(index_t n, index_t per_row) {
        M.nrows = M.ncols = n;
        M.row_ptr.clear();
        M.row_ptr.reserve(n + 1);
        M.row_ptr.push_back(0);
        M.col_idx.reserve(n * per_row);
        M.values.reserve(n * per_row);
    }
    void put(index_t c, double v) {
        M.col_idx.push_back(c);
        M.values.push_back(v);
    }
    void end_row() { M.row_ptr.push_back(static_cast<index_t>(M.values.size())); }
};

CsrMatrix nine_point(index_t nx, index_t ny, double a, double b, double c) {
    if (nx < 2 || ny < 2) throw std::invalid_argument("grid must be at least 2x2");
    const double hx = 1.0 / static_cast<double>(nx + 1);
    const double hy = 1.0 / static_cast<double>(ny + 1);
    const double east_west = -a / (hx * hx);
    const double north_south = -b / (hy * hy);
    const double corner = -2.0 * c / (4.0 * hx * hy);
    const double centre = 2.0 * a / (hx * hx) + 2.0 * b / (hy * hy);
    // stencil in ascending column order: (di, dj, weight)
    const struct {
        int di, dj;
        double w;
    } st[9] = {{-1, -1, corner},  {0, -1, north_south}, {1, -1, -corner},
               {-1, 0, east_west}, {0, 0, centre},      {1, 0, east_west},
               {-1, 1, -corner},  {0, 1, north_south},  {1, 1, corner}};
    RowBuilder B(nx * ny, 9);
    for (index_t y = 0; y < ny; ++y)
        for (index_t x = 0; x < nx; ++x) {
            for (const auto& s : st) {
                const index_t xx = x + s.di, yy = y + s.dj;
                if (s.w == 0.0 || xx < 0 || xx >= nx || yy < 0 || yy >= ny) continue;
                B.put(yy * nx + xx, s.w);
            }
            B.end_row();
        }
    return std::move(B.M);
}

// splitmix64 stream -> 53-bit uniforms -> Box-Muller pairs (cached spare)
class Gaussian {
public:
    explicit Gaussian(std::uint64_t seed) : s_(seed) {}
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
        const double phi = 2.0 * std::numbers::pi * u2;
        spare_ = r * std::sin(phi);
        cached_ = true;
        return r * std::cos(phi);
    }

private:
    std::uint64_t bits() {
        std::uint64_t z = (s_ += 0x9E3779B97F4A7C15ULL);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
        return z ^ (z >> 31);
    }
    double unit() { return static_cast<double>(bits() >> 11) * 0x1.0p-53; }

    std::uint64_t s_;
    bool cached_ = false;
    double spare_ = 0.0;
};

} // namespace

CsrMatrix gen_anisotropic_2d(const AniSpec& spec) {
    if (!(spec.epsilon > 0.0)) throw std::invalid_argument("gen_anisotropic_2d: epsilon must be > 0");
    const double co = std::cos(spec.theta), si = std::sin(spec.theta);
    return nine_point(spec.nx, spec.ny, spec.epsilon + co * co, spec.epsilon + si * si, co * si);
}

CsrMatrix gen_poisson_2d(index_t nx, index_t ny) { return nine_point(nx, ny, 1.0, 1.0, 0.0); }

namespace {

// Cell-centred FV assembly of -div(K grad u) on the unit cube shared by the
// cfg 2 (lognormal K) and cfg 4 (jump K) generators: harmonic face means,
// Dirichlet closure at h/2 (proj/src/problems.cpp:150-190 evaluation order).
CsrMatrix fv7(index_t nx, index_t ny, index_t nz, const std::vector<double>& perm) {
    const index_t n = nx * ny * nz;
    const double h[3] = {1.0 / static_cast<double>(nx), 1.0 / static_cast<double>(ny),
                         1.0 / static_cast<double>(nz)};
    const index_t plane = nx * ny;
    RowBuilder B(n, 7);
    for (index_t k = 0; k < nz; ++k)
        for (index_t j = 0; j < ny; ++j)
            for (index_t i = 0; i < nx; ++i) {
                const index_t row = (k * ny + j) * nx + i;
                const double kc = perm[row];
                // faces in ascending neighbour order: -z, -y, -x | +x, +y, +z
                const struct {
                    bool inside;
                    index_t nbr;
                    int axis;
                } faces[6] = {{k > 0, row - plane, 2},   {j > 0, row - nx, 1},
                              {i > 0, row - 1, 0},       {i + 1 < nx, row + 1, 0},
                              {j + 1 < ny, row + nx, 1}, {k + 1 < nz, row + plane, 2}};
                double diag = 0.0;
                double off[6];
                index_t col[6];
                int m = 0, below = 0;
                for (int f = 0; f < 6; ++f) {
                    const double hh = h[faces[f].axis];
                    if (faces[f].inside) {
                        const double kn = perm[faces[f].nbr];
                        const double t = 2.0 / (1.0 / kc + 1.0 / kn) / (hh * hh);
                        off[m] = -t;
                        col[m] = faces[f].nbr;
                        ++m;
                        diag += t;
                    } else {
                        diag += 2.0 * kc / (hh * hh); // boundary face at h/2
                    }
                    if (f == 2) below = m;
                }
                for (int t = 0; t < below; ++t) B.put(col[t], off[t]);
                B.put(row, diag);
                for (int t = below; t < m; ++t) B.put(col[t], off[t]);
                B.end_row();
            }
    return std::move(B.M);
}

// Row-parallel CSR fill: fill(row, cols, vals) writes <= max_per_row entries
// (ascending columns) and returns the count. Rows are cut into contiguous
// chunks, one per worker; the result does not depend on the worker count.
template <class F>
CsrMatrix build_rows(index_t n, int max_per_row, F&& fill) {
    const int hw = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
    const int T = static_cast<int>(std::min<index_t>(hw, std::max<index_t>(1, n / 4096)));
    std::vector<std::vector<index_t>> cols(T);
    std::vector<std::vector<double>> vals(T);
    std::vector<index_t> cnt(n + 1, 0);
    auto work = [&](int t) {
        const index_t r0 = n * t / T, r1 = n * (t + 1) / T;
        std::vector<index_t>& C = cols[t];
        std::vector<double>& V = vals[t];
        C.reserve((r1 - r0) * max_per_row);
        V.reserve((r1 - r0) * max_per_row);
        std::vector<index_t> c(max_per_row);
        std::vector<double> v(max_per_row);
        for (index_t r = r0; r < r1; ++r) {
            const int m = fill(r, c.data(), v.data());
            cnt[r + 1] = m;
            C.insert(C.end(), c.begin(), c.begin() + m);
            V.insert(V.end(), v.begin(), v.begin() + m);
        }
    };
    std::vector<std::thread> th;
    for (int t = 1; t < T; ++t) th.emplace_back(work, t);
    work(0);
    for (auto& x : th) x.join();
    CsrMatrix M;
    M.nrows = M.ncols = n;
    M.row_ptr.assign(n + 1, 0);
    for (index_t r = 0; r < n; ++r) M.row_ptr[r + 1] = M.row_ptr[r] + cnt[r + 1];
    M.col_idx.resize(M.row_ptr[n]);
    M.values.resize(M.row_ptr[n]);
    std::vector<std::thread> cp;
    auto copy = [&](int t) {
        const index_t at = M.row_ptr[n * t / T];
        std::memcpy(M.col_idx.data() + at, cols[t].data(), sizeof(index_t) * cols[t].size());
        std::memcpy(M.values.data() + at, vals[t].data(), sizeof(double) * vals[t].size());
    };
    for (int t = 1; t < T; ++t) cp.emplace_back(copy, t);
    copy(0);
    for (auto& x : cp) x.join();
    return M;
}

std::uint64_t splitmix64(std::uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

} // namespace

CsrMatrix gen_poisson_3d_randk(const RandPermSpec& spec) {
    const index_t nx = spec.nx, ny = spec.ny, nz = spec.nz;
    if (nx < 2 || ny < 2 || nz < 2)
        throw std::invalid_argument("gen_poisson_3d_randk: grid must be >= 2^3");
    if (spec.sigma < 0.0) throw std::invalid_argument("gen_poisson_3d_randk: sigma must be >= 0");
    // ln K ~ N(mu, s^2), s^2 = ln(1 + sigma^2), mu = -s^2 / 2  (mean 1)
    const double var = std::log1p(spec.sigma * spec.sigma);
    const double sd = std::sqrt(var);
    const double mu = -0.5 * var;
    const index_t n = nx * ny * nz;
    std::vector<double> perm(n);
    Gaussian g(spec.seed);
    for (index_t c = 0; c < n; ++c) perm[c] = std::exp(mu + sd * g());
    return fv7(nx, ny, nz, perm);
}

CsrMatrix gen_jump_3d(const JumpSpec& spec) {
    const index_t nx = spec.nx, ny = spec.ny, nz = spec.nz;
    if (nx < 2 || ny < 2 || nz < 2) throw std::invalid_argument("gen_jump_3d: grid must be >= 2^3");
    if (spec.block < 1) throw std::invalid_argument("gen_jump_3d: block must be >= 1");
    if (!(spec.lo > 0.0) || !(spec.hi > 0.0))
        throw std::invalid_argument("gen_jump_3d: coefficients must be > 0");
    const double K[3] = {spec.lo, 1.0, spec.hi};
    const index_t bx = (nx + spec.block - 1) / spec.block, by = (ny + spec.block - 1) / spec.block;
    std::vector<double> perm(nx * ny * nz);
    for (index_t k = 0; k < nz; ++k)
        for (index_t j = 0; j < ny; ++j)
            for (index_t i = 0; i < nx; ++i) {
                const index_t cube = ((k / spec.block) * by + j / spec.block) * bx + i / spec.block;
                const std::uint64_t hsh =
                    splitmix64(spec.seed * 0x100000001B3ULL ^ static_cast<std::uint64_t>(cube));
                perm[(k * ny + j) * nx + i] = K[hsh % 3];
            }
    return fv7(nx, ny, nz, perm);
}

CsrMatrix gen_anisotropic_3d_q1(const Aniso27Spec& spec) {
    const index_t nx = spec.nx, ny = spec.ny, nz = spec.nz;
    if (nx < 2 || ny < 2 || nz < 2)
        throw std::invalid_argument("gen_anisotropic_3d_q1: grid must be >= 2^3");
    if (!(spec.kx > 0.0) || !(spec.ky > 0.0) || !(spec.kz > 0.0))
        throw std::invalid_argument("gen_anisotropic_3d_q1: coefficients must be > 0");
    const double hx = 1.0 / static_cast<double>(nx + 1), hy = 1.0 / static_cast<double>(ny + 1),
                 hz = 1.0 / static_cast<double>(nz + 1);
    // assembled 1D stiffness (x h) and mass (/ h) stencils, offsets -1, 0, +1
    const double K1[3] = {-1.0, 2.0, -1.0};
    const double M1[3] = {1.0 / 6.0, 2.0 / 3.0, 1.0 / 6.0};
    const double sx = spec.kx * ((hy * hz) / hx), sy = spec.ky * ((hx * hz) / hy),
                 sz = spec.kz * ((hx * hy) / hz);
    double S[27]; // S[(dz+1)*9 + (dy+1)*3 + (dx+1)]
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b)
            for (int c = 0; c < 3; ++c)
                S[a * 9 + b * 3 + c] = (sx * ((K1[c] * M1[b]) * M1[a]) +
                                        sy * ((M1[c] * K1[b]) * M1[a])) +
                                       sz * ((M1[c] * M1[b]) * K1[a]);
    const index_t plane = nx * ny;
    return build_rows(nx * ny * nz, 27, [&](index_t row, index_t* col, double* val) {
        const index_t i = row % nx, j = (row / nx) % ny, k = row / plane;
        int m = 0;
        for (int dz = -1; dz <= 1; ++dz)
            for (int dy = -1; dy <= 1; ++dy)
                for (int dx = -1; dx <= 1; ++dx) {
                    const index_t ii = i + dx, jj = j + dy, kk = k + dz;
                    if (ii < 0 || ii >= nx || jj < 0 || jj >= ny || kk < 0 || kk >= nz) continue;
                    const double s = S[(dz + 1) * 9 + (dy + 1) * 3 + (dx + 1)];
                    const bool diag = dx == 0 && dy == 0 && dz == 0;
                    if (s == 0.0 && !diag) continue;
                    col[m] = (kk * ny + jj) * nx + ii;
                    val[m++] = s;
                }
        return m;
    });
}

CsrMatrix gen_elasticity_3d(const ElasticitySpec& spec) {
    const index_t nx = spec.nx, ny = spec.ny, nz = spec.nz;
    if (nx < 1 || ny < 2 || nz < 2)
        throw std::invalid_argument("gen_elasticity_3d: need nx >= 1, ny >= 2, nz >= 2");
    if (!(spec.mu > 0.0) || !(spec.lambda >= 0.0))
        throw std::invalid_argument("gen_elasticity_3d: need mu > 0, lambda >= 0");
    const double h = 1.0 / static_cast<double>(nx);
    // Q1 element matrix on an h-cube, exact tensor-product integrals:
    // J(a,b,p,q) = int d_p phi_a d_q phi_b = prod_d F_d, with per axis
    //   F = (a==b ? 1 : -1)/h (d==p==q), +-1/2 (d in {p,q} once), h(1/3 | 1/6)
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
    // Ke[(a*3+i)*24 + b*3+j] = lambda J(a,b,i,j) + mu (delta_ij sum_d J(a,b,d,d) + J(a,b,j,i))
    std::vector<double> Ke(24 * 24);
    for (int a = 0; a < 8; ++a)
        for (int i = 0; i < 3; ++i)
            for (int b = 0; b < 8; ++b)
                for (int j = 0; j < 3; ++j) {
                    const double lap = i == j ? (J(a, b, 0, 0) + J(a, b, 1, 1)) + J(a, b, 2, 2) : 0.0;
                    Ke[(a * 3 + i) * 24 + b * 3 + j] =
                        spec.lambda * J(a, b, i, j) + spec.mu * (lap + J(a, b, j, i));
                }
    const index_t plane = nx * ny;
    return build_rows(3 * nx * ny * nz, 81, [&](index_t row, index_t* col, double* val) {
        const int r = static_cast<int>(row % 3);
        const index_t node = row / 3;
        const index_t i = node % nx, j = (node / nx) % ny, k = node / plane;
        int m = 0;
        for (int dz = -1; dz <= 1; ++dz)
            for (int dy = -1; dy <= 1; ++dy)
                for (int dx = -1; dx <= 1; ++dx) {
                    const index_t ii = i + dx, jj = j + dy, kk = k + dz;
                    if (ii < 0 || ii >= nx || jj < 0 || jj >= ny || kk < 0 || kk >= nz) continue;
                    for (int c = 0; c < 3; ++c) {
                        // elements (lower corners ex, ey, ez) holding both nodes, ascending
                        double s = 0.0;
                        bool first = true;
                        for (index_t ez = std::max(k, kk) - 1; ez <= std::min(k, kk); ++ez) {
                            if (ez < 0 || ez > nz - 2) continue;
                            for (index_t ey = std::max(j, jj) - 1; ey <= std::min(j, jj); ++ey) {
                                if (ey < 0 || ey > ny - 2) continue;
                                for (index_t ex = std::max(i, ii) - 1; ex <= std::min(i, ii); ++ex) {
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
                        col[m] = 3 * ((kk * ny + jj) * nx + ii) + c;
                        val[m++] = s;
                    }
                }
        return m;
    });
}

} // namespace matchamg

// ------------------------------------------------------------------ C ABI --
namespace {
thread_local std::string g_host_err;

int export_csr(const matchamg::CsrMatrix& A, mamg_host_csr* out) {
    out->nrows = A.nrows;
    out->ncols = A.ncols;
    out->nnz = A.nnz();
    out->rp = static_cast<int64_t*>(std::malloc(sizeof(int64_t) * (A.nrows + 1)));
    out->ci = static_cast<int64_t*>(std::malloc(sizeof(int64_t) * (A.nnz() ? A.nnz() : 1)));
    out->v = static_cast<double*>(std::malloc(sizeof(double) * (A.nnz() ? A.nnz() : 1)));
    if (!out->rp || !out->ci || !out->v) return 2;
    std::memcpy(out->rp, A.row_ptr.data(), sizeof(int64_t) * (A.nrows + 1));
    std::memcpy(out->ci, A.col_idx.data(), sizeof(int64_t) * A.nnz());
    std::memcpy(out->v, A.values.data(), sizeof(double) * A.nnz());
    return 0;
}

template <class F>
int run(F&& f, mamg_host_csr* out) {
    try {
        return export_csr(f(), out);
    } catch (const std::invalid_argument& e) {
        g_host_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_host_err = e.what();
        return 2;
    }
}
} // namespace

extern "C" {
int mamg_gen_poisson2d(int64_t nx, int64_t ny, mamg_host_csr* out) {
    return run([&] { return matchamg::gen_poisson_2d(nx, ny); }, out);
}
int mamg_gen_aniso2d(int64_t nx, int64_t ny, double eps, double theta, mamg_host_csr* out) {
    return run([&] { return matchamg::gen_anisotropic_2d({nx, ny, eps, theta}); }, out);
}
int mamg_gen_randk3d(int64_t nx, int64_t ny, int64_t nz, double sigma, uint64_t seed,
                     mamg_host_csr* out) {
    return run([&] { return matchamg::gen_poisson_3d_randk({nx, ny, nz, sigma, seed}); }, out);
}
int mamg_gen_aniso27(int64_t nx, int64_t ny, int64_t nz, double kx, double ky, double kz,
                     mamg_host_csr* out) {
    return run([&] { return matchamg::gen_anisotropic_3d_q1({nx, ny, nz, kx, ky, kz}); }, out);
}
int mamg_gen_jump3d(int64_t nx, int64_t ny, int64_t nz, int64_t block, uint64_t seed, double lo,
                    double hi, mamg_host_csr* out) {
    return run([&] { return matchamg::gen_jump_3d({nx, ny, nz, block, seed, lo, hi}); }, out);
}
int mamg_gen_elast3d(int64_t nx, int64_t ny, int64_t nz, double mu, double lambda,
                     mamg_host_csr* out) {
    return run([&] { return matchamg::gen_elasticity_3d({nx, ny, nz, mu, lambda}); }, out);
}
int mamg_read_mm(const char* path, mamg_host_csr* out) {
    return run([&] { return matchamg::read_matrix_market(path); }, out);
}
int mamg_write_mm(int64_t nrows, int64_t ncols, const int64_t* rp, const int64_t* ci,
                  const double* v, const char* path, int symmetric) {
    try {
        matchamg::CsrMatrix A;
        A.nrows = nrows;
        A.ncols = ncols;
        A.row_ptr.assign(rp, rp + nrows + 1);
        A.col_idx.assign(ci, ci + rp[nrows]);
        A.values.assign(v, v + rp[nrows]);
        matchamg::write_matrix_market(A, path, symmetric != 0);
        return 0;
    } catch (const std::invalid_argument& e) {
        g_host_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_host_err = e.what();
        return 2;
    }
}
void mamg_host_csr_free(mamg_host_csr* m) {
    if (!m) return;
    std::free(m->rp);
    std::free(m->ci);
    std::free(m->v);
    m->rp = m->ci = nullptr;
    m->v = nullptr;
}
const char* mamg_host_last_error(void) { return g_host_err.c_str(); }
}
