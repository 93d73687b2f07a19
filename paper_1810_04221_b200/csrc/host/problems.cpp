// problems.cpp — model-problem generators of the matchamg API, written to
// reproduce the reference's matrices bit for bit (same formulas, same
// left-to-right evaluation, glibc libm for exp/log/sin/cos):
//   * gen_anisotropic_2d / gen_poisson_2d: proj/src/problems.cpp:13-69
//   * gen_poisson_3d_randk:                proj/src/problems.cpp:73-193
// These are host input producers for the B200 path.
#include "matchamg/problems.hpp"

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <numbers>
#include <stdexcept>
#include <string>

#include "mamg_host.h"

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
