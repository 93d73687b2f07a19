/* mamg_host.h — C entry points of the HOST library libmatchamg.so (the
 * matchamg C++ facade). They expose the model-problem generators
 * (proj/include/matchamg/problems.hpp) to non-C++ callers (ctypes in bench.py
 * and the tests) so every caller feeds identical matrices to the reference
 * and to the B200 path. Arrays are malloc'ed; release with mamg_host_csr_free. */
#ifndef MAMG_HOST_H
#define MAMG_HOST_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    int64_t nrows, ncols, nnz;
    int64_t* rp;
    int64_t* ci;
    double* v;
} mamg_host_csr;

/* 0 ok, 1 invalid argument (message via mamg_host_last_error) */
int mamg_gen_poisson2d(int64_t nx, int64_t ny, mamg_host_csr* out);
int mamg_gen_aniso2d(int64_t nx, int64_t ny, double epsilon, double theta, mamg_host_csr* out);
int mamg_gen_randk3d(int64_t nx, int64_t ny, int64_t nz, double sigma, uint64_t seed,
                     mamg_host_csr* out);
/* BASELINE configs 3-5 (matchamg/problems.hpp) */
int mamg_gen_aniso27(int64_t nx, int64_t ny, int64_t nz, double kx, double ky, double kz,
                     mamg_host_csr* out);
int mamg_gen_jump3d(int64_t nx, int64_t ny, int64_t nz, int64_t block, uint64_t seed, double lo,
                    double hi, mamg_host_csr* out);
int mamg_gen_elast3d(int64_t nx, int64_t ny, int64_t nz, double mu, double lambda,
                     mamg_host_csr* out);
/* MatrixMarket coordinate I/O (matchamg/matrix_market.hpp); 2 = runtime
 * error (I/O or parse; message "path:line: what"), 1 = invalid argument */
int mamg_read_mm(const char* path, mamg_host_csr* out);
int mamg_write_mm(int64_t nrows, int64_t ncols, const int64_t* rp, const int64_t* ci,
                  const double* v, const char* path, int symmetric);
void mamg_host_csr_free(mamg_host_csr* m);
const char* mamg_host_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
