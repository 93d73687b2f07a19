/* matchamg_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C, single-threaded restatement of the reference's hot path
 * (/root/reference/proj/src, the AMG-PCG setup+solve of arXiv 1810.04221),
 * used as the parity CHECKER for the B200 kernels. Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it; the
 * product (paper_1810_04221_b200/) never links or calls it.
 *
 * Parity is pinned: tests/test_oracle.py checks every function here bit for
 * bit against the unmodified reference library built by oracle/Makefile
 * (oracle/_ref/libmatchamg_ref.so) and against the committed golden fixtures
 * in tests/golden/ (generated from that library by tests/golden/make_golden.py).
 *
 * Index type is int64 (proj/include/matchamg/csr.hpp:14); all arithmetic is
 * IEEE binary64 without contraction, in the reference's evaluation order.
 */
#ifndef MAMG_ORACLE_H
#define MAMG_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    int64_t nrows, ncols;
    int64_t* rp; /* nrows + 1 */
    int64_t* ci; /* nnz */
    double* v;   /* nnz */
} orc_csr;

orc_csr* orc_csr_new(int64_t nrows, int64_t ncols, int64_t nnz);
orc_csr* orc_csr_copy_from(int64_t nrows, int64_t ncols, const int64_t* rp,
                           const int64_t* ci, const double* v);
void orc_csr_free(orc_csr* A);
int64_t orc_csr_nnz(const orc_csr* A);

/* sparse kernels */
int orc_lane_policy(const orc_csr* A);
void orc_spmv(const orc_csr* A, int group, const double* x, double* y);
int64_t orc_l1_diagonal(const orc_csr* A, double* d); /* -1 ok, else bad row */
int orc_has_symmetric_pattern(const orc_csr* A);
orc_csr* orc_transpose(const orc_csr* A);
orc_csr* orc_spgemm(const orc_csr* A, const orc_csr* B);

/* matching; status: 0 ok, 1 non-positive diagonal, 2 asymmetric pattern,
 * 3 non-finite weight; *bad_row receives the row */
int orc_build_weights(const orc_csr* A, const double* w, int64_t* xadj,
                      int64_t* adjncy, double* weight, int64_t* zero_edges,
                      int64_t* bad_row);
void orc_suitor(int64_t n, const int64_t* xadj, const int64_t* adjncy,
                const double* weight, int64_t* mate);

/* coarsening */
/* 0 ok, 1 invalid matching */
int orc_pairwise_aggregate(int64_t n, const int64_t* mate, int64_t* agg_of,
                           int64_t* counts /* n_c, n_p, n_s */);
/* 0 ok; 1 aggregate id out of range (*bad = vertex); 2 w vanishes on an
 * aggregate of size > 1 (*bad = aggregate) */
int orc_build_prolongator(int64_t n, int64_t n_c, const int64_t* agg_of,
                          const double* w, orc_csr** P, int64_t* bad);
/* NULL when a row of P does not hold exactly one entry */
orc_csr* orc_galerkin_by_aggregates(const orc_csr* A, const orc_csr* P);
void orc_restrict_vector(const orc_csr* P, const double* w, double* wc);

typedef struct {
    orc_csr* A;
    orc_csr* P; /* NULL on the coarsest level */
    orc_csr* R;
    double* l1;
    double* w;
} orc_level;

typedef struct {
    int nl;
    orc_level* lv;
    int stalled;
    int64_t zero_edges;
} orc_hier;

/* mode 1 = Pairwise, 2 = DoublePairwise; status as build_weights, plus
 * 4 = l1 diagonal error, 5 = prolongator error, 6 = asymmetric pattern at
 * level 0; *bad receives the row/aggregate */
int orc_build_hierarchy(const orc_csr* A, const double* w, int max_levels,
                        double coarse_factor, int mode, orc_hier** out,
                        int64_t* bad);
void orc_hier_free(orc_hier* h);

/* multigrid; cycle 0 = V, 1 = W, 2 = K (K-cycle: an extension, not in the
 * reference; see kcycle_coarse in matchamg_oracle.c) */
void orc_l1_jacobi(const orc_csr* A, const double* d, const double* b,
                   double* x, int k);
void orc_apply_cycle(const orc_hier* h, int level, const double* b, double* x,
                     int cycle, int pre, int post, int coarsest);

/* vector ops */
double orc_dot(int64_t n, const double* x, const double* y);
double orc_norm2(int64_t n, const double* x);
void orc_axpy(int64_t n, double* y, double a, const double* x);
void orc_triple_dot(int64_t n, const double* w, const double* r,
                    const double* v, const double* q, double* out3);
void orc_axpy_pair(int64_t n, double* y1, double* y2, const double* x,
                   double a, double b);

typedef struct {
    int64_t iterations;
    double final_relres;
    int32_t converged;
    int32_t pad;
    double solve_ms;
    int64_t audit_checks;
    int64_t audit_failures;
    double audit_max_rel;
    int64_t breakdown_iteration;
} orc_report;

/* returns 0 ok, 3 breakdown; h == NULL -> unpreconditioned; u0 NULL -> 0;
 * hist holds itmax + 1 entries */
int orc_pcg(const orc_csr* A, const orc_hier* h, int cycle, int pre, int post,
            int coarsest, const double* b, const double* u0, double rtol,
            int64_t itmax, double* u, double* hist, orc_report* rep);

#ifdef __cplusplus
}
#endif
#endif
