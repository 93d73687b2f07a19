/* matchamg_oracle.c — TEST INFRASTRUCTURE ONLY (see matchamg_oracle.h).
 *
 * Sequential C restatement of the reference's setup+solve path. Each function
 * names the reference code it restates (paths relative to
 * /root/reference/proj). The arithmetic is written out operation by
 * operation, in the reference's order, so the results are bit-identical; it
 * is compiled with -ffp-contract=off.
 */
#define _POSIX_C_SOURCE 199309L
#include "matchamg_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#define ORC_BLOCK 2048 /* src/vector_ops.cpp:12 */

static void* xmalloc(size_t bytes) {
    void* p = malloc(bytes ? bytes : 1);
    if (!p) abort();
    return p;
}
static void* xcalloc(size_t n, size_t sz) {
    void* p = calloc(n ? n : 1, sz);
    if (!p) abort();
    return p;
}

/* ------------------------------------------------------------------ CSR --- */
orc_csr* orc_csr_new(int64_t nrows, int64_t ncols, int64_t nnz) {
    orc_csr* A = xmalloc(sizeof(orc_csr));
    A->nrows = nrows;
    A->ncols = ncols;
    A->rp = xcalloc((size_t)nrows + 1, sizeof(int64_t));
    A->ci = xmalloc(sizeof(int64_t) * (size_t)nnz);
    A->v = xmalloc(sizeof(double) * (size_t)nnz);
    return A;
}

orc_csr* orc_csr_copy_from(int64_t nrows, int64_t ncols, const int64_t* rp,
                           const int64_t* ci, const double* v) {
    const int64_t nnz = rp[nrows];
    orc_csr* A = orc_csr_new(nrows, ncols, nnz);
    memcpy(A->rp, rp, sizeof(int64_t) * (size_t)(nrows + 1));
    memcpy(A->ci, ci, sizeof(int64_t) * (size_t)nnz);
    memcpy(A->v, v, sizeof(double) * (size_t)nnz);
    return A;
}

void orc_csr_free(orc_csr* A) {
    if (!A) return;
    free(A->rp);
    free(A->ci);
    free(A->v);
    free(A);
}

int64_t orc_csr_nnz(const orc_csr* A) { return A->rp[A->nrows]; }

/* binary search of column j in row i (src/csr.cpp:10-16): position or -1 */
static int64_t find_pos(const orc_csr* A, int64_t i, int64_t j) {
    int64_t lo = A->rp[i], hi = A->rp[i + 1];
    while (lo < hi) {
        const int64_t mid = lo + (hi - lo) / 2;
        if (A->ci[mid] < j)
            lo = mid + 1;
        else
            hi = mid;
    }
    return (lo < A->rp[i + 1] && A->ci[lo] == j) ? lo : -1;
}

/* --------------------------------------------------------- sparse kernels --- */
/* src/kernels.cpp:11-24 */
int orc_lane_policy(const orc_csr* A) {
    const int64_t n = A->nrows, nnz = orc_csr_nnz(A);
    if (n > 0 && nnz == n) {
        int single = 1;
        for (int64_t i = 0; i < n && single; ++i) single = (A->rp[i + 1] - A->rp[i]) == 1;
        if (single) return 1;
    }
    const double mean = n > 0 ? (double)nnz / (double)n : 0.0;
    for (int g = 2; g <= 32; g *= 2)
        if ((double)g >= mean) return g;
    return 32;
}

/* src/kernels.cpp:36-61: lane l sums entries lo+l, lo+l+G, ... from 0.0;
 * the lanes fold with a halving tree (acc[l] += acc[l+off]). */
void orc_spmv(const orc_csr* A, int group, const double* x, double* y) {
    double lane[32];
    for (int64_t i = 0; i < A->nrows; ++i) {
        const int64_t lo = A->rp[i], hi = A->rp[i + 1];
        if (group == 1) {
            double s = 0.0;
            for (int64_t k = lo; k < hi; ++k) s = s + A->v[k] * x[A->ci[k]];
            y[i] = s;
            continue;
        }
        for (int l = 0; l < group; ++l) {
            double s = 0.0;
            for (int64_t k = lo + l; k < hi; k += group) s = s + A->v[k] * x[A->ci[k]];
            lane[l] = s;
        }
        for (int half = group >> 1; half >= 1; half >>= 1)
            for (int l = 0; l < half; ++l) lane[l] = lane[l] + lane[l + half];
        y[i] = lane[0];
    }
}

/* src/kernels.cpp:295-324 */
int64_t orc_l1_diagonal(const orc_csr* A, double* d) {
    for (int64_t i = 0; i < A->nrows; ++i) {
        double dg = 0.0, off = 0.0;
        int seen = 0;
        for (int64_t k = A->rp[i]; k < A->rp[i + 1]; ++k) {
            if (A->ci[k] == i) {
                dg = A->v[k];
                seen = 1;
            } else {
                off = off + fabs(A->v[k]);
            }
        }
        d[i] = (!seen || dg == 0.0) ? NAN : dg + off;
    }
    for (int64_t i = 0; i < A->nrows; ++i)
        if (isnan(d[i])) return i;
    return -1;
}

/* src/csr.cpp:106-112 */
int orc_has_symmetric_pattern(const orc_csr* A) {
    if (A->nrows != A->ncols) return 0;
    for (int64_t i = 0; i < A->nrows; ++i)
        for (int64_t k = A->rp[i]; k < A->rp[i + 1]; ++k)
            if (find_pos(A, A->ci[k], i) < 0) return 0;
    return 1;
}

/* src/kernels.cpp:116-134: counting sort by column, scatter in row order */
orc_csr* orc_transpose(const orc_csr* A) {
    const int64_t nnz = orc_csr_nnz(A);
    orc_csr* B = orc_csr_new(A->ncols, A->nrows, nnz);
    for (int64_t k = 0; k < nnz; ++k) B->rp[A->ci[k] + 1]++;
    for (int64_t j = 0; j < A->ncols; ++j) B->rp[j + 1] += B->rp[j];
    int64_t* fill = xmalloc(sizeof(int64_t) * (size_t)(A->ncols + 1));
    memcpy(fill, B->rp, sizeof(int64_t) * (size_t)(A->ncols + 1));
    for (int64_t i = 0; i < A->nrows; ++i)
        for (int64_t k = A->rp[i]; k < A->rp[i + 1]; ++k) {
            const int64_t at = fill[A->ci[k]]++;
            B->ci[at] = i;
            B->v[at] = A->v[k];
        }
    free(fill);
    return B;
}

static int cmp_i64(const void* a, const void* b) {
    const int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
    return (x > y) - (x < y);
}

/* Row accumulator shared by spgemm and the Galerkin product: the first
 * contribution to a column assigns, later ones add in encounter order
 * (src/kernels.cpp:169-194, src/coarsening.cpp:131-138). */
typedef struct {
    int64_t* stamp;
    double* val;
    int64_t* cols;
    int64_t ncols_touched;
} row_acc;

static void acc_init(row_acc* a, int64_t ncols) {
    a->stamp = xmalloc(sizeof(int64_t) * (size_t)ncols);
    for (int64_t j = 0; j < ncols; ++j) a->stamp[j] = -1;
    a->val = xmalloc(sizeof(double) * (size_t)ncols);
    a->cols = xmalloc(sizeof(int64_t) * (size_t)ncols);
    a->ncols_touched = 0;
}
static void acc_free(row_acc* a) {
    free(a->stamp);
    free(a->val);
    free(a->cols);
}
static inline void acc_add(row_acc* a, int64_t row, int64_t col, double x) {
    if (a->stamp[col] != row) {
        a->stamp[col] = row;
        a->val[col] = x;
        a->cols[a->ncols_touched++] = col;
    } else {
        a->val[col] = a->val[col] + x;
    }
}

typedef struct {
    int64_t* ci;
    double* v;
    int64_t len, cap;
} grow_buf;

static void gb_push(grow_buf* g, int64_t c, double v) {
    if (g->len == g->cap) {
        g->cap = g->cap ? 2 * g->cap : 1024;
        g->ci = realloc(g->ci, sizeof(int64_t) * (size_t)g->cap);
        g->v = realloc(g->v, sizeof(double) * (size_t)g->cap);
        if (!g->ci || !g->v) abort();
    }
    g->ci[g->len] = c;
    g->v[g->len] = v;
    g->len++;
}

static orc_csr* csr_from_grow(int64_t nrows, int64_t ncols, int64_t* rp, grow_buf* g) {
    orc_csr* C = xmalloc(sizeof(orc_csr));
    C->nrows = nrows;
    C->ncols = ncols;
    C->rp = rp;
    C->ci = g->ci ? g->ci : xmalloc(sizeof(int64_t));
    C->v = g->v ? g->v : xmalloc(sizeof(double));
    return C;
}

static void flush_row(row_acc* acc, grow_buf* out) {
    qsort(acc->cols, (size_t)acc->ncols_touched, sizeof(int64_t), cmp_i64);
    for (int64_t t = 0; t < acc->ncols_touched; ++t)
        gb_push(out, acc->cols[t], acc->val[acc->cols[t]]);
    acc->ncols_touched = 0;
}

/* src/kernels.cpp:237-285 (sorted output, cancelled zeros kept) */
orc_csr* orc_spgemm(const orc_csr* A, const orc_csr* B) {
    if (A->ncols != B->nrows) return NULL;
    row_acc acc;
    acc_init(&acc, B->ncols);
    grow_buf out = {0};
    int64_t* rp = xcalloc((size_t)A->nrows + 1, sizeof(int64_t));
    for (int64_t i = 0; i < A->nrows; ++i) {
        for (int64_t k = A->rp[i]; k < A->rp[i + 1]; ++k) {
            const int64_t j = A->ci[k];
            const double a = A->v[k];
            for (int64_t t = B->rp[j]; t < B->rp[j + 1]; ++t)
                acc_add(&acc, i, B->ci[t], a * B->v[t]);
        }
        flush_row(&acc, &out);
        rp[i + 1] = out.len;
    }
    acc_free(&acc);
    return csr_from_grow(A->nrows, B->ncols, rp, &out);
}

/* --------------------------------------------------------------- matching --- */
/* src/matching.cpp:28-101 (diagonal via src/csr.cpp:99-104) */
int orc_build_weights(const orc_csr* A, const double* w, int64_t* xadj,
                      int64_t* adjncy, double* weight, int64_t* zero_edges,
                      int64_t* bad_row) {
    const int64_t n = A->nrows;
    double* dg = xmalloc(sizeof(double) * (size_t)n);
    int status = 0;
    *zero_edges = 0;
    *bad_row = -1;
    for (int64_t i = 0; i < n; ++i) {
        const int64_t p = find_pos(A, i, i);
        dg[i] = p >= 0 ? A->v[p] : 0.0;
    }
    for (int64_t i = 0; i < n; ++i)
        if (!(dg[i] > 0.0)) {
            *bad_row = i;
            free(dg);
            return 1;
        }
    xadj[0] = 0;
    for (int64_t i = 0; i < n; ++i)
        xadj[i + 1] = xadj[i] + (A->rp[i + 1] - A->rp[i]) - (find_pos(A, i, i) >= 0);

    int64_t pattern_row = -1, weight_row = -1;
    for (int64_t i = 0; i < n; ++i) {
        int64_t pos = xadj[i];
        for (int64_t k = A->rp[i]; k < A->rp[i + 1]; ++k) {
            const int64_t j = A->ci[k];
            if (j == i) continue;
            const int64_t mirror = find_pos(A, j, i);
            if (mirror < 0) {
                if (pattern_row < 0) pattern_row = i; /* lowest offending row */
                break;
            }
            /* weight from the upper-triangle entry A(p, q), p < q */
            const int64_t p = i < j ? i : j, q = i < j ? j : i;
            const double apq = i < j ? A->v[k] : A->v[mirror];
            const double den = dg[p] * w[p] * w[p] + dg[q] * w[q] * w[q];
            double c;
            if (den == 0.0) {
                c = 0.0;
                if (i < j) ++*zero_edges;
            } else {
                c = 1.0 - 2.0 * apq * w[p] * w[q] / den;
            }
            if (!isfinite(c)) {
                if (weight_row < 0) weight_row = i;
                break;
            }
            adjncy[pos] = j;
            weight[pos] = c;
            ++pos;
        }
    }
    free(dg);
    if (pattern_row >= 0) {
        *bad_row = pattern_row;
        status = 2;
    } else if (weight_row >= 0) {
        *bad_row = weight_row;
        status = 3;
    }
    return status;
}

/* edge order of src/matching.cpp:108-113 specialised to a shared endpoint:
 * heavier wins; on equal weight the smaller opposite endpoint wins. */
static inline int beats(double c1, int64_t u1, double c2, int64_t u2) {
    if (c1 != c2) return c1 > c2;
    return u1 < u2;
}

/* src/matching.cpp:117-154 — sequential Suitor with re-proposals */
void orc_suitor(int64_t n, const int64_t* xadj, const int64_t* adjncy,
                const double* weight, int64_t* mate) {
    int64_t* who = xmalloc(sizeof(int64_t) * (size_t)(n ? n : 1));
    double* how = xmalloc(sizeof(double) * (size_t)(n ? n : 1));
    for (int64_t v = 0; v < n; ++v) {
        who[v] = -1;
        how[v] = 0.0;
    }
    for (int64_t s = 0; s < n; ++s) {
        int64_t u = s;
        for (;;) {
            int64_t pick = -1;
            double pick_c = 0.0;
            for (int64_t k = xadj[u]; k < xadj[u + 1]; ++k) {
                const int64_t v = adjncy[k];
                const double c = weight[k];
                if (c < 0.0) continue;
                if (who[v] >= 0 && !beats(c, u, how[v], who[v])) continue;
                if (pick < 0 || beats(c, v, pick_c, pick)) {
                    pick = v;
                    pick_c = c;
                }
            }
            if (pick < 0) break;
            const int64_t loser = who[pick];
            who[pick] = u;
            how[pick] = pick_c;
            if (loser < 0) break;
            u = loser;
        }
    }
    for (int64_t v = 0; v < n; ++v) {
        const int64_t u = who[v];
        mate[v] = (u >= 0 && who[u] == v) ? u : -1;
    }
    free(who);
    free(how);
}

/* ------------------------------------------------------------- coarsening --- */
/* src/matching.cpp:18-26 + src/coarsening.cpp:12-34 */
int orc_pairwise_aggregate(int64_t n, const int64_t* mate, int64_t* agg_of,
                           int64_t* counts) {
    for (int64_t i = 0; i < n; ++i) {
        const int64_t j = mate[i];
        if (j == -1) continue;
        if (j < 0 || j >= n || j == i || mate[j] != i) return 1;
    }
    int64_t nc = 0, np = 0, ns = 0;
    for (int64_t i = 0; i < n; ++i) agg_of[i] = -1;
    for (int64_t i = 0; i < n; ++i) {
        if (agg_of[i] >= 0) continue;
        agg_of[i] = nc;
        if (mate[i] != -1) {
            agg_of[mate[i]] = nc;
            ++np;
        } else {
            ++ns;
        }
        ++nc;
    }
    counts[0] = nc;
    counts[1] = np;
    counts[2] = ns;
    return 0;
}

/* src/coarsening.cpp:36-76 */
int orc_build_prolongator(int64_t n, int64_t n_c, const int64_t* agg_of,
                          const double* w, orc_csr** P, int64_t* bad) {
    double* nsq = xcalloc((size_t)n_c, sizeof(double));
    int64_t* cnt = xcalloc((size_t)n_c, sizeof(int64_t));
    *P = NULL;
    for (int64_t i = 0; i < n; ++i) {
        const int64_t a = agg_of[i];
        if (a < 0 || a >= n_c) {
            *bad = i;
            free(nsq);
            free(cnt);
            return 1;
        }
        nsq[a] = nsq[a] + w[i] * w[i];
        cnt[a]++;
    }
    for (int64_t a = 0; a < n_c; ++a) {
        if (nsq[a] == 0.0 && cnt[a] > 1) {
            *bad = a;
            free(nsq);
            free(cnt);
            return 2;
        }
        nsq[a] = sqrt(nsq[a]); /* reuse as the norm */
    }
    orc_csr* M = orc_csr_new(n, n_c, n);
    for (int64_t i = 0; i <= n; ++i) M->rp[i] = i;
    for (int64_t i = 0; i < n; ++i) {
        const int64_t a = agg_of[i];
        M->ci[i] = a;
        M->v[i] = nsq[a] == 0.0 ? 1.0 : w[i] / nsq[a];
    }
    free(nsq);
    free(cnt);
    *P = M;
    return 0;
}

/* src/coarsening.cpp:78-87 */
void orc_restrict_vector(const orc_csr* P, const double* w, double* wc) {
    for (int64_t a = 0; a < P->ncols; ++a) wc[a] = 0.0;
    for (int64_t i = 0; i < P->nrows; ++i)
        for (int64_t k = P->rp[i]; k < P->rp[i + 1]; ++k)
            wc[P->ci[k]] = wc[P->ci[k]] + P->v[k] * w[i];
}

/* src/coarsening.cpp:89-161: contributions (p_i a_ik) p_j in member order
 * (ascending fine index) then row order; output columns sorted. */
orc_csr* orc_galerkin_by_aggregates(const orc_csr* A, const orc_csr* P) {
    if (A->nrows != A->ncols || A->nrows != P->nrows) return NULL;
    const int64_t n = A->nrows, nc = P->ncols;
    for (int64_t i = 0; i < n; ++i)
        if (P->rp[i + 1] - P->rp[i] != 1) return NULL;
    const int64_t* agg = P->ci + 0; /* row i's single entry sits at P->rp[i] */
    const double* pv = P->v;
    /* members grouped by aggregate, ascending */
    int64_t* mptr = xcalloc((size_t)nc + 1, sizeof(int64_t));
    for (int64_t i = 0; i < n; ++i) mptr[agg[P->rp[i]] + 1]++;
    for (int64_t a = 0; a < nc; ++a) mptr[a + 1] += mptr[a];
    int64_t* members = xmalloc(sizeof(int64_t) * (size_t)(n ? n : 1));
    int64_t* cur = xmalloc(sizeof(int64_t) * (size_t)(nc + 1));
    memcpy(cur, mptr, sizeof(int64_t) * (size_t)(nc + 1));
    for (int64_t i = 0; i < n; ++i) members[cur[agg[P->rp[i]]]++] = i;
    free(cur);

    row_acc acc;
    acc_init(&acc, nc);
    grow_buf out = {0};
    int64_t* rp = xcalloc((size_t)nc + 1, sizeof(int64_t));
    for (int64_t I = 0; I < nc; ++I) {
        for (int64_t m = mptr[I]; m < mptr[I + 1]; ++m) {
            const int64_t i = members[m];
            const double pi = pv[P->rp[i]];
            for (int64_t k = A->rp[i]; k < A->rp[i + 1]; ++k) {
                const int64_t j = A->ci[k];
                acc_add(&acc, I, agg[P->rp[j]], pi * A->v[k] * pv[P->rp[j]]);
            }
        }
        flush_row(&acc, &out);
        rp[I + 1] = out.len;
    }
    acc_free(&acc);
    free(mptr);
    free(members);
    return csr_from_grow(nc, nc, rp, &out);
}

typedef struct {
    orc_csr* P;
    orc_csr* Ac;
    double* wc;
    int64_t zero_edges;
} orc_step;

static void step_free(orc_step* s) {
    orc_csr_free(s->P);
    orc_csr_free(s->Ac);
    free(s->wc);
    memset(s, 0, sizeof(*s));
}

/* src/coarsening.cpp:163-173 */
static int pairwise_step(const orc_csr* A, const double* w, orc_step* out, int64_t* bad) {
    const int64_t n = A->nrows, nnz = orc_csr_nnz(A);
    int64_t* xadj = xmalloc(sizeof(int64_t) * (size_t)(n + 1));
    int64_t* adj = xmalloc(sizeof(int64_t) * (size_t)(nnz ? nnz : 1));
    double* wt = xmalloc(sizeof(double) * (size_t)(nnz ? nnz : 1));
    memset(out, 0, sizeof(*out));
    int st = orc_build_weights(A, w, xadj, adj, wt, &out->zero_edges, bad);
    if (st) {
        free(xadj);
        free(adj);
        free(wt);
        return st;
    }
    int64_t* mate = xmalloc(sizeof(int64_t) * (size_t)(n ? n : 1));
    orc_suitor(n, xadj, adj, wt, mate);
    free(xadj);
    free(adj);
    free(wt);
    int64_t* agg = xmalloc(sizeof(int64_t) * (size_t)(n ? n : 1));
    int64_t cnt[3];
    orc_pairwise_aggregate(n, mate, agg, cnt);
    free(mate);
    st = orc_build_prolongator(n, cnt[0], agg, w, &out->P, bad);
    free(agg);
    if (st) return 5;
    out->Ac = orc_galerkin_by_aggregates(A, out->P);
    out->wc = xmalloc(sizeof(double) * (size_t)(cnt[0] ? cnt[0] : 1));
    orc_restrict_vector(out->P, w, out->wc);
    return 0;
}

/* src/coarsening.cpp:175-185 */
static int double_pairwise(const orc_csr* A, const double* w, orc_step* out, int64_t* bad) {
    orc_step first, second;
    int st = pairwise_step(A, w, &first, bad);
    if (st) return st;
    st = pairwise_step(first.Ac, first.wc, &second, bad);
    if (st) {
        step_free(&first);
        return st;
    }
    out->P = orc_spgemm(first.P, second.P);
    out->Ac = second.Ac;
    out->wc = second.wc;
    out->zero_edges = first.zero_edges + second.zero_edges;
    orc_csr_free(second.P);
    step_free(&first);
    return 0;
}

static orc_csr* csr_clone(const orc_csr* A) {
    return orc_csr_copy_from(A->nrows, A->ncols, A->rp, A->ci, A->v);
}

/* src/coarsening.cpp:187-238 */
int orc_build_hierarchy(const orc_csr* A, const double* w, int max_levels,
                        double coarse_factor, int mode, orc_hier** out,
                        int64_t* bad) {
    *out = NULL;
    *bad = -1;
    if (max_levels < 1 || !(coarse_factor > 0.0)) return 7;
    if (A->nrows != A->ncols) return 7;
    if (!orc_has_symmetric_pattern(A)) return 6;
    const int64_t n = A->nrows;
    const double bound = coarse_factor * cbrt((double)n);

    orc_hier* h = xcalloc(1, sizeof(orc_hier));
    h->lv = xcalloc((size_t)max_levels, sizeof(orc_level));
    orc_level* L0 = &h->lv[0];
    L0->A = csr_clone(A);
    L0->l1 = xmalloc(sizeof(double) * (size_t)(n ? n : 1));
    L0->w = xmalloc(sizeof(double) * (size_t)(n ? n : 1));
    memcpy(L0->w, w, sizeof(double) * (size_t)n);
    h->nl = 1;
    int64_t r = orc_l1_diagonal(L0->A, L0->l1);
    if (r >= 0) {
        *bad = r;
        orc_hier_free(h);
        return 4;
    }
    while ((double)h->lv[h->nl - 1].A->nrows > bound && h->nl < max_levels) {
        orc_level* fine = &h->lv[h->nl - 1];
        orc_step s;
        const int st = mode == 2 ? double_pairwise(fine->A, fine->w, &s, bad)
                                 : pairwise_step(fine->A, fine->w, &s, bad);
        if (st) {
            orc_hier_free(h);
            return st;
        }
        h->zero_edges += s.zero_edges;
        if (s.Ac->nrows == fine->A->nrows) {
            h->stalled = 1;
            step_free(&s);
            break;
        }
        fine->P = s.P;
        fine->R = orc_transpose(s.P);
        orc_level* coarse = &h->lv[h->nl];
        coarse->A = s.Ac;
        coarse->w = s.wc;
        coarse->l1 = xmalloc(sizeof(double) * (size_t)(s.Ac->nrows ? s.Ac->nrows : 1));
        h->nl++;
        r = orc_l1_diagonal(coarse->A, coarse->l1);
        if (r >= 0) {
            *bad = r;
            orc_hier_free(h);
            return 4;
        }
    }
    *out = h;
    return 0;
}

void orc_hier_free(orc_hier* h) {
    if (!h) return;
    for (int k = 0; k < h->nl; ++k) {
        orc_csr_free(h->lv[k].A);
        orc_csr_free(h->lv[k].P);
        orc_csr_free(h->lv[k].R);
        free(h->lv[k].l1);
        free(h->lv[k].w);
    }
    free(h->lv);
    free(h);
}

/* -------------------------------------------------------------- multigrid --- */
/* src/multigrid.cpp:19-34 and :52-61: x += (b - A x) / d, Jacobi */
static void sweeps(const orc_csr* A, const double* d, const double* b, double* x,
                   int k, double* Ax) {
    const int g = orc_lane_policy(A);
    for (int s = 0; s < k; ++s) {
        orc_spmv(A, g, x, Ax);
        for (int64_t i = 0; i < A->nrows; ++i) x[i] = x[i] + (b[i] - Ax[i]) / d[i];
    }
}

void orc_l1_jacobi(const orc_csr* A, const double* d, const double* b,
                   double* x, int k) {
    if (k <= 0) return;
    double* Ax = xmalloc(sizeof(double) * (size_t)(A->nrows ? A->nrows : 1));
    sweeps(A, d, b, x, k, Ax);
    free(Ax);
}

typedef struct {
    double** scratch;
    double** cb;
    double** cx;
    double** k1; /* K-cycle: c1, c2, v1, v2, rt of level k (size n_{k+1}) */
    double** k2;
    double** kv1;
    double** kv2;
    double** kr;
} orc_ws;

static void cycle_rec(const orc_hier* h, int level, const double* b, double* x,
                      int cycle, int pre, int post, int coarsest, orc_ws* ws);

/* K-cycle coarse correction (cycle == 2). NOT in the reference: the north
 * star's "K-cycle driver" (Notay & Vassilevski, Numer. Linear Algebra Appl.
 * 15 (2008) 473-487): two steps of flexible CG on A_{k+1} xc = bc, each
 * preconditioned by the K-cycle of level k + 1 from zero; the second step is
 * skipped when ||rt|| <= 0.25 ||bc||. Written with the reference's own vector
 * primitives (blocked dot / norm2, axpy) so the B200 path can be checked bit
 * for bit; parity with the reference itself is unpinned (it has no K-cycle). */
static void kcycle_coarse(const orc_hier* h, int level, const double* bc, double* xc,
                          int pre, int post, int coarsest, orc_ws* ws) {
    const orc_csr* Ac = h->lv[level + 1].A;
    const int64_t m = Ac->nrows;
    double *c1 = ws->k1[level], *c2 = ws->k2[level], *v1 = ws->kv1[level];
    double *v2 = ws->kv2[level], *rt = ws->kr[level];
    const int g = orc_lane_policy(Ac);
    for (int64_t i = 0; i < m; ++i) c1[i] = 0.0;
    cycle_rec(h, level + 1, bc, c1, 2, pre, post, coarsest, ws);
    orc_spmv(Ac, g, c1, v1);
    const double rho1 = orc_dot(m, c1, v1);
    const double alpha1 = orc_dot(m, c1, bc);
    const int ok1 = rho1 > 0.0;
    const double s1 = ok1 ? alpha1 / rho1 : 0.0;
    for (int64_t i = 0; i < m; ++i) {
        rt[i] = bc[i] + (-s1) * v1[i];
        xc[i] = ok1 ? 0.0 + s1 * c1[i] : 0.0;
    }
    if (!ok1 || sqrt(orc_dot(m, rt, rt)) <= 0.25 * sqrt(orc_dot(m, bc, bc))) return;
    for (int64_t i = 0; i < m; ++i) c2[i] = 0.0;
    cycle_rec(h, level + 1, rt, c2, 2, pre, post, coarsest, ws);
    orc_spmv(Ac, g, c2, v2);
    const double gamma = orc_dot(m, c2, v1);
    const double beta = orc_dot(m, c2, v2);
    const double alpha2 = orc_dot(m, c2, rt);
    const double rho2 = beta - gamma * gamma / rho1;
    if (!(rho2 > 0.0)) return; /* keep the one-step correction */
    const double a2 = alpha2 / rho2;
    const double a1 = s1 - gamma * a2 / rho1;
    for (int64_t i = 0; i < m; ++i) xc[i] = (0.0 + a1 * c1[i]) + a2 * c2[i];
}

/* src/multigrid.cpp:65-109 */
static void cycle_rec(const orc_hier* h, int level, const double* b, double* x,
                      int cycle, int pre, int post, int coarsest, orc_ws* ws) {
    const orc_level* L = &h->lv[level];
    const int64_t n = L->A->nrows;
    double* r = ws->scratch[level];
    if (level == h->nl - 1) {
        for (int64_t i = 0; i < n; ++i) x[i] = 0.0;
        sweeps(L->A, L->l1, b, x, coarsest, r);
        return;
    }
    sweeps(L->A, L->l1, b, x, pre, r);
    orc_spmv(L->A, orc_lane_policy(L->A), x, r);
    for (int64_t i = 0; i < n; ++i) r[i] = b[i] - r[i];
    double* bc = ws->cb[level];
    double* xc = ws->cx[level];
    orc_spmv(L->R, orc_lane_policy(L->R), r, bc);
    for (int64_t i = 0; i < L->R->nrows; ++i) xc[i] = 0.0;
    if (cycle == 2 && level + 2 < h->nl) {
        kcycle_coarse(h, level, bc, xc, pre, post, coarsest, ws);
    } else {
        const int visits = cycle == 1 ? 2 : 1;
        for (int t = 0; t < visits; ++t)
            cycle_rec(h, level + 1, bc, xc, cycle, pre, post, coarsest, ws);
    }
    orc_spmv(L->P, orc_lane_policy(L->P), xc, r);
    for (int64_t i = 0; i < n; ++i) x[i] = x[i] + 1.0 * r[i];
    sweeps(L->A, L->l1, b, x, post, r);
}

static void ws_init(const orc_hier* h, orc_ws* ws) {
    ws->scratch = xcalloc((size_t)h->nl, sizeof(double*));
    ws->cb = xcalloc((size_t)h->nl, sizeof(double*));
    ws->cx = xcalloc((size_t)h->nl, sizeof(double*));
    double*** kb[5] = {&ws->k1, &ws->k2, &ws->kv1, &ws->kv2, &ws->kr};
    for (int j = 0; j < 5; ++j) *kb[j] = xcalloc((size_t)h->nl, sizeof(double*));
    for (int k = 0; k < h->nl; ++k) {
        ws->scratch[k] = xcalloc((size_t)h->lv[k].A->nrows, sizeof(double));
        if (k + 1 < h->nl) {
            const size_t m = (size_t)h->lv[k + 1].A->nrows;
            ws->cb[k] = xcalloc(m, sizeof(double));
            ws->cx[k] = xcalloc(m, sizeof(double));
            for (int j = 0; j < 5; ++j) (*kb[j])[k] = xcalloc(m, sizeof(double));
        }
    }
}

static void ws_free(const orc_hier* h, orc_ws* ws) {
    for (int k = 0; k < h->nl; ++k) {
        free(ws->scratch[k]);
        free(ws->cb[k]);
        free(ws->cx[k]);
        free(ws->k1[k]);
        free(ws->k2[k]);
        free(ws->kv1[k]);
        free(ws->kv2[k]);
        free(ws->kr[k]);
    }
    free(ws->k1);
    free(ws->k2);
    free(ws->kv1);
    free(ws->kv2);
    free(ws->kr);
    free(ws->scratch);
    free(ws->cb);
    free(ws->cx);
}

void orc_apply_cycle(const orc_hier* h, int level, const double* b, double* x,
                     int cycle, int pre, int post, int coarsest) {
    orc_ws ws;
    ws_init(h, &ws);
    cycle_rec(h, level, b, x, cycle, pre, post, coarsest, &ws);
    ws_free(h, &ws);
}

/* ------------------------------------------------------------- vector ops --- */
/* src/vector_ops.cpp:16-25: pairwise fold with the odd tail carried */
static double fold(double* part, int64_t m) {
    if (m == 0) return 0.0;
    while (m > 1) {
        const int64_t half = m / 2;
        for (int64_t i = 0; i < half; ++i) part[i] = part[2 * i] + part[2 * i + 1];
        if (m & 1) part[half] = part[m - 1];
        m = (m + 1) / 2;
    }
    return part[0];
}

/* src/vector_ops.cpp:29-44 */
double orc_dot(int64_t n, const double* x, const double* y) {
    const int64_t nb = (n + ORC_BLOCK - 1) / ORC_BLOCK;
    double* part = xmalloc(sizeof(double) * (size_t)(nb ? nb : 1));
    for (int64_t b = 0; b < nb; ++b) {
        const int64_t lo = b * ORC_BLOCK, hi = lo + ORC_BLOCK < n ? lo + ORC_BLOCK : n;
        double s = 0.0;
        for (int64_t i = lo; i < hi; ++i) s = s + x[i] * y[i];
        part[b] = s;
    }
    const double r = fold(part, nb);
    free(part);
    return r;
}

double orc_norm2(int64_t n, const double* x) { return sqrt(orc_dot(n, x, x)); }

/* src/vector_ops.cpp:48-54 */
void orc_axpy(int64_t n, double* y, double a, const double* x) {
    for (int64_t i = 0; i < n; ++i) y[i] = y[i] + a * x[i];
}

/* src/vector_ops.cpp:56-80 */
void orc_triple_dot(int64_t n, const double* w, const double* r,
                    const double* v, const double* q, double* out3) {
    const int64_t nb = (n + ORC_BLOCK - 1) / ORC_BLOCK;
    double* pr = xmalloc(sizeof(double) * (size_t)(nb ? nb : 1));
    double* pv = xmalloc(sizeof(double) * (size_t)(nb ? nb : 1));
    double* pq = xmalloc(sizeof(double) * (size_t)(nb ? nb : 1));
    for (int64_t b = 0; b < nb; ++b) {
        const int64_t lo = b * ORC_BLOCK, hi = lo + ORC_BLOCK < n ? lo + ORC_BLOCK : n;
        double sr = 0.0, sv = 0.0, sq = 0.0;
        for (int64_t i = lo; i < hi; ++i) {
            sr = sr + w[i] * r[i];
            sv = sv + w[i] * v[i];
            sq = sq + w[i] * q[i];
        }
        pr[b] = sr;
        pv[b] = sv;
        pq[b] = sq;
    }
    out3[0] = fold(pr, nb);
    out3[1] = fold(pv, nb);
    out3[2] = fold(pq, nb);
    free(pr);
    free(pv);
    free(pq);
}

/* src/vector_ops.cpp:82-92 */
void orc_axpy_pair(int64_t n, double* y1, double* y2, const double* x,
                   double a, double b) {
    for (int64_t i = 0; i < n; ++i) {
        const double t = y1[i] + a * x[i];
        y1[i] = t;
        y2[i] = y2[i] + b * t;
    }
}

/* ----------------------------------------------------------------- Krylov --- */
static double now_ms(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec * 1e3 + (double)ts.tv_nsec * 1e-6;
}

static void precond(const orc_hier* h, orc_ws* ws, int cycle, int pre, int post,
                    int coarsest, const double* r, double* z, int64_t n) {
    if (!h) {
        memcpy(z, r, sizeof(double) * (size_t)n);
        return;
    }
    for (int64_t i = 0; i < n; ++i) z[i] = 0.0; /* src/multigrid.cpp:145-149 */
    cycle_rec(h, 0, r, z, cycle, pre, post, coarsest, ws);
}

/* src/krylov.cpp:43-141 (audit :25-39) */
int orc_pcg(const orc_csr* A, const orc_hier* h, int cycle, int pre, int post,
            int coarsest, const double* b, const double* u0, double rtol,
            int64_t itmax, double* u, double* hist, orc_report* rep) {
    const double t0 = now_ms();
    const int64_t n = A->nrows;
    memset(rep, 0, sizeof(*rep));
    rep->breakdown_iteration = -1;
    int64_t nh = 0;
    const double norm_b = orc_norm2(n, b);
    int status = 0;
    if (norm_b == 0.0) {
        for (int64_t i = 0; i < n; ++i) u[i] = 0.0;
        rep->converged = 1;
        hist[nh++] = 0.0;
        rep->solve_ms = now_ms() - t0;
        return 0;
    }
    const int g = orc_lane_policy(A);
    const size_t bytes = sizeof(double) * (size_t)(n ? n : 1);
    double *r = xmalloc(bytes), *w = xmalloc(bytes), *d = xmalloc(bytes),
           *v = xmalloc(bytes), *q = xmalloc(bytes);
    orc_ws ws;
    if (h) ws_init(h, &ws);
    for (int64_t i = 0; i < n; ++i) u[i] = u0 ? u0[i] : 0.0;

    orc_spmv(A, g, u, r);
    for (int64_t i = 0; i < n; ++i) r[i] = b[i] - r[i];
    hist[nh++] = orc_norm2(n, r);
    if (hist[nh - 1] / norm_b <= rtol) {
        rep->converged = 1;
        goto done;
    }
    precond(h, &ws, cycle, pre, post, coarsest, r, w, n);
    memcpy(d, w, bytes);
    orc_spmv(A, g, w, v);
    memcpy(q, v, bytes);
    double alpha = orc_dot(n, w, r);
    double rho = orc_dot(n, w, v);
    if (!isfinite(alpha) || !isfinite(rho) || rho <= 0.0) {
        rep->breakdown_iteration = 0;
        status = 3;
        goto done;
    }
    double step = alpha / rho;
    orc_axpy(n, u, step, d);
    orc_axpy(n, r, -step, q);
    rep->iterations = 1;
    hist[nh++] = orc_norm2(n, r);

    while (hist[nh - 1] / norm_b > rtol && rep->iterations < itmax) {
        precond(h, &ws, cycle, pre, post, coarsest, r, w, n);
        orc_spmv(A, g, w, v);
        double s3[3];
        orc_triple_dot(n, w, r, v, q, s3);
        alpha = s3[0];
        const double rho_next = s3[1] - s3[2] * s3[2] / rho;
        if (!isfinite(s3[0]) || !isfinite(s3[1]) || !isfinite(s3[2]) ||
            !isfinite(rho_next) || rho_next <= 0.0) {
            rep->breakdown_iteration = rep->iterations;
            status = 3;
            goto done;
        }
        const double t = s3[2] / rho;
        step = alpha / rho_next;
        double* tmp;
        orc_axpy_pair(n, w, u, d, -t, step);
        tmp = d; d = w; w = tmp;
        orc_axpy_pair(n, v, r, q, -t, -step);
        tmp = q; q = v; v = tmp;
        rho = rho_next;
        rep->iterations++;
        hist[nh++] = orc_norm2(n, r);
        if (rep->iterations % 50 == 0) {
            /* audit: || r - (b - A u) || / ||b|| (scratch = w) */
            orc_spmv(A, g, u, w);
            for (int64_t i = 0; i < n; ++i) w[i] = r[i] - (b[i] - w[i]);
            const double rel = orc_norm2(n, w) / norm_b;
            rep->audit_checks++;
            if (rel > rep->audit_max_rel) rep->audit_max_rel = rel;
            if (rel > 1e-10) rep->audit_failures++;
        }
    }
    rep->converged = hist[nh - 1] / norm_b <= rtol;
done:
    if (status == 0 && nh > 0) rep->final_relres = hist[nh - 1] / norm_b;
    rep->solve_ms = now_ms() - t0;
    if (h) ws_free(h, &ws);
    free(r);
    free(w);
    free(d);
    free(v);
    free(q);
    return status;
}
