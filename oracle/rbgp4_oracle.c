/*
 * rbgp4_oracle.c -- CPU restatement of the reference RBGP4 multiply.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product package links or calls
 * this file; only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
 * / --impl reference legs load it, as the checker and as the CPU baseline.
 *
 * Restates, loop for loop, the two numba kernels of the reference:
 *   oracle_rbgp4mm_*  <- kronsparse.sdmm._tile_worker   (sdmm.py:148-205)
 *   oracle_csr_*      <- kronsparse.sdmm._csr_rows      (sdmm.py:297-304)
 * Arithmetic is IEEE multiply-then-add with no contraction (numba's default;
 * SURVEY Appendix A), so this file MUST be compiled with -ffp-contract=off
 * and without -ffast-math.  Pinned against the reference's own outputs by
 * tests/test_oracle.py (golden hashes in tests/golden/golden.json).
 *
 * The tile loop is split over pthreads exactly like the reference's worker
 * pool (sdmm.py:274-283): worker t owns tiles t, t+T, t+2T, ...; results are
 * bit-identical for any worker count.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <unistd.h>

typedef struct {
    int64_t rows, cols, n_cols;   /* W is rows x cols, I is cols x n_cols */
    int32_t d_o;                  /* outer degree: steps per tile          */
    int32_t tm, tk, tn;           /* W tile and output column tile         */
    int32_t rm, rk, bm, bk;       /* complete factors g_r and g_b          */
    int32_t rn, bn;               /* column register blocking (tn knobs)   */
    int32_t n_ui, n_vi, d_i;      /* inner factor g_i                      */
} oracle_dims;

/* Run fn(arg, w, nthreads) for w in [0, nthreads) on nthreads pthreads. */
typedef void (*worker_fn)(void *arg, int64_t w, int64_t nthreads);
typedef struct { worker_fn fn; void *arg; int64_t w, n; } worker_job;

static void *worker_main(void *p)
{
    worker_job *j = (worker_job *)p;
    j->fn(j->arg, j->w, j->n);
    return NULL;
}

static void run_workers(worker_fn fn, void *arg, int nthreads)
{
    if (nthreads < 1) nthreads = 1;
    pthread_t *tid = (pthread_t *)malloc(sizeof(pthread_t) * nthreads);
    worker_job *jobs = (worker_job *)malloc(sizeof(worker_job) * nthreads);
    for (int w = 0; w < nthreads; ++w) {
        jobs[w] = (worker_job){fn, arg, w, nthreads};
        if (w > 0) pthread_create(&tid[w], NULL, worker_main, &jobs[w]);
    }
    worker_main(&jobs[0]);
    for (int w = 1; w < nthreads; ++w) pthread_join(tid[w], NULL);
    free(tid);
    free(jobs);
}

#define DEFINE_TILE_WORKER(T, SUFFIX)                                                   \
static void tile_worker_##SUFFIX(const T *values, const int32_t *adj_o,                 \
                                 const int32_t *adj_i, const T *inp, T *out,            \
                                 const oracle_dims *p, int64_t start, int64_t stride)   \
{                                                                                        \
    const int64_t row_nnz = (int64_t)p->d_o * p->rk * p->d_i * p->bk;                   \
    const int32_t d_t = p->rk * p->d_i * p->bk;                                         \
    const int64_t n_tile_cols = p->n_cols / p->tn;                                       \
    const int64_t n_tiles = (p->rows / p->tm) * n_tile_cols;                             \
    const int32_t strides_n = p->tn / (p->rn * p->bn);                                   \
    const int32_t col_stride = p->tn / p->rn;                                            \
    const int32_t g = p->rm * p->bm, cw = p->rn * p->bn;                                 \
    T *wbuf = (T *)malloc(sizeof(T) * (size_t)p->tm * d_t);                              \
    T *ibuf = (T *)malloc(sizeof(T) * (size_t)p->tk * p->tn);                            \
    T *acc = (T *)malloc(sizeof(T) * (size_t)p->tm * p->tn);                             \
    T *creg = (T *)malloc(sizeof(T) * (size_t)g * cw);                                   \
    for (int64_t tile = start; tile < n_tiles; tile += stride) {                         \
        const int64_t tbm = tile / n_tile_cols, tbn = tile % n_tile_cols;                \
        memset(acc, 0, sizeof(T) * (size_t)p->tm * p->tn);                               \
        for (int32_t s = 0; s < p->d_o; ++s) {                                           \
            const int64_t oind = adj_o[tbm * p->d_o + s];                                \
            for (int32_t r = 0; r < p->tm; ++r)  /* W tile -> scratch */                 \
                memcpy(wbuf + (size_t)r * d_t,                                           \
                       values + (tbm * p->tm + r) * row_nnz + (int64_t)s * d_t,          \
                       sizeof(T) * d_t);                                                 \
            for (int32_t r = 0; r < p->tk; ++r)  /* I tile -> scratch */                 \
                memcpy(ibuf + (size_t)r * p->tn,                                         \
                       inp + (oind * p->tk + r) * p->n_cols + tbn * p->tn,               \
                       sizeof(T) * p->tn);                                               \
            for (int32_t ui = 0; ui < p->n_ui; ++ui) {                                   \
                for (int32_t thn = 0; thn < strides_n; ++thn) {                          \
                    memset(creg, 0, sizeof(T) * (size_t)g * cw);                         \
                    for (int32_t rk = 0; rk < p->rk; ++rk)                               \
                    for (int32_t ink = 0; ink < p->d_i; ++ink) {                         \
                        const int32_t wcol = (rk * p->d_i + ink) * p->bk;                \
                        const int32_t kbase =                                            \
                            (rk * p->n_vi + adj_i[ui * p->d_i + ink]) * p->bk;           \
                        for (int32_t rm = 0; rm < p->rm; ++rm) {                         \
                            const int32_t rbase = (rm * p->n_ui + ui) * p->bm;           \
                            for (int32_t m = 0; m < p->bm; ++m)                          \
                            for (int32_t k = 0; k < p->bk; ++k) {                        \
                                const T a = wbuf[(size_t)(rbase + m) * d_t + wcol + k];  \
                                const T *irow = ibuf + (size_t)(kbase + k) * p->tn;      \
                                T *c = creg + (size_t)(rm * p->bm + m) * cw;             \
                                for (int32_t rn = 0; rn < p->rn; ++rn) {                 \
                                    const int32_t cbase = rn * col_stride + thn * p->bn; \
                                    for (int32_t n = 0; n < p->bn; ++n)                  \
                                        c[rn * p->bn + n] += a * irow[cbase + n];        \
                                }                                                        \
                            }                                                            \
                        }                                                                \
                    }                                                                    \
                    for (int32_t rm = 0; rm < p->rm; ++rm) {                             \
                        const int32_t rbase = (rm * p->n_ui + ui) * p->bm;               \
                        for (int32_t m = 0; m < p->bm; ++m)                              \
                        for (int32_t rn = 0; rn < p->rn; ++rn) {                         \
                            const int32_t cbase = rn * col_stride + thn * p->bn;         \
                            T *a = acc + (size_t)(rbase + m) * p->tn + cbase;            \
                            const T *c = creg + (size_t)(rm * p->bm + m) * cw            \
                                         + rn * p->bn;                                   \
                            for (int32_t n = 0; n < p->bn; ++n) a[n] += c[n];            \
                        }                                                                \
                    }                                                                    \
                }                                                                        \
            }                                                                            \
        }                                                                                \
        for (int32_t r = 0; r < p->tm; ++r)                                              \
            memcpy(out + (tbm * p->tm + r) * p->n_cols + tbn * p->tn,                    \
                   acc + (size_t)r * p->tn, sizeof(T) * p->tn);                          \
    }                                                                                    \
    free(wbuf); free(ibuf); free(acc); free(creg);                                       \
}                                                                                        \
                                                                                         \
typedef struct { const T *values; const int32_t *adj_o, *adj_i; const T *inp; T *out;   \
                 const oracle_dims *p; } tile_args_##SUFFIX;                             \
static void tile_entry_##SUFFIX(void *arg, int64_t w, int64_t n)                         \
{                                                                                        \
    tile_args_##SUFFIX *a = (tile_args_##SUFFIX *)arg;                                   \
    tile_worker_##SUFFIX(a->values, a->adj_o, a->adj_i, a->inp, a->out, a->p, w, n);     \
}                                                                                        \
int oracle_rbgp4mm_##SUFFIX(const T *values, const int32_t *adj_o, const int32_t *adj_i, \
                            const T *inp, T *out, const oracle_dims *p, int nthreads)    \
{                                                                                        \
    tile_args_##SUFFIX a = {values, adj_o, adj_i, inp, out, p};                          \
    run_workers(tile_entry_##SUFFIX, &a, nthreads);                                      \
    return 0;                                                                            \
}

DEFINE_TILE_WORKER(float, f32)
DEFINE_TILE_WORKER(double, f64)

/* _csr_rows (sdmm.py:297-304): out[i, j] += v * inp[c, j] over ascending nonzeros. */
#define DEFINE_CSR(T, SUFFIX)                                                            \
typedef struct { const int64_t *indptr; const int32_t *indices; const T *values;         \
                 const T *inp; T *out; int64_t rows, n_cols; } csr_args_##SUFFIX;        \
static void csr_entry_##SUFFIX(void *arg, int64_t w, int64_t nw)                         \
{                                                                                        \
    csr_args_##SUFFIX *a = (csr_args_##SUFFIX *)arg;                                     \
    const int64_t *indptr = a->indptr; const int32_t *indices = a->indices;              \
    const T *values = a->values, *inp = a->inp; T *out = a->out;                         \
    const int64_t n_cols = a->n_cols;                                                    \
    for (int64_t i = w; i < a->rows; i += nw) {                                          \
        T *o = out + i * n_cols;                                                         \
        for (int64_t p = indptr[i]; p < indptr[i + 1]; ++p) {                            \
            const T v = values[p];                                                       \
            const T *x = inp + (int64_t)indices[p] * n_cols;                             \
            for (int64_t j = 0; j < n_cols; ++j) o[j] += v * x[j];                       \
        }                                                                                \
    }                                                                                    \
}                                                                                        \
int oracle_csr_##SUFFIX(const int64_t *indptr, const int32_t *indices, const T *values,  \
                        const T *inp, T *out, int64_t rows, int64_t n_cols, int nthreads)\
{                                                                                        \
    csr_args_##SUFFIX a = {indptr, indices, values, inp, out, rows, n_cols};             \
    run_workers(csr_entry_##SUFFIX, &a, nthreads);                                       \
    return 0;                                                                            \
}

DEFINE_CSR(float, f32)
DEFINE_CSR(double, f64)

int oracle_max_threads(void)
{
    long n = sysconf(_SC_NPROCESSORS_ONLN);
    return n > 0 ? (int)n : 1;
}
