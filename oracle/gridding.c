/* Plain-C restatement of the reference window loops -- TEST INFRASTRUCTURE ONLY.
 *
 * Follows _gridding.py:53-74 (_gather_kernel) and _gridding.py:77-95
 * (_scatter_kernel) of the reference package, with the wrap-padding of
 * pad_wrap / fold_wrap (_gridding.py:29-50) expressed as modular indexing
 * into the un-padded oversampled grid (cell lo - q + o, taken mod N).
 * Used only by tests/, smoke() and bench.py's CPU-baseline arms.
 * threads <= 0 means "all OpenMP threads"; threads == 1 is the serial,
 * deterministic order of the reference.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static inline int64_t wrap(int64_t i, int64_t n) {
    i %= n;
    return i < 0 ? i + n : i;
}

int oracle_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* order[] = node indices sorted by a blocked key (4x4 cell columns along
 * axis 2, blocks in axis-0 order): consecutive nodes then share most of their
 * window rows in cache.  Returned through qsort on (key, index) pairs. */
typedef struct {
    int64_t key, idx;
} keyed_t;

static int cmp_keyed(const void *x, const void *y) {
    const keyed_t *a = x, *b = y;
    if (a->key != b->key) return a->key < b->key ? -1 : 1;
    return a->idx < b->idx ? -1 : (a->idx > b->idx);
}

static int64_t *sort_nodes(const int64_t *b0, const int64_t *b1, const int64_t *b2, int64_t m,
                           int64_t n0, int64_t n1, int64_t n2) {
    keyed_t *kv = malloc(sizeof(keyed_t) * (size_t)(m ? m : 1));
    for (int64_t i = 0; i < m; ++i) {
        const int64_t l0 = wrap(b0[i], n0), l1 = wrap(b1[i], n1), l2 = wrap(b2[i], n2);
        kv[i].key = ((l0 >> 2) * ((n1 >> 2) + 1) + (l1 >> 2)) * n2 + l2;
        kv[i].idx = i;
    }
    qsort(kv, (size_t)m, sizeof(keyed_t), cmp_keyed);
    int64_t *order = malloc(sizeof(int64_t) * (size_t)(m ? m : 1));
    for (int64_t i = 0; i < m; ++i) order[i] = kv[i].idx;
    free(kv);
    return order;
}

static void gather_one(const double *grid, int64_t N0, int64_t N1, int64_t N2, int64_t P, int64_t q,
                       int64_t i, const int64_t *b0, const int64_t *b1, const int64_t *b2,
                       const double *w0, const double *w1, const double *w2, double *out) {
    double ar = 0.0, ai = 0.0;
    for (int64_t a = 0; a < P; ++a) {
        const double wa = w0[i * P + a];
        if (wa == 0.0) continue;
        const int64_t g0 = wrap(b0[i] - q + a, N0);
        for (int64_t b = 0; b < P; ++b) {
            const double wab = wa * w1[i * P + b];
            const int64_t g1 = wrap(b1[i] - q + b, N1);
            const double *row = grid + 2 * ((g0 * N1 + g1) * N2);
            double sr = 0.0, si = 0.0;
            for (int64_t c = 0; c < P; ++c) {
                const int64_t g2 = wrap(b2[i] - q + c, N2);
                const double wc = w2[i * P + c];
                sr += wc * row[2 * g2];
                si += wc * row[2 * g2 + 1];
            }
            ar += wab * sr;
            ai += wab * si;
        }
    }
    out[2 * i] = ar;
    out[2 * i + 1] = ai;
}

void oracle_gather(const double *grid, const int64_t *shape, int64_t m,
                   const int64_t *b0, const int64_t *b1, const int64_t *b2,
                   const double *w0, const double *w1, const double *w2,
                   int64_t q, double *out, int threads) {
    const int64_t P = 2 * q + 1, N0 = shape[0], N1 = shape[1], N2 = shape[2];
    int nt = 1;
#ifdef _OPENMP
    nt = threads > 0 ? threads : omp_get_max_threads();
#endif
    if (nt == 1) {   /* the reference order (_gridding.py:53-74) */
        for (int64_t i = 0; i < m; ++i) gather_one(grid, N0, N1, N2, P, q, i, b0, b1, b2, w0, w1, w2, out);
        return;
    }
    /* per-node sums are independent: visit nodes in axis-0 order for cache reuse */
    int64_t *order = sort_nodes(b0, b1, b2, m, N0, N1, N2);
#ifdef _OPENMP
#pragma omp parallel for schedule(dynamic, 16) num_threads(nt)
#endif
    for (int64_t k = 0; k < m; ++k) gather_one(grid, N0, N1, N2, P, q, order[k], b0, b1, b2, w0, w1, w2, out);
    free(order);
}

void oracle_scatter(double *grid, const int64_t *shape, int64_t m,
                    const int64_t *b0, const int64_t *b1, const int64_t *b2,
                    const double *w0, const double *w1, const double *w2,
                    int64_t q, const double *values, int threads) {
    const int64_t P = 2 * q + 1, N0 = shape[0], N1 = shape[1], N2 = shape[2];
    int nt = 1;
#ifdef _OPENMP
    nt = threads > 0 ? threads : omp_get_max_threads();
#endif
    if (nt == 1) {
        for (int64_t i = 0; i < m; ++i) {
            const double vr = values[2 * i], vi = values[2 * i + 1];
            for (int64_t a = 0; a < P; ++a) {
                const double wa = w0[i * P + a];
                if (wa == 0.0) continue;
                const int64_t g0 = wrap(b0[i] - q + a, N0);
                for (int64_t b = 0; b < P; ++b) {
                    const double wab = wa * w1[i * P + b];
                    const double tr = wab * vr, ti = wab * vi;
                    const int64_t g1 = wrap(b1[i] - q + b, N1);
                    double *row = grid + 2 * ((g0 * N1 + g1) * N2);
                    for (int64_t c = 0; c < P; ++c) {
                        const int64_t g2 = wrap(b2[i] - q + c, N2);
                        const double wc = w2[i * P + c];
                        row[2 * g2] += wc * tr;
                        row[2 * g2 + 1] += wc * ti;
                    }
                }
            }
        }
        return;
    }
    /* row ownership instead of atomics: thread t accumulates only the taps
     * whose axis-0 cell lies in its slab range; nodes in axis-0 order */
    int64_t *order = sort_nodes(b0, b1, b2, m, N0, N1, N2);
#ifdef _OPENMP
#pragma omp parallel num_threads(nt)
    {
        const int t = omp_get_thread_num(), T = omp_get_num_threads();
        const int64_t r0 = N0 * t / T, r1 = N0 * (t + 1) / T;
        for (int64_t k = 0; k < m; ++k) {
            const int64_t i = order[k];
            const double vr = values[2 * i], vi = values[2 * i + 1];
            for (int64_t a = 0; a < P; ++a) {
                const int64_t g0 = wrap(b0[i] - q + a, N0);
                if (g0 < r0 || g0 >= r1) continue;
                const double wa = w0[i * P + a];
                if (wa == 0.0) continue;
                for (int64_t b = 0; b < P; ++b) {
                    const double wab = wa * w1[i * P + b];
                    const double tr = wab * vr, ti = wab * vi;
                    const int64_t g1 = wrap(b1[i] - q + b, N1);
                    double *row = grid + 2 * ((g0 * N1 + g1) * N2);
                    for (int64_t c = 0; c < P; ++c) {
                        const int64_t g2 = wrap(b2[i] - q + c, N2);
                        const double wc = w2[i * P + c];
                        row[2 * g2] += wc * tr;
                        row[2 * g2 + 1] += wc * ti;
                    }
                }
            }
        }
    }
#endif
    free(order);
}
