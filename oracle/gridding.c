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

void oracle_gather(const double *grid, const int64_t *shape, int64_t m,
                   const int64_t *b0, const int64_t *b1, const int64_t *b2,
                   const double *w0, const double *w1, const double *w2,
                   int64_t q, double *out, int threads) {
    const int64_t P = 2 * q + 1, N0 = shape[0], N1 = shape[1], N2 = shape[2];
#ifdef _OPENMP
    int nt = threads > 0 ? threads : omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 64) num_threads(nt)
#endif
    for (int64_t i = 0; i < m; ++i) {
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
#ifdef _OPENMP
#pragma omp parallel for schedule(dynamic, 16) num_threads(nt)
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
#pragma omp atomic
                    row[2 * g2] += wc * tr;
#pragma omp atomic
                    row[2 * g2 + 1] += wc * ti;
                }
            }
        }
    }
#endif
}
