/* The C ABI used from C alone (no Python): what a non-Python consumer of
 * include/sgl_b200.h does.  Plans a seeded B = 8 problem, runs forward and
 * adjoint on host buffers, and checks
 *   - the pairing <y, F x> = <F^H y, x>          (test_transform.py:305-315)
 *   - the fast forward against the device direct sums sgl_direct_forward
 *     (transform.py:95-117) to the window error (q = 16: < 1e-9 relative)
 *   - the error path: a radius beyond rho -> SGL_EINVAL + the reference text
 *   - a two-sub-plan multi-device plan (devices {0, 0}) against the single plan.
 * Exit code 0 on success.  Build: gcc -O2 sgl_c_smoke.c -I include -L <lib dir> -lsgl_b200 -lm */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "sgl_b200.h"

static uint64_t rng_state = 0x9E3779B97F4A7C15ull;
static double urand(void) { /* splitmix64 -> [0, 1) */
    uint64_t z = (rng_state += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    return (double)(z >> 11) * 0x1.0p-53;
}

#define CHECK(x)                                                                          \
    do {                                                                                  \
        int _rc = (x);                                                                    \
        if (_rc != SGL_OK) {                                                              \
            fprintf(stderr, "%s failed: rc=%d (%s)\n", #x, _rc, sgl_last_error());       \
            return 1;                                                                     \
        }                                                                                 \
    } while (0)

int main(void) {
    const int32_t B = 8;
    const int64_t M = 300, count = (int64_t)B * (B + 1) * (2 * B + 1) / 6;
    int32_t ndev = 0;
    sgl_device_count(&ndev);
    printf("%s, %d device(s)\n", sgl_version(), ndev);
    if (ndev < 1) return 2;
    double *pts = malloc(sizeof(double) * 3 * M);
    for (int64_t i = 0; i < M; ++i) {
        pts[3 * i] = 3.0 * cbrt(urand());
        pts[3 * i + 1] = acos(2.0 * urand() - 1.0);
        pts[3 * i + 2] = 2.0 * M_PI * urand();
    }
    sgl_cdouble *x = malloc(sizeof(sgl_cdouble) * count), *ax = malloc(sizeof(sgl_cdouble) * count);
    sgl_cdouble *y = malloc(sizeof(sgl_cdouble) * M), *fx = malloc(sizeof(sgl_cdouble) * M);
    sgl_cdouble *fd = malloc(sizeof(sgl_cdouble) * M), *fm = malloc(sizeof(sgl_cdouble) * M);
    sgl_cdouble *am = malloc(sizeof(sgl_cdouble) * count);
    for (int64_t i = 0; i < count; ++i) x[i] = (sgl_cdouble){2 * urand() - 1, 2 * urand() - 1};
    for (int64_t i = 0; i < M; ++i) y[i] = (sgl_cdouble){2 * urand() - 1, 2 * urand() - 1};

    sgl_plan *p = NULL;
    CHECK(sgl_plan_create(B, M, pts, 2, 16, 0.0, 0, NULL, &p));
    sgl_plan_info info;
    CHECK(sgl_plan_get_info(p, &info));
    CHECK(sgl_forward(p, x, 1, fx, NULL));
    CHECK(sgl_adjoint(p, y, ax, NULL));
    /* <y, F x> and <F^H y, x> (conjugate-linear in the first argument) */
    double lr = 0, li = 0, rr = 0, ri = 0, ny = 0, nx = 0, nf = 0;
    for (int64_t i = 0; i < M; ++i) {
        lr += y[i].re * fx[i].re + y[i].im * fx[i].im;
        li += y[i].re * fx[i].im - y[i].im * fx[i].re;
        ny += y[i].re * y[i].re + y[i].im * y[i].im;
        nf += fx[i].re * fx[i].re + fx[i].im * fx[i].im;
    }
    for (int64_t i = 0; i < count; ++i) {
        rr += ax[i].re * x[i].re + ax[i].im * x[i].im;
        ri += ax[i].re * x[i].im - ax[i].im * x[i].re;
        nx += x[i].re * x[i].re + x[i].im * x[i].im;
    }
    const double pair = hypot(lr - rr, li - ri) / (sqrt(ny) * (sqrt(nx) + sqrt(nf)));
    CHECK(sgl_direct_forward(B, M, pts, x, fd, NULL));
    double dmax = 0, fmax_ = 0;
    for (int64_t i = 0; i < M; ++i) {
        dmax = fmax(dmax, hypot(fx[i].re - fd[i].re, fx[i].im - fd[i].im));
        fmax_ = fmax(fmax_, hypot(fd[i].re, fd[i].im));
    }
    const double fast_vs_direct = dmax / fmax_;
    /* the reference's ValueError path: radius > rho */
    sgl_plan *bad = NULL;
    const int rc_bad = sgl_plan_create(B, M, pts, 2, 16, 1.0, 0, NULL, &bad);
    char bad_msg[256];
    snprintf(bad_msg, sizeof bad_msg, "%s", sgl_last_error());   /* the message of THIS call */
    /* multi-device plan: two sub-plans (on device 0 twice when only one GPU exists) */
    int32_t devs[2] = {0, ndev > 1 ? 1 : 0};
    sgl_plan *pm = NULL;
    CHECK(sgl_plan_create_multi(B, M, pts, 2, 16, 0.0, 0, 2, devs, &pm));
    CHECK(sgl_forward(pm, x, 1, fm, NULL));
    CHECK(sgl_adjoint(pm, y, am, NULL));
    double mf = 0, ma = 0, na = 0;
    for (int64_t i = 0; i < M; ++i) mf = fmax(mf, hypot(fm[i].re - fx[i].re, fm[i].im - fx[i].im));
    for (int64_t i = 0; i < count; ++i) {
        ma = fmax(ma, hypot(am[i].re - ax[i].re, am[i].im - ax[i].im));
        na = fmax(na, hypot(ax[i].re, ax[i].im));
    }
    printf("plan: rho %.6f grid %d x %d x %d, int8 gather %d, plan %.1f ms\n", info.rho, info.grid[0], info.grid[1],
           info.grid[2], info.i8_gather, info.plan_ms);
    printf("pairing %.2e, fast vs direct %.2e, bad rho rc %d (%s), multi fwd %.2e adj %.2e\n", pair, fast_vs_direct,
           rc_bad, bad_msg, mf / fmax_, ma / na);
    const int ok = pair < 1e-11 && fast_vs_direct < 1e-9 && rc_bad == SGL_EINVAL && bad == NULL &&
                   strstr(bad_msg, "radius exceeds") != NULL && mf / fmax_ < 1e-11 && ma / na < 1e-11;
    sgl_plan_destroy(pm);
    sgl_plan_destroy(p);
    free(pts), free(x), free(ax), free(y), free(fx), free(fd), free(fm), free(am);
    printf("%s\n", ok ? "C ABI smoke: OK" : "C ABI smoke: FAILED");
    return ok ? 0 : 1;
}
