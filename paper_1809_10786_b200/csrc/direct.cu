// Direct summation of the spherical Gauss-Laguerre expansion on the device:
// the reference's `evaluate_direct` / `evaluate_direct_adjoint`
// (transform.py:95-139), i.e. the "naive" method of its CLI (cli.py:154-176).
//
//   f(x_i) = sum_{n,l,m} c[mu(n,l,m)] R_{l,n-l-1}(r_i) Qs(l,m) P_{l,|m|}(cos t_i) e^{i m p_i}
//   c[mu]  = sum_i v_i conj(...)
//
// R_{l,k}: the normalised Laguerre family of recurrences.py:85-106 (the same
// recurrence as the plan's K_l in basal.cu); Qs(l,m) P_{l,|m|}: Q(l,|m|)
// P_{l,|m|} from the normalised degree recurrence (no overflow at B = 128),
// negated for odd negative m (transform.py:84-92).
//
// One thread per node; |m| outer, degree l middle (Legendre recurrence in
// registers), radial order k inner (the radial recurrence restarts per
// (|m|, l), so nothing is tabulated).  O(M * count) FP64: a verification
// path, as in the reference.  The adjoint reduces each coefficient over the
// warp's 32 nodes with shuffles and adds the sum with one FP64 atomic.
#include <cuda_runtime.h>

#include <cmath>

#include "sgl_internal.cuh"

namespace sgl {
namespace {

constexpr int DT = 128;   // threads (nodes) per block

__device__ __forceinline__ int64_t mu_nlm(int n, int l, int m) {
    return (int64_t)n * (n - 1) * (2 * n - 1) / 6 + (int64_t)l * (l + 1) + m;   // indexing.py:41-69
}

struct NodeGeom {
    double r, x, s, phi;
};

__device__ __forceinline__ NodeGeom node_geom(const double *pts, int64_t i, int64_t M) {
    NodeGeom g{0.0, 1.0, 0.0, 0.0};
    if (i < M) {
        g.r = pts[3 * i];
        const double t = pts[3 * i + 1];
        g.x = cos(t);
        // sin t as the reference forms it, sqrt(clip(1 - x^2, 0)) (special.py:84-85)
        g.s = sqrt(fmax(0.0, 1.0 - g.x * g.x));
        g.phi = pts[3 * i + 2];
    }
    return g;
}

// Q(am,am) P_{am,am}(x) with the Condon-Shortley sign (special.py:66-90)
__device__ __forceinline__ double legendre_seed(int am, double s) {
    if (am == 0) return sqrt(1.0 / (4.0 * kPi));
    const double lg = lgamma(2.0 * am + 1) - am * log(2.0) - lgamma(am + 1.0) +
                      0.5 * (log((2.0 * am + 1) / (4.0 * kPi)) - lgamma(2.0 * am + 1));
    const double v = (s > 0.0) ? exp(lg + am * log(s)) : 0.0;
    return (am & 1) ? -v : v;
}

// Walks (l, k) for one |m|: calls f(l, k, y_l * R_{l,k}) for l = am..B-1,
// k = 0..B-l-1, where y_l = Q(l,am) P_{l,am}(x).
template <typename F>
__device__ __forceinline__ void walk_am(int B, int am, const NodeGeom &g, F &&f) {
    const double r2 = g.r * g.r;
    double rl = (am == 0) ? 1.0 : pow(g.r, (double)am);
    double ym = 0.0, y = legendre_seed(am, g.s), a_prev = 0.0;
    for (int l = am; l < B; ++l) {
        if (l == am + 1) {
            a_prev = sqrt(2.0 * am + 3.0);
            const double yn = g.x * a_prev * y;
            ym = y;
            y = yn;
        } else if (l > am + 1) {
            const double al = sqrt((4.0 * l * l - 1.0) / ((double)l * l - (double)am * am));
            const double yn = al * (g.x * y - ym / a_prev);
            ym = y;
            y = yn;
            a_prev = al;
        }
        // radial family of order l (recurrences.py:85-106)
        const double a = l + 0.5;
        const double c0 = exp(0.5 * (log(2.0) - lgamma(l + 1.5)));
        double fm = c0 * rl;
        double fk = c0 / sqrt(1.0 + a) * (1.0 + a - r2) * rl;
        f(l, 0, y * fm);
        if (B - l > 1) f(l, 1, y * fk);
        for (int k = 2; k < B - l; ++k) {
            const int kk = k - 1;
            const double al = (2 * kk + 1 + a - r2) / (kk + 1) * sqrt((kk + 1) / (kk + 1 + a));
            const double be = -sqrt(kk * (kk + a) / ((kk + 1) * (kk + 1 + a)));
            const double fn = al * fk + be * fm;
            fm = fk;
            fk = fn;
            f(l, k, y * fn);
        }
        rl *= g.r;
    }
}

__global__ void __launch_bounds__(DT) k_direct_fwd(int B, int64_t M, const double *__restrict__ pts,
                                                   const double2 *__restrict__ c, double2 *__restrict__ out) {
    const int64_t i = blockIdx.x * (int64_t)DT + threadIdx.x;
    const NodeGeom g = node_geom(pts, i, M);
    double vr = 0.0, vi = 0.0;
    for (int am = 0; am < B; ++am) {
        double sn, cs;
        sincos(am * g.phi, &sn, &cs);
        const double sg = (am & 1) ? -1.0 : 1.0;   // odd negative m
        walk_am(B, am, g, [&](int l, int k, double h) {
            const int n = k + l + 1;
            const double2 cp = c[mu_nlm(n, l, am)];
            // e^{i am phi} c_+ h
            double tr = cp.x * cs - cp.y * sn, ti = cp.x * sn + cp.y * cs;
            if (am > 0) {   // + sg e^{-i am phi} c_- h
                const double2 cm = c[mu_nlm(n, l, -am)];
                tr += sg * (cm.x * cs + cm.y * sn);
                ti += sg * (cm.y * cs - cm.x * sn);
            }
            vr = fma(h, tr, vr);
            vi = fma(h, ti, vi);
        });
    }
    if (i < M) out[i] = make_double2(vr, vi);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__global__ void __launch_bounds__(DT) k_direct_adj(int B, int64_t M, const double *__restrict__ pts,
                                                   const double2 *__restrict__ v, double2 *__restrict__ c) {
    const int64_t i = blockIdx.x * (int64_t)DT + threadIdx.x;
    const int lane = threadIdx.x & 31;
    const NodeGeom g = node_geom(pts, i, M);
    const double2 vi = (i < M) ? v[i] : make_double2(0.0, 0.0);
    for (int am = 0; am < B; ++am) {
        double sn, cs;
        sincos(am * g.phi, &sn, &cs);
        const double sg = (am & 1) ? -1.0 : 1.0;
        // v e^{-i am phi} (m = +am) and sg v e^{+i am phi} (m = -am)
        const double pr = vi.x * cs + vi.y * sn, pi = vi.y * cs - vi.x * sn;
        const double nr = sg * (vi.x * cs - vi.y * sn), ni = sg * (vi.y * cs + vi.x * sn);
        walk_am(B, am, g, [&](int l, int k, double h) {
            const int n = k + l + 1;
            const double ar = warp_sum(h * pr), ai = warp_sum(h * pi);
            if (lane == 0) {
                double2 *dst = c + mu_nlm(n, l, am);
                atomicAdd(&dst->x, ar);
                atomicAdd(&dst->y, ai);
            }
            if (am > 0) {
                const double br = warp_sum(h * nr), bi = warp_sum(h * ni);
                if (lane == 0) {
                    double2 *dst = c + mu_nlm(n, l, -am);
                    atomicAdd(&dst->x, br);
                    atomicAdd(&dst->y, bi);
                }
            }
        });
    }
}

}  // namespace

int launch_direct_forward(int B, int64_t M, const double *pts, const double2 *c, double2 *out, cudaStream_t st) {
    if (M == 0) return SGL_OK;
    k_direct_fwd<<<(unsigned)((M + DT - 1) / DT), DT, 0, st>>>(B, M, pts, c, out);
    return cudaGetLastError() == cudaSuccess ? SGL_OK : SGL_ECUDA;
}

int launch_direct_adjoint(int B, int64_t M, const double *pts, const double2 *v, double2 *c, int64_t count,
                          cudaStream_t st) {
    if (cudaMemsetAsync(c, 0, sizeof(double2) * count, st) != cudaSuccess) return SGL_ECUDA;
    if (M == 0) return SGL_OK;
    k_direct_adj<<<(unsigned)((M + DT - 1) / DT), DT, 0, st>>>(B, M, pts, v, c);
    return cudaGetLastError() == cudaSuccess ? SGL_OK : SGL_ECUDA;
}

}  // namespace sgl
