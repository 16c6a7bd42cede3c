// Accuracy guard of the int8 window engines (gather_i8.cu, scatter_i8.cu).
//
// The digit-split engines reproduce the FP64 window sums to ~2^-46 of their
// fixed-point reference scales; the transform's own gains (the deconvolution
// exp(2 lam (pi k / N)^2) of the spectral edge, the basal stage) can amplify
// that to the output.  The reference's FP64 loops (_gridding.py:53-95) have no
// such error, and it ships a closed-form bound for its own window error
// (nfft_error_bound, nfft.py:85-98).  Here, per call:
//
// * forward: est = kappa 2^-46 W_mass max|G| / max|out| (W_mass = the largest
//   L1 mass of a node's window, max|G| from the per-slab maxima the digit
//   split computes anyway, max|out| reduced from the int8 result).  This
//   bounds |out_int8 - out_fp64| / max|out| (the rel-linf of the parity bar)
//   because every digit-split error term is <= 2^-46 of its slab's scale
//   times the weight of its tap.  est > SGL_GUARD_BOUND raises the plan's
//   device flag and the gated FP64 DMMA gather (k_gather_tiled, launched
//   right after, returning at once when the flag is clear) recomputes the
//   values.  No host round trip: graph-capturable.
// * adjoint: est = kappa_s 2^-46 rms(v) A_p / max|c|, where A_p is the
//   plan-time response of the adjoint's linear tail (FFT, crop,
//   deconvolution, basal adjoint) to white grid noise of the spread's per-cell
//   rms (measured once when the plan selects the int8 scatter).  The result is
//   known only after the tail, so the check reads the flag on the host (not
//   inside a CUDA-graph capture) and reruns the adjoint on the FP64 scatter.
// * non-finite input (NaN / Inf in the grid or the values): the int8 kernels
//   would map it to zero weights; their setup kernels raise the flag before
//   the int8 kernel runs (it then returns at once) and the gated FP64 kernel
//   propagates NaN / Inf as the reference does.  Always on.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "sgl_internal.cuh"

namespace sgl {

constexpr double kGuardBound = 1e-11;    // switch to FP64 above this estimate (the parity bar is 1e-10)
// Constants from tools/guard_calib.py and tools/guard_full.py
// (profiles/r02/guard_calib.txt): over the BASELINE configs, single SGL
// coefficients at the (n, l, m) corners, edge spectra, raw-NFFT families and
// smooth / sparse / uniform adjoint inputs, the measured int8-vs-FP64 rel-linf
// stays below the estimate (forward: >= 1.9x margin; adjoint: >= 1.6x at
// config 3 with all 1e7 nodes, 4x at config 4 with 1e8), while the BASELINE
// configurations stay below the 1e-11 switch (config 3: 4.2e-13 / 4.0e-12,
// config 4 adjoint: 5.7e-12).  The floors cover the output-independent
// rounding (~1.4e-13) of single-coefficient spectra.
constexpr double kGuardKappaF = 8.0;
constexpr double kGuardFloorF = 3e-13;
constexpr double kGuardKappaA = 32.0;
constexpr double kGuardFloorA = 3e-13;
constexpr double k2m46 = 1.4210854715202004e-14;   // 2^-46

namespace {

// bits of max(|Re|, |Im|) over n complex values; NaN counts as +Inf
__global__ void k_absmax_c(const double2 *__restrict__ v, int64_t n, unsigned long long *out) {
    double m = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double2 x = v[i];
        m = fmax(m, cabsmax_naninf(x));   // NaN counts as +Inf
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
}

// sum |v 2^-ev|^2 with max|v| < 2^ev (FP64 atomics, one per warp): scaled so
// that neither tiny (1e-300) nor huge (1e300) values under- / overflow the sum
// (r02 fix: the unscaled sum read 0 or Inf there, i.e. no check or a fallback
// on every call)
__device__ __forceinline__ int vmax_exp(unsigned long long bits) {
    const double vm = __longlong_as_double((long long)bits);
    int ev = 0;
    if (vm > 0.0 && isfinite(vm)) frexp(vm, &ev);
    return ev;
}

__global__ void k_sumsq_c(const double2 *__restrict__ v, int64_t n, const unsigned long long *__restrict__ vmax,
                          double *out) {
    const int ev = vmax_exp(*vmax);
    const double f1 = ldexp(1.0, -(ev / 2)), f2 = ldexp(1.0, -(ev - ev / 2));
    double s = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        double2 x = v[i];
        x.x = (x.x * f1) * f2;
        x.y = (x.y * f1) * f2;
        s = fma(x.x, x.x, fma(x.y, x.y, s));
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(out, s);
}

// forward decision (one warp): grid max from the per-slab maxima
__global__ void k_guard_fwd(GuardState *g, const unsigned long long *__restrict__ slabmax, int n0, double wk,
                            int on) {
    const int lane = threadIdx.x;
    double gm = 0.0;
    for (int a = lane; a < n0; a += 32) gm = fmax(gm, __longlong_as_double((long long)slabmax[a]));
#pragma unroll
    for (int o = 16; o; o >>= 1) gm = fmax(gm, __shfl_xor_sync(0xffffffffu, gm, o));
    if (lane) return;
    const double om = __longlong_as_double((long long)g->outmax);
    double est;
    if (!isfinite(om) || !isfinite(gm)) est = INFINITY;
    else if (om > 0.0) est = wk * gm / om + (gm > 0.0 ? kGuardFloorF : 0.0);
    else est = gm > 0.0 ? INFINITY : 0.0;   // all-zero output from a nonzero grid: not trusted
    g->est_fwd = est;
    if (on && est > kGuardBound) g->fwd = 1;   // on = 0 (SGL_FLAG_NO_GUARD): estimate only
    if (g->fwd) g->fwd_count += 1;
}

// adjoint decision (one thread): rms of the values, max of the result
__global__ void k_guard_adj(GuardState *g, const double *__restrict__ sumsq, double inv_m, double ak, int on) {
    const double cm = __longlong_as_double((long long)g->amax);
    const double rms = sqrt(*sumsq * inv_m);   // in units of 2^ev (k_sumsq_c)
    const int ev = vmax_exp(g->vmax);
    double est;
    if (!isfinite(cm) || !isfinite(rms)) {
        est = INFINITY;
    } else if (cm > 0.0) {
        int ec;
        const double mc = frexp(cm, &ec);   // cm = mc 2^ec: the ratio without over- / underflow
        est = ldexp(ak * rms / mc, ev - ec) + (rms > 0.0 ? kGuardFloorA : 0.0);
    } else {
        est = rms > 0.0 ? INFINITY : 0.0;
    }
    g->est_adj = est;
    // (a non-finite input already ran on the FP64 scatter: nothing to redo)
    g->adj_redo = (on && est > kGuardBound && !g->adj) ? 1 : 0;
    if (g->adj || g->adj_redo) g->adj_count += 1;
}

// white noise of the given rms on the interior of the halo-padded grid (zero halo)
__global__ void k_noise_grid(WindowParams wp, double rms, double2 *__restrict__ grid) {
    const int64_t total = (int64_t)wp.N0 * wp.N1p * wp.N2p;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int c2 = (int)(i % wp.N2p);
        const int c1 = (int)((i / wp.N2p) % wp.N1p);
        double2 v = make_double2(0.0, 0.0);
        if (c1 >= wp.pad && c1 < wp.pad + wp.N1 && c2 >= wp.pad && c2 < wp.pad + wp.N2) {
            uint64_t h = (uint64_t)i * 0x9E3779B97F4A7C15ull + 0x632BE59BD9B4E019ull;
            h ^= h >> 31;
            h *= 0xBF58476D1CE4E5B9ull;
            h ^= h >> 27;
            h *= 0x94D049BB133111EBull;
            h ^= h >> 31;
            const double u0 = (double)(h >> 11) * 0x1.0p-53, u1 = (double)((h << 21) >> 11) * 0x1.0p-53;
            // uniform on [-sqrt(3), sqrt(3)): unit variance per component
            v = make_double2(rms * 1.7320508075688772 * (2.0 * u0 - 1.0), rms * 1.7320508075688772 * (2.0 * u1 - 1.0));
        }
        grid[i] = v;
    }
}

// per-axis max over the sub-cell offset of sum_taps w and sum_taps w^2
void axis_mass(double c, double h, int q, double &l1, double &l2) {
    l1 = l2 = 0.0;
    for (int s = 0; s <= 100; ++s) {
        const double f = s / 100.0;
        double a = 0.0, b = 0.0;
        for (int j = -q; j <= q + 1; ++j) {
            const double w = c * std::exp(-h * (j - f) * (j - f));
            a += w;
            b += w * w;
        }
        l1 = std::max(l1, a);
        l2 = std::max(l2, b);
    }
}

}  // namespace

int setup_guard(Plan &p) {
    if (cudaMalloc(&p.guard, sizeof(GuardState)) != cudaSuccess) {
        cudaGetLastError();
        set_error("out of device memory for the guard state");
        return SGL_ENOMEM;
    }
    SGL_CUDA_CHECK(cudaMemset(p.guard, 0, sizeof(GuardState)));
    p.guard_on = !(p.flags & SGL_FLAG_NO_GUARD);
    double m1 = 1.0, t2 = 1.0;
    const double cs[3] = {p.wp.c0, p.wp.c1, p.wp.c2}, hs[3] = {p.wp.h0, p.wp.h1, p.wp.h2};
    const int qs[3] = {p.wp.qa0, p.wp.qa1, p.wp.qa2};
    for (int ax = 0; ax < 3; ++ax) {
        double a, b;
        axis_mass(cs[ax], hs[ax], qs[ax], a, b);
        m1 *= a;
        // the weight digits are fixed point at the plan scale c0 c2 (c1 for the
        // values' w1): every tap carries the same absolute rounding, however
        // small its weight -- hence (2q+1) c^2 per axis, not sum w^2
        t2 *= cs[ax] * cs[ax] * (2.0 * qs[ax] + 1.0);
    }
    p.guard_wmass = m1;
    p.guard_tap2 = t2;
    return SGL_OK;
}

int launch_noise_grid(const Plan &p, double rms, cudaStream_t st) {
    k_noise_grid<<<num_sms() * 8, 256, 0, st>>>(p.wp, rms, p.grid_buf);
    SGL_CUDA_CHECK(cudaGetLastError());
    return SGL_OK;
}

// host copy of max(|Re|, |Im|) over n device values (synchronises st)
int launch_absmax(const double2 *v, int64_t n, unsigned long long *out, cudaStream_t st) {
    k_absmax_c<<<256, 256, 0, st>>>(v, n, out);
    SGL_CUDA_CHECK(cudaGetLastError());
    return SGL_OK;
}

int read_absmax(const Plan &p, const double2 *v, int64_t n, cudaStream_t st, double *out) {
    SGL_CUDA_CHECK(cudaMemsetAsync(&p.guard->amax, 0, sizeof(unsigned long long), st));
    k_absmax_c<<<256, 256, 0, st>>>(v, n, &p.guard->amax);
    SGL_CUDA_CHECK(cudaGetLastError());
    unsigned long long bits = 0;
    SGL_CUDA_CHECK(cudaMemcpyAsync(&bits, &p.guard->amax, sizeof(bits), cudaMemcpyDeviceToHost, st));
    SGL_CUDA_CHECK(cudaStreamSynchronize(st));
    memcpy(out, &bits, sizeof(double));
    return SGL_OK;
}

int launch_gather_guarded(const Plan &p, const double2 *grid, double2 *values, cudaStream_t st) {
    if (p.M == 0) return SGL_OK;
    GuardState *g = p.guard;
    SGL_CUDA_CHECK(cudaMemsetAsync(&g->fwd, 0, sizeof(int), st));
    SGL_CUDA_CHECK(cudaMemsetAsync(&g->outmax, 0, sizeof(unsigned long long), st));
    int rc = launch_gather_i8(p, grid, values, st);   // raises g->fwd on a non-finite grid (and skips)
    if (rc) return rc;
    k_absmax_c<<<num_sms() * 4, 256, 0, st>>>(values, p.M, &g->outmax);
    SGL_CUDA_CHECK(cudaGetLastError());
    const unsigned long long *slabmax = reinterpret_cast<const unsigned long long *>(p.gmax);
    k_guard_fwd<<<1, 32, 0, st>>>(g, slabmax, p.wp.N0, kGuardKappaF * k2m46 * p.guard_wmass, p.guard_on ? 1 : 0);
    SGL_CUDA_CHECK(cudaGetLastError());
    return launch_gather_tiled_gated(p, values, &g->fwd, st);
}

int guard_adjoint_estimate(const Plan &p, const double2 *values, const double2 *coeffs, cudaStream_t st) {
    GuardState *g = p.guard;
    double *ss = &g->vsumsq;
    SGL_CUDA_CHECK(cudaMemsetAsync(ss, 0, sizeof(double), st));
    SGL_CUDA_CHECK(cudaMemsetAsync(&g->amax, 0, sizeof(unsigned long long), st));
    SGL_CUDA_CHECK(cudaMemsetAsync(&g->vmax, 0, sizeof(unsigned long long), st));
    k_absmax_c<<<256, 256, 0, st>>>(values, p.M, &g->vmax);
    k_sumsq_c<<<num_sms() * 4, 256, 0, st>>>(values, p.M, &g->vmax, ss);
    SGL_CUDA_CHECK(cudaGetLastError());
    k_absmax_c<<<256, 256, 0, st>>>(coeffs, p.count, &g->amax);
    SGL_CUDA_CHECK(cudaGetLastError());
    k_guard_adj<<<1, 1, 0, st>>>(g, ss, 1.0 / (double)std::max<int64_t>(1, p.M), kGuardKappaA * k2m46 * p.guard_ap,
                                 p.guard_on ? 1 : 0);
    SGL_CUDA_CHECK(cudaGetLastError());
    return SGL_OK;
}

int launch_scatter_guarded(const Plan &p, const double2 *values, double2 *grid, cudaStream_t st) {
    if (p.M == 0) return SGL_OK;
    SGL_CUDA_CHECK(cudaMemsetAsync(&p.guard->adj, 0, sizeof(int), st));
    int rc = launch_scatter_i8(p, values, grid, st);   // raises g->adj on non-finite values (and skips)
    if (rc) return rc;
    return launch_scatter_tiled_gated(p, values, grid, &p.guard->adj, st);
}

}  // namespace sgl
