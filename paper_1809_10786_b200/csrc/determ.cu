// Deterministic adjoint (SGL_FLAG_DETERMINISTIC).
//
// The reference's spreading loop (_gridding.py:77-95) is serial, so its
// adjoint is bitwise reproducible.  The window kernels here reduce into the
// grid with RED.E.ADD.F64 from many CTAs; FP64 addition is not associative,
// so the arrival order changes the last bits run to run (~1e-13 relative).
// With this flag every window kernel reduces 64-bit fixed-point integers
// instead (RED.E.ADD.U64: two's-complement addition is associative, so the
// grid is the same bit pattern whatever the order), converted back to FP64
// once after the spread.  Everything downstream (halo fold: one thread per
// target cell in a fixed order; cuFFT; the basal adjoint) is already
// order-fixed, so the whole adjoint is reproducible.
//
// Fixed-point unit 2^-E per call: E = 61 - ceil(log2(max|v| * D)), with
// D = max over grid cells of sum_n w_n(cell) (the window density, measured
// once at plan time by spreading unit values).  Every per-cell sum -- and
// every single contribution (one node, one tile or one DMMA fragment) -- is
// bounded by max|v| D, so no sum leaves [-2^61, 2^61].  Each contribution is
// rounded once to the unit: relative to max|v| D that is <= 2^-62 per
// contribution, far below the digit split's 2^-46 (int8 engines) and the
// FP64 accumulation error (FP64 kernels).
#include "sgl_internal.cuh"

#include <cfloat>

namespace sgl {

namespace {

__global__ void k_det_exponent(const unsigned long long *__restrict__ vmax_bits, double dens, int *__restrict__ e) {
    const double vm = __longlong_as_double((long long)*vmax_bits);
    int r;
    if (!(vm <= DBL_MAX)) {
        r = kDetOff;   // non-finite input: FP64 REDs, NaN / Inf propagate as in the reference
    } else if (vm == 0.0 || dens == 0.0) {
        r = 0;
    } else {
        int ev, ed;
        frexp(vm, &ev);
        frexp(dens, &ed);        // vm * dens < 2^(ev + ed), without overflow
        r = 61 - ev - ed;
    }
    *e = r;
}

// int64 fixed point -> FP64 in place (the grid's two 8-byte words per cell)
__global__ void k_det_convert(longlong2 *__restrict__ g, int64_t n, const int *__restrict__ e) {
    const int E = *e;
    if (E == kDetOff) return;
    const double ua = ldexp(1.0, -(E / 2)), ub = ldexp(1.0, -(E - E / 2));   // 2^-E in two exact factors
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const longlong2 x = g[i];
        double2 d;
        d.x = ((double)x.x * ua) * ub;
        d.y = ((double)x.y * ua) * ub;
        reinterpret_cast<double2 *>(g)[i] = d;
    }
}

__global__ void k_fill_ones(double2 *__restrict__ v, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        v[i] = make_double2(1.0, 0.0);
}

}  // namespace

int setup_det(Plan &p, cudaStream_t st) {
    if (!(p.flags & SGL_FLAG_DETERMINISTIC) || p.exact || p.M == 0) return SGL_OK;
    // window density D: spread unit values with the FP64 kernels (p.det not yet
    // set, so plain FP64 REDs), max over the padded grid's cells (before the
    // halo fold: the REDs land on the physical cells)
    const unsigned blocks = (unsigned)std::min<int64_t>((p.M + 255) / 256, (int64_t)num_sms() * 8);
    k_fill_ones<<<blocks, 256, 0, st>>>(p.val_buf, p.M);
    SGL_CUDA_CHECK(cudaGetLastError());
    SGL_CUDA_CHECK(cudaMemsetAsync(p.grid_buf, 0, sizeof(double2) * p.grid_elems, st));
    int rc = launch_scatter(p, p.val_buf, p.grid_buf, st);
    if (rc) return rc;
    double d = 0.0;
    rc = read_absmax(p, p.grid_buf, (int64_t)p.grid_elems, st, &d);
    if (rc) return rc;
    if (cudaMalloc(&p.det, sizeof(DetState)) != cudaSuccess) {
        cudaGetLastError();
        set_error("out of device memory for the deterministic-adjoint state");
        return SGL_ENOMEM;
    }
    p.det_density = d * (1.0 + 1e-6);   // FP64 rounding of the measurement
    return SGL_OK;
}

int det_begin(const Plan &p, const double2 *v, cudaStream_t st) {
    if (!p.det) return SGL_OK;
    SGL_CUDA_CHECK(cudaMemsetAsync(&p.det->vmax, 0, sizeof(unsigned long long), st));
    int rc = launch_absmax(v, p.M, &p.det->vmax, st);
    if (rc) return rc;
    k_det_exponent<<<1, 1, 0, st>>>(&p.det->vmax, p.det_density, &p.det->e);
    SGL_CUDA_CHECK(cudaGetLastError());
    return SGL_OK;
}

int det_finish(const Plan &p, double2 *grid, cudaStream_t st) {
    if (!p.det) return SGL_OK;
    const int64_t n = (int64_t)p.grid_elems;
    const unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * 16));
    k_det_convert<<<blocks, 256, 0, st>>>(reinterpret_cast<longlong2 *>(grid), n, &p.det->e);
    SGL_CUDA_CHECK(cudaGetLastError());
    return SGL_OK;
}

int spread_stage(Plan &p, const double2 *v, cudaStream_t st, bool allow_i8) {
    SGL_CUDA_CHECK(cudaMemsetAsync(p.grid_buf, 0, sizeof(double2) * p.grid_elems, st));
    int rc = det_begin(p, v, st);
    if (rc) return rc;
    rc = (allow_i8 && p.i8s_live()) ? launch_scatter_guarded(p, v, p.grid_buf, st)
                                    : launch_scatter(p, v, p.grid_buf, st);
    if (rc) return rc;
    return det_finish(p, p.grid_buf, st);
}

}  // namespace sgl
