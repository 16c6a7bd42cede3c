// Stage entry points of the grid-partitioned multi-GPU adjoint
// (BASELINE north star: "each GPU spreads its own nodes locally,
// then a reduce-scatter combines the oversampled grid before a slab-decomposed
// FFT").  The collectives run in the caller (torch.distributed / NCCL over
// NVLink, paper_1809_10786_b200/distributed.py); the library provides the
// per-rank compute around them, all on the plan's own padded grid:
//
//   sgl_adjoint_spread      zero + window scatter (+ halo fold) of the rank's
//                           node shard (_gridding.py:77-95, fold_wrap :34-50)
//   [reduce-scatter of axis-0 plane blocks of the grid]
//   sgl_adjoint_slab_fft    forward 2-D FFT (axes 1, 2) of the rank's planes,
//                           then the crop to the spectral box the basal stage
//                           reads (kappa1 in I_n1, kappa2 in [-B, B)), packed
//   [gather of the packed planes to the root rank]
//   sgl_adjoint_from_packed (root) unpack, 1-D FFT along axis 0, crop +
//                           deconvolution + basal adjoint (nfft.py:254-273,
//                           transform.py:408-429) -> coefficients
//   [broadcast of the coefficients]
//
// The 2-D-then-1-D order is the separable forward FFT of the reference's
// fftn (nfft.py:268) split at the slab boundary.
#include <cufft.h>

#include <algorithm>
#include <string>
#include <vector>

#include "sgl_internal.cuh"

namespace sgl {
namespace {

__device__ __forceinline__ int wrapk(int k, int n) {
    k %= n;
    return k < 0 ? k + n : k;
}

// packed[(a - a0), p1, p2] <- grid[a, g1 + pad, g2 + pad],
// g1 = (p1 - n1 / 2) mod N1, g2 = (p2 - B) mod N2
__global__ void k_pack_crop(const double2 *__restrict__ grid, WindowParams wp, int n1, int n2c, int B, int a0,
                            int planes, double2 *__restrict__ out) {
    const int64_t total = (int64_t)planes * n1 * n2c;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int p2 = (int)(i % n2c);
        const int p1 = (int)((i / n2c) % n1);
        const int a = a0 + (int)(i / ((int64_t)n2c * n1));
        const int g1 = wrapk(p1 - n1 / 2, wp.N1), g2 = wrapk(p2 - B, wp.N2);
        out[i] = grid[((size_t)a * wp.N1p + g1 + wp.pad) * wp.N2p + g2 + wp.pad];
    }
}

__global__ void k_unpack_crop(const double2 *__restrict__ in, WindowParams wp, int n1, int n2c, int B,
                              double2 *__restrict__ grid) {
    const int64_t total = (int64_t)wp.N0 * n1 * n2c;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int p2 = (int)(i % n2c);
        const int p1 = (int)((i / n2c) % n1);
        const int a = (int)(i / ((int64_t)n2c * n1));
        const int g1 = wrapk(p1 - n1 / 2, wp.N1), g2 = wrapk(p2 - B, wp.N2);
        grid[((size_t)a * wp.N1p + g1 + wp.pad) * wp.N2p + g2 + wp.pad] = in[i];
    }
}

// axis-0 planes a node's window touches (the reference's taps, nfft.py:131-141)
__global__ void k_planes(NodeSet nodes, int64_t M, WindowParams wp, int *__restrict__ mask) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= M) return;
    int lo, hi;
    window_cells(nodes.u0[i], wp.qa0, lo, hi);
    for (int a = lo; a <= hi; ++a) {
        const int w = wrapk(a, wp.N0);
        if (!mask[w]) mask[w] = 1;   // benign race: every writer stores 1
    }
}

// eta_t columns [col0, col0 + nc) of the cropped, deconvolved spectrum after
// the 1-D FFT along axis 0: eta[k0][j] = X[(k0 - 2B) mod N0][j] d0 d1 d2
// (nfft.py:268-273), column j = p1 * crop2 + p2 of the packed box
__global__ void k_axis0_crop(const double2 *__restrict__ X, int64_t nc, int64_t col0, int N0, int B, int crop2,
                             const double *__restrict__ d0, const double *__restrict__ d1,
                             const double *__restrict__ d2, double2 *__restrict__ eta) {
    const int64_t total = (int64_t)4 * B * nc;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = i % nc;
        const int k0 = (int)(i / nc);
        const int64_t col = col0 + j;
        const int p1 = (int)(col / crop2), p2 = (int)(col % crop2);
        const double2 x = X[(int64_t)wrapk(k0 - 2 * B, N0) * nc + j];
        const double s = d0[k0] * d1[p1] * d2[p2];
        eta[i] = make_double2(x.x * s, x.y * s);
    }
}

// eta[k0][p1][p2] (deconvolved) -> zeta[mi][p1][k0], m = p2 - B (the layout k_sph_adj reads)
__global__ void k_eta_to_zeta(const double2 *__restrict__ eta, int B, int n1, double2 *__restrict__ zeta) {
    const int W = 4 * B, NM = 2 * B - 1, C2 = 2 * B;
    const int64_t total = (int64_t)NM * n1 * W;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int k0 = (int)(i % W);
        const int p1 = (int)((i / W) % n1);
        const int mi = (int)(i / ((int64_t)W * n1));
        zeta[i] = eta[((int64_t)k0 * n1 + p1) * C2 + (mi + 1)];   // p2 = m + B = mi + 1
    }
}

// The plan's call serialisation (as PlanGuard in capi.cu): host threads by the
// mutex, streams by waiting on the previous call's completion event.
struct StageGuard {
    Plan &p;
    cudaStream_t st;
    std::lock_guard<std::mutex> lock;
    bool capturing = false;
    StageGuard(Plan &pl, cudaStream_t s) : p(pl), st(s), lock(pl.mu) {
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        if (cudaStreamIsCapturing(st, &cs) != cudaSuccess) cudaGetLastError();
        capturing = cs != cudaStreamCaptureStatusNone;
        if (p.done && !capturing) cudaStreamWaitEvent(st, p.done, 0);
    }
    ~StageGuard() {
        if (p.done && !capturing) cudaEventRecord(p.done, st);
    }
};

int check_sgl(const Plan &p) {
    if (p.raw || p.exact || p.M < 0) {
        set_error("the partitioned adjoint needs a fast SGL plan (not an NFFT or exact-stage plan)");
        return SGL_EINVAL;
    }
    return SGL_OK;
}

int fft_rc(cufftResult r, const char *what) {
    if (r != CUFFT_SUCCESS) {
        set_error(std::string("cuFFT error ") + std::to_string((int)r) + " in " + what);
        return SGL_ECUDA;
    }
    return SGL_OK;
}

}  // namespace
}  // namespace sgl

using namespace sgl;

extern "C" {

int sgl_plan_grid(const sgl_plan *plan, sgl_grid_info *info) {
    if (!plan || !info) {
        set_error("NULL plan or info");
        return SGL_EINVAL;
    }
    const Plan &p = *reinterpret_cast<const Plan *>(plan);
    info->data = p.grid_buf;
    info->N0 = p.wp.N0;
    info->N1 = p.wp.N1;
    info->N2 = p.wp.N2;
    info->N1p = p.wp.N1p;
    info->N2p = p.wp.N2p;
    info->pad = p.wp.pad;
    info->plane_elems = (int64_t)p.wp.N1p * p.wp.N2p;
    info->crop1 = p.n_axis[1];
    info->crop2 = 2 * p.B;
    return SGL_OK;
}

int sgl_adjoint_spread(sgl_plan *plan, const sgl_cdouble *values, void *stream) {
    if (!plan) {
        set_error("NULL plan");
        return SGL_EINVAL;
    }
    Plan &p = *reinterpret_cast<Plan *>(plan);
    int rc = check_sgl(p);
    if (rc) return rc;
    if (p.M > 0 && !values) {
        set_error("values length does not match the plan");
        return SGL_EINVAL;
    }
    SGL_CUDA_CHECK(cudaSetDevice(p.device));
    cudaStream_t st = (cudaStream_t)stream;
    StageGuard guard(p, st);
    const double2 *v = reinterpret_cast<const double2 *>(values);
    cudaPointerAttributes a;
    const bool dev = values && cudaPointerGetAttributes(&a, values) == cudaSuccess &&
                     (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged);
    cudaGetLastError();
    if (p.M > 0 && !dev) {
        SGL_CUDA_CHECK(cudaMemcpyAsync(p.val_buf, v, sizeof(double2) * p.M, cudaMemcpyHostToDevice, st));
        v = p.val_buf;
    }
    rc = spread_stage(p, v, st, true);
    if (rc) return rc;
    rc = launch_halo_fold(p, p.grid_buf, st);
    if (rc) return rc;
    SGL_CUDA_CHECK(cudaGetLastError());
    return SGL_OK;
}

int sgl_adjoint_slab_fft(sgl_plan *plan, int32_t a0, int32_t a1, sgl_cdouble *packed, void *stream) {
    if (!plan) {
        set_error("NULL plan");
        return SGL_EINVAL;
    }
    Plan &p = *reinterpret_cast<Plan *>(plan);
    int rc = check_sgl(p);
    if (rc) return rc;
    if (a0 < 0 || a1 > p.wp.N0 || a0 > a1 || (a1 > a0 && !packed)) {
        set_error("slab [a0, a1) outside the grid's axis-0 planes");
        return SGL_EINVAL;
    }
    if (a1 == a0) return SGL_OK;
    SGL_CUDA_CHECK(cudaSetDevice(p.device));
    cudaStream_t st = (cudaStream_t)stream;
    StageGuard guard(p, st);
    const int planes = a1 - a0;
    // 2-D plans over the slab's planes, cached by plane count
    cufftHandle h = 0;
    for (auto &e : p.slab_ffts)
        if (e.first == planes) h = e.second;
    if (!h) {
        long long n2[2] = {p.wp.N1, p.wp.N2}, e2[2] = {p.wp.N1p, p.wp.N2p};
        const long long pl = (long long)p.wp.N1p * p.wp.N2p;
        size_t work = 0;
        rc = fft_rc(cufftCreate(&h), "cufftCreate");
        if (rc) return rc;
        rc = fft_rc(cufftMakePlanMany64(h, 2, n2, e2, 1, pl, e2, 1, pl, CUFFT_Z2Z, planes, &work),
                    "cufftMakePlanMany64(slab)");
        if (rc) {
            cufftDestroy(h);
            return rc;
        }
        p.slab_ffts.emplace_back(planes, h);
    }
    rc = fft_rc(cufftSetStream(h, st), "cufftSetStream");
    if (rc) return rc;
    cufftDoubleComplex *first = reinterpret_cast<cufftDoubleComplex *>(
        p.grid_buf + ((size_t)a0 * p.wp.N1p + p.wp.pad) * p.wp.N2p + p.wp.pad);
    rc = fft_rc(cufftExecZ2Z(h, first, first, CUFFT_FORWARD), "cufftExecZ2Z(slab)");
    if (rc) return rc;
    const int n1 = p.n_axis[1], n2c = 2 * p.B;
    k_pack_crop<<<num_sms() * 8, 256, 0, st>>>(p.grid_buf, p.wp, n1, n2c, p.B, a0, planes,
                                               reinterpret_cast<double2 *>(packed));
    SGL_CUDA_CHECK(cudaGetLastError());
    return SGL_OK;
}

int sgl_plan_planes(const sgl_plan *plan, uint8_t *mask) {
    if (!plan || !mask) {
        set_error("NULL plan or mask");
        return SGL_EINVAL;
    }
    const Plan &p = *reinterpret_cast<const Plan *>(plan);
    int rc = check_sgl(p);
    if (rc) return rc;
    SGL_CUDA_CHECK(cudaSetDevice(p.device));
    std::vector<int> h(p.wp.N0, 0);
    if (p.M > 0) {
        int *d = nullptr;
        SGL_CUDA_CHECK(cudaMalloc(&d, sizeof(int) * p.wp.N0));
        SGL_CUDA_CHECK(cudaMemset(d, 0, sizeof(int) * p.wp.N0));
        k_planes<<<(unsigned)((p.M + 255) / 256), 256>>>(p.nodes, p.M, p.wp, d);
        const cudaError_t e = cudaMemcpy(h.data(), d, sizeof(int) * p.wp.N0, cudaMemcpyDeviceToHost);
        cudaFree(d);
        SGL_CUDA_CHECK(e);
    }
    for (int a = 0; a < p.wp.N0; ++a) mask[a] = h[a] ? 1 : 0;
    return SGL_OK;
}

int sgl_adjoint_axis0(sgl_plan *plan, const sgl_cdouble *cols, int64_t ncols, int64_t col0, sgl_cdouble *eta,
                      void *stream) {
    if (!plan) {
        set_error("NULL plan");
        return SGL_EINVAL;
    }
    Plan &p = *reinterpret_cast<Plan *>(plan);
    int rc = check_sgl(p);
    if (rc) return rc;
    const int64_t C = (int64_t)p.n_axis[1] * 2 * p.B;
    if (ncols < 0 || col0 < 0 || col0 + ncols > C || (ncols > 0 && (!cols || !eta))) {
        set_error("column block outside the packed spectral box");
        return SGL_EINVAL;
    }
    if (ncols == 0) return SGL_OK;
    SGL_CUDA_CHECK(cudaSetDevice(p.device));
    cudaStream_t st = (cudaStream_t)stream;
    StageGuard guard(p, st);
    // the plan's grid serves as scratch (N0 x ncols <= N0 x C fits it)
    double2 *X = p.grid_buf;
    SGL_CUDA_CHECK(cudaMemcpyAsync(X, cols, sizeof(double2) * (size_t)p.wp.N0 * ncols, cudaMemcpyDeviceToDevice, st));
    cufftHandle h = 0;
    for (auto &e : p.axis0_ffts)
        if (e.first == ncols) h = e.second;
    if (!h) {
        long long n1d[1] = {p.wp.N0};
        size_t work = 0;
        rc = fft_rc(cufftCreate(&h), "cufftCreate");
        if (rc) return rc;
        rc = fft_rc(cufftMakePlanMany64(h, 1, n1d, n1d, ncols, 1, n1d, ncols, 1, CUFFT_Z2Z, ncols, &work),
                    "cufftMakePlanMany64(axis 0 columns)");
        if (rc) {
            cufftDestroy(h);
            return rc;
        }
        p.axis0_ffts.emplace_back(ncols, h);
    }
    rc = fft_rc(cufftSetStream(h, st), "cufftSetStream");
    if (rc) return rc;
    cufftDoubleComplex *x = reinterpret_cast<cufftDoubleComplex *>(X);
    rc = fft_rc(cufftExecZ2Z(h, x, x, CUFFT_FORWARD), "cufftExecZ2Z(axis 0 columns)");
    if (rc) return rc;
    k_axis0_crop<<<num_sms() * 8, 256, 0, st>>>(X, ncols, col0, p.wp.N0, p.B, 2 * p.B, p.dec0, p.dec1, p.dec2,
                                                reinterpret_cast<double2 *>(eta));
    SGL_CUDA_CHECK(cudaGetLastError());
    return SGL_OK;
}

int sgl_adjoint_from_eta(sgl_plan *plan, const sgl_cdouble *eta, sgl_cdouble *coeffs, void *stream) {
    if (!plan) {
        set_error("NULL plan");
        return SGL_EINVAL;
    }
    Plan &p = *reinterpret_cast<Plan *>(plan);
    int rc = check_sgl(p);
    if (rc) return rc;
    if (!eta || !coeffs) {
        set_error("NULL spectrum or coefficient array");
        return SGL_EINVAL;
    }
    SGL_CUDA_CHECK(cudaSetDevice(p.device));
    cudaStream_t st = (cudaStream_t)stream;
    StageGuard guard(p, st);
    k_eta_to_zeta<<<num_sms() * 8, 256, 0, st>>>(reinterpret_cast<const double2 *>(eta), p.B, p.n_axis[1], p.zeta);
    SGL_CUDA_CHECK(cudaGetLastError());
    cudaPointerAttributes a;
    const bool dev = cudaPointerGetAttributes(&a, coeffs) == cudaSuccess &&
                     (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged);
    cudaGetLastError();
    double2 *c = dev ? reinterpret_cast<double2 *>(coeffs) : p.coef_buf;
    rc = launch_basal_adjoint_from_zeta(p, c, st);
    if (rc) return rc;
    if (!dev) {
        SGL_CUDA_CHECK(cudaMemcpyAsync(coeffs, p.coef_buf, sizeof(double2) * p.count, cudaMemcpyDeviceToHost, st));
        SGL_CUDA_CHECK(cudaStreamSynchronize(st));
    }
    SGL_CUDA_CHECK(cudaGetLastError());
    return SGL_OK;
}

int sgl_adjoint_from_packed(sgl_plan *plan, const sgl_cdouble *packed, sgl_cdouble *coeffs, void *stream) {
    if (!plan) {
        set_error("NULL plan");
        return SGL_EINVAL;
    }
    Plan &p = *reinterpret_cast<Plan *>(plan);
    int rc = check_sgl(p);
    if (rc) return rc;
    if (!packed || !coeffs) {
        set_error("NULL packed spectrum or coefficient array");
        return SGL_EINVAL;
    }
    SGL_CUDA_CHECK(cudaSetDevice(p.device));
    cudaStream_t st = (cudaStream_t)stream;
    StageGuard guard(p, st);
    SGL_CUDA_CHECK(cudaMemsetAsync(p.grid_buf, 0, sizeof(double2) * p.grid_elems, st));
    const int n1 = p.n_axis[1], n2c = 2 * p.B;
    k_unpack_crop<<<num_sms() * 8, 256, 0, st>>>(reinterpret_cast<const double2 *>(packed), p.wp, n1, n2c, p.B,
                                                 p.grid_buf);
    SGL_CUDA_CHECK(cudaGetLastError());
    // 1-D forward FFT along axis 0 over every column of the padded planes
    if (!p.dist_fft1) {
        long long n1d[1] = {p.wp.N0}, e1[1] = {p.wp.N0};
        const long long pl = (long long)p.wp.N1p * p.wp.N2p;
        size_t work = 0;
        cufftHandle h = 0;
        rc = fft_rc(cufftCreate(&h), "cufftCreate");
        if (rc) return rc;
        rc = fft_rc(cufftMakePlanMany64(h, 1, n1d, e1, pl, 1, e1, pl, 1, CUFFT_Z2Z, pl, &work),
                    "cufftMakePlanMany64(axis 0)");
        if (rc) {
            cufftDestroy(h);
            return rc;
        }
        p.dist_fft1 = h;
    }
    rc = fft_rc(cufftSetStream(p.dist_fft1, st), "cufftSetStream");
    if (rc) return rc;
    cufftDoubleComplex *all = reinterpret_cast<cufftDoubleComplex *>(p.grid_buf);
    rc = fft_rc(cufftExecZ2Z(p.dist_fft1, all, all, CUFFT_FORWARD), "cufftExecZ2Z(axis 0)");
    if (rc) return rc;
    cudaPointerAttributes a;
    const bool dev = cudaPointerGetAttributes(&a, coeffs) == cudaSuccess &&
                     (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged);
    cudaGetLastError();
    double2 *c = dev ? reinterpret_cast<double2 *>(coeffs) : p.coef_buf;
    rc = launch_basal_adjoint(p, p.grid_buf, c, st);
    if (rc) return rc;
    if (!dev) {
        SGL_CUDA_CHECK(cudaMemcpyAsync(coeffs, p.coef_buf, sizeof(double2) * p.count, cudaMemcpyDeviceToHost, st));
        SGL_CUDA_CHECK(cudaStreamSynchronize(st));
    }
    SGL_CUDA_CHECK(cudaGetLastError());
    return SGL_OK;
}

}  // extern "C"
