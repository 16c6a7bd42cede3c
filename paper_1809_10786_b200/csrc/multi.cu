// Single-process multi-GPU plans through the C ABI (the plan
// creation takes n_gpus): sgl_plan_create_multi shards the caller's points
// into contiguous, count-balanced node ranges, one sub-plan per device, all
// on the global rho (transform.py:39-43, 345-348).  Forward: each device
// evaluates its shard into its slice of the caller's values (no exchange).
// Adjoint: each device runs the whole adjoint of its shard and the
// coefficient vectors are summed (the "coeffs" partition of
// distributed.py; the FFT and basal adjoint are linear).  One host thread per
// device drives its sub-plan, so devices run concurrently.  Device-resident
// caller buffers are staged through host memory (one copy of the
// coefficients per call); the fastest multi-GPU path is one process per GPU
// over torch.distributed (distributed.py), which this entry point mirrors for
// consumers without Python.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "sgl_internal.cuh"

namespace sgl {
namespace {

bool dev_ptr(const void *p) {
    if (!p) return false;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// run f(k) on one host thread per sub-plan; first failure wins
template <typename F>
int per_device(size_t n, F f) {
    std::vector<int> rc(n, SGL_OK);
    std::vector<std::string> err(n);
    std::vector<std::thread> th;
    for (size_t k = 0; k < n; ++k)
        th.emplace_back([&, k]() {
            rc[k] = f(k);
            if (rc[k]) err[k] = sgl_last_error();
        });
    for (auto &t : th) t.join();
    for (size_t k = 0; k < n; ++k)
        if (rc[k]) {
            set_error(err[k]);
            return rc[k];
        }
    return SGL_OK;
}

}  // namespace

int multi_forward(Plan &p, const sgl_cdouble *coeffs, int64_t K, sgl_cdouble *values, void *stream) {
    if (K < 1 || !coeffs || (!values && p.M > 0)) {
        set_error("coefficient length does not match the bandwidth");
        return SGL_EINVAL;
    }
    const size_t n = p.subs.size();
    std::vector<sgl_cdouble> ch, vh;
    const sgl_cdouble *c = coeffs;
    if (dev_ptr(coeffs)) {   // stage device coefficients through the host once
        ch.resize((size_t)K * p.count);
        SGL_CUDA_CHECK(cudaStreamSynchronize((cudaStream_t)stream));
        SGL_CUDA_CHECK(cudaMemcpy(ch.data(), coeffs, sizeof(sgl_cdouble) * ch.size(), cudaMemcpyDefault));
        c = ch.data();
    }
    const bool vdev = dev_ptr(values);
    if (vdev) vh.resize((size_t)K * p.M);
    sgl_cdouble *vout = vdev ? vh.data() : values;
    // K > 1: per-vector calls (the values of vector k are a contiguous M-slice per shard)
    int rc = per_device(n, [&](size_t k) -> int {
        Plan &s = *p.subs[k];
        const int64_t m = s.M, off = p.sub_start[k];
        if (m == 0) return SGL_OK;
        std::vector<sgl_cdouble> tmp(K > 1 ? (size_t)K * m : 0);
        int r = sgl_forward(reinterpret_cast<sgl_plan *>(&s), c, K, K > 1 ? tmp.data() : vout + off, nullptr);
        if (r) return r;
        for (int64_t v = 0; K > 1 && v < K; ++v)
            memcpy(vout + v * p.M + off, tmp.data() + v * m, sizeof(sgl_cdouble) * m);
        return SGL_OK;
    });
    if (rc) return rc;
    if (vdev && p.M > 0)
        SGL_CUDA_CHECK(cudaMemcpyAsync(values, vh.data(), sizeof(sgl_cdouble) * vh.size(), cudaMemcpyDefault,
                                       (cudaStream_t)stream));
    if (vdev) SGL_CUDA_CHECK(cudaStreamSynchronize((cudaStream_t)stream));
    return SGL_OK;
}

int multi_adjoint(Plan &p, const sgl_cdouble *values, sgl_cdouble *coeffs, void *stream) {
    if (!coeffs || (!values && p.M > 0)) {
        set_error("values length does not match the plan");
        return SGL_EINVAL;
    }
    const size_t n = p.subs.size();
    std::vector<sgl_cdouble> vh;
    const sgl_cdouble *v = values;
    if (p.M > 0 && dev_ptr(values)) {
        vh.resize(p.M);
        SGL_CUDA_CHECK(cudaStreamSynchronize((cudaStream_t)stream));
        SGL_CUDA_CHECK(cudaMemcpy(vh.data(), values, sizeof(sgl_cdouble) * p.M, cudaMemcpyDefault));
        v = vh.data();
    }
    std::vector<std::vector<sgl_cdouble>> part(n, std::vector<sgl_cdouble>(p.count));
    int rc = per_device(n, [&](size_t k) -> int {
        Plan &s = *p.subs[k];
        if (s.M == 0) {
            std::fill(part[k].begin(), part[k].end(), sgl_cdouble{0.0, 0.0});
            return SGL_OK;
        }
        return sgl_adjoint(reinterpret_cast<sgl_plan *>(&s), v + p.sub_start[k], part[k].data(), nullptr);
    });
    if (rc) return rc;
    // the exchange: sum of the shard adjoints (in shard order: deterministic)
    std::vector<sgl_cdouble> sum(part[0]);
    for (size_t k = 1; k < n; ++k)
        for (int64_t i = 0; i < p.count; ++i) {
            sum[i].re += part[k][i].re;
            sum[i].im += part[k][i].im;
        }
    if (dev_ptr(coeffs)) {
        SGL_CUDA_CHECK(cudaMemcpyAsync(coeffs, sum.data(), sizeof(sgl_cdouble) * p.count, cudaMemcpyDefault,
                                       (cudaStream_t)stream));
        SGL_CUDA_CHECK(cudaStreamSynchronize((cudaStream_t)stream));
    } else {
        memcpy(coeffs, sum.data(), sizeof(sgl_cdouble) * p.count);
    }
    return SGL_OK;
}

}  // namespace sgl

using namespace sgl;

extern "C" {

int sgl_plan_create_multi(int32_t B, int64_t M, const double *points, int32_t sigma, int32_t q, double rho,
                          uint32_t flags, int32_t n_gpus, const int32_t *devices, sgl_plan **out) {
    if (!out) {
        set_error("output plan pointer is NULL");
        return SGL_EINVAL;
    }
    *out = nullptr;
    if (n_gpus < 1) {
        set_error("n_gpus must be >= 1");
        return SGL_EINVAL;
    }
    if (M < 0 || (M > 0 && !points)) {
        set_error("points must be (M, 3) spherical coordinates");
        return SGL_EINVAL;
    }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess) {
        cudaGetLastError();
        ndev = 0;
    }
    std::vector<int> devs(n_gpus);
    for (int k = 0; k < n_gpus; ++k) {
        devs[k] = devices ? devices[k] : k;
        if (devs[k] < 0 || devs[k] >= ndev) {
            set_error("device " + std::to_string(devs[k]) + " is not visible (" + std::to_string(ndev) +
                      " CUDA devices)");
            return SGL_EINVAL;
        }
    }
    // host copy of device points; the global rho (choose_rho, transform.py:39-43)
    std::vector<double> ph;
    const double *pts = points;
    if (M > 0 && dev_ptr(points)) {
        ph.resize((size_t)3 * M);
        SGL_CUDA_CHECK(cudaDeviceSynchronize());
        SGL_CUDA_CHECK(cudaMemcpy(ph.data(), points, sizeof(double) * ph.size(), cudaMemcpyDefault));
        pts = ph.data();
    }
    if (!(rho > 0)) {
        double r = 0.0;
        for (int64_t i = 0; i < M; ++i) r = std::max(r, pts[3 * i]);
        rho = r > 0 ? r : 1.0;
    }
    Plan *p = new Plan();
    cudaGetDevice(&p->device);
    p->B = B;
    p->M = M;
    p->rho = rho;
    p->sigma = sigma;
    p->q = q;
    p->flags = flags;
    p->count = B >= 1 ? (int64_t)B * (B + 1) * (2 * B + 1) / 6 : 0;
    p->subs.assign(n_gpus, nullptr);
    p->sub_start.assign(n_gpus + 1, 0);
    for (int k = 0; k < n_gpus; ++k) {   // shard_bounds (distributed.py)
        const int64_t base = M / n_gpus, extra = M % n_gpus;
        p->sub_start[k] = k * base + std::min<int64_t>(k, extra);
    }
    p->sub_start[n_gpus] = M;
    int rc = per_device(n_gpus, [&](size_t k) -> int {
        SGL_CUDA_CHECK(cudaSetDevice(devs[k]));
        const int64_t s = p->sub_start[k], m = p->sub_start[k + 1] - s;
        sgl_plan *h = nullptr;
        const int r = sgl_plan_create(B, m, m ? pts + 3 * s : nullptr, sigma, q, rho, flags, nullptr, &h);
        p->subs[k] = reinterpret_cast<Plan *>(h);
        return r;
    });
    cudaSetDevice(p->device);
    if (rc) {
        for (Plan *s : p->subs)
            if (s) sgl_plan_destroy(reinterpret_cast<sgl_plan *>(s));
        p->subs.clear();
        delete p;
        return rc;
    }
    const Plan &s0 = *p->subs[0];
    for (int i = 0; i < 3; ++i) {
        p->n_axis[i] = s0.n_axis[i];
        p->grid[i] = s0.grid[i];
        p->sig_axes[i] = s0.sig_axes[i];
        p->s_eff[i] = s0.s_eff[i];
        p->lam[i] = s0.lam[i];
    }
    p->q = s0.q;
    p->sigma = s0.sigma;
    p->exact = s0.exact;
    p->generic = s0.generic;
    *out = reinterpret_cast<sgl_plan *>(p);
    return SGL_OK;
}

}  // extern "C"
