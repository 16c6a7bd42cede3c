// C ABI of the B200 NFSGLFT (include/sgl_b200.h).
//
// Mirrors the reference surface transform.plan / forward / adjoint
// (transform.py:320-429) with the same argument meaning and the same
// ValueError conditions, reported as SGL_EINVAL + sgl_last_error().
#include <cufft.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>

#include "sgl_internal.cuh"

namespace sgl {

static thread_local std::string g_err;

void set_error(const std::string &msg) { g_err = msg; }

void plan_lap(Plan &p, cudaStream_t st, const char *what) {
    if (!(p.flags & SGL_FLAG_I8_PROF)) return;
    cudaStreamSynchronize(st);
    const double now =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
    if (p.lap_ms >= 0) fprintf(stderr, "plan %-28s %9.2f ms\n", what, now - p.lap_ms);
    p.lap_ms = now;
}

namespace {

bool is_device_ptr(const void *p) {
    if (!p) return false;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// page-locked (cudaHostAlloc / cudaHostRegister) host memory
bool is_pinned_host(const void *p) {
    if (!p) return false;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

int fft_check(cufftResult r, const char *what) {
    if (r != CUFFT_SUCCESS) {
        set_error(std::string("cuFFT error ") + std::to_string((int)r) + " in " + what);
        return SGL_ECUDA;
    }
    return SGL_OK;
}

void free_plan(Plan *p) {
    if (!p) return;
    if (!p->subs.empty()) {   // multi-GPU plan: only its sub-plans own device state
        for (Plan *s : p->subs) free_plan(s);
        delete p;
        return;
    }
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(p->device);
    if (p->snodes_shared) p->snodes = NodeSet();
    void *bufs[] = {p->nodes.u0, p->nodes.u1, p->nodes.u2, p->nodes.perm, p->snodes.u0, p->snodes.u1, p->snodes.u2,
                    p->snodes.perm, p->tiles, p->stiles, p->Kl, p->Km,
                    p->Kl_off_d, p->Km_off_d, p->dec0, p->dec1, p->dec2, p->grid_buf, p->beta,
                    p->coef_buf, p->val_buf, p->zeta, p->inodes.u0, p->inodes.u1, p->inodes.u2, p->inodes.perm,
                    p->itiles, p->digits, p->gmax, p->gplist, p->istiles, p->tsv, p->vdig, p->guard, p->prof, p->det};
    for (void *b : bufs)
        if (b) cudaFree(b);
    if (p->fft_ready) cufftDestroy(p->fft);
    if (p->pruned) {
        cufftDestroy(p->fft2);
        cufftDestroy(p->fft1);
    }
    if (p->fft_work) cudaFree(p->fft_work);
    for (auto &e : p->slab_ffts) cufftDestroy(e.second);
    for (auto &e : p->axis0_ffts) cufftDestroy(e.second);
    if (p->dist_fft1) cufftDestroy(p->dist_fft1);
    for (int k = 0; k < p->n_fft1r; ++k) cufftDestroy(p->fft1r[k]);
    if (p->done) cudaEventDestroy(p->done);
    if (p->ev_a) cudaEventDestroy(p->ev_a);
    if (p->ev_b) cudaEventDestroy(p->ev_b);
    if (p->ev_c) cudaEventDestroy(p->ev_c);
    if (p->ev_d) cudaEventDestroy(p->ev_d);
    if (p->copy_stream) cudaStreamDestroy(p->copy_stream);
    if (p->val_buf2) cudaFree(p->val_buf2);
    for (auto &t : p->timers)
        if (t.ready)
            for (auto &e : t.ev) cudaEventDestroy(e);
    cudaSetDevice(cur);
    delete p;
}

struct PlanGuard {
    // Serialises calls on one plan: host threads by the mutex, streams by
    // waiting on the previous call's completion event.  Inside a CUDA-graph
    // capture the graph's own dependencies order the work, and an event
    // recorded outside the capture may not be waited on, so the event is
    // left alone there.
    Plan &p;
    cudaStream_t st;
    std::lock_guard<std::mutex> lock;
    bool capturing = false;
    PlanGuard(Plan &pl, cudaStream_t s) : p(pl), st(s), lock(pl.mu) {
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        if (cudaStreamIsCapturing(st, &cs) != cudaSuccess) cudaGetLastError();
        capturing = cs != cudaStreamCaptureStatusNone;
        if (p.done && !capturing) cudaStreamWaitEvent(st, p.done, 0);
    }
    ~PlanGuard() {
        if (p.done && !capturing) cudaEventRecord(p.done, st);
    }
};

struct StageRec {
    // events recorded in call order; slot i..i+1 is charged to stage_of[i]
    Plan &p;
    int dir;
    cudaStream_t st;
    bool on;
    int n = 0;
    int stage_of[SGL_STAGE_COUNT + 1];
    StageRec(Plan &pl, int d, cudaStream_t s) : p(pl), dir(d), st(s), on(pl.profile) {
        for (float &x : p.stage_ms[dir]) x = 0.f;
    }
    void mark(int stage) {
        if (!on || n > SGL_STAGE_COUNT) return;
        stage_of[n] = stage;
        cudaEventRecord(p.timers[dir].ev[n], st);
        ++n;
    }
    void flush() {   // accumulate and restart (one forward vector / one adjoint)
        if (!on || n < 2) {
            n = 0;
            return;
        }
        cudaEventSynchronize(p.timers[dir].ev[n - 1]);
        for (int i = 0; i + 1 < n; ++i) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, p.timers[dir].ev[i], p.timers[dir].ev[i + 1]);
            p.stage_ms[dir][stage_of[i]] += ms;
        }
        n = 0;
    }
};


// ---------------------------------------------------------------------------
// device-pointer cores shared by the entry points

// side stream, events and the second value buffer for copy/compute overlap
// (created on first use)
cudaError_t ensure_side(Plan &p) {
    if (p.copy_stream) return cudaSuccess;
    cudaError_t e = cudaMalloc(&p.val_buf2, sizeof(double2) * (p.M ? p.M : 1));
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p.ev_a, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p.ev_b, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p.ev_c, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p.ev_d, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&p.copy_stream, cudaStreamNonBlocking);
    return e;
}

// The oversampled 3-D FFT of the padded interior (in place).  Pruned plans
// skip the 2-D transforms of the axis-0 planes outside the n0 spectral
// planes [0, n0/2) U [N0 - n0/2, N0): zero on input of the inverse
// transform, not read after the forward one.
int grid_fft(Plan &p, cudaStream_t st, int dir) {
    cufftDoubleComplex *interior = reinterpret_cast<cufftDoubleComplex *>(p.grid_buf + (size_t)p.wp.pad * p.wp.N2p + p.wp.pad);
    if (!p.pruned) {
        int rc = fft_check(cufftSetStream(p.fft, st), "cufftSetStream");
        if (rc) return rc;
        return fft_check(cufftExecZ2Z(p.fft, interior, interior, dir), "cufftExecZ2Z");
    }
    const size_t plane = (size_t)p.wp.N1p * p.wp.N2p;
    const int h = p.n_axis[0] / 2;
    cufftDoubleComplex *all = reinterpret_cast<cufftDoubleComplex *>(p.grid_buf);
    int rc = fft_check(cufftSetStream(p.fft2, st), "cufftSetStream");
    if (!rc) rc = fft_check(cufftSetStream(p.fft1, st), "cufftSetStream");
    if (rc) return rc;
    auto planes = [&]() {
        int r = fft_check(cufftExecZ2Z(p.fft2, interior, interior, dir), "cufftExecZ2Z(2d)");
        if (!r) {
            cufftDoubleComplex *hi = interior + (size_t)(p.wp.N0 - h) * plane;
            r = fft_check(cufftExecZ2Z(p.fft2, hi, hi, dir), "cufftExecZ2Z(2d)");
        }
        return r;
    };
    auto axis0 = [&]() {   // all columns, or only the rows the window stages touch
        if (!(p.fft_rows_on && p.n_fft1r > 0))
            return fft_check(cufftExecZ2Z(p.fft1, all, all, dir), "cufftExecZ2Z(1d)");
        int r = SGL_OK;
        for (int k = 0; k < p.n_fft1r && !r; ++k) {
            r = fft_check(cufftSetStream(p.fft1r[k], st), "cufftSetStream");
            cufftDoubleComplex *rows = all + (size_t)p.fft1r_row0[k] * p.wp.N2p;
            if (!r) r = fft_check(cufftExecZ2Z(p.fft1r[k], rows, rows, dir), "cufftExecZ2Z(1d rows)");
        }
        return r;
    };
    if (dir == CUFFT_INVERSE) {
        rc = planes();
        if (!rc) rc = axis0();
    } else {
        rc = axis0();
        if (!rc) rc = planes();
    }
    return rc;
}

int forward_core(Plan &p, const double2 *c, double2 *v, cudaStream_t st, StageRec *rec) {
    auto mark = [&](int s) {
        if (rec) rec->mark(s);
    };
    mark(SGL_STAGE_BASAL);
    int rc = p.raw ? launch_place_raw(p, c, p.grid_buf, st) : launch_basal_forward(p, c, p.grid_buf, st, nullptr);
    if (rc) return rc;
    if (p.exact) {   // direct NDFT of eta (transform.py:393-394)
        mark(SGL_STAGE_WINDOW);
        return launch_exact_forward(p, p.grid_buf, v, st);
    }
    mark(SGL_STAGE_FFT);
    rc = grid_fft(p, st, CUFFT_INVERSE);
    if (rc) return rc;
    rc = launch_halo_fill(p, p.grid_buf, st);
    if (rc) return rc;
    mark(SGL_STAGE_WINDOW);
    // int8 gather with its accuracy guard (gated FP64 gather; guard.cu)
    return p.i8 ? launch_gather_guarded(p, p.grid_buf, v, st) : launch_gather(p, p.grid_buf, v, st);
}

// the adjoint's linear tail after the window stage: halo fold, FFT, crop +
// deconvolution (+ basal adjoint)
int adjoint_tail(Plan &p, double2 *c, cudaStream_t st, StageRec *rec) {
    if (rec) rec->mark(SGL_STAGE_FFT);
    int rc = launch_halo_fold(p, p.grid_buf, st);
    if (rc) return rc;
    rc = grid_fft(p, st, CUFFT_FORWARD);
    if (rc) return rc;
    if (rec) rec->mark(SGL_STAGE_BASAL);
    return p.raw ? launch_crop_raw(p, p.grid_buf, c, st) : launch_basal_adjoint(p, p.grid_buf, c, st);
}

// the int8 scatter's accuracy decision (after guard_adjoint_estimate): read
// the flag on the host; above the bound, rerun the adjoint on the FP64 scatter
int adjoint_guard_resolve(Plan &p, const double2 *v, double2 *c, cudaStream_t st) {
    if (!(p.i8s_live() && p.guard_on && p.guard_ap > 0.0 && p.M > 0)) return SGL_OK;
    int redo = 0;
    SGL_CUDA_CHECK(cudaMemcpyAsync(&redo, &p.guard->adj_redo, sizeof(int), cudaMemcpyDeviceToHost, st));
    SGL_CUDA_CHECK(cudaStreamSynchronize(st));
    p.i8s_streak = redo ? p.i8s_streak + 1 : 0;
    if (p.i8s_auto && p.i8s_streak >= 2) p.i8s_off = true;   // the FP64 scatter from the next call on
    if (!redo) return SGL_OK;
    int rc = spread_stage(p, v, st, false);
    if (rc) return rc;
    return adjoint_tail(p, c, st, nullptr);
}

// may_sync: the int8 scatter's accuracy check reads its flag on the host
// (not possible inside a CUDA-graph capture, where it is skipped)
int adjoint_core(Plan &p, const double2 *v, double2 *c, cudaStream_t st, StageRec *rec, bool may_sync = true) {
    auto mark = [&](int s) {
        if (rec) rec->mark(s);
    };
    mark(SGL_STAGE_WINDOW);
    int rc = SGL_OK;
    if (p.exact) {   // direct adjoint NDFT (transform.py:404-405)
        rc = launch_exact_adjoint(p, v, p.grid_buf, st);
        if (rc) return rc;
        mark(SGL_STAGE_BASAL);
        return p.raw ? launch_crop_raw(p, p.grid_buf, c, st) : launch_basal_adjoint(p, p.grid_buf, c, st);
    }
    rc = spread_stage(p, v, st, true);
    if (rc) return rc;
    rc = adjoint_tail(p, c, st, rec);
    if (rc || !(p.i8s_live() && p.guard_ap > 0.0 && p.M > 0)) return rc;
    // int8 scatter accuracy check (guard.cu): estimate from the result, rerun on FP64 above the bound
    rc = guard_adjoint_estimate(p, v, c, st);
    if (rc || !(p.guard_on && may_sync)) return rc;
    return adjoint_guard_resolve(p, v, c, st);
}

}  // namespace
}  // namespace sgl

using namespace sgl;

namespace {
int plan_finish(Plan *p, const double *points, cudaStream_t st, sgl_plan **out,
                std::chrono::steady_clock::time_point t0);
}  // namespace

extern "C" {

const char *sgl_last_error(void) { return g_err.c_str(); }

int sgl_set_device(int32_t device) {
    SGL_CUDA_CHECK(cudaSetDevice(device));
    return SGL_OK;
}

int sgl_device_count(int32_t *n) {
    int c = 0;
    cudaError_t e = cudaGetDeviceCount(&c);
    if (e != cudaSuccess) {
        cudaGetLastError();
        c = 0;
    }
    if (n) *n = c;
    return SGL_OK;
}

const char *sgl_version(void) {
    return "sgl-b200 0.2.0 (sm_100a: int8 tcgen05 window engines with an FP64 accuracy guard, FP64 DMMA gridding)";
}

int sgl_plan_create(int32_t B, int64_t M, const double *points, int32_t sigma, int32_t q, double rho,
                    uint32_t flags, void *stream, sgl_plan **out) {
    g_err.clear();
    if (!out) {
        set_error("output plan pointer is NULL");
        return SGL_EINVAL;
    }
    *out = nullptr;
    if (B < 1) {
        set_error("bandwidth must be >= 1");
        return SGL_EINVAL;
    }
    if (M < 0 || (M > 0 && !points)) {
        set_error("points must be (M, 3) spherical coordinates");
        return SGL_EINVAL;
    }
    if (M > (int64_t)INT32_MAX) {
        set_error("more than 2^31-1 points per plan: shard the node set");
        return SGL_EUNSUPPORTED;
    }
    const bool exact = flags & SGL_FLAG_EXACT_LAST_STAGE;
    if (!exact) {   // the window parameters are only checked for the fast path (transform.py:352-356)
        if (q < 1) {
            set_error("cutoff parameter q must be >= 1");
            return SGL_EINVAL;
        }
        if (sigma < 2) {
            set_error("oversampling factor must be an integer >= 2");
            return SGL_EINVAL;
        }
        if ((int64_t)q >= 4LL * sigma * B) {
            set_error("cutoff q = " + std::to_string(q) + " must be below 4*sigma*B = " +
                      std::to_string(4LL * sigma * B));
            return SGL_EINVAL;
        }
    } else {
        q = 0;
        sigma = 1;
    }
    auto t0 = std::chrono::steady_clock::now();
    Plan *p = new Plan();
    cudaGetDevice(&p->device);
    cudaStream_t st = (cudaStream_t)stream;
    p->B = B;
    p->M = M;
    p->rho = rho;
    p->sigma = sigma;
    p->q = q;
    p->compact = flags & SGL_FLAG_COMPACT_K1;
    p->profile = flags & SGL_FLAG_PROFILE;
    // basal matrices in x87 extended precision unless FP64 tables are asked
    // for (FP64 construction error dominates the ill-conditioned large-rho
    // configurations: config 4 is 4.7e-9 from the extended-precision truth
    // with FP64 tables, 1.2e-9 with extended ones; the reference: 2.6e-9)
    p->precise = (flags & SGL_FLAG_PRECISE) || !(flags & SGL_FLAG_FP64_TABLES);
    p->exact = exact;
    p->flags = flags;
    p->generic = exact || (flags & SGL_FLAG_GENERIC_GRIDDING) || q > kMaxQTiled;
    {
        // int8 tensor-core gather unless the FP64 kernels are asked for;
        // int8 scatter automatic for dense node sets (see build_nodes), forced
        // by SGL_FLAG_I8_SCATTER, off with SGL_FLAG_FP64_SCATTER / FP64_WINDOW
        p->i8 = !p->generic && !(flags & SGL_FLAG_FP64_WINDOW);
        p->i8s = p->i8 && (flags & SGL_FLAG_I8_SCATTER);
        p->i8s_auto = p->i8 && !p->i8s && !(flags & SGL_FLAG_FP64_SCATTER);
    }
    p->n_axis[0] = 4 * B;
    p->n_axis[1] = p->compact ? 2 * B : 4 * B;
    p->n_axis[2] = 2 * B;
    p->count = (int64_t)B * (B + 1) * (2 * B + 1) / 6;
    // sigma escalation (transform.py:357-362) and geometry (nfft.py:174-182)
    for (int ax = 0; ax < 3; ++ax) {
        int s = sigma;
        auto pow2 = [](int64_t v) {
            int64_t g = 1;
            while (g < v) g <<= 1;
            return g;
        };
        if (exact) {   // eta on I_n itself: no oversampling, no window
            p->sig_axes[ax] = 1;
            p->grid[ax] = p->n_axis[ax];
            p->s_eff[ax] = 1.0;
            p->lam[ax] = 0.0;
            continue;
        }
        while (pow2((int64_t)s * p->n_axis[ax]) <= q) s *= 2;
        p->sig_axes[ax] = s;
        p->grid[ax] = (int)pow2((int64_t)s * p->n_axis[ax]);
        p->s_eff[ax] = (double)p->grid[ax] / p->n_axis[ax];
        p->lam[ax] = p->s_eff[ax] * q / ((2 * p->s_eff[ax] - 1) * kPi);
    }
    return plan_finish(p, points, st, out, t0);
}

}  // extern "C"

namespace {

// Shared second half of plan creation: window constants, halo geometry,
// nodes, tables, buffers, cuFFT plan, TMA descriptor.
int plan_finish(Plan *p, const double *points, cudaStream_t st, sgl_plan **out,
                std::chrono::steady_clock::time_point t0) {
    const int64_t M = p->M;
    const int q = p->q;
    const bool exact = p->exact;
    WindowParams &wp = p->wp;
    wp.N0 = p->grid[0];
    wp.N1 = p->grid[1];
    wp.N2 = p->grid[2];
    // halo width: q, widened on grids whose padded plane would be smaller than
    // the TMA slab box (kBoxMax^2) so that the box always fits the plane
    int pad = q;
    if (!exact && q > 0 && std::min(wp.N1, wp.N2) + 2 * q < kBoxMax)
        pad = (kBoxMax - std::min(wp.N1, wp.N2) + 1) / 2;
    wp.N1p = wp.N1 + 2 * pad;
    wp.N2p = wp.N2 + 2 * pad;
    wp.q = q;
    wp.pad = pad;
    p->grid_elems = (size_t)wp.N0 * wp.N1p * wp.N2p;
    if (wp.N1p < kBoxMax || wp.N2p < kBoxMax) p->generic = true;   // (not reached: pad widens the plane)
    if (wp.N1p < kI8Box1 || pad != q) p->i8 = false;   // digit TMA box within the plane; aligned K ranges
    if (!p->i8) p->i8s = p->i8s_auto = false;
    double *cs[3] = {&wp.c0, &wp.c1, &wp.c2}, *hs[3] = {&wp.h0, &wp.h1, &wp.h2};
    for (int ax = 0; ax < 3; ++ax) {
        if (exact) {
            *cs[ax] = *hs[ax] = 0.0;
            continue;
        }
        const double N = p->grid[ax], a = N / kTwoPi, lam = p->lam[ax];
        *cs[ax] = a / std::sqrt(kTwoPi * lam);                          // nfft.py:137
        *hs[ax] = ((kTwoPi / N) * (kTwoPi / N)) * (a * a) / (2.0 * lam);  // nfft.py:138
    }
    int *qas[3] = {&wp.qa0, &wp.qa1, &wp.qa2};
    for (int ax = 0; ax < 3; ++ax) {
        *qas[ax] = q;
        if (p->raw && ax < 3 - p->d) {   // dummy axis of a d < 3 NFFT: one tap of weight 1
            *qas[ax] = 0;
            *cs[ax] = 1.0;
            *hs[ax] = 0.0;
        }
    }
    wp.r0_1 = std::exp(-2.0 * wp.h0);
    wp.r0_8 = std::exp(-2.0 * wp.h0 * 64.0);
    wp.r1_1 = std::exp(-2.0 * wp.h1);
    wp.r1_4 = std::exp(-2.0 * wp.h1 * 16.0);
    wp.r2_1 = std::exp(-2.0 * wp.h2);
    wp.r2_4 = std::exp(-2.0 * wp.h2 * 16.0);
    int rc = SGL_OK;
    const double *dpts = points;
    double *owned = nullptr;
    if (M > 0 && !is_device_ptr(points)) {
        const int cols = p->raw ? p->d : 3;   // (M, d) torus nodes of an NFFT plan
        if (cudaMalloc(&owned, sizeof(double) * cols * M) != cudaSuccess ||
            cudaMemcpyAsync(owned, points, sizeof(double) * cols * M, cudaMemcpyHostToDevice, st) != cudaSuccess) {
            set_error("CUDA error while uploading points");
            rc = SGL_ECUDA;
        }
        dpts = owned;
    }
    plan_lap(*p, st, "start");
    if (rc == SGL_OK) rc = resolve_rho(*p, dpts, st);
    // the basal matrices depend on (B, rho) only: built on a host thread while
    // the device sorts and tiles the nodes
    std::vector<double> Kl, Km;
    std::thread tables;
    if (rc == SGL_OK && !p->raw) tables = std::thread([&]() { basal_tables_host(*p, Kl, Km); });
    if (rc == SGL_OK) rc = build_nodes(*p, dpts, st);
    plan_lap(*p, st, "nodes (total)");
    if (tables.joinable()) tables.join();
    plan_lap(*p, st, "basal tables (host, join)");
    if (owned) {
        cudaStreamSynchronize(st);
        cudaFree(owned);
    }
    if (rc == SGL_OK) rc = p->raw ? build_deconv_tables(*p) : upload_basal_tables(*p, Kl, Km);
    plan_lap(*p, st, "basal tables upload");
    if (rc == SGL_OK) {
        if (cudaMalloc(&p->grid_buf, sizeof(double2) * p->grid_elems) != cudaSuccess ||
            cudaMalloc(&p->beta, sizeof(double2) * (size_t)std::max(1, p->B * p->B * 4 * p->B)) != cudaSuccess ||
            cudaMalloc(&p->coef_buf, sizeof(double2) * p->count) != cudaSuccess ||
            cudaMalloc(&p->val_buf, sizeof(double2) * (M ? M : 1)) != cudaSuccess ||
            (!p->raw &&
             cudaMalloc(&p->zeta, sizeof(double2) * (size_t)(2 * p->B - 1) * p->n_axis[1] * (4 * p->B)) !=
                 cudaSuccess)) {
            cudaGetLastError();
            set_error("out of device memory for the plan's grid / staging buffers");
            rc = SGL_ENOMEM;
        }
    }
    if (rc == SGL_OK && !exact) {
        // transform the interior of the halo-padded grid in place
        // 64-bit plan: the padded grid exceeds 2^31 elements from B = 256 on
        // rank d over the active (trailing) axes; the SGL transform is 3-D
        const int rank = p->raw ? p->d : 3;
        // Pruned FFT when at most half the axis-0 planes carry the spectrum:
        // a batched 2-D plan and a 1-D plan sharing one work area; otherwise
        // (or if those plans fail) a single rank-d plan
        const bool want = rank == 3 && 2 * p->n_axis[0] <= p->grid[0] && !(p->flags & SGL_FLAG_FULL_FFT);
        if (want) {
            long long n2[2] = {p->grid[1], p->grid[2]}, e2[2] = {wp.N1p, wp.N2p};
            const long long pl = (long long)wp.N1p * wp.N2p;
            long long n1[1] = {p->grid[0]}, e1[1] = {p->grid[0]};
            size_t w2 = 0, w1 = 0;
            bool made2 = false, made1 = false;
            bool ok = cufftCreate(&p->fft2) == CUFFT_SUCCESS;
            made2 = ok;
            ok = ok && cufftCreate(&p->fft1) == CUFFT_SUCCESS;
            made1 = ok;
            ok = ok && cufftSetAutoAllocation(p->fft2, 0) == CUFFT_SUCCESS &&
                 cufftSetAutoAllocation(p->fft1, 0) == CUFFT_SUCCESS;
            ok = ok && cufftMakePlanMany64(p->fft2, 2, n2, e2, 1, pl, e2, 1, pl, CUFFT_Z2Z, p->n_axis[0] / 2, &w2) ==
                           CUFFT_SUCCESS;
            ok = ok && cufftMakePlanMany64(p->fft1, 1, n1, e1, pl, 1, e1, pl, 1, CUFFT_Z2Z, pl, &w1) == CUFFT_SUCCESS;
            const size_t wmax = std::max(w2, w1);
            ok = ok && (wmax == 0 || cudaMalloc(&p->fft_work, wmax) == cudaSuccess);
            ok = ok && cufftSetWorkArea(p->fft2, p->fft_work) == CUFFT_SUCCESS &&
                 cufftSetWorkArea(p->fft1, p->fft_work) == CUFFT_SUCCESS;
            p->pruned = ok;
            if (!ok) {
                cudaGetLastError();
                if (made2) cufftDestroy(p->fft2);
                if (made1) cufftDestroy(p->fft1);
                if (p->fft_work) cudaFree(p->fft_work);
    for (auto &e : p->slab_ffts) cufftDestroy(e.second);
    for (auto &e : p->axis0_ffts) cufftDestroy(e.second);
    if (p->dist_fft1) cufftDestroy(p->dist_fft1);
                p->fft_work = nullptr;
            }
        }
        if (!p->pruned) {
            long long n[3] = {p->grid[0], p->grid[1], p->grid[2]};
            long long emb[3] = {wp.N0, wp.N1p, wp.N2p};
            const long long dist = (long long)p->grid_elems;
            size_t work = 0;
            rc = fft_check(cufftCreate(&p->fft), "cufftCreate");
            if (rc == SGL_OK) {
                p->fft_ready = true;
                rc = fft_check(cufftMakePlanMany64(p->fft, rank, n + 3 - rank, emb + 3 - rank, 1, dist,
                                                   emb + 3 - rank, 1, dist, CUFFT_Z2Z, 1, &work),
                               "cufftMakePlanMany64");
            }
        }
    }
    plan_lap(*p, st, "buffers + cuFFT plans");
    if (rc == SGL_OK && !p->generic && !exact) rc = make_grid_tmap(*p);
    if (rc == SGL_OK && p->i8) rc = setup_i8(*p);
    plan_lap(*p, st, "setup int8 gather");
    if (rc == SGL_OK && p->i8s) rc = setup_scatter_i8(*p);
    plan_lap(*p, st, "setup int8 scatter");
    if (rc == SGL_OK) rc = setup_guard(*p);
    if (rc == SGL_OK && (p->flags & SGL_FLAG_I8_PROF) && (p->i8 || p->i8s) &&
        cudaMalloc(&p->prof, sizeof(unsigned long long) * 8 * num_sms()) != cudaSuccess) {
        cudaGetLastError();
        set_error("out of device memory for the profile counters");
        rc = SGL_ENOMEM;
    }
    if (rc == SGL_OK && p->i8s && M > 0) {
        // adjoint guard: response A_p of the tail to white grid noise of the
        // spread's per-cell rms for unit-rms values (guard.cu)
        const double cells = (double)p->grid[0] * p->grid[1] * p->grid[2];
        rc = launch_noise_grid(*p, std::sqrt((double)M * p->guard_tap2 / cells), st);
        if (rc == SGL_OK) rc = adjoint_tail(*p, p->coef_buf, st, nullptr);
        if (rc == SGL_OK) rc = read_absmax(*p, p->coef_buf, p->count, st, &p->guard_ap);
        plan_lap(*p, st, "guard calibration");
    }
    if (rc == SGL_OK) rc = setup_det(*p, st);   // SGL_FLAG_DETERMINISTIC: window density (determ.cu)
    plan_lap(*p, st, "deterministic-adjoint density");
    p->fft_rows_on = p->n_fft1r > 0;   // (after the guard calibration's full-grid transform)
    if (rc == SGL_OK && cudaEventCreateWithFlags(&p->done, cudaEventDisableTiming) != cudaSuccess) {
        set_error("cudaEventCreate failed");
        rc = SGL_ECUDA;
    }
    if (rc == SGL_OK && p->profile) {
        for (auto &t : p->timers) {
            for (auto &e : t.ev) cudaEventCreate(&e);
            t.ready = true;
        }
    }
    cudaStreamSynchronize(st);   // the plan is complete (and the caller's points are free) on return
    auto t1 = std::chrono::steady_clock::now();
    p->plan_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
    if (rc != SGL_OK) {
        free_plan(p);
        return rc;
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error(std::string("CUDA error: ") + cudaGetErrorString(e));
        free_plan(p);
        return SGL_ECUDA;
    }
    *out = reinterpret_cast<sgl_plan *>(p);
    return SGL_OK;
}

}  // namespace

extern "C" {

int sgl_nfft_plan_create(int32_t d, const int32_t *n_axis_d, int64_t M, const double *nodes,
                         const int32_t *sigma_d, int32_t q, uint32_t flags, void *stream, sgl_plan **out) {
    g_err.clear();
    if (!out || !n_axis_d || !sigma_d) {
        set_error("NULL n_axis, sigma or output plan pointer");
        return SGL_EINVAL;
    }
    *out = nullptr;
    if (d < 1 || d > 3) {
        set_error("only d <= 3 supported");
        return SGL_EINVAL;
    }
    // nfft.py:164-176; leading axes 0 .. 2-d are length-1 dummies
    int32_t n_axis[3] = {1, 1, 1}, sigma[3] = {2, 2, 2};
    for (int j = 0; j < d; ++j) {
        n_axis[3 - d + j] = n_axis_d[j];
        sigma[3 - d + j] = sigma_d[j];
        if (n_axis_d[j] < 2 || n_axis_d[j] % 2) {
            set_error("per-axis degree must be even and >= 2");
            return SGL_EINVAL;
        }
    }
    if (M < 0 || (M > 0 && !nodes)) {
        set_error("nodes must be (m, d)");
        return SGL_EINVAL;
    }
    if (M > (int64_t)INT32_MAX) {
        set_error("more than 2^31-1 points per plan: shard the node set");
        return SGL_EUNSUPPORTED;
    }
    const bool exact = flags & SGL_FLAG_EXACT_LAST_STAGE;
    auto pow2 = [](int64_t v) {
        int64_t g = 1;
        while (g < v) g <<= 1;
        return g;
    };
    int32_t sig[3] = {sigma[0], sigma[1], sigma[2]};
    if (!exact) {
        for (int ax = 0; ax < 3; ++ax)
            if (sig[ax] < 2) {
                set_error("oversampling factor must be an integer >= 2");
                return SGL_EINVAL;
            }
        if (q < 1) {
            set_error("cutoff parameter must be >= 1");
            return SGL_EINVAL;
        }
        int64_t gmin = INT64_MAX;
        for (int ax = 3 - d; ax < 3; ++ax) gmin = std::min<int64_t>(gmin, pow2((int64_t)sig[ax] * n_axis[ax]));
        if (q >= gmin) {
            set_error("cutoff q = " + std::to_string(q) + " must be below sigma*n = " + std::to_string(gmin));
            return SGL_EINVAL;
        }
    } else {
        q = 0;
        sig[0] = sig[1] = sig[2] = 1;
    }
    auto t0 = std::chrono::steady_clock::now();
    Plan *p = new Plan();
    cudaGetDevice(&p->device);
    p->raw = true;
    p->d = d;
    p->B = 0;
    p->M = M;
    p->rho = 1.0;
    p->sigma = sig[0];
    p->q = q;
    p->profile = flags & SGL_FLAG_PROFILE;
    p->exact = exact;
    p->flags = flags;
    p->generic = exact || (flags & SGL_FLAG_GENERIC_GRIDDING) || q > kMaxQTiled || d < 3;
    {
        // The int8 gather's digit-split error (~1e-15 of the local grid scale) is
        // amplified by the deconvolution gain of the spectrum's edge (up to
        // ~65 per axis at sigma = 2): harmless for SGL spectra (<= 2.5e-12 even
        // for edge-concentrated coefficients, tools/i8_adversarial.py) but 1.8e-10
        // for a white raw NFFT spectrum at q = 16.  Raw NFFT plans therefore keep
        // the FP64 gather unless SGL_FLAG_I8_GATHER asks for it (the accuracy
        // guard then still switches a call to FP64 when its bound is exceeded).
        p->i8 = !p->generic && (flags & SGL_FLAG_I8_GATHER);
    }
    p->count = (int64_t)n_axis[0] * n_axis[1] * n_axis[2];
    for (int ax = 0; ax < 3; ++ax) {   // nfft.py:174, 181-182 (no sigma escalation in the NFFT layer)
        const bool dummy = ax < 3 - d;
        p->n_axis[ax] = n_axis[ax];
        p->sig_axes[ax] = dummy ? 1 : sig[ax];
        p->grid[ax] = (exact || dummy) ? n_axis[ax] : (int)pow2((int64_t)sig[ax] * n_axis[ax]);
        p->s_eff[ax] = (double)p->grid[ax] / n_axis[ax];
        p->lam[ax] = (exact || dummy) ? 0.0 : p->s_eff[ax] * q / ((2 * p->s_eff[ax] - 1) * kPi);
    }
    return plan_finish(p, nodes, (cudaStream_t)stream, out, t0);
}

void sgl_plan_destroy(sgl_plan *plan) { free_plan(reinterpret_cast<Plan *>(plan)); }

int sgl_plan_get_info(const sgl_plan *plan, sgl_plan_info *info) {
    if (!plan || !info) {
        set_error("NULL plan or info");
        return SGL_EINVAL;
    }
    const Plan &p = *reinterpret_cast<const Plan *>(plan);
    if (!p.subs.empty()) {   // multi-GPU plan: sub-plan 0's geometry, node totals over the shards
        int rc = sgl_plan_get_info(reinterpret_cast<const sgl_plan *>(p.subs[0]), info);
        if (rc) return rc;
        info->M = p.M;
        info->n_gpus = (int32_t)p.subs.size();
        for (size_t k = 1; k < p.subs.size(); ++k) {
            sgl_plan_info s;
            rc = sgl_plan_get_info(reinterpret_cast<const sgl_plan *>(p.subs[k]), &s);
            if (rc) return rc;
            info->n_tiles += s.n_tiles;
            info->tile_nodes += s.tile_nodes;
            info->tile_dmma += s.tile_dmma;
            info->i8_tiles += s.i8_tiles;
            info->i8_ksteps += s.i8_ksteps;
            info->i8_sksteps += s.i8_sksteps;
            info->plan_ms = std::max(info->plan_ms, s.plan_ms);
            info->guard_fwd_fallbacks += s.guard_fwd_fallbacks;
            info->guard_adj_fallbacks += s.guard_adj_fallbacks;
        }
        return SGL_OK;
    }
    info->n_gpus = 1;
    info->B = p.B;
    info->M = p.M;
    info->rho = p.rho;
    info->sigma = p.sigma;
    info->q = p.q;
    for (int i = 0; i < 3; ++i) {
        info->n_axis[i] = p.n_axis[i];
        info->grid[i] = p.grid[i];
        info->sigma_axes[i] = p.sig_axes[i];
        info->sigma_eff[i] = p.s_eff[i];
        info->lam[i] = p.lam[i];
    }
    info->coeff_count = p.count;
    info->n_tiles = p.n_tiles;
    info->tile_nodes = p.tile_nodes;
    info->tile_dmma = p.tile_dmma;
    info->generic = p.generic ? 1 : 0;
    info->exact = p.exact ? 1 : 0;
    info->plan_ms = p.plan_ms;
    info->i8_gather = p.i8 ? 1 : 0;
    info->i8_tiles = p.n_itiles;
    info->i8_ksteps = p.i8_ksteps;
    info->i8_scatter = p.i8s_live() ? 1 : 0;   // the engine the adjoint uses now (Plan::i8s_off)
    info->i8_sksteps = p.i8_sksteps;
    info->guard = p.guard_on ? 1 : 0;
    info->guard_ap = p.guard_ap;
    info->guard_fwd_fallbacks = info->guard_adj_fallbacks = 0;
    info->guard_est_fwd = info->guard_est_adj = 0.0;
    if (p.guard) {   // diagnostics: a synchronous read of the device state
        GuardState g;
        int cur = 0;
        cudaGetDevice(&cur);
        cudaSetDevice(p.device);
        if (cudaMemcpy(&g, p.guard, sizeof(g), cudaMemcpyDeviceToHost) == cudaSuccess) {
            info->guard_fwd_fallbacks = (int64_t)g.fwd_count;
            info->guard_adj_fallbacks = (int64_t)g.adj_count;
            info->guard_est_fwd = g.est_fwd;
            info->guard_est_adj = g.est_adj;
        } else {
            cudaGetLastError();
        }
        cudaSetDevice(cur);
    }
    return SGL_OK;
}

int sgl_plan_stage_ms(const sgl_plan *plan, int32_t dir, float *ms, int32_t n) {
    if (!plan || !ms || dir < 0 || dir > 1) {
        set_error("bad arguments to sgl_plan_stage_ms");
        return SGL_EINVAL;
    }
    const Plan &p = *reinterpret_cast<const Plan *>(plan);
    for (int i = 0; i < n && i < SGL_STAGE_COUNT; ++i) ms[i] = p.stage_ms[dir][i];
    return SGL_OK;
}

int sgl_forward(sgl_plan *plan, const sgl_cdouble *coeffs, int64_t K, sgl_cdouble *values, void *stream) {
    g_err.clear();
    if (!plan) {
        set_error("NULL plan");
        return SGL_EINVAL;
    }
    Plan &p = *reinterpret_cast<Plan *>(plan);
    if (!p.subs.empty()) return multi_forward(p, coeffs, K, values, stream);
    SGL_CUDA_CHECK(cudaSetDevice(p.device));
    PlanGuard guard(p, (cudaStream_t)stream);
    if (K < 1 || !coeffs || (!values && p.M > 0)) {
        set_error("coefficient length does not match the bandwidth");
        return SGL_EINVAL;
    }
    cudaStream_t st = (cudaStream_t)stream;
    const bool cdev = is_device_ptr(coeffs), vdev = values ? is_device_ptr(values) : true;
    // K > 1 into host memory: double-buffer the values and download vector k
    // on the side stream while vector k+1 is computed.  Vector k+1 is enqueued
    // BEFORE the download of vector k is issued: with pageable (not pinned)
    // user memory the download call blocks the host until it completes, and
    // the GPU must already hold the next vector's work by then.
    const bool overlap = !vdev && p.M > 0 && K > 1;
    if (overlap) SGL_CUDA_CHECK(ensure_side(p));
    StageRec rec(p, 0, st);
    cudaEvent_t drained[2] = {p.ev_a, p.ev_b}, computed[2] = {p.ev_c, p.ev_d};
    auto download = [&](int64_t k) -> int {   // vector k: val_buf / val_buf2 -> host, side stream
        double2 *v = (k & 1) ? p.val_buf2 : p.val_buf;
        SGL_CUDA_CHECK(cudaStreamWaitEvent(p.copy_stream, computed[k & 1], 0));
        SGL_CUDA_CHECK(cudaMemcpyAsync(reinterpret_cast<double2 *>(values) + k * p.M, v, sizeof(double2) * p.M,
                                       cudaMemcpyDeviceToHost, p.copy_stream));
        SGL_CUDA_CHECK(cudaEventRecord(drained[k & 1], p.copy_stream));
        return SGL_OK;
    };
    for (int64_t k = 0; k < K; ++k) {
        rec.mark(SGL_STAGE_H2D);
        const double2 *c = reinterpret_cast<const double2 *>(coeffs) + k * p.count;
        if (!cdev) {
            SGL_CUDA_CHECK(cudaMemcpyAsync(p.coef_buf, c, sizeof(double2) * p.count, cudaMemcpyHostToDevice, st));
            c = p.coef_buf;
        }
        double2 *v = vdev ? reinterpret_cast<double2 *>(values) + k * p.M : ((overlap && (k & 1)) ? p.val_buf2 : p.val_buf);
        if (overlap && k >= 2) SGL_CUDA_CHECK(cudaStreamWaitEvent(st, drained[k & 1], 0));   // download of k-2 done
        const int rc = forward_core(p, c, v, st, &rec);
        if (rc) return rc;
        rec.mark(SGL_STAGE_D2H);
        if (overlap) {
            SGL_CUDA_CHECK(cudaEventRecord(computed[k & 1], st));
            if (k >= 1) {
                const int r = download(k - 1);
                if (r) return r;
            }
        } else if (!vdev && p.M > 0) {
            SGL_CUDA_CHECK(cudaMemcpyAsync(reinterpret_cast<double2 *>(values) + k * p.M, v, sizeof(double2) * p.M,
                                           cudaMemcpyDeviceToHost, st));
        }
        rec.mark(SGL_STAGE_COUNT);
        rec.flush();
    }
    if (overlap) {   // the last vector, then join the side stream back into st
        const int r = download(K - 1);
        if (r) return r;
        SGL_CUDA_CHECK(cudaEventRecord(p.ev_c, p.copy_stream));
        SGL_CUDA_CHECK(cudaStreamWaitEvent(st, p.ev_c, 0));
    }
    if (!vdev) SGL_CUDA_CHECK(cudaStreamSynchronize(st));
    SGL_CUDA_CHECK(cudaGetLastError());
    return SGL_OK;
}

int sgl_adjoint(sgl_plan *plan, const sgl_cdouble *values, sgl_cdouble *coeffs, void *stream) {
    g_err.clear();
    if (!plan) {
        set_error("NULL plan");
        return SGL_EINVAL;
    }
    Plan &p = *reinterpret_cast<Plan *>(plan);
    if (!p.subs.empty()) return multi_adjoint(p, values, coeffs, stream);
    SGL_CUDA_CHECK(cudaSetDevice(p.device));
    PlanGuard guard(p, (cudaStream_t)stream);
    if (!coeffs || (!values && p.M > 0)) {
        set_error("values length does not match the plan");
        return SGL_EINVAL;
    }
    cudaStream_t st = (cudaStream_t)stream;
    const bool vdev = values ? is_device_ptr(values) : true, cdev = is_device_ptr(coeffs);
    StageRec rec(p, 1, st);
    rec.mark(SGL_STAGE_H2D);
    const double2 *v = reinterpret_cast<const double2 *>(values);
    if (!vdev && p.M > 0) {
        SGL_CUDA_CHECK(cudaMemcpyAsync(p.val_buf, v, sizeof(double2) * p.M, cudaMemcpyHostToDevice, st));
        v = p.val_buf;
    }
    double2 *c = cdev ? reinterpret_cast<double2 *>(coeffs) : p.coef_buf;
    const int rc = adjoint_core(p, v, c, st, &rec, !guard.capturing);
    if (rc) return rc;
    rec.mark(SGL_STAGE_D2H);
    if (!cdev) {
        SGL_CUDA_CHECK(cudaMemcpyAsync(coeffs, p.coef_buf, sizeof(double2) * p.count, cudaMemcpyDeviceToHost, st));
        SGL_CUDA_CHECK(cudaStreamSynchronize(st));
    }
    rec.mark(SGL_STAGE_COUNT);
    rec.flush();
    SGL_CUDA_CHECK(cudaGetLastError());
    return SGL_OK;
}

int sgl_forward_adjoint(sgl_plan *plan, const sgl_cdouble *coeffs, sgl_cdouble *values_out,
                        const sgl_cdouble *values_in, sgl_cdouble *coeffs_out, void *stream) {
    g_err.clear();
    if (!plan) {
        set_error("NULL plan");
        return SGL_EINVAL;
    }
    Plan &p = *reinterpret_cast<Plan *>(plan);
    if (!p.subs.empty()) {
        const int rc = multi_forward(p, coeffs, 1, values_out, stream);
        return rc ? rc : multi_adjoint(p, values_in, coeffs_out, stream);
    }
    SGL_CUDA_CHECK(cudaSetDevice(p.device));
    PlanGuard guard(p, (cudaStream_t)stream);
    if (!coeffs || !coeffs_out || (p.M > 0 && (!values_out || !values_in))) {
        set_error("coefficient / value arrays do not match the plan");
        return SGL_EINVAL;
    }
    cudaStream_t st = (cudaStream_t)stream;
    SGL_CUDA_CHECK(ensure_side(p));
    cudaStream_t cs = p.copy_stream;
    const bool cdev = is_device_ptr(coeffs), codev = is_device_ptr(coeffs_out);
    const bool vodev = values_out ? is_device_ptr(values_out) : true;
    const bool videv = values_in ? is_device_ptr(values_in) : true;
    // Pinned host buffers: copies are truly asynchronous, queued on the side
    // stream up front.  Pageable ones: cudaMemcpyAsync blocks the host until
    // the copy is done, so each is issued only after the kernels it should
    // overlap are enqueued (value upload after the forward, value download
    // after the adjoint).
    const bool vin_pinned = !videv && is_pinned_host(values_in), vout_pinned = !vodev && is_pinned_host(values_out);
    // coefficients first: a copy queued behind the large value upload would
    // hold up the forward (copies in one direction share an engine queue)
    const double2 *c = reinterpret_cast<const double2 *>(coeffs);
    if (!cdev) {
        SGL_CUDA_CHECK(cudaMemcpyAsync(p.coef_buf, c, sizeof(double2) * p.count, cudaMemcpyHostToDevice, st));
        c = p.coef_buf;
    }
    const double2 *vin = reinterpret_cast<const double2 *>(values_in);
    auto upload = [&]() -> int {   // adjoint input: H2D on the side stream, overlapped with the forward
        SGL_CUDA_CHECK(cudaEventRecord(p.ev_a, st));   // the plan's previous work is ordered before
        SGL_CUDA_CHECK(cudaStreamWaitEvent(cs, p.ev_a, 0));
        SGL_CUDA_CHECK(cudaMemcpyAsync(p.val_buf2, values_in, sizeof(double2) * p.M, cudaMemcpyHostToDevice, cs));
        SGL_CUDA_CHECK(cudaEventRecord(p.ev_a, cs));   // the adjoint waits on this upload only
        return SGL_OK;
    };
    if (!videv && p.M > 0) {
        if (vin_pinned) {
            const int r = upload();
            if (r) return r;
        }
        vin = p.val_buf2;
    }
    double2 *vout = vodev ? reinterpret_cast<double2 *>(values_out) : p.val_buf;
    int rc = forward_core(p, c, vout, st, nullptr);
    if (rc) return rc;
    if (!videv && p.M > 0 && !vin_pinned) {
        rc = upload();   // pageable: blocks the host while the GPU runs the forward
        if (rc) return rc;
    }
    // forward output: D2H on the side stream, overlapped with the adjoint
    SGL_CUDA_CHECK(cudaEventRecord(p.ev_b, st));
    SGL_CUDA_CHECK(cudaStreamWaitEvent(cs, p.ev_b, 0));
    if (!vodev && p.M > 0 && vout_pinned)
        SGL_CUDA_CHECK(cudaMemcpyAsync(values_out, p.val_buf, sizeof(double2) * p.M, cudaMemcpyDeviceToHost, cs));
    if (!videv && p.M > 0) SGL_CUDA_CHECK(cudaStreamWaitEvent(st, p.ev_a, 0));
    double2 *cout = codev ? reinterpret_cast<double2 *>(coeffs_out) : p.coef_buf;
    rc = adjoint_core(p, vin, cout, st, nullptr, false);   // enqueue only; the guard decision follows
    if (rc) return rc;
    if (!vodev && p.M > 0 && !vout_pinned)   // pageable: blocks the host while the GPU runs the adjoint
        SGL_CUDA_CHECK(cudaMemcpyAsync(values_out, p.val_buf, sizeof(double2) * p.M, cudaMemcpyDeviceToHost, cs));
    if (!guard.capturing) {
        rc = adjoint_guard_resolve(p, vin, cout, st);
        if (rc) return rc;
    }
    if (!codev)
        SGL_CUDA_CHECK(cudaMemcpyAsync(coeffs_out, p.coef_buf, sizeof(double2) * p.count, cudaMemcpyDeviceToHost, st));
    // join the side stream back into st (the next call on this plan reuses val_buf)
    SGL_CUDA_CHECK(cudaEventRecord(p.ev_b, cs));
    SGL_CUDA_CHECK(cudaStreamWaitEvent(st, p.ev_b, 0));
    if (!codev || !vodev) SGL_CUDA_CHECK(cudaStreamSynchronize(st));
    SGL_CUDA_CHECK(cudaGetLastError());
    return SGL_OK;
}

// ---------------------------------------------------------------------------
// direct sums (transform.py:95-139)

}  // extern "C"

namespace {

struct DeviceScratch {
    std::vector<void *> ptrs;
    cudaStream_t st;
    explicit DeviceScratch(cudaStream_t s) : st(s) {}
    ~DeviceScratch() {
        for (void *p : ptrs) cudaFreeAsync(p, st);
    }
    // device copy of a host input (or the pointer itself when on the device)
    template <typename T>
    int input(const T *src, size_t n, const T **dst) {
        if (!src || n == 0 || is_device_ptr(src)) {
            *dst = src;
            return SGL_OK;
        }
        void *d = nullptr;
        SGL_CUDA_CHECK(cudaMallocAsync(&d, sizeof(T) * n, st));
        ptrs.push_back(d);
        SGL_CUDA_CHECK(cudaMemcpyAsync(d, src, sizeof(T) * n, cudaMemcpyHostToDevice, st));
        *dst = reinterpret_cast<const T *>(d);
        return SGL_OK;
    }
    template <typename T>
    int output(T *user, size_t n, T **dst) {
        if (!user || n == 0 || is_device_ptr(user)) {
            *dst = user;
            return SGL_OK;
        }
        void *d = nullptr;
        SGL_CUDA_CHECK(cudaMallocAsync(&d, sizeof(T) * n, st));
        ptrs.push_back(d);
        *dst = reinterpret_cast<T *>(d);
        return SGL_OK;
    }
};

int direct_check(int32_t B, int64_t M, const double *points) {
    if (B < 1) {
        set_error("bandwidth must be >= 1");
        return SGL_EINVAL;
    }
    if (M < 0 || (M > 0 && !points)) {
        set_error("points must be (M, 3) spherical coordinates");
        return SGL_EINVAL;
    }
    return SGL_OK;
}

}  // namespace

extern "C" {

int sgl_direct_forward(int32_t B, int64_t M, const double *points, const sgl_cdouble *coeffs,
                       sgl_cdouble *values, void *stream) {
    g_err.clear();
    int rc = direct_check(B, M, points);
    if (rc) return rc;
    if (!coeffs || (M > 0 && !values)) {
        set_error("coefficient length does not match the bandwidth");
        return SGL_EINVAL;
    }
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t count = (int64_t)B * (B + 1) * (2 * B + 1) / 6;
    DeviceScratch sc(st);
    const double *dp;
    const double2 *dc;
    double2 *dv;
    if ((rc = sc.input(points, (size_t)M * 3, &dp))) return rc;
    if ((rc = sc.input(reinterpret_cast<const double2 *>(coeffs), (size_t)count, &dc))) return rc;
    if ((rc = sc.output(reinterpret_cast<double2 *>(values), (size_t)M, &dv))) return rc;
    if ((rc = launch_direct_forward(B, M, dp, dc, dv, st))) {
        set_error("CUDA error in the direct forward kernel");
        return rc;
    }
    if (M > 0 && dv != reinterpret_cast<double2 *>(values)) {
        SGL_CUDA_CHECK(cudaMemcpyAsync(values, dv, sizeof(double2) * M, cudaMemcpyDeviceToHost, st));
        SGL_CUDA_CHECK(cudaStreamSynchronize(st));
    }
    SGL_CUDA_CHECK(cudaGetLastError());
    return SGL_OK;
}

int sgl_direct_adjoint(int32_t B, int64_t M, const double *points, const sgl_cdouble *values,
                       sgl_cdouble *coeffs, void *stream) {
    g_err.clear();
    int rc = direct_check(B, M, points);
    if (rc) return rc;
    if (!coeffs || (M > 0 && !values)) {
        set_error("values length does not match the point count");
        return SGL_EINVAL;
    }
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t count = (int64_t)B * (B + 1) * (2 * B + 1) / 6;
    DeviceScratch sc(st);
    const double *dp;
    const double2 *dv;
    double2 *dc;
    if ((rc = sc.input(points, (size_t)M * 3, &dp))) return rc;
    if ((rc = sc.input(reinterpret_cast<const double2 *>(values), (size_t)M, &dv))) return rc;
    if ((rc = sc.output(reinterpret_cast<double2 *>(coeffs), (size_t)count, &dc))) return rc;
    if ((rc = launch_direct_adjoint(B, M, dp, dv, dc, count, st))) {
        set_error("CUDA error in the direct adjoint kernel");
        return rc;
    }
    if (dc != reinterpret_cast<double2 *>(coeffs)) {
        SGL_CUDA_CHECK(cudaMemcpyAsync(coeffs, dc, sizeof(double2) * count, cudaMemcpyDeviceToHost, st));
        SGL_CUDA_CHECK(cudaStreamSynchronize(st));
    }
    SGL_CUDA_CHECK(cudaGetLastError());
    return SGL_OK;
}

}  // extern "C"
