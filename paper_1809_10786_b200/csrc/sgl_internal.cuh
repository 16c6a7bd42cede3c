// Internal definitions shared by the NFSGLFT CUDA sources (sm_100a).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <cufft.h>
#include <stdint.h>

#include <mutex>
#include <string>
#include <vector>

#include "../../include/sgl_b200.h"

namespace sgl {

constexpr double kPi = 3.14159265358979323846;
constexpr double kTwoPi = 6.28318530717958647692;

// ---------------------------------------------------------------------------
// window tiles:  a tile is <= kTileNodes sorted
// nodes from one pencil (lo1, lo2 in a W x W cell block), consecutive in lo0.
// Its box covers the union of the nodes' window supports.
constexpr int kTileNodes = 64;   // gather tiles: GEMM M-dim (8 warps x 8 nodes)
constexpr int kBoxMax = 36;      // max box extent on axes 1 and 2 (== the TMA slab box)
constexpr int kBox0Max = 96;     // gather: max box extent on axis 0 (slabs; no smem cost)
constexpr int kSTileNodes = 128; // scatter tiles: GEMM K-dim (more nodes per RED)
constexpr int kSBox0Max = 96;    // scatter: max box extent on axis 0 (no smem cost)
constexpr int kMaxQTiled = 16;   // tiled kernels need 2q + W - 1 <= kBoxMax

// int8 tensor-core gather tiles (gather_i8.cu)
constexpr int kI8Nodes = 128;    // tcgen05 M
constexpr int kI8Box1 = 40;      // axis-1 box (80 re|im rows per digit = MMA N)
constexpr int kI8Box2 = 48;      // axis-2 box (3 K-chunks of 16 cells per slab)
constexpr int kI8SNodes = 512;   // int8 scatter tiles (MMA K: more nodes per RED)

struct Tile {
    int32_t start;    // first sorted node
    int32_t count;    // nodes in tile (1..kTileNodes)
    int32_t o0, o1, o2;  // box origin (unwrapped cell coordinates)
    int32_t e0, e1, e2;  // box extents
};

struct NodeSet {
    // sorted order (tile order); u_j = N_j * tau_j / (2 pi) in [0, N_j)
    double *u0 = nullptr, *u1 = nullptr, *u2 = nullptr;
    int32_t *perm = nullptr;   // sorted position -> caller index
    int64_t n = 0;             // node count (bounds of perm / the caller arrays)
};

// The oversampled grid is stored with a periodic halo of q cells on both
// sides of axes 1 and 2 (pitches N1p = N1 + 2q, N2p = N2 + 2q): interior cell
// (g0, g1, g2) sits at padded (g0, g1 + q, g2 + q).  This is the reference's
// pad_wrap / fold_wrap (_gridding.py:29-50) restricted to axes 1-2, so window
// boxes never wrap there and one TMA box load fetches a whole slab.
struct WindowParams {
    int32_t N0, N1, N2;
    int32_t N1p, N2p;
    int32_t q;
    int32_t pad;                // halo width on axes 1-2 (>= q; wider on grids smaller than the TMA box)
    int32_t qa0, qa1, qa2;      // per-axis tap half-width of the generic kernels (0 on the
                                // dummy axes of a d < 3 NFFT plan: one tap of weight 1)
    double c0, c1, c2;          // (N/2pi)/sqrt(2 pi lam)
    double h0, h1, h2;          // 1/(2 lam)
    // recurrence ratios e^{-2 h s^2} of the Gaussian walks (stride s in cells)
    double r0_1, r0_8;          // axis 0: s = 1 (gather), s = 8 (scatter warp stride)
    double r1_1, r1_4;          // axis 1: s = 1 (scatter table), s = 4 (gather fragments)
    double r2_1, r2_4;          // axis 2
};

// The cells a node's window covers on one axis, exactly as the reference
// decides them (nfft.py:131-141): the 2q+1 offsets lo-q .. lo+q, lo = floor(u),
// minus those with |fl(u - cell)| > q.  Only the first offset can drop out
// (u - (lo+q) = frac(u) - q >= -q always); it stays in when u sits on, or
// within rounding of, a grid line.  [c_lo, c_hi] inclusive.
__host__ __device__ inline void window_cells(double u, int q, int &c_lo, int &c_hi) {
    const double f = floor(u);
    const int lo = (int)f;
    c_lo = lo - q + ((u - (double)(lo - q) <= (double)q) ? 0 : 1);
    c_hi = lo + q;
}

// max(|Re|, |Im|) with a NaN in either part as +Inf: fmax alone returns the
// other operand (r02 fix: NaN + 0i values were seen as 0 by the int8 engines'
// non-finite checks)
__device__ __forceinline__ double cabsmax_naninf(double2 v) {
    const double a = fmax(fabs(v.x), fabs(v.y));
    return (v.x != v.x || v.y != v.y) ? INFINITY : a;
}

// SGL_FLAG_DETERMINISTIC (determ.cu): per-call fixed-point exponent E of the
// spread (grid unit 2^-E; kDetOff = FP64 REDs for non-finite input) and the
// max |v| it is derived from
constexpr int kDetOff = -(1 << 20);
struct DetState {
    int e, pad_;
    unsigned long long vmax;
};

struct StageTimer {
    cudaEvent_t ev[SGL_STAGE_COUNT + 1];
    bool ready = false;
};

// Per-plan device state of the int8 accuracy guard (guard.cu): per call, the
// int8 window kernels raise `fwd` / `adj` when their input is non-finite or
// the digit-split error estimate exceeds the bound; the gated FP64 kernel then
// recomputes the stage (it returns at once when the flag is clear).
struct GuardState {
    int fwd, adj;                       // this call: 1 = the gated FP64 kernel recomputes the stage
    int adj_redo, pad_;                 // adjoint estimate above the bound: rerun on the FP64 scatter
    unsigned long long fwd_count, adj_count;   // calls that fell back (diagnostics)
    unsigned long long outmax;          // bits of max |Re|, |Im| of the int8 gather output
    double vsumsq;                      // sum |v 2^-ev|^2 of the adjoint input (max|v| < 2^ev)
    unsigned long long vmax;            // bits of max |Re|, |Im| of the adjoint input
    unsigned long long amax;            // bits of max |Re|, |Im| of the adjoint output
    double est_fwd, est_adj;            // last estimates (relative to the output's max)
};

struct Plan {
    uint32_t flags = 0;
    int B = 0;
    int64_t M = 0;
    double rho = 0;
    int sigma = 2, q = 16;
    bool compact = false;
    bool generic = false;
    bool exact = false;           // exact last stage: direct NDFT on I_n (no window, no FFT)
    bool raw = false;
    int d = 3;                    // NFFT dimension (raw plans); axes 0 .. 2-d are length-1 dummies
    bool precise = false;         // basal tables built in x87 extended precision (precise=True)             // plain 3-D NFFT plan (nfft.py): torus nodes, coefficients on I_n, no basal
    bool profile = false;
    int n_axis[3];
    int grid[3];
    int sig_axes[3];
    double s_eff[3];
    double lam[3];
    int64_t count = 0;
    int device = 0;

    WindowParams wp;
    NodeSet nodes;                // gather order (also the generic kernels)
    NodeSet snodes;               // scatter order (== nodes when snodes_shared)
    bool snodes_shared = false;
    Tile *tiles = nullptr;        // gather tiles (<= kTileNodes nodes)
    int64_t n_tiles = 0;
    Tile *stiles = nullptr;       // scatter tiles (<= kSTileNodes nodes)
    int64_t n_stiles = 0;
    int64_t tile_nodes = 0;
    int64_t tile_dmma = 0;
    int tile_box = kBoxMax;       // widest gather-tile box on axes 1-2 (cells): fragment loop extent
    double plan_ms = 0;
    // per-node u (caller order) for the generic kernels
    double *gu0 = nullptr, *gu1 = nullptr, *gu2 = nullptr;

    // basal matrices (device)
    double *Kl = nullptr;        // concat over l of (B-l) x 4B
    int64_t *Kl_off = nullptr;   // host offsets (B+1)
    double *Km = nullptr;        // concat over m=-(B-1)..B-1 of (B-|m|) x 4B
    std::vector<int64_t> Kl_off_h, Km_off_h;
    int64_t *Kl_off_d = nullptr, *Km_off_d = nullptr;
    double *dec0 = nullptr, *dec1 = nullptr, *dec2 = nullptr;  // deconv incl. (2pi)^3/prod N

    // scratch
    double2 *grid_buf = nullptr;   // N0 x N1p x N2p complex (halo-padded)
    alignas(64) CUtensorMap tmap;  // TMA descriptor of grid_buf (FLOAT64 view)
    bool tmap_ready = false;
    double2 *beta = nullptr;       // B^2 x 4B complex
    double2 *zeta = nullptr;       // (2B-1) x n1 x 4B complex: the adjoint's cropped spectrum, m-major
    double2 *coef_buf = nullptr;   // count complex (staging)
    double2 *val_buf = nullptr;    // M complex (staging)
    size_t grid_elems = 0;
    cufftHandle fft = 0;
    bool fft_ready = false;
    // pruned 3-D FFT: 2-D transforms over the planes that hold (forward) or
    // receive (adjoint) the n0 spectral planes, 1-D transforms along axis 0
    cufftHandle fft2 = 0, fft1 = 0;
    bool pruned = false;
    void *fft_work = nullptr;       // shared cuFFT work area of fft2 / fft1

    // int8 tensor-core window stage (gather_i8.cu): FP64 reproduced from
    // byte digits of the window weights and of the grid (Ozaki split) on
    // tcgen05.mma kind::i8; own node order / tiles (8 x 16 pencils, 128 nodes)
    bool i8 = false;
    NodeSet inodes;
    Tile *itiles = nullptr;
    int64_t n_itiles = 0;
    int64_t i8_ksteps = 0;         // K-steps of one gather pass (sum over tiles)
    bool i8s = false;              // int8 tensor-core scatter (scatter_i8.cu), same node order
    bool i8s_auto = false;         // decide i8s from the tiles' density at plan time
    // run time: an automatically chosen int8 scatter whose accuracy guard made
    // two calls in a row recompute on FP64 (inputs it cannot resolve, e.g. the
    // config-2 lattice) is switched off for the plan's later adjoints
    bool i8s_off = false;
    int i8s_streak = 0;
    bool i8s_live() const { return i8s && !i8s_off; }
    Tile *istiles = nullptr;       // its 512-node tiles
    int64_t n_istiles = 0;
    int *tsv = nullptr;            // per scatter tile: value fixed-point shift
    int64_t i8_sksteps = 0;        // int8 scatter K-steps per pass
    uint8_t *vdig = nullptr;       // value-digit ring of the int8 scatter: 2 tiles (2 x 240 KB) per CTA
    uint8_t *digits = nullptr;     // N0 x P2 x 6 x N1p x 2 x 16 signed bytes
    int P2 = 0;                    // 16-cell column blocks of a padded row
    uint64_t *gmax = nullptr;      // device scratch: bits of max |Re G|, |Im G|
    // the grid region the int8 gather's tiles read (plan time): their axis-0
    // planes (device list) and padded axis-1 rows [grow0, grow1); slab maxima
    // and digit planes are made for it only
    int *gplist = nullptr;
    int n_gplanes = 0, grow0 = 0, grow1 = 0;
    // the pruned FFT's axis-0 pass over those rows only (plus the interior rows
    // whose images fill the region's halo rows): no window stage reads or
    // writes the other rows.  Plans per row interval (setup_i8); enabled after
    // the adjoint guard's calibration, which transforms the full grid.
    cufftHandle fft1r[3] = {0, 0, 0};
    int fft1r_row0[3] = {0, 0, 0};
    int n_fft1r = 0;
    bool fft_rows_on = false;
    alignas(64) CUtensorMap dmap;  // TMA descriptor of the digit planes

    // int8 accuracy guard and debug counters (guard.cu)
    GuardState *guard = nullptr;   // device
    bool guard_on = false;
    double guard_wmass = 0.0;      // max window L1 mass sum |w0 w1 w2| over a node's taps
    double guard_tap2 = 0.0;       // per-node error variance of the int8 spread in units of
                                   // (2^-46 |v|)^2: (c0 c1 c2)^2 (2q+1)^3 (uniform per-tap error)
    double guard_ap = 0.0;         // adjoint tail's response to the spread noise model (plan time)
    unsigned long long *prof = nullptr;   // SGL_FLAG_I8_PROF: clock64 counters (device, per plan)
    // SGL_FLAG_DETERMINISTIC (determ.cu): fixed-point spread state (device) and
    // the window density max_cell sum_n w_n(cell) measured at plan time
    DetState *det = nullptr;
    double det_density = 0.0;
    const int *det_e() const { return det ? &det->e : nullptr; }
    double lap_ms = -1.0;          // SGL_FLAG_I8_PROF: plan-construction stage clock (plan_lap)

    // single-process multi-GPU plan (multi.cu): one sub-plan per device over a
    // contiguous node shard [sub_start[k], sub_start[k + 1]); empty otherwise
    std::vector<Plan *> subs;
    std::vector<int64_t> sub_start;

    // grid-partitioned multi-GPU adjoint (dist.cu): slab 2-D plans by plane count, axis-0 plan
    std::vector<std::pair<int, cufftHandle>> slab_ffts;
    std::vector<std::pair<int64_t, cufftHandle>> axis0_ffts;   // 1-D axis-0 plans by column count
    cufftHandle dist_fft1 = 0;

    StageTimer timers[2];
    float stage_ms[2][SGL_STAGE_COUNT] = {{0}};

    // Calls on a plan are serialised across host threads (mutex) and across
    // CUDA streams (each call's stream waits for the previous call's event),
    // so a plan can be shared like the reference's (README.md:66-67).
    std::mutex mu;
    cudaEvent_t done = nullptr;

    // copy/compute overlap (sgl_forward_adjoint, batched sgl_forward into
    // host memory): side stream for the host copies, events, a second value
    // buffer; created on first use
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t ev_a = nullptr, ev_b = nullptr, ev_c = nullptr, ev_d = nullptr;
    double2 *val_buf2 = nullptr;
};

// Checked builds (python -m paper_1809_10786_b200.build --checked, -DSGL_CHECKED):
// device-side bounds checks of every grid / TMA / output index the window
// kernels form, trapping with the failing condition -- the stand-in for
// compute-sanitizer memcheck, which this GPU pool does not allow.
#ifdef SGL_CHECKED
#define SGL_DCHECK(cond)                                                                    \
    do {                                                                                    \
        if (!(cond)) {                                                                      \
            printf("SGL_CHECKED: %s failed at %s:%d (block %d thread %d)\n", #cond, __FILE__, \
                   __LINE__, (int)blockIdx.x, (int)threadIdx.x);                            \
            __trap();                                                                       \
        }                                                                                   \
    } while (0)
#else
#define SGL_DCHECK(cond) \
    do {                 \
    } while (0)
#endif

// error state
void set_error(const std::string &msg);
#define SGL_CUDA_CHECK(x)                                                        \
    do {                                                                         \
        cudaError_t _e = (x);                                                    \
        if (_e != cudaSuccess) {                                                 \
            ::sgl::set_error(std::string("CUDA error: ") + cudaGetErrorString(_e) + \
                             " at " + __FILE__ + ":" + std::to_string(__LINE__)); \
            return SGL_ECUDA;                                                    \
        }                                                                        \
    } while (0)

// kernels / launchers (defined in the .cu files)
int build_nodes(Plan &p, const double *points_dev, cudaStream_t st);
// device statistics of a tile list: mode 0 = FP64 gather tiles (work = DMMA
// count, box = widest axis-1/2 extent), 1 = int8 gather tiles (work = K-steps),
// 2 = int8 scatter tiles (work = K-steps x M-blocks); bad = a tile outside its
// kernel's limits
struct TileStats {
    int64_t nodes = 0, work = 0;
    bool bad = false;
    int box = 0;
};
int tile_stats(const Tile *tiles, int64_t n, int mode, const WindowParams &wp, cudaStream_t st, TileStats *out);
int build_basal_tables(Plan &p);
// the host half (no CUDA calls; uses B, rho, precise) and the upload half,
// so plan creation can overlap the host tables with the device node work
void basal_tables_host(Plan &p, std::vector<double> &Kl, std::vector<double> &Km);
int upload_basal_tables(Plan &p, const std::vector<double> &Kl, const std::vector<double> &Km);
// rho (choose_rho, transform.py:39-43) and the radius check (transform.py:50-51)
int resolve_rho(Plan &p, const double *points_dev, cudaStream_t st);
int build_deconv_tables(Plan &p);
int launch_place_raw(const Plan &p, const double2 *coeffs, double2 *grid, cudaStream_t st);
int launch_crop_raw(const Plan &p, const double2 *grid, double2 *coeffs, cudaStream_t st);
int launch_gather(const Plan &p, const double2 *grid, double2 *values, cudaStream_t st);
int launch_scatter(const Plan &p, const double2 *values, double2 *grid, cudaStream_t st);
int launch_basal_forward(const Plan &p, const double2 *coeffs, double2 *grid, cudaStream_t st,
                         cudaEvent_t mid);
int launch_basal_adjoint(const Plan &p, const double2 *grid, double2 *coeffs, cudaStream_t st);
int launch_basal_adjoint_from_zeta(const Plan &p, double2 *coeffs, cudaStream_t st);
int make_grid_tmap(Plan &p);
int launch_exact_forward(const Plan &p, const double2 *eta, double2 *values, cudaStream_t st);
int launch_exact_adjoint(const Plan &p, const double2 *values, double2 *eta, cudaStream_t st);
int launch_direct_forward(int B, int64_t M, const double *pts, const double2 *c, double2 *out, cudaStream_t st);
int launch_direct_adjoint(int B, int64_t M, const double *pts, const double2 *v, double2 *c, int64_t count,
                          cudaStream_t st);
int launch_halo_fill(const Plan &p, double2 *grid, cudaStream_t st);
int launch_halo_fold(const Plan &p, double2 *grid, cudaStream_t st);
int launch_gather_i8(const Plan &p, const double2 *grid, double2 *values, cudaStream_t st);
int launch_scatter_i8(const Plan &p, const double2 *values, double2 *grid, cudaStream_t st);
int setup_scatter_i8(Plan &p);
int setup_guard(Plan &p);
int multi_forward(Plan &p, const sgl_cdouble *coeffs, int64_t K, sgl_cdouble *values, void *stream);
int multi_adjoint(Plan &p, const sgl_cdouble *values, sgl_cdouble *coeffs, void *stream);
// SGL_FLAG_I8_PROF: synchronise and print the host time since the previous lap
// of this plan's construction to stderr (diagnostics of plan time)
void plan_lap(Plan &p, cudaStream_t st, const char *what);
int launch_gather_guarded(const Plan &p, const double2 *grid, double2 *values, cudaStream_t st);
int launch_noise_grid(const Plan &p, double rms, cudaStream_t st);
int read_absmax(const Plan &p, const double2 *v, int64_t n, cudaStream_t st, double *out);
int guard_adjoint_estimate(const Plan &p, const double2 *values, const double2 *coeffs, cudaStream_t st);
int launch_scatter_guarded(const Plan &p, const double2 *values, double2 *grid, cudaStream_t st);
int launch_gather_tiled_gated(const Plan &p, double2 *values, const int *gate, cudaStream_t st);
int launch_scatter_tiled_gated(const Plan &p, const double2 *values, double2 *grid, const int *gate,
                               cudaStream_t st);
int setup_i8(Plan &p);
int num_sms();
// max(|Re|, |Im|) bits into *out (atomicMax; *out zeroed by the caller; NaN counts as +Inf)
int launch_absmax(const double2 *v, int64_t n, unsigned long long *out, cudaStream_t st);
// SGL_FLAG_DETERMINISTIC (determ.cu)
int setup_det(Plan &p, cudaStream_t st);
int det_begin(const Plan &p, const double2 *v, cudaStream_t st);
int det_finish(const Plan &p, double2 *grid, cudaStream_t st);
// the adjoint's window stage into the zeroed p.grid_buf (int8 scatter with its
// guard when allow_i8 and live, else the FP64 / per-node scatter), in fixed
// point under SGL_FLAG_DETERMINISTIC
int spread_stage(Plan &p, const double2 *v, cudaStream_t st, bool allow_i8);

}  // namespace sgl
