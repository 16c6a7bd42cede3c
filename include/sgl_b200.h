/*
 * sgl_b200.h -- C ABI of the B200-native NFSGLFT (forward + adjoint).
 *
 * Drop-in boundary for the hot path of the reference `sglnufft` package
 * (arXiv 1809.10786).  Plain pointers and sizes only; no torch types.
 * Each entry point replaces one reference interface (paths relative to the
 * reference's pkg/src/sglnufft/):
 *
 *   sgl_plan_create   <- transform.plan            (transform.py:320-382)
 *                        + nfft.nfft_plan          (nfft.py:147-207)
 *   sgl_forward       <- transform.forward         (transform.py:385-395)
 *                        (batched: K coefficient vectors on one plan)
 *   sgl_adjoint       <- transform.adjoint         (transform.py:398-429)
 *   sgl_plan_destroy  <- (garbage collection of SglPlan)
 *   sgl_last_error    <- the ValueError message text raised by the above
 *   sgl_plan_get_info <- SglPlan / NfftPlan fields (transform.py:292-317,
 *                        nfft.py:101-120)
 *   sgl_nfft_plan_create <- nfft.nfft_plan (nfft.py:147-207): a plain 3-D
 *                        NFFT plan; sgl_forward / sgl_adjoint on it are
 *                        nfft_execute / nfft_adjoint_execute (nfft.py:234-273)
 *                        (with SGL_FLAG_EXACT_LAST_STAGE: ndft / ndft_adjoint,
 *                        nfft.py:51-82)
 *   sgl_direct_forward  <- transform.evaluate_direct         (transform.py:95-117)
 *   sgl_direct_adjoint  <- transform.evaluate_direct_adjoint (transform.py:120-139)
 *
 * Pointers to points / coefficients / values may be host or device
 * (CUDA) memory; the library detects which.  Host outputs are complete when
 * the call returns; device outputs are complete in stream order.
 *
 * A plan may be shared by host threads and streams like the reference's
 * (README.md:66-67): calls on one plan are serialised by a mutex and by
 * stream-ordering on the previous call (the plan owns its scratch grid).
 */
#ifndef SGL_B200_H
#define SGL_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct sgl_plan sgl_plan;

typedef struct {
    double re, im;
} sgl_cdouble;

/* return codes; SGL_EINVAL corresponds to the reference's ValueError */
enum {
    SGL_OK = 0,
    SGL_EINVAL = 1,
    SGL_ECUDA = 2,
    SGL_ENOMEM = 3,
    SGL_EUNSUPPORTED = 4
};

/* plan flags */
enum {
    SGL_FLAG_COMPACT_K1 = 1u << 0,        /* compact_k1=True (transform.py:350)     */
    SGL_FLAG_EXACT_LAST_STAGE = 1u << 1,  /* exact_last_stage=True: direct NDFT      */
    SGL_FLAG_GENERIC_GRIDDING = 1u << 2,  /* force the per-node window kernels      */
    SGL_FLAG_PROFILE = 1u << 3,           /* record per-stage CUDA-event timings    */
    SGL_FLAG_PRECISE = 1u << 4,           /* basal tables in 80-bit extended precision
                                             (precise=True, recurrences.py:13); the
                                             default since round 2 unless
                                             SGL_FLAG_FP64_TABLES                   */
    SGL_FLAG_FP64_WINDOW = 1u << 5,       /* both window stages on the FP64 DMMA
                                             kernels instead of the int8 tensor-core
                                             (digit-split) engines                  */
    SGL_FLAG_I8_SCATTER = 1u << 6,        /* adjoint window stage on the int8 tensor
                                             cores for any node set (default: only
                                             large dense sets, chosen at plan time) */
    SGL_FLAG_FP64_SCATTER = 1u << 7,      /* adjoint window stage on the FP64 DMMA
                                             kernel (the int8 gather is kept)       */
    SGL_FLAG_FULL_FFT = 1u << 8,          /* one 3-D cuFFT plan instead of the pruned
                                             2-D + 1-D passes                      */
    SGL_FLAG_I8_GATHER = 1u << 9,         /* sgl_nfft_plan_create only: int8 gather
                                             (off by default on raw NFFT plans)     */
    SGL_FLAG_SCATTER_WIDE = 1u << 10,     /* FP64 scatter tiles in the gather's W x W
                                             pencils (default: by node density)     */
    SGL_FLAG_SCATTER_NARROW = 1u << 11,   /* FP64 scatter tiles in W x W2 pencils   */
    SGL_FLAG_I8_PROF = 1u << 12,          /* debug: clock64 wait counters of the int8
                                             kernels, printed to stderr per call    */
    SGL_FLAG_NO_GUARD = 1u << 13,         /* disable the int8 accuracy guard (the
                                             per-call switch to the FP64 kernels;
                                             estimates are still recorded)          */
    SGL_FLAG_FP64_TABLES = 1u << 14,      /* build the basal matrices in FP64 (the
                                             reference's default arithmetic) instead
                                             of x87 extended precision: config 4 is
                                             4.7e-9 from the truth this way, 1.2e-9
                                             with extended tables (reference: 2.6e-9) */
    SGL_FLAG_DETERMINISTIC = 1u << 15     /* bitwise reproducible adjoint: the window
                                             kernels reduce 64-bit fixed-point
                                             integers into the grid (order-independent
                                             sums; unit 2^-62 of max|v| x the window
                                             density) instead of FP64 atomics, as the
                                             reference's serial loop
                                             (_gridding.py:77-95) is reproducible   */
};

typedef struct {
    int32_t B;
    int64_t M;
    double rho;
    int32_t sigma;
    int32_t q;
    int32_t n_axis[3];
    int32_t grid[3];
    int32_t sigma_axes[3];
    double sigma_eff[3];
    double lam[3];
    int64_t coeff_count;
    int64_t n_tiles;          /* window tiles built by the plan (0 if generic) */
    int64_t tile_nodes;       /* nodes covered by tiles                        */
    int64_t tile_dmma;        /* DMMA m8n8k4 issued per gather pass            */
    int32_t generic;          /* 1 if the per-node window kernels are used     */
    int32_t exact;            /* 1 for exact_last_stage plans (direct NDFT)    */
    double plan_ms;           /* device time of plan construction              */
    int32_t i8_gather;        /* 1 if the forward window stage runs on the int8
                                 tensor cores (tcgen05, FP64 by digit split)   */
    int64_t i8_tiles;         /* its 128-node tiles                            */
    int64_t i8_ksteps;        /* K-steps of 32 per gather pass (9 MMAs each,
                                 M = 128, N = 1680 digit columns in total)     */
    int32_t i8_scatter;       /* 1 if the adjoint window stage runs on the int8
                                 tensor cores (chosen for >= 1e5 nodes at < 1.5
                                 K-steps per node, or forced); 0 again once an
                                 automatic choice switched itself off after two
                                 consecutive accuracy-guard fallbacks          */
    int64_t i8_sksteps;       /* its K-steps (32 nodes x 128 cells) per pass   */
    int32_t guard;            /* 1 if the int8 accuracy guard is on            */
    double guard_ap;          /* adjoint guard: the tail's noise response (plan time) */
    int64_t guard_fwd_fallbacks;  /* forward calls whose window stage ran on the
                                     FP64 kernel (estimate above 1e-11, or a
                                     non-finite grid)                          */
    int64_t guard_adj_fallbacks;  /* adjoint calls likewise                     */
    double guard_est_fwd;     /* last forward's digit-split error estimate     */
    double guard_est_adj;     /* last adjoint's estimate                       */
    int32_t n_gpus;           /* devices of the plan (sgl_plan_create_multi)   */
} sgl_plan_info;

/* stage indices for sgl_plan_stage_ms (valid with SGL_FLAG_PROFILE) */
enum {
    SGL_STAGE_H2D = 0,
    SGL_STAGE_BASAL = 1,      /* radial + spherical stage (fwd) / their adjoints */
    SGL_STAGE_FFT = 2,        /* zero + cuFFT (+ place / crop fused in basal)    */
    SGL_STAGE_WINDOW = 3,     /* gather (fwd) / scatter (adj)                    */
    SGL_STAGE_D2H = 4,
    SGL_STAGE_COUNT = 5
};

/* Create a plan for M points given as (r, theta, phi) rows (M x 3, C order,
 * float64).  rho <= 0 selects max r (choose_rho, transform.py:39-43).
 * stream may be NULL (legacy default stream). */
int sgl_plan_create(int32_t B, int64_t M, const double *points, int32_t sigma, int32_t q,
                    double rho, uint32_t flags, void *stream, sgl_plan **out);

/* The same plan over n_gpus devices of this process (devices: n_gpus ids, or
 * NULL for 0 .. n_gpus-1): the points are split into contiguous,
 * count-balanced shards, one sub-plan per device, all on the global rho
 * (rho <= 0: max r over ALL points).  sgl_forward / sgl_adjoint /
 * sgl_forward_adjoint / sgl_plan_get_info / sgl_plan_destroy accept the
 * result: the forward evaluates each shard on its device into its slice of
 * the values; the adjoint sums the shards' coefficient vectors.  One host
 * thread per device per call; device-resident caller buffers are staged
 * through host memory.  Reference signature: transform.plan
 * (transform.py:320-330) + SURVEY 8(b)'s n_gpus. */
int sgl_plan_create_multi(int32_t B, int64_t M, const double *points, int32_t sigma, int32_t q, double rho,
                          uint32_t flags, int32_t n_gpus, const int32_t *devices, sgl_plan **out);

/* Forward: coeffs is K x coeff_count(B) complex128 (mu order), values is
 * K x M complex128 in the caller's point order. */
int sgl_forward(sgl_plan *plan, const sgl_cdouble *coeffs, int64_t K, sgl_cdouble *values,
                void *stream);

/* Adjoint: values is M complex128, coeffs receives coeff_count(B). */
int sgl_adjoint(sgl_plan *plan, const sgl_cdouble *values, sgl_cdouble *coeffs, void *stream);

/* Forward of `coeffs` and adjoint of `values_in` on one plan in one call
 * (independent inputs, e.g. a benchmark or a block solver step).  With host
 * buffers the value H2D overlaps the forward and the value D2H overlaps the
 * adjoint on a side stream.  values_out: M, coeffs_out: coeff_count(B). */
int sgl_forward_adjoint(sgl_plan *plan, const sgl_cdouble *coeffs, sgl_cdouble *values_out,
                        const sgl_cdouble *values_in, sgl_cdouble *coeffs_out, void *stream);

void sgl_plan_destroy(sgl_plan *plan);

/* Plain d-dimensional NFFT on the torus (the reference's NFFT layer, d <= 3):
 * trigonometric polynomial coefficients on I_n = prod [-n_j/2, n_j/2) in the
 * centred layout (position p on axis j holds frequency p - n_j/2), nodes
 * (M x d) reduced into [0, 2 pi).  n_axis[j] even >= 2, sigma[j] >= 2
 * (length-d arrays); oversampled length pow2(sigma_j n_j); q must be below
 * every oversampled length (no escalation).  Use sgl_forward (coefficients:
 * prod n_j per vector, K vectors) and sgl_adjoint on the plan.  d = 3 runs
 * the tiled window kernels; d < 3 the per-node ones.
 * Flags: SGL_FLAG_EXACT_LAST_STAGE (direct NDFT), SGL_FLAG_GENERIC_GRIDDING,
 * SGL_FLAG_PROFILE. */
int sgl_nfft_plan_create(int32_t d, const int32_t *n_axis, int64_t M, const double *nodes, const int32_t *sigma,
                         int32_t q, uint32_t flags, void *stream, sgl_plan **out);

/* Direct summation of the expansion (no plan, O(M * count) FP64; the
 * reference's verification path and the CLI's --method naive).
 * points: M x 3 (r, theta, phi); coeffs: coeff_count(B); values: M.
 * Errors as the reference: bandwidth < 1, length mismatches (SGL_EINVAL). */
int sgl_direct_forward(int32_t B, int64_t M, const double *points, const sgl_cdouble *coeffs,
                       sgl_cdouble *values, void *stream);
int sgl_direct_adjoint(int32_t B, int64_t M, const double *points, const sgl_cdouble *values,
                       sgl_cdouble *coeffs, void *stream);

int sgl_plan_get_info(const sgl_plan *plan, sgl_plan_info *info);

/* ---- grid-partitioned multi-GPU adjoint (one process per GPU) ----------
 * Stage entry points of the north star's adjoint partition: each rank
 * spreads its node shard into its plan's own oversampled grid; the caller
 * reduce-scatters axis-0 plane blocks of that grid (NCCL over NVLink); each
 * rank FFTs its planes over axes 1-2 and packs the spectral box the basal
 * stage reads; the caller gathers the packed planes to one rank, which
 * finishes (1-D FFT along axis 0, crop, deconvolution, basal adjoint) and
 * broadcasts the coefficients.  Replaces nfft_adjoint_execute +
 * transform.adjoint (nfft.py:254-273, transform.py:398-429) split across
 * ranks; see paper_1809_10786_b200/distributed.py.  All pointers device
 * memory except `values` / `coeffs`, which may be host. */
typedef struct {
    void *data;               /* the plan's grid: N0 x N1p x N2p complex128 */
    int32_t N0, N1, N2;       /* oversampled grid                           */
    int32_t N1p, N2p, pad;    /* halo-padded pitches; interior at +pad      */
    int64_t plane_elems;      /* N1p * N2p complex per axis-0 plane         */
    int32_t crop1, crop2;     /* packed spectrum per plane: crop1 x crop2   */
} sgl_grid_info;

int sgl_plan_grid(const sgl_plan *plan, sgl_grid_info *info);
/* zero the grid, spread `values` (M, this plan's nodes), fold the halo */
int sgl_adjoint_spread(sgl_plan *plan, const sgl_cdouble *values, void *stream);
/* 2-D forward FFT of planes [a0, a1) (in place), then pack their spectral box
 * into `packed` ((a1 - a0) x crop1 x crop2, device) */
int sgl_adjoint_slab_fft(sgl_plan *plan, int32_t a0, int32_t a1, sgl_cdouble *packed, void *stream);
/* `packed`: all N0 planes (N0 x crop1 x crop2, device) -> coeff_count(B) */
int sgl_adjoint_from_packed(sgl_plan *plan, const sgl_cdouble *packed, sgl_cdouble *coeffs, void *stream);
/* The all-to-all variant: the axis-0 planes this plan's node
 * windows touch (mask: N0 bytes, host; the caller ORs the ranks' masks and
 * reduce-scatters only those planes); after an all-to-all of the packed box
 * by columns, the 1-D FFT along axis 0 of a column block (cols: N0 x ncols,
 * columns col0 .. col0+ncols-1 of the crop1 x crop2 box, device), cropped to
 * kappa0 in [-2B, 2B) and deconvolved -> eta (4B x ncols, device); and the
 * basal adjoint from the gathered eta (4B x crop1 x crop2, device). */
int sgl_plan_planes(const sgl_plan *plan, uint8_t *mask);
int sgl_adjoint_axis0(sgl_plan *plan, const sgl_cdouble *cols, int64_t ncols, int64_t col0, sgl_cdouble *eta,
                      void *stream);
int sgl_adjoint_from_eta(sgl_plan *plan, const sgl_cdouble *eta, sgl_cdouble *coeffs, void *stream);

/* per-stage device milliseconds of the last forward / adjoint call
 * (dir 0 = forward, 1 = adjoint); needs SGL_FLAG_PROFILE */
int sgl_plan_stage_ms(const sgl_plan *plan, int32_t dir, float *ms, int32_t n);

/* Message of the most recent failing call on this thread ("" if none). */
const char *sgl_last_error(void);

/* Select the CUDA device for subsequent plan creation on this thread
 * (plans remember their device). */
int sgl_set_device(int32_t device);

/* Number of visible CUDA devices (0 when none; never fails). */
int sgl_device_count(int32_t *n);

/* Library version string. */
const char *sgl_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SGL_B200_H */
