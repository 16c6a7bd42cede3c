// Gaussian-window gather (forward NFFT interpolation) and scatter (adjoint
// spreading) on the oversampled grid, FP64, sm_100a.
//
// Reference: _gridding.py:53-74 (_gather_kernel), :77-95 (_scatter_kernel)
// with the wrap padding of :29-50 kept as a resident periodic halo on axes
// 1-2 (see sgl_internal.cuh) and modular addressing on axis 0, and the
// window of nfft.py:123-144:
//     w_j(delta) = (N_j/2pi)/sqrt(2 pi lam_j) * exp(-delta^2/(2 lam_j)),
//     delta = u_j - cell, zero where |delta| > q.
//
// Tiled kernels (q <= 16): a tile is a run of sorted nodes (64 for the
// gather, 128 for the scatter) from one pencil of cells, whose window boxes
// overlap almost entirely.  Per axis-0 slab of the tile's box the contraction
// over axis 2 is a real GEMM on the FP64 tensor cores (DMMA m8n8k4):
//     gather : D[node, (b,re|im)] = sum_c W2[c,node] * G[a,b,c]
//     scatter: D[(b,re|im), c]    = sum_node V[(b,re|im),node] * W2[c,node]
// and the axis-1 / axis-0 weights are applied in the epilogue (gather) or
// folded into V (scatter).  Gather slabs arrive by TMA (one
// cp.async.bulk.tensor.3d box per slab) in a 4-deep mbarrier ring fed by a
// producer warp; scatter fragments are reduced into the grid with
// RED.E.ADD.F64.
//
// Generic kernels (any q, tiny grids, or forced): one warp per node, lanes
// over axis-2 taps, exactly the reference loop nest.
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <atomic>

#include "sgl_internal.cuh"

namespace sgl {
namespace {

__device__ __forceinline__ int wrapi(int i, int n) {
    i %= n;
    return i < 0 ? i + n : i;
}

__device__ __forceinline__ double wfun(double u, int cell, double c, double h, int q) {
    double d = u - (double)cell;
    return (fabs(d) <= (double)q) ? c * exp(-d * d * h) : 0.0;
}

// w(j) = wfun(u, o + S j) for j = 0 .. N-1 (j < n live, 0 beyond) by the
// Gaussian's two-term recurrence w(j+1) = w(j) r(j), r(j+1) = r(j) e^{-2 h S^2},
// seeded at the first cell of the node's window (window_cells: the
// reference's own tap rule, decided on fl(u - cell)); values differ from
// wfun's by a few ulps.  3 exps instead of N.
template <int N, int S>
__device__ __forceinline__ void wwalk(double u, int o, int n, double c, double h, double rs, int q, double (&w)[N]) {
    int c_lo, c_hi;
    window_cells(u, q, c_lo, c_hi);
    // first j with o + S j >= c_lo (integer ceiling; c_lo - o may be negative)
    const int num = c_lo - o;
    const int j0 = num <= 0 ? 0 : (num + S - 1) / S;
    const double d0 = u - (double)(o + S * j0);
    double cur = c * exp(-d0 * d0 * h), r = exp(h * (2.0 * S * d0 - (double)(S * S)));
#pragma unroll
    for (int j = 0; j < N; ++j) {
        const int cell = o + S * j;
        w[j] = (j >= j0 && j < n && cell >= c_lo && cell <= c_hi) ? cur : 0.0;
        if (j >= j0) {
            cur *= r;
            r *= rs;
        }
    }
}

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ bool mbar_try(uint64_t *bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}

// Wait for the phase of `parity` to complete.  A watchdog turns a lost
// phase (a pipeline bug) into a trapped kernel instead of a hung GPU.
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t spins = 0;
    while (!mbar_try(bar, parity)) {
        if (++spins == (1u << 24)) __trap();
    }
}

__device__ __forceinline__ void red_add(double *addr, double v) {
    asm volatile("red.global.add.f64 [%0], %1;\n" ::"l"(addr), "d"(v) : "memory");
}

// SGL_FLAG_DETERMINISTIC (determ.cu): v rounded to the call's fixed-point
// unit 2^-E and reduced as a 64-bit integer (order-independent).  2^E as two
// factors (a, b) so that E beyond the FP64 exponent range of one factor (inputs
// near 1e-300) scales exactly; a == 0: plain FP64 REDs.
struct DScale {
    double a, b;
};

__device__ __forceinline__ void red_add_det(double *addr, double v, DScale ds) {
    if (ds.a != 0.0) {
        const long long x = __double2ll_rn((v * ds.a) * ds.b);
        if (x != 0) asm volatile("red.global.add.u64 [%0], %1;\n" ::"l"(addr), "l"(x) : "memory");
    } else {
        red_add(addr, v);
    }
}

__device__ __forceinline__ DScale det_scale(const int *det) {
    if (!det) return DScale{0.0, 0.0};
    const int e = *det;
    if (e == kDetOff) return DScale{0.0, 0.0};
    return DScale{ldexp(1.0, e / 2), ldexp(1.0, e - e / 2)};
}

// ---------------------------------------------------------------------------
// tiled gather
//
// CTA = 8 consumer warps (one per 8-node M-tile of the 64-node tile) + 1
// producer warp.  Per box slab a (axis 0), consumer warp w computes
//     D[node, (b, re|im)] = sum_c W2[c, node] * G[a, b, c]       (DMMA)
// with the W2 fragments resident in registers and the G fragments read from
// the shared-memory slab, then applies W1[b, node] (registers) and W0[a, node]
// (a per-thread recurrence along the slabs).  The
// producer lane streams one TMA box per slab (cp.async.bulk.tensor.3d, the
// halo-padded grid needs no wrap on axes 1-2) into a 5-deep ring guarded by
// full / empty mbarriers; it walks the CTA's tile sequence on its own, so the
// next tile's first slabs are in flight while the consumers finish a tile.

constexpr int GCW = kTileNodes / 8;   // consumer warps
constexpr int GT = (GCW + 1) * 32;    // + producer warp
constexpr int GCPS = 2;               // resident CTAs per SM (3 with NST = 3 and 72 registers: no faster)
constexpr int NST = 5;                // slab ring depth
constexpr int SROWS = kBoxMax;        // TMA box rows (axis 1)
constexpr int SSTR = kBoxMax;         // TMA box width in complex (== 4 mod 8: conflict-free B reads)
static_assert(SSTR % 8 == 4, "slab row stride must be 4 mod 8 complex");
constexpr int KSMAX = kBoxMax / 4;    // k-steps over axis 2
constexpr int NTMAX = kBoxMax / 4;    // 4-row (8 re|im column) tiles over axis 1
static_assert(NTMAX % 3 == 0, "gather N-tile loop runs in groups of 3");
constexpr uint32_t SLAB_BYTES = SROWS * SSTR * 16;

struct GatherSmem {
    double2 slab[NST][SROWS * SSTR];
    double nu[3][kTileNodes];
    uint64_t full[NST];
    uint64_t empty[NST];
    Tile t;
};

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *map, int c0, int c1, int c2,
                                            uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];\n" ::"r"(smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void consumers_sync() {
    asm volatile("bar.sync 1, %0;\n" ::"n"(GCW * 32) : "memory");
}

// One slab of one warp's 8 nodes: fixed NTMAX x NKS fragment loops with no
// predicates around the DMMAs (a .sync.aligned MMA under a runtime guard costs
// a WARPSYNC, a branch and a NOP each); fragments beyond the tile's box have
// zero W2 weights and multiply finite smem data.  NKS is 8 for boxes of
// <= 32 columns (narrow pencils) and 9 otherwise.  W0[a, node] is folded
// into the A fragments, so the NTMAX accumulators run over the whole tile
// (K = slabs x columns) and W1 is applied once per tile.
template <int NKS, int NT>
__device__ __forceinline__ void gather_slab(const double *sl, const double (&afr)[NT], double w0, int rb, int cc,
                                            int part, double (&d)[NT][2]) {
    // B fragments double-buffered one k-step ahead, so no DMMA waits on the
    // shared-memory load feeding it
    double bf[2][NT];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) bf[0][nt] = sl[((nt * 4 + rb) * SSTR + cc) * 2 + part];
#pragma unroll
    for (int ks = 0; ks < NKS; ++ks) {
        if (ks + 1 < NKS) {
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
                bf[(ks + 1) & 1][nt] = sl[((nt * 4 + rb) * SSTR + (ks + 1) * 4 + cc) * 2 + part];
        }
        const double a = w0 * afr[ks];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) dmma(d[nt], a, bf[ks & 1][nt]);
    }
}

template <int NT>   // fragment tiles per slab axis: ceil(box / 4) of the plan's widest tile (9 at q = 16)
__global__ void __launch_bounds__(GT, GCPS)
    k_gather_tiled(const __grid_constant__ CUtensorMap tmap, const Tile *__restrict__ tiles, int64_t ntiles,
                   NodeSet nodes, WindowParams wp, double2 *__restrict__ out, const int *__restrict__ gate) {
    // gated launch (accuracy guard of the int8 gather): nothing to do unless raised
    if (gate && *gate == 0) return;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    GatherSmem &S = *reinterpret_cast<GatherSmem *>(smem_raw);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

    for (int i = tid; i < NST * SROWS * SSTR; i += GT) (&S.slab[0][0])[i] = make_double2(0.0, 0.0);
    if (tid == 0) {
        for (int s = 0; s < NST; ++s) {
            mbar_init(&S.full[s], 1);
            mbar_init(&S.empty[s], GCW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncthreads();

    if (warp == GCW) {
        // producer: one lane walks the tile sequence and streams slabs
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tmap) : "memory");
            uint32_t q = 0;
            for (int64_t ti = blockIdx.x; ti < ntiles; ti += gridDim.x) {
                const Tile t = tiles[ti];
                const int c0 = 2 * (t.o2 + wp.pad), c1 = t.o1 + wp.pad;
                SGL_DCHECK(c0 >= 0 && c0 + 2 * t.e2 <= 2 * wp.N2p && c1 >= 0 && c1 + t.e1 <= wp.N1p &&
                           t.e0 <= kBox0Max);
                for (int a = 0; a < t.e0; ++a, ++q) {
                    const int buf = (int)(q % NST);
                    const uint32_t use = q / NST;
                    if (use > 0) mbar_wait(&S.empty[buf], (use - 1) & 1);
                    mbar_expect_tx(&S.full[buf], SLAB_BYTES);
                    tma_load_3d(S.slab[buf], &tmap, c0, c1, wrapi(t.o0 + a, wp.N0), &S.full[buf]);
                }
            }
        }
        return;
    }

    uint32_t seq = 0;                           // slabs consumed by this CTA so far
    // warp w owns the 8 consecutive nodes 8w .. 8w+7 of the lo0-sorted tile:
    // its active slab range is short and inactive slabs are skipped; the
    // 4-deep ring absorbs the few slabs of skew between warps
    const int node = warp * 8 + (lane >> 2);    // this lane's node
    const int cc = lane & 3;
    const int rb = lane >> 3, part = (lane >> 2) & 1;

    for (int64_t ti = blockIdx.x; ti < ntiles; ti += gridDim.x) {
        consumers_sync();   // previous tile's readers of S.t / S.nu are done
        if (tid == 0) S.t = tiles[ti];
        consumers_sync();
        const Tile t = S.t;
        if (tid < kTileNodes) {
            const bool ok = tid < t.count;
            const int64_t s = (int64_t)t.start + tid;
            // far-away sentinel: every weight of a missing node is exactly zero
            S.nu[0][tid] = ok ? nodes.u0[s] : -1e9;
            S.nu[1][tid] = ok ? nodes.u1[s] : -1e9;
            S.nu[2][tid] = ok ? nodes.u2[s] : -1e9;
        }
        consumers_sync();
        // W0[a, node] by the Gaussian's two-term recurrence along axis 0:
        // w(a+1) = w(a) r(a), r(a+1) = r(a) exp(-2h), seeded exactly at the
        // node's first in-window slab (relative drift <= e0 ulps); the
        // truncation |delta| <= q is applied exactly
        const double u0n = S.nu[0][node];
        int c_lo0, c_hi0;
        window_cells(u0n, wp.q, c_lo0, c_hi0);
        const int a_first = max(0, c_lo0 - t.o0), a_last = c_hi0 - t.o0;
        double w0r, r0r;
        {
            const double d = u0n - (double)(t.o0 + a_first);
            w0r = wp.c0 * exp(-d * d * wp.h0);
            r0r = exp(wp.h0 * (2.0 * d - 1.0));
        }
        const double r0step = wp.r0_1;
        const int Mt = (t.e1 + 3) >> 2;
        const int KS = (t.e2 + 3) >> 2;
        double afr[NT];
        wwalk<NT, 4>(S.nu[2][node], t.o2 + cc, KS, wp.c2, wp.h2, wp.r2_4, wp.q, afr);
        consumers_sync();
        const bool col_live = warp * 8 < t.count;
        double d[NT][2];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) d[nt][0] = d[nt][1] = 0.0;
        for (int a = 0; a < t.e0; ++a) {
            const uint32_t q = seq + a;
            const int buf = (int)(q % NST);
            double w0 = 0.0;
            if (a >= a_first) {
                w0 = (a <= a_last) ? w0r : 0.0;
                w0r *= r0r;
                r0r *= r0step;
            }
            // every consumer observes every phase (keeps the ring's parity
            // bookkeeping exact); the math is skipped where none of this
            // warp's 8 nodes has weight on the slab (warp-uniform)
            mbar_wait(&S.full[buf], (q / NST) & 1);
            if (col_live && __any_sync(0xffffffffu, w0 != 0.0)) {
                const double *sl = reinterpret_cast<const double *>(S.slab[buf]);
                if (KS <= NT - 1)
                    gather_slab<NT - 1, NT>(sl, afr, w0, rb, cc, part, d);
                else
                    gather_slab<NT, NT>(sl, afr, w0, rb, cc, part, d);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&S.empty[buf]);
        }
        double acc_re = 0.0, acc_im = 0.0;
        {
            // W1 once per tile, evaluated here so it holds no registers in the slab loop
            double w1[NT];
            wwalk<NT, 4>(S.nu[1][node], t.o1 + cc, Mt, wp.c1, wp.h1, wp.r1_4, wp.q, w1);
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
                acc_re = fma(w1[nt], d[nt][0], acc_re);
                acc_im = fma(w1[nt], d[nt][1], acc_im);
            }
        }
        seq += (uint32_t)t.e0;
        // reduce over the 4 lanes of a node (their rows b differ)
        acc_re += __shfl_xor_sync(0xffffffffu, acc_re, 1);
        acc_im += __shfl_xor_sync(0xffffffffu, acc_im, 1);
        acc_re += __shfl_xor_sync(0xffffffffu, acc_re, 2);
        acc_im += __shfl_xor_sync(0xffffffffu, acc_im, 2);
        if (cc == 0 && node < t.count) out[nodes.perm[t.start + node]] = make_double2(acc_re, acc_im);
    }
}

// ---------------------------------------------------------------------------
// tiled scatter
//
// Scatter tiles hold up to 128 nodes (twice the gather's) so that each RED
// of an output fragment carries the sum over more nodes.  A warp owns whole
// axis-0 slabs of the tile's box.  Per slab it forms W0[a, node] (one exp
// per node, staged through a per-warp smem row), finds the active node
// k-steps (nodes are sorted by lo0 inside a tile), and for groups of 3
// four-row M-tiles computes
//     D[(b, re|im), c] = sum_node V[(b, re|im), node] * W2[c, node]  (DMMA)
// with V = W0 W1 v formed on the fly and every W2 fragment feeding 3 DMMAs.
// D is reduced into the halo-padded grid with RED.E.ADD.F64 (no wrap on
// axes 1-2; the halo is folded back by k_halo_fold).

constexpr int SN = kSTileNodes;       // nodes per scatter tile
constexpr int SW = 8;                 // warps per CTA
constexpr int STH = SW * 32;
constexpr int WS = SN + 4;            // w1/w2 row stride (doubles): == 4 mod 16, conflict-free
constexpr int CTMAX = (kBoxMax + 7) / 8;   // 8-column tiles over axis 2
constexpr int SMT = 3;                // M-tiles per group (reuse of each W2 fragment)
constexpr int SKS = SN / 4;           // node k-steps
static_assert(CTMAX * 8 >= kBoxMax, "scatter column tiles must cover the box");
static_assert(KSMAX * 4 >= kBoxMax && NTMAX * 4 >= kBoxMax, "gather tiles must cover the box");
static_assert(SN == 128, "the active-k-step mask below assumes 4 x 32 nodes");
static_assert(CTMAX == 5 && kBoxMax > 32, "scatter column tiles: 4 (box <= 32) or 5 (box <= 40)");
static_assert(((kBoxMax / 4 + SMT - 1) / SMT) * SMT * 4 <= kBoxMax, "padded M-tile groups fit the W1 table");

struct ScatterSmem {
    double w1[kBoxMax][WS];
    double w2[CTMAX * 8][WS];
    double w0[SW][2][WS];             // per-warp rows: W0 v (re, im) of the warp's current slab
                                      // (pitch WS: the re and im rows sit in different banks)
    double2 v[SN];
    double nu[3][SN];
    int clo0[SN], chi0[SN];           // axis-0 window cells per node (window_cells)
    Tile t;
};

// One group of SMT four-row M-tiles x NCT eight-column tiles of slab a,
// accumulated over the active node k-steps, then reduced into the grid.
// NCT is a template parameter so no runtime predicate sits around a DMMA.
template <int NCT, int G, bool DET>
__device__ __forceinline__ void scatter_group(const ScatterSmem &S, const double (*w0row)[WS], int mt0, int ks0, int ks1,
                                              int g0, const Tile &t, const WindowParams &wp, double *grid,
                                              int lane, DScale dscale) {
    const int rb = lane >> 3, part = (lane >> 2) & 1, kk = lane & 3, cr = lane >> 2;
    double d[G][NCT][2];
#pragma unroll
    for (int i = 0; i < G; ++i)
#pragma unroll
        for (int ct = 0; ct < NCT; ++ct) d[i][ct][0] = d[i][ct][1] = 0.0;
#pragma unroll 2
    for (int ks = ks0; ks < ks1; ++ks) {
        const int n = ks * 4 + kk;
        const double wv = w0row[part][n];
        double av[G];
#pragma unroll
        for (int i = 0; i < G; ++i) av[i] = wv * S.w1[(mt0 + i) * 4 + rb][n];
#pragma unroll
        for (int ct = 0; ct < NCT; ++ct) {
            const double bv = S.w2[ct * 8 + cr][n];
#pragma unroll
            for (int i = 0; i < G; ++i) dmma(d[i][ct], av[i], bv);
        }
    }
#pragma unroll
    for (int i = 0; i < G; ++i) {
        const int b = (mt0 + i) * 4 + rb;
        if (b < t.e1) {
            // halo-padded grid: rows / columns of the box never wrap
            double *row = grid + 2 * (((size_t)g0 * wp.N1p + (t.o1 + b + wp.pad)) * wp.N2p + (t.o2 + wp.pad));
#pragma unroll
            for (int ct = 0; ct < NCT; ++ct) {
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    const int c = ct * 8 + 2 * kk + j;
                    SGL_DCHECK(c >= t.e2 || (g0 >= 0 && g0 < wp.N0 && t.o1 + b + wp.pad >= 0 &&
                                             t.o1 + b + wp.pad < wp.N1p && t.o2 + wp.pad + c >= 0 &&
                                             t.o2 + wp.pad + c < wp.N2p));
                    // DET == false: the plain RED, no per-RED branch on the scale (the
                    // branch cost the FP64 scatter 7 % at config 2: 5.17 -> 5.53 ms)
                    if (c < t.e2) {
                        if constexpr (DET) red_add_det(row + 2 * c + part, d[i][ct][j], dscale);
                        else red_add(row + 2 * c + part, d[i][ct][j]);
                    }
                }
            }
        }
    }
}

// the group's column tiles (box width / 8) and M-tiles (<= SMT; fewer for the
// last group of a short box) as template parameters: no DMMA on padding tiles
template <bool DET>
__device__ __forceinline__ void scatter_group_any(int nct, int g, const ScatterSmem &S, const double (*w0row)[WS],
                                                  int mt0, int ks0, int ks1, int g0, const Tile &t,
                                                  const WindowParams &wp, double *grid, int lane, DScale dscale) {
#define SGL_SG(NC, GG) scatter_group<NC, GG, DET>(S, w0row, mt0, ks0, ks1, g0, t, wp, grid, lane, dscale)
    switch (nct * 4 + g) {
    case 1 * 4 + 1: SGL_SG(1, 1); break;
    case 1 * 4 + 2: SGL_SG(1, 2); break;
    case 1 * 4 + 3: SGL_SG(1, 3); break;
    case 2 * 4 + 1: SGL_SG(2, 1); break;
    case 2 * 4 + 2: SGL_SG(2, 2); break;
    case 2 * 4 + 3: SGL_SG(2, 3); break;
    case 3 * 4 + 1: SGL_SG(3, 1); break;
    case 3 * 4 + 2: SGL_SG(3, 2); break;
    case 3 * 4 + 3: SGL_SG(3, 3); break;
    case 4 * 4 + 1: SGL_SG(4, 1); break;
    case 4 * 4 + 2: SGL_SG(4, 2); break;
    case 4 * 4 + 3: SGL_SG(4, 3); break;
    case 5 * 4 + 1: SGL_SG(5, 1); break;
    case 5 * 4 + 2: SGL_SG(5, 2); break;
    default: SGL_SG(5, 3); break;
    }
#undef SGL_SG
}

template <bool DET>
__global__ void __launch_bounds__(STH, 2)
    k_scatter_tiled(const Tile *__restrict__ tiles, int64_t ntiles, NodeSet nodes, WindowParams wp,
                    const double2 *__restrict__ values, double *__restrict__ grid, const int *__restrict__ gate,
                    const int *__restrict__ det) {
    if (gate && *gate == 0) return;   // gated launch (fallback of the int8 scatter)
    const DScale dscale = DET ? det_scale(det) : DScale{0.0, 0.0};
    extern __shared__ __align__(128) unsigned char smem_raw[];
    ScatterSmem &S = *reinterpret_cast<ScatterSmem *>(smem_raw);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    double (*w0row)[WS] = S.w0[warp];

    for (int64_t ti = blockIdx.x; ti < ntiles; ti += gridDim.x) {
        __syncthreads();   // previous tile's readers are done
        if (tid == 0) S.t = tiles[ti];
        __syncthreads();
        const Tile t = S.t;
        if (tid < SN) {
            const bool ok = tid < t.count;
            const int64_t s = (int64_t)t.start + tid;
            S.nu[0][tid] = ok ? nodes.u0[s] : -1e9;
            S.nu[1][tid] = ok ? nodes.u1[s] : -1e9;
            S.nu[2][tid] = ok ? nodes.u2[s] : -1e9;
            S.v[tid] = ok ? values[nodes.perm[s]] : make_double2(0.0, 0.0);
            int clo = 1 << 30, chi = -(1 << 30);   // no window for a padding node
            if (ok) window_cells(nodes.u0[s], wp.q, clo, chi);
            S.clo0[tid] = clo;
            S.chi0[tid] = chi;
        }
        __syncthreads();
        const int Mt = (t.e1 + 3) >> 2;
        const int CT = (t.e2 + 7) >> 3;
        // W1 / W2 tables: one thread per (node, axis) walks the rows with the
        // Gaussian recurrence (every row up to the groups' extent; 0 outside the box)
        static_assert(STH == 2 * SN, "one thread per node and table");
        {
            const int k = tid % SN;
            if (tid < SN) {
                double w[kBoxMax];
                wwalk<kBoxMax, 1>(S.nu[1][k], t.o1, kBoxMax, wp.c1, wp.h1, wp.r1_1, wp.q, w);
                const int rows = ((Mt + SMT - 1) / SMT) * SMT * 4;
#pragma unroll
                for (int y = 0; y < kBoxMax; ++y)
                    if (y < rows) S.w1[y][k] = w[y];
            } else {
                double w[CTMAX * 8];
                wwalk<CTMAX * 8, 1>(S.nu[2][k], t.o2, CTMAX * 8, wp.c2, wp.h2, wp.r2_1, wp.q, w);
#pragma unroll
                for (int y = 0; y < CTMAX * 8; ++y)
                    if (y < CT * 8) S.w2[y][k] = w[y];
            }
        }
        __syncthreads();
        const int nks = (t.count + 3) >> 2;
        // W0 along this warp's slabs a = warp, warp + SW, ...: per node the
        // Gaussian recurrence with stride SW, seeded exactly at the node's
        // first in-window slab of the warp (2 exps per node instead of one
        // per slab); the truncation |d| <= q is tested on the exact d
        double w0s[SN / 32], r0s[SN / 32];
        int a0s[SN / 32];
        static_assert(SW == 8, "the stride-8 ratio wp.r0_8 assumes 8 warps");
        const double r0step = wp.r0_8;
#pragma unroll
        for (int j = 0; j < SN / 32; ++j) {
            const int clo = S.clo0[32 * j + lane] - t.o0;           // first in-window slab
            const int k0 = clo > warp ? (clo - warp + SW - 1) / SW : 0;
            a0s[j] = warp + SW * k0;
            const double df = S.nu[0][32 * j + lane] - (double)(t.o0 + a0s[j]);
            w0s[j] = wp.c0 * exp(-df * df * wp.h0);
            r0s[j] = exp(wp.h0 * (2.0 * SW * df - (double)(SW * SW)));
        }
        for (int a = warp; a < t.e0; a += SW) {
            // W0 of this slab for all nodes; active k-steps from the nonzero mask
            int kfirst = SKS, klast = -1;
#pragma unroll
            for (int j = 0; j < SN / 32; ++j) {
                const double w = (a >= a0s[j] && a + t.o0 <= S.chi0[32 * j + lane]) ? w0s[j] : 0.0;
                if (a >= a0s[j]) {
                    w0s[j] *= r0s[j];
                    r0s[j] *= r0step;
                }
                const double2 v = S.v[32 * j + lane];
                w0row[0][32 * j + lane] = w * v.x;
                w0row[1][32 * j + lane] = w * v.y;
                const unsigned m = __ballot_sync(0xffffffffu, w != 0.0);
                if (m) {
                    kfirst = min(kfirst, (32 * j + __ffs(m) - 1) >> 2);
                    klast = max(klast, (32 * j + 31 - __clz(m)) >> 2);
                }
            }
            __syncwarp();
            if (klast < 0) continue;
            const int ks0 = kfirst, ks1 = min(nks, klast + 1);
            const int g0 = wrapi(t.o0 + a, wp.N0);
            for (int mt0 = 0; mt0 < Mt; mt0 += SMT)
                scatter_group_any<DET>(CT, min(SMT, Mt - mt0), S, w0row, mt0, ks0, ks1, g0, t, wp, grid, lane, dscale);
            __syncwarp();   // w0row is rewritten for the warp's next slab
        }
    }
}

// ---------------------------------------------------------------------------
// generic per-node kernels (any q): the reference loop nest, one warp per node

constexpr int NW_GEN = 4;

__global__ void __launch_bounds__(NW_GEN * 32)
    k_gather_generic(int64_t M, NodeSet nodes, WindowParams wp, const double2 *__restrict__ grid,
                     double2 *__restrict__ out) {
    extern __shared__ __align__(16) double gsm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int P0 = 2 * wp.qa0 + 1, P1 = 2 * wp.qa1 + 1, P2 = 2 * wp.qa2 + 1;
    double *w0 = gsm + warp * (P0 + P1 + P2), *w1 = w0 + P0, *w2 = w1 + P1;
    const int64_t i = blockIdx.x * (int64_t)NW_GEN + warp;
    if (i >= M) return;
    const double u0 = nodes.u0[i], u1 = nodes.u1[i], u2 = nodes.u2[i];
    const int l0 = (int)floor(u0), l1 = (int)floor(u1), l2 = (int)floor(u2);
    for (int o = lane; o < P0; o += 32) w0[o] = wfun(u0, l0 - wp.qa0 + o, wp.c0, wp.h0, wp.qa0);
    for (int o = lane; o < P1; o += 32) w1[o] = wfun(u1, l1 - wp.qa1 + o, wp.c1, wp.h1, wp.qa1);
    for (int o = lane; o < P2; o += 32) w2[o] = wfun(u2, l2 - wp.qa2 + o, wp.c2, wp.h2, wp.qa2);
    __syncwarp();
    double ar = 0.0, ai = 0.0;
    for (int a = 0; a < P0; ++a) {
        const double wa = w0[a];
        if (wa == 0.0) continue;
        const int g0 = wrapi(l0 - wp.qa0 + a, wp.N0);
        for (int b = 0; b < P1; ++b) {
            const double wab = wa * w1[b];
            const int g1 = wrapi(l1 - wp.qa1 + b, wp.N1);
            const double2 *row = grid + ((size_t)g0 * wp.N1p + g1 + wp.pad) * wp.N2p + wp.pad;
            double sr = 0.0, si = 0.0;
            for (int c = lane; c < P2; c += 32) {
                const double2 g = row[wrapi(l2 - wp.qa2 + c, wp.N2)];
                sr = fma(w2[c], g.x, sr);
                si = fma(w2[c], g.y, si);
            }
            ar = fma(wab, sr, ar);
            ai = fma(wab, si, ai);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        ar += __shfl_xor_sync(0xffffffffu, ar, o);
        ai += __shfl_xor_sync(0xffffffffu, ai, o);
    }
    SGL_DCHECK(nodes.perm[i] >= 0 && nodes.perm[i] < M);
    if (lane == 0) out[nodes.perm[i]] = make_double2(ar, ai);
}

__global__ void __launch_bounds__(NW_GEN * 32)
    k_scatter_generic(int64_t M, NodeSet nodes, WindowParams wp, const double2 *__restrict__ values,
                      double *__restrict__ grid, const int *__restrict__ det) {
    extern __shared__ __align__(16) double gsm[];
    const DScale dscale = det_scale(det);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int P0 = 2 * wp.qa0 + 1, P1 = 2 * wp.qa1 + 1, P2 = 2 * wp.qa2 + 1;
    double *w0 = gsm + warp * (P0 + P1 + P2), *w1 = w0 + P0, *w2 = w1 + P1;
    const int64_t i = blockIdx.x * (int64_t)NW_GEN + warp;
    if (i >= M) return;
    const double u0 = nodes.u0[i], u1 = nodes.u1[i], u2 = nodes.u2[i];
    const int l0 = (int)floor(u0), l1 = (int)floor(u1), l2 = (int)floor(u2);
    for (int o = lane; o < P0; o += 32) w0[o] = wfun(u0, l0 - wp.qa0 + o, wp.c0, wp.h0, wp.qa0);
    for (int o = lane; o < P1; o += 32) w1[o] = wfun(u1, l1 - wp.qa1 + o, wp.c1, wp.h1, wp.qa1);
    for (int o = lane; o < P2; o += 32) w2[o] = wfun(u2, l2 - wp.qa2 + o, wp.c2, wp.h2, wp.qa2);
    __syncwarp();
    const double2 v = values[nodes.perm[i]];
    for (int a = 0; a < P0; ++a) {
        const double wa = w0[a];
        if (wa == 0.0) continue;
        const int g0 = wrapi(l0 - wp.qa0 + a, wp.N0);
        for (int b = 0; b < P1; ++b) {
            const double wab = wa * w1[b];
            const double tr = wab * v.x, tim = wab * v.y;
            const int g1 = wrapi(l1 - wp.qa1 + b, wp.N1);
            double *row = grid + 2 * (((size_t)g0 * wp.N1p + g1 + wp.pad) * wp.N2p + wp.pad);
            for (int c = lane; c < P2; c += 32) {
                const int g2 = wrapi(l2 - wp.qa2 + c, wp.N2);
                red_add_det(row + 2 * g2, w2[c] * tr, dscale);
                red_add_det(row + 2 * g2 + 1, w2[c] * tim, dscale);
            }
        }
    }
}

// ---------------------------------------------------------------------------
// periodic halo of the padded grid (axes 1-2)

// copy interior images into the halo (after the inverse FFT, before gather)
// copy interior images into the halo (after the inverse FFT).  One thread
// per halo cell of a plane (blockIdx.y = axis-0 plane): the q-row bands above
// and below the interior (full padded width) and the q-column strips beside
// it; 32-bit index math, no pass over the interior.
__global__ void k_halo_fill(WindowParams wp, double2 *__restrict__ grid) {
    const int q = wp.pad, band = 2 * q * wp.N2p, per_plane = band + 2 * q * wp.N1;
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= per_plane) return;
    int p1, p2;
    if (r < band) {
        const int k = r / wp.N2p;
        p1 = k < q ? k : wp.N1 + k;            // rows [0, q) and [N1 + q, N1 + 2q)
        p2 = r - k * wp.N2p;
    } else {
        const int s = r - band, k = s / (2 * q), cc = s - k * (2 * q);
        p1 = q + k;
        p2 = cc < q ? cc : wp.N2 + cc;          // columns [0, q) and [N2 + q, N2 + 2q)
    }
    const int s1 = wrapi(p1 - q, wp.N1) + q, s2 = wrapi(p2 - q, wp.N2) + q;
    double2 *plane = grid + (size_t)blockIdx.y * wp.N1p * wp.N2p;
    plane[(size_t)p1 * wp.N2p + p2] = plane[(size_t)s1 * wp.N2p + s2];
}

// add the halo images back into the interior (after scatter, before FFT).
// Only interior cells within q of an axis-1/2 edge have images: thread over
// that edge set (rows i1 < q or i1 >= N1 - q in full, plus the q-wide column
// strips of the other rows) instead of the whole plane.
__device__ __forceinline__ void fold_cell(const WindowParams &wp, double2 *grid, int64_t g0, int i1, int i2) {
    double2 acc = make_double2(0.0, 0.0);
    bool any = false;
    // every padded position p = i + q + k N inside [0, N + 2q), except k = 0 on both axes
    for (int p1 = (i1 + wp.pad) % wp.N1; p1 < wp.N1p; p1 += wp.N1) {
        for (int p2 = (i2 + wp.pad) % wp.N2; p2 < wp.N2p; p2 += wp.N2) {
            if (p1 == i1 + wp.pad && p2 == i2 + wp.pad) continue;
            const double2 v = grid[((size_t)g0 * wp.N1p + p1) * wp.N2p + p2];
            acc.x += v.x;
            acc.y += v.y;
            any = true;
        }
    }
    if (any) {
        double2 &dst = grid[((size_t)g0 * wp.N1p + i1 + wp.pad) * wp.N2p + i2 + wp.pad];
        dst.x += acc.x;
        dst.y += acc.y;
    }
}

__global__ void k_halo_fold(WindowParams wp, double2 *__restrict__ grid) {
    // blockIdx.y = axis-0 plane; 32-bit index math within the plane
    const int q1 = min(wp.pad, wp.N1), q2 = min(wp.pad, wp.N2);
    const int band_rows = min(wp.N1, 2 * q1);              // rows [0,q) and [N1-q, N1)
    const int strip = min(wp.N2, 2 * q2);                   // columns [0,q) and [N2-q, N2)
    const int per_plane = band_rows * wp.N2 + (wp.N1 - band_rows) * strip;
    int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= per_plane) return;
    int i1, i2;
    if (r < band_rows * wp.N2) {
        const int k = r / wp.N2;
        i1 = k < q1 ? k : wp.N1 - band_rows + k;
        i2 = r - k * wp.N2;
    } else {
        r -= band_rows * wp.N2;
        const int k = r / strip;
        i1 = q1 + k;
        const int cc = r - k * strip;
        i2 = cc < q2 ? cc : wp.N2 - strip + cc;
    }
    fold_cell(wp, grid, blockIdx.y, i1, i2);
}

}  // namespace

// SM count of the current device (cached per device; benign concurrent fill)
int num_sms() {
    static std::atomic<int> cache[64];
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    int n = cache[dev].load(std::memory_order_relaxed);
    if (n <= 0) {
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
        cache[dev].store(n, std::memory_order_relaxed);
    }
    return n;
}

namespace {

}  // namespace

namespace {
template <int NT>
cudaError_t launch_gather_nt(const Plan &p, double2 *values, unsigned blocks, const int *gate, cudaStream_t st) {
    const size_t sm = sizeof(GatherSmem);
    cudaError_t e = cudaFuncSetAttribute(k_gather_tiled<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    k_gather_tiled<NT><<<blocks, GT, sm, st>>>(p.tmap, p.tiles, p.n_tiles, p.nodes, p.wp, values, gate);
    return cudaGetLastError();
}
}  // namespace

int launch_gather_tiled_gated(const Plan &p, double2 *values, const int *gate, cudaStream_t st) {
    if (p.M == 0 || p.generic) return SGL_OK;
    int64_t blocks = std::min<int64_t>(p.n_tiles, (int64_t)num_sms() * GCPS);
    if (blocks < 1) blocks = 1;
    switch (std::max(3, std::min(NTMAX, (p.tile_box + 3) / 4))) {
    case 3: SGL_CUDA_CHECK(launch_gather_nt<3>(p, values, (unsigned)blocks, gate, st)); break;
    case 4: SGL_CUDA_CHECK(launch_gather_nt<4>(p, values, (unsigned)blocks, gate, st)); break;
    case 5: SGL_CUDA_CHECK(launch_gather_nt<5>(p, values, (unsigned)blocks, gate, st)); break;
    case 6: SGL_CUDA_CHECK(launch_gather_nt<6>(p, values, (unsigned)blocks, gate, st)); break;
    case 7: SGL_CUDA_CHECK(launch_gather_nt<7>(p, values, (unsigned)blocks, gate, st)); break;
    case 8: SGL_CUDA_CHECK(launch_gather_nt<8>(p, values, (unsigned)blocks, gate, st)); break;
    default: SGL_CUDA_CHECK(launch_gather_nt<NTMAX>(p, values, (unsigned)blocks, gate, st)); break;
    }
    return SGL_OK;
}

int launch_gather(const Plan &p, const double2 *grid, double2 *values, cudaStream_t st) {
    if (p.M == 0) return SGL_OK;
    if (!p.generic) {
        return launch_gather_tiled_gated(p, values, nullptr, st);
    } else {
        const size_t sm = (size_t)NW_GEN * (3 + 2 * (p.wp.qa0 + p.wp.qa1 + p.wp.qa2)) * sizeof(double);
        if (sm > 48 * 1024) SGL_CUDA_CHECK(cudaFuncSetAttribute(k_gather_generic, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        k_gather_generic<<<(unsigned)((p.M + NW_GEN - 1) / NW_GEN), NW_GEN * 32, sm, st>>>(p.M, p.nodes, p.wp,
                                                                                           grid, values);
    }
    SGL_CUDA_CHECK(cudaGetLastError());
    return SGL_OK;
}

int make_grid_tmap(Plan &p) {
    // FLOAT64 view of the padded grid: dims {2 N2p, N1p, N0}; one box = one slab
    // driver entry point, looked up once (thread-safe static initialisation)
    static const PFN_cuTensorMapEncodeTiled_v12000 encode = []() -> PFN_cuTensorMapEncodeTiled_v12000 {
        cudaDriverEntryPointQueryResult qr;
        void *fn = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr) != cudaSuccess ||
            qr != cudaDriverEntryPointSuccess)
            return nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }();
    if (!encode) {
        cudaGetLastError();
        set_error("cuTensorMapEncodeTiled is unavailable");
        return SGL_ECUDA;
    }
    const WindowParams &w = p.wp;
    cuuint64_t dims[3] = {(cuuint64_t)2 * w.N2p, (cuuint64_t)w.N1p, (cuuint64_t)w.N0};
    cuuint64_t strides[2] = {(cuuint64_t)w.N2p * 16, (cuuint64_t)w.N1p * w.N2p * 16};
    cuuint32_t box[3] = {2 * SSTR, SROWS, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = encode(&p.tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, p.grid_buf, dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        set_error("cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
        return SGL_ECUDA;
    }
    p.tmap_ready = true;
    return SGL_OK;
}

int launch_halo_fill(const Plan &p, double2 *grid, cudaStream_t st) {
    if (p.wp.pad == 0) return SGL_OK;
    const int per_plane = 2 * p.wp.pad * p.wp.N2p + 2 * p.wp.pad * p.wp.N1;
    k_halo_fill<<<dim3((per_plane + 255) / 256, p.wp.N0), 256, 0, st>>>(p.wp, grid);
    SGL_CUDA_CHECK(cudaGetLastError());
    return SGL_OK;
}

int launch_halo_fold(const Plan &p, double2 *grid, cudaStream_t st) {
    if (p.wp.pad == 0) return SGL_OK;
    const int q1 = std::min(p.wp.pad, p.wp.N1), q2 = std::min(p.wp.pad, p.wp.N2);
    const int band_rows = std::min(p.wp.N1, 2 * q1), strip = std::min(p.wp.N2, 2 * q2);
    const int per_plane = band_rows * p.wp.N2 + (p.wp.N1 - band_rows) * strip;
    k_halo_fold<<<dim3((per_plane + 255) / 256, p.wp.N0), 256, 0, st>>>(p.wp, grid);
    SGL_CUDA_CHECK(cudaGetLastError());
    return SGL_OK;
}

int launch_scatter_tiled_gated(const Plan &p, const double2 *values, double2 *grid, const int *gate,
                               cudaStream_t st) {
    if (p.M == 0 || p.generic) return SGL_OK;
    const size_t sm = sizeof(ScatterSmem);
    const int *det = p.det_e();
    auto kern = det ? k_scatter_tiled<true> : k_scatter_tiled<false>;
    SGL_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    int64_t blocks = std::min<int64_t>(p.n_stiles, (int64_t)num_sms() * 2 * 8);
    if (blocks < 1) blocks = 1;
    kern<<<(unsigned)blocks, STH, sm, st>>>(p.stiles, p.n_stiles, p.snodes, p.wp, values,
                                            reinterpret_cast<double *>(grid), gate, det);
    SGL_CUDA_CHECK(cudaGetLastError());
    return SGL_OK;
}

int launch_scatter(const Plan &p, const double2 *values, double2 *grid, cudaStream_t st) {
    if (p.M == 0) return SGL_OK;
    if (!p.generic) {
        return launch_scatter_tiled_gated(p, values, grid, nullptr, st);
    } else {
        const size_t sm = (size_t)NW_GEN * (3 + 2 * (p.wp.qa0 + p.wp.qa1 + p.wp.qa2)) * sizeof(double);
        if (sm > 48 * 1024) SGL_CUDA_CHECK(cudaFuncSetAttribute(k_scatter_generic, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        k_scatter_generic<<<(unsigned)((p.M + NW_GEN - 1) / NW_GEN), NW_GEN * 32, sm, st>>>(
            p.M, p.nodes, p.wp, values, reinterpret_cast<double *>(grid), p.det_e());
    }
    SGL_CUDA_CHECK(cudaGetLastError());
    return SGL_OK;
}

}  // namespace sgl
