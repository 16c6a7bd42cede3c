// Gaussian-window gather (forward NFFT interpolation, _gridding.py:53-74) on
// the int8 tensor cores (tcgen05.mma kind::i8), reproducing FP64 results by an
// exact integer digit split (Ozaki scheme).  sm_100a.
//
// Per tile of <= 128 sorted nodes (one 8 x 16 pencil of cells on axes 1-2,
// consecutive in lo0) and its box of e0 x 40 x 48 cells, the window sum
//     out[n] = sum_b w1[n,b] sum_{a,c} w0[n,a] w2[n,c] G[a,b,c]
// is a GEMM with M = nodes, N = (b, re|im) = 80 and K = (a, c) = e0 x 48:
//     D[n, (b,ri)] = sum_k A[n,k] G_ri[k,b],  A[n,(a,c)] = w0[n,a] w2[n,c].
// Both operands are scaled to fixed point and split into 6 balanced signed
// bytes (digits in [-128, 127]: zero-mean truncation error):
//     A * 2^sA = sum_p a_p 256^p,   G * 2^sG(a) = sum_q g_q 256^q,
// so A G = 2^-(sA+sG) sum_{p,q} 256^(p+q) (a_p . g_q), every a_p . g_q an
// exact int32 dot product.  The grid scale is per slab (sG(a), from the slab's
// max |G|: the slab envelope spans up to 1e15 at B = 64); a tile works at the
// scale of its largest slab, sG_t = min_a sG(a), and the weight digits absorb
// the slab factor, A'[n,(a,c)] = A 2^(sG_t - sG(a)) <= A.  The 21 digit pairs
// with p + q >= 5 are kept (tools/ozaki_sim.py: ~1e-12 relative on the
// reference goldens, the dropped pairs being the leading error); pairs with equal
// p + q share one int32 TMEM accumulator (6 "diagonals" x 80 columns = 480
// of the 512 TMEM columns), and one MMA multiplies A digit p with up to
// three consecutive B digits stacked along N (N = 240), 9 MMAs per K-step of
// 32.  The epilogue combines the diagonals of a column into one exact int64,
// converts it, applies the axis-1 weights w1[n,b] and the scale and writes
// the node values in caller order.
//
// Grid digits are produced once per forward (k_slice_grid, after the halo
// fill) as [a][c/16][digit][b][re|im][c%16] and reach shared memory by TMA
// (one 6-digit x 1280-byte box per K-chunk).  The weight digits are
// built per tile by 12 generator warps directly in the UMMA K-major layout.
//
// CTA (one per SM, persistent over tiles): warp 0 TMA producer, warp 1 MMA
// issuer (one lane), warps 2-13 weight-digit generators, warps 14-17 epilogue
// (TMEM lane quarters).  4-stage weight-digit ring and 8-stage grid-digit
// ring (full / empty mbarriers), TMEM full / empty mbarriers between the MMA
// issuer and the epilogue.
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "sgl_internal.cuh"
#include "umma.cuh"
#include "i8_common.cuh"

namespace sgl {
namespace {

using namespace i8;

constexpr int IM = kI8Nodes;              // MMA M (nodes)
static_assert(kMaxQTiled <= 16, "combine6_i64 in the gather needs (2q + 1)^2 <= 2^11 window cells");
constexpr int ROWS = 2 * kI8Box1;         // MMA N per digit: (b, re|im)
constexpr int NSTG = 4;                   // weight-digit ring depth (K-steps of 32)
constexpr int NSTGB = 8;                  // grid-digit (TMA) ring depth: hides the L2 latency
constexpr int A_DIGIT = IM * 16;          // one K-chunk of one weight digit (2048 B)
constexpr int A_CHUNK = ND * A_DIGIT;
constexpr int A_STAGE = 2 * A_CHUNK;
constexpr int B_DIGIT = ROWS * 16;        // one K-chunk of one grid digit (1280 B)
constexpr int B_CHUNK = ND * B_DIGIT;     // one TMA box
constexpr int B_STAGE = 2 * B_CHUNK;
constexpr int NGW = 12;                   // generator warps (3 chunk columns x 128 nodes)
constexpr int NEW = 4;                    // epilogue warps
constexpr int IT = (2 + NGW + NEW) * 32;
static_assert(NBLK * ROWS <= (int)TCOLS, "diagonal accumulators must fit TMEM");
static_assert(CHUNKS == 3, "K-chunk bookkeeping assumes 48-cell slabs");

struct I8Smem {
    uint8_t a[NSTG][A_STAGE];     // weight digits, [chunk][digit][node][16 cells]
    uint8_t b[NSTGB][B_STAGE];    // grid digits,   [chunk][digit][b][re|im][16 cells]
    uint64_t fullA[NSTG], empty[NSTG], fullB[NSTGB], emptyB[NSTGB];
    uint64_t tfull, tempty;
    uint32_t tbase;
};

// MMA schedule of one K-step (SGL_I8_OP list in the issuer): A digit p times
// B digits q0 .. q0+nq-1 (stacked along N) into the diagonal accumulators
// p+q0-DMIN .. ; 21 digit pairs with p + q >= DMIN in 9 MMAs.


__device__ __forceinline__ void st_async_v4(void *dst, const uint32_t (&v)[4], uint64_t *bar) {
    asm volatile(
        "st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];\n" ::"r"(
            umma::smem_addr(dst)),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(umma::smem_addr(bar))
        : "memory");
}

__device__ __forceinline__ int64_t tile_steps(const Tile &t) { return (CHUNKS * t.e0 + 1) >> 1; }

template <bool P>
__device__ __forceinline__ long long tick() {
    if constexpr (P) return clock64();
    else return 0;
}

template <bool PROF>   // PROF: clock64 wait counters (SGL_FLAG_I8_PROF); compiled out otherwise
__global__ void __cluster_dims__(1, 1, 1) __launch_bounds__(IT, 1)
    k_gather_i8(const __grid_constant__ CUtensorMap dmap, const Tile *__restrict__ tiles, int64_t ntiles,
                NodeSet nodes, WindowParams wp, double s0, double s2, int sA,
                const int *__restrict__ gsh, const int *__restrict__ tsh, double2 *__restrict__ out,
                unsigned long long *__restrict__ prof, const int *__restrict__ skip) {
    if (*skip) return;   // non-finite grid: the gated FP64 gather runs instead (guard.cu)
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    I8Smem &S = *reinterpret_cast<I8Smem *>(smem_raw);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

    if (tid == 0) {
        for (int s = 0; s < NSTG; ++s) {
            mbar_init(&S.fullA[s], 1);   // one expect_tx arrive + the st.async bytes of a K-step
            mbar_init(&S.empty[s], 1);
        }
        for (int s = 0; s < NSTGB; ++s) {
            mbar_init(&S.fullB[s], 1);
            mbar_init(&S.emptyB[s], 1);
        }
        mbar_init(&S.tfull, 1);
        mbar_init(&S.tempty, NEW);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (warp == 1) umma::tmem_alloc(&S.tbase, TCOLS);
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    const uint32_t tbase = S.tbase;

    if (warp == 0) {
        // ---- TMA producer: grid digits, two 16-cell K-chunks per stage
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];\n" ::"l"(&dmap) : "memory");
            uint32_t g = 0;
            for (int64_t ti = blockIdx.x; ti < ntiles; ti += gridDim.x) {
                const Tile t = tiles[ti];
                const int ns = (int)tile_steps(t);
                const int cb = kstart2(t, wp), bb = t.o1 + wp.pad;   // TMA rows are (b, re|im) pairs
                for (int s = 0; s < ns; ++s, ++g) {
                    const int stg = (int)(g % NSTGB);
                    const uint32_t use = g / NSTGB;
                    if (use) mbar_wait(&S.emptyB[stg], (use - 1) & 1, 1);
                    mbar_expect_tx(&S.fullB[stg], B_STAGE);
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int kc = 2 * s + h, al = kc / CHUNKS, cc = kc - CHUNKS * al;
                        // the tile's live cells inside the padded plane (box parts beyond it are
                        // TMA out-of-bounds reads: zero-filled, and their weights are zero)
                        SGL_DCHECK(bb >= 0 && bb + t.e1 <= wp.N1p && t.o2 + wp.pad >= 0 &&
                                   t.o2 + wp.pad + t.e2 <= wp.N2p && (cb >> 4) + cc >= 0 && al <= t.e0 &&
                                   wrap1(t.o0 + al, wp.N0) >= 0 && wrap1(t.o0 + al, wp.N0) < wp.N0);
                        tma_load_4d(S.b[stg] + h * B_CHUNK, &dmap, 4 * bb, 0, (cb >> 4) + cc, wrap1(t.o0 + al, wp.N0),
                                    &S.fullB[stg]);
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ---- MMA issuer: the warp waits, one elected lane issues.  The 9
        // MMAs of a K-step use compile-time digit offsets and instruction
        // descriptors on top of two per-stage base descriptors.
        const uint64_t a0 = umma::desc_kmajor(umma::smem_addr(S.a[0]), A_CHUNK, 128);
        const uint64_t b0 = umma::desc_kmajor(umma::smem_addr(S.b[0]), B_CHUNK, 128);
        uint32_t g = 0, tc = 0;
        long long pw_a = 0, pw_b = 0, pw_e = 0, pt0 = tick<PROF>();
        for (int64_t ti = blockIdx.x; ti < ntiles; ti += gridDim.x, ++tc) {
            const int ns = (int)tile_steps(tiles[ti]);
            long long t0 = tick<PROF>();
            if (tc) mbar_wait(&S.tempty, (tc - 1) & 1, 2);
            umma::fence_after();
            long long t1 = tick<PROF>();
            pw_e += t1 - t0;
            for (int s = 0; s < ns; ++s, ++g) {
                const int stg = (int)(g % NSTG), stgb = (int)(g % NSTGB);
                t0 = tick<PROF>();
                mbar_wait(&S.fullB[stgb], (g / NSTGB) & 1, 3);
                t1 = tick<PROF>();
                mbar_wait(&S.fullA[stg], (g / NSTG) & 1, 4);
                long long t2 = tick<PROF>();
                pw_b += t1 - t0;
                pw_a += t2 - t1;
                umma::fence_after();
                if (umma::elect_one()) {
                    const uint64_t ad = a0 + (uint64_t)(stg * (A_STAGE >> 4));
                    const uint64_t bd = b0 + (uint64_t)(stgb * (B_STAGE >> 4));
                    const bool acc = s > 0;
                    {
#define SGL_I8_OP(P, Q0, NQ, ACC)                                                                              \
    umma::mma_i8(tbase + (uint32_t)(((P) + (Q0)-DMIN) * ROWS), ad + (uint64_t)((P)*A_DIGIT >> 4),             \
                 bd + (uint64_t)((Q0)*B_DIGIT >> 4), umma::idesc_i8(IM, (NQ)*ROWS, true, true), ACC)
                        // the two p = 5 MMAs cover every accumulator and carry the per-tile reset
                        SGL_I8_OP(5, 0, 3, acc);
                        SGL_I8_OP(5, 3, 3, acc);
                        SGL_I8_OP(4, 1, 3, true);
                        SGL_I8_OP(4, 4, 2, true);
                        SGL_I8_OP(3, 2, 3, true);
                        SGL_I8_OP(3, 5, 1, true);
                        SGL_I8_OP(2, 3, 3, true);
                        SGL_I8_OP(1, 4, 2, true);
                        SGL_I8_OP(0, 5, 1, true);
#undef SGL_I8_OP
                    }
                    umma::commit(&S.empty[stg]);
                    umma::commit(&S.emptyB[stgb]);
                }
                __syncwarp();
            }
            if (umma::elect_one()) umma::commit(&S.tfull);
            __syncwarp();
        }
        if (PROF && prof && lane == 0) {
            prof[blockIdx.x * 4 + 0] = tick<PROF>() - pt0;
            prof[blockIdx.x * 4 + 1] = pw_a;
            prof[blockIdx.x * 4 + 2] = pw_b;
            prof[blockIdx.x * 4 + 3] = pw_e;
        }
    } else if (warp < 2 + NGW) {
        // ---- weight-digit generators: thread = (node n, chunk column cc of a
        // slab): its 16 W2 values stay in registers for the whole tile and its
        // chunks kc = cc, cc + 3, ... visit the slabs one by one (W0 by the
        // Gaussian recurrence); chunk kc goes to half kc % 2 of K-step kc / 2
        const int gt = tid - 64, n = gt % IM, cc = gt / IM;
        uint32_t g = 0;   // K-steps of the previous tiles
        for (int64_t ti = blockIdx.x; ti < ntiles; ti += gridDim.x) {
            const Tile t = tiles[ti];
            const bool live = n < t.count;
            const int64_t si = (int64_t)t.start + n;
            const double u0 = live ? nodes.u0[si] : -1e9, u2 = live ? nodes.u2[si] : -1e9;
            int lo0, hi0, lo2, hi2;
            window_cells(u0, wp.q, lo0, hi0);
            window_cells(u2, wp.q, lo2, hi2);
            const int cell2 = kstart2(t, wp) - wp.pad + 16 * cc;   // cell of this thread's first column
            double w2[16];
            {
                const int efirst = max(0, lo2 - cell2);
                const double d = u2 - (double)(cell2 + efirst);
                double w = s2 * (wp.c2 * exp(-d * d * wp.h2)), r = exp(wp.h2 * (2.0 * d - 1.0));
#pragma unroll
                for (int e = 0; e < 16; ++e) {
                    w2[e] = (live && e >= efirst && cell2 + e <= hi2) ? w : 0.0;
                    if (e >= efirst) {
                        w *= r;
                        r *= wp.r2_1;
                    }
                }
            }
            const int ns = (int)tile_steps(t);
            const int a_first = max(0, lo0 - t.o0), a_last = hi0 - t.o0;
            const int sGt = __ldg(tsh + ti);
            double wcur = 0.0, rcur = 0.0;
            // slab shifts loaded one slab ahead (their L1/L2 latency off the digit chain)
            int sh_next = __ldg(gsh + wrap1(t.o0, wp.N0));
            for (int kc = cc, al = 0; kc < 2 * ns; kc += CHUNKS, ++al) {
                const int sh_al = sh_next;
                if (kc + CHUNKS < 2 * ns) sh_next = __ldg(gsh + wrap1(t.o0 + al + 1, wp.N0));
                // W0 of slab al (recurrence from the node's first window slab)
                if (al == a_first) {
                    const double d0 = u0 - (double)(t.o0 + al);
                    wcur = s0 * (wp.c0 * exp(-d0 * d0 * wp.h0));
                    rcur = exp(wp.h0 * (2.0 * d0 - 1.0));
                } else if (al > a_first) {
                    wcur *= rcur;
                    rcur *= wp.r0_1;
                }
                const double fslab = pow2n(sGt - sh_al);   // slab -> tile scale
                const double w0 = (live && al >= a_first && al <= a_last) ? wcur * fslab : 0.0;
                const uint32_t gs = g + (uint32_t)(kc >> 1);
                const int stg = (int)(gs % NSTG), h = kc & 1;
                const uint32_t use = gs / NSTG;
                uint32_t dw[ND][4];
#pragma unroll
                for (int q4 = 0; q4 < 4; ++q4) {
                    uint32_t L[4], H[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const double y = fma(w0, w2[q4 * 4 + e], MAGIC_BAL);
                        L[e] = (uint32_t)__double2loint(y);
                        H[e] = (uint32_t)__double2hiint(y);
                    }
                    // byte transpose: digit p of the 4 entries -> one word
                    const uint32_t t0 = prmt(L[0], L[1], 0x5140), t1 = prmt(L[2], L[3], 0x5140);
                    const uint32_t t2 = prmt(L[0], L[1], 0x7362), t3 = prmt(L[2], L[3], 0x7362);
                    const uint32_t h0 = prmt(H[0], H[1], 0x5140), h1 = prmt(H[2], H[3], 0x5140);
                    dw[0][q4] = prmt(t0, t1, 0x5410) ^ 0x80808080u;   // offset bytes -> balanced digits
                    dw[1][q4] = prmt(t0, t1, 0x7632) ^ 0x80808080u;
                    dw[2][q4] = prmt(t2, t3, 0x5410) ^ 0x80808080u;
                    dw[3][q4] = prmt(t2, t3, 0x7632) ^ 0x80808080u;
                    dw[4][q4] = prmt(h0, h1, 0x5410) ^ 0x80808080u;
                    dw[5][q4] = prmt(h0, h1, 0x7632) ^ 0x80808080u;
                }
                if (use) mbar_wait(&S.empty[stg], (use - 1) & 1, 5);
                // st.async: async-proxy stores that complete_tx on the stage's
                // barrier (no proxy fence, no per-warp arrive); one thread per
                // K-step registers the stage's byte count
                if (h == 0 && n == 0) mbar_expect_tx(&S.fullA[stg], A_STAGE);
                uint8_t *dst = S.a[stg] + h * A_CHUNK + n * 16;
#pragma unroll
                for (int p = 0; p < ND; ++p) st_async_v4(dst + p * A_DIGIT, dw[p], &S.fullA[stg]);
            }
            g += (uint32_t)ns;
        }
    } else {
        // ---- epilogue: thread = node = TMEM lane
        const int quarter = warp & 3, n = quarter * 32 + lane;
        const uint32_t tl = tbase + ((uint32_t)(quarter * 32) << 16);
        uint32_t tc = 0;
        for (int64_t ti = blockIdx.x; ti < ntiles; ti += gridDim.x, ++tc) {
            const Tile t = tiles[ti];
            const bool live = n < t.count;
            const int64_t si = (int64_t)t.start + n;
            const double u1 = live ? nodes.u1[si] : -1e9;
            int lo1, hi1;
            window_cells(u1, wp.q, lo1, hi1);
            const int sGt = __ldg(tsh + ti);
            const double unit = ldexp(1.0, 8 * DMIN - sA - sGt);   // value of diagonal DMIN
            // W1 along axis 1 by the Gaussian recurrence, seeded before the wait
            const int bfirst = max(0, lo1 - t.o1), blast = hi1 - t.o1;
            double w1 = 0.0, r1 = 0.0;
            {
                const double d = u1 - (double)(t.o1 + bfirst);
                w1 = wp.c1 * exp(-d * d * wp.h1);
                r1 = exp(wp.h1 * (2.0 * d - 1.0));
            }
            mbar_wait(&S.tfull, tc & 1, 6);
            umma::fence_after();
            double acc_re = 0.0, acc_im = 0.0;
            // software-pipelined drain, 4 columns (2 axis-1 cells x re|im) per step:
            // the TMEM loads of step i+1 are in flight while step i converts
            int32_t D[2][NBLK][4];
            __syncwarp();   // tcgen05.ld is .sync.aligned: the warp must be converged
#pragma unroll
            for (int k = 0; k < NBLK; ++k) umma::tmem_ld4(tl + (uint32_t)(k * ROWS), D[0][k]);
            umma::tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < ROWS / 4; ++i) {
                const int cur = i & 1;
                if (i + 1 < ROWS / 4) {
#pragma unroll
                    for (int k = 0; k < NBLK; ++k) umma::tmem_ld4(tl + (uint32_t)(k * ROWS + (i + 1) * 4), D[cur ^ 1][k]);
                }
                double v[4];
                // one exact int64 per column (a node's weights are nonzero on at most
                // (2q + 1)^2 <= 33^2 cells, so |sum| < 2^(46 + 46 + 10.1 - 40) < 2^63
                // for any K); the power-of-two unit is applied once per node
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    v[j] = (double)combine6_i64(D[cur][0][j], D[cur][1][j], D[cur][2][j], D[cur][3][j], D[cur][4][j],
                                                D[cur][5][j]);
#pragma unroll
                for (int jb = 0; jb < 2; ++jb) {
                    const int b = i * 2 + jb;
                    const double w = (live && b >= bfirst && b <= blast) ? w1 : 0.0;
                    if (b >= bfirst) {
                        w1 *= r1;
                        r1 *= wp.r1_1;
                    }
                    acc_re = fma(w, v[2 * jb], acc_re);
                    acc_im = fma(w, v[2 * jb + 1], acc_im);
                }
                umma::tmem_ld_wait();
            }
            umma::fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&S.tempty);
            SGL_DCHECK(!live || (si < nodes.n && nodes.perm[si] >= 0 && nodes.perm[si] < nodes.n));
            if (live) out[nodes.perm[si]] = make_double2(acc_re * unit, acc_im * unit);
        }
    }

    umma::fence_before();
    __syncthreads();
    if (warp == 1) {
        __syncwarp();
        umma::fence_after();
        umma::tmem_free(tbase, TCOLS);
    }
}

// per slab a: max(|Re G|, |Im G|) (bits of a non-negative double order like
// the double; NaN counts as +Inf); grid = (N0 slabs) x (blocks per slab)
__global__ void k_slab_absmax(const double2 *__restrict__ g, size_t per_slab, const int *__restrict__ plist,
                              size_t i0, size_t i1, unsigned long long *out) {
    const int a = plist[blockIdx.y];   // a plane of the gather's region, its rows [i0, i1) / N2p
    const double2 *s = g + (size_t)a * per_slab;
    double m = 0.0;
    for (size_t i = i0 + blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < i1; i += (size_t)gridDim.x * blockDim.x) {
        const double2 v = s[i];
        m = fmax(m, cabsmax_naninf(v));   // NaN counts as +Inf
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(out + a, (unsigned long long)__double_as_longlong(m));
}

// the int8 gather's grid region (plan time): planes and padded rows its tiles'
// TMA boxes read (slab e0 of a tile with an odd chunk count is read with zero
// weights and needs no digits)
__global__ void k_gather_region(const Tile *__restrict__ tiles, int64_t n, WindowParams wp, int *planes,
                                int *rows) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const Tile t = tiles[i];
    for (int a = 0; a < t.e0; ++a) planes[wrap1(t.o0 + a, wp.N0)] = 1;
    atomicMin(rows, t.o1 + wp.pad);
    atomicMax(rows + 1, min(wp.N1p, t.o1 + wp.pad + kI8Box1));
}

// per tile: the shift of its largest slab (the tile's fixed-point reference)
__global__ void k_tile_shift(const Tile *__restrict__ tiles, int64_t n, WindowParams wp, const int *__restrict__ gsh,
                             int *__restrict__ tsh) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const Tile t = tiles[i];
    int m = NOSLAB;
    for (int a = 0; a < t.e0; ++a) m = min(m, gsh[wrap1(t.o0 + a, wp.N0)]);
    tsh[i] = m;
}

__global__ void k_slab_shift(const unsigned long long *__restrict__ mx, int n, int *__restrict__ sh,
                             int *__restrict__ nonfinite) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        sh[i] = slab_shift(mx[i]);
        if (!isfinite(__longlong_as_double((long long)mx[i]))) *nonfinite = 1;   // FP64 gather propagates it
    }
}

// Grid -> balanced byte digits: G 2^sG(a) = sum_j d_j 256^j, d_j in [-128, 127],
// layout [a][c / 16][j][b][re|im][c % 16] (zero beyond N2p): one K-chunk of one
// digit for a tile's 40 axis-1 cells is 1280 contiguous bytes, so a TMA box
// row is 1280 B (6 rows per box) instead of 480 rows of 16 B.  Thread = 4
// consecutive cells.
__global__ void k_slice_grid(const double2 *__restrict__ g, WindowParams wp, int ncb, const int *__restrict__ gsh,
                             const int *__restrict__ plist, int nplanes, int row0, int nrows,
                             uint8_t *__restrict__ dig) {
    // the gather's region only: planes plist[0 .. nplanes), rows row0 .. row0 + nrows
    const int64_t total = (int64_t)nplanes * ncb * nrows * 4;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int c4 = (int)(i & 3);
        int64_t r = i >> 2;
        const int b = row0 + (int)(r % nrows);
        r /= nrows;
        const int cb = (int)(r % ncb);
        const int a = plist[r / ncb];
        const int sh = gsh[a];
        // 2^sh in two factors: slabs below ~1e-290 need sh > 1023
        const int sh1 = min(sh, 960);
        const double sc = sh == NOSLAB ? 0.0 : ldexp(1.0, sh1), sc2 = sh == NOSLAB ? 0.0 : ldexp(1.0, sh - sh1);
        const double2 *row = g + ((size_t)a * wp.N1p + b) * wp.N2p;
        uint32_t w[ND][2] = {};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int c = cb * 16 + c4 * 4 + e;
            double2 v = make_double2(0.0, 0.0);
            if (c < wp.N2p) v = row[c];
#pragma unroll
            for (int ri = 0; ri < 2; ++ri) {
                const double y = fma((ri ? v.y : v.x) * sc2, sc, MAGIC);
                long long f = __double_as_longlong(y) - __double_as_longlong(MAGIC);   // rint(x 2^sG)
#pragma unroll
                for (int j = 0; j < ND; ++j) {
                    const long long d = (long long)(int8_t)(f & 0xff);   // balanced digit
                    w[j][ri] |= ((uint32_t)(uint8_t)d) << (8 * e);
                    f = (f - d) >> 8;
                }
            }
        }
        uint8_t *base = dig + (((size_t)a * ncb + cb) * ND * wp.N1p + b) * 32 + c4 * 4;
#pragma unroll
        for (int j = 0; j < ND; ++j) {
            *reinterpret_cast<uint32_t *>(base + (size_t)j * wp.N1p * 32) = w[j][0];
            *reinterpret_cast<uint32_t *>(base + (size_t)j * wp.N1p * 32 + 16) = w[j][1];
        }
    }
}

void i8_scales(const Plan &p, double &s0, double &s2, int &sA) {
    // A 2^sA = w0 w2 2^sA <= c0 c2 2^sA <= 2^46 (6 balanced bytes)
    const int e = (int)std::ceil(std::log2(p.wp.c0 * p.wp.c2));
    sA = 46 - e;
    const int a0 = sA / 2;
    s0 = std::ldexp(1.0, a0);
    s2 = std::ldexp(1.0, sA - a0);
}

}  // namespace

// The pruned FFT's axis-0 pass over the rows the window stages can touch:
// the region rows inside the interior, and the interior rows whose periodic
// images are the region's halo rows (k_halo_fill / k_halo_fold).  The FP64
// tiled gather (the guard's fallback) loads 36-row TMA boxes that may end up
// to a few rows past its nodes' windows; the region gets that margin.  Rows
// outside are never read by a window kernel after the forward and never
// written with nonzero values by the adjoint's spread, so their axis-0
// transforms are skipped (the adjoint's are transforms of zeros).
void setup_fft_rows(Plan &p) {
    const WindowParams &w = p.wp;
    // small grids: the extra cuFFT launches outweigh the skipped rows
    // (config 1, 128 x 128 x 64: 0.253 -> 0.271 ms per forward)
    if (!p.pruned || p.raw || p.grid_elems < ((size_t)1 << 24)) return;
    const int pad = w.pad, N1 = p.grid[1];
    const int g0 = std::max(0, p.grow0 - 4), g1 = std::min(w.N1p, p.grow1 + 4);
    std::vector<std::pair<int, int>> iv;
    auto add = [&](int a, int b) {
        a = std::max(a, pad);
        b = std::min(b, pad + N1);
        if (b > a) iv.emplace_back(a, b);
    };
    add(g0, g1);
    add(g0 + N1, std::min(g1, pad) + N1);            // images of the low halo rows
    add(std::max(g0, pad + N1) - N1, g1 - N1);      // images of the high halo rows
    std::sort(iv.begin(), iv.end());
    std::vector<std::pair<int, int>> m;
    for (auto &x : iv) {
        if (!m.empty() && x.first <= m.back().second) m.back().second = std::max(m.back().second, x.second);
        else m.push_back(x);
    }
    int rows = 0;
    for (auto &x : m) rows += x.second - x.first;
    if (m.empty() || m.size() > 3 || rows > N1 * 9 / 10) return;   // little to gain
    long long n1[1] = {p.grid[0]}, e1[1] = {p.grid[0]};
    const long long pl = (long long)w.N1p * w.N2p;
    size_t wfull = 0;
    cufftGetSize(p.fft1, &wfull);
    int k = 0;
    for (auto &x : m) {
        cufftHandle h = 0;
        size_t ws = 0;
        bool ok = cufftCreate(&h) == CUFFT_SUCCESS;
        ok = ok && cufftSetAutoAllocation(h, 0) == CUFFT_SUCCESS &&
             cufftMakePlanMany64(h, 1, n1, e1, pl, 1, e1, pl, 1, CUFFT_Z2Z, (long long)(x.second - x.first) * w.N2p,
                                 &ws) == CUFFT_SUCCESS &&
             ws <= wfull && cufftSetWorkArea(h, p.fft_work) == CUFFT_SUCCESS;
        if (!ok) {   // keep the full axis-0 pass
            if (h) cufftDestroy(h);
            for (int j = 0; j < k; ++j) cufftDestroy(p.fft1r[j]);
            p.n_fft1r = 0;
            cudaGetLastError();
            return;
        }
        p.fft1r[k] = h;
        p.fft1r_row0[k] = x.first;
        ++k;
    }
    p.n_fft1r = k;
}

int setup_i8(Plan &p) {
    const WindowParams &w = p.wp;
    if (p.n_itiles > 0) {
        TileStats ts;
        const int rc = tile_stats(p.itiles, p.n_itiles, 1, w, nullptr, &ts);
        if (rc) return rc;
        if (ts.bad) {
            set_error("internal: int8 gather tile outside its K range");
            return SGL_ECUDA;
        }
        p.i8_ksteps = ts.work;
    }
    p.P2 = (w.N2p + 15) / 16;   // 16-cell column blocks per row
    const size_t bytes = (size_t)w.N0 * p.P2 * ND * w.N1p * 32;
    // per slab: max bits (N0 x u64), shift (N0 x int); per tile: shift (n_itiles x int)
    if (cudaMalloc(&p.digits, bytes) != cudaSuccess ||
        cudaMalloc(&p.gmax, (sizeof(unsigned long long) + sizeof(int)) * w.N0 + sizeof(int) * (p.n_itiles + 1)) !=
            cudaSuccess) {
        // not enough memory for the grid digits (0.75x the grid): fall back to
        // the FP64 DMMA gather, which needs none
        cudaGetLastError();
        if (p.digits) cudaFree(p.digits);
        if (p.gmax) cudaFree(p.gmax);
        p.digits = nullptr;
        p.gmax = nullptr;
        p.i8 = false;
        p.i8s = false;
        return SGL_OK;
    }
    // the grid region the tiles read
    p.n_gplanes = 0;
    p.grow0 = 0;
    p.grow1 = 0;
    if (p.n_itiles > 0) {
        int *d = nullptr;
        SGL_CUDA_CHECK(cudaMalloc(&d, sizeof(int) * (w.N0 + 2)));
        std::vector<int> h(w.N0 + 2, 0);
        h[w.N0] = w.N1p;   // row min, row max
        SGL_CUDA_CHECK(cudaMemcpy(d, h.data(), sizeof(int) * (w.N0 + 2), cudaMemcpyHostToDevice));
        k_gather_region<<<(unsigned)((p.n_itiles + 255) / 256), 256>>>(p.itiles, p.n_itiles, w, d, d + w.N0);
        const cudaError_t e = cudaMemcpy(h.data(), d, sizeof(int) * (w.N0 + 2), cudaMemcpyDeviceToHost);
        cudaFree(d);
        SGL_CUDA_CHECK(e);
        std::vector<int> pl;
        for (int a = 0; a < w.N0; ++a)
            if (h[a]) pl.push_back(a);
        p.n_gplanes = (int)pl.size();
        p.grow0 = h[w.N0];
        p.grow1 = std::max(h[w.N0 + 1], h[w.N0]);
        SGL_CUDA_CHECK(cudaMalloc(&p.gplist, sizeof(int) * std::max<size_t>(1, pl.size())));
        if (!pl.empty())
            SGL_CUDA_CHECK(cudaMemcpy(p.gplist, pl.data(), sizeof(int) * pl.size(), cudaMemcpyHostToDevice));
        setup_fft_rows(p);
    }
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
    // 8-byte elements; dims (innermost first): (b, re|im, c % 16), digit, c / 16, a
    cuuint64_t dims[4] = {(cuuint64_t)4 * w.N1p, (cuuint64_t)ND, (cuuint64_t)p.P2, (cuuint64_t)w.N0};
    cuuint64_t strides[3] = {(cuuint64_t)32 * w.N1p, (cuuint64_t)ND * 32 * w.N1p,
                             (cuuint64_t)p.P2 * ND * 32 * w.N1p};
    cuuint32_t box[4] = {(cuuint32_t)(ROWS * 2), (cuuint32_t)ND, 1, 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = encode(&p.dmap, CU_TENSOR_MAP_DATA_TYPE_UINT64, 4, p.digits, dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        set_error("cuTensorMapEncodeTiled (digits) failed: " + std::to_string((int)r));
        return SGL_ECUDA;
    }
    return SGL_OK;
}

int launch_gather_i8(const Plan &p, const double2 *grid, double2 *values, cudaStream_t st) {
    if (p.M == 0) return SGL_OK;
    const int sms = num_sms();
    unsigned long long *mx = reinterpret_cast<unsigned long long *>(p.gmax);
    int *gsh = reinterpret_cast<int *>(mx + p.wp.N0);
    SGL_CUDA_CHECK(cudaMemsetAsync(mx, 0, sizeof(unsigned long long) * p.wp.N0, st));
    const size_t per_slab = (size_t)p.wp.N1p * p.wp.N2p;
    const int nrows = p.grow1 - p.grow0;
    const size_t region = (size_t)nrows * p.wp.N2p;   // slab elements the gather reads
    const unsigned bx = (unsigned)std::max<size_t>(1, std::min<size_t>(64, (region + 8191) / 8192));
    if (p.n_gplanes > 0 && nrows > 0)
        k_slab_absmax<<<dim3(bx, p.n_gplanes), 256, 0, st>>>(grid, per_slab, p.gplist, (size_t)p.grow0 * p.wp.N2p,
                                                             (size_t)p.grow1 * p.wp.N2p, mx);
    SGL_CUDA_CHECK(cudaGetLastError());
    k_slab_shift<<<(p.wp.N0 + 255) / 256, 256, 0, st>>>(mx, p.wp.N0, gsh, &p.guard->fwd);
    SGL_CUDA_CHECK(cudaGetLastError());
    if (p.n_gplanes > 0 && nrows > 0)   // P2 = column blocks
        k_slice_grid<<<sms * 16, 256, 0, st>>>(grid, p.wp, p.P2, gsh, p.gplist, p.n_gplanes, p.grow0, nrows, p.digits);
    SGL_CUDA_CHECK(cudaGetLastError());
    int *tsh = gsh + p.wp.N0;
    k_tile_shift<<<(unsigned)((p.n_itiles + 255) / 256), 256, 0, st>>>(p.itiles, p.n_itiles, p.wp, gsh, tsh);
    SGL_CUDA_CHECK(cudaGetLastError());
    double s0, s2;
    int sA;
    i8_scales(p, s0, s2, sA);
    const size_t sm = sizeof(I8Smem);
    unsigned long long *prof = p.prof;   // SGL_FLAG_I8_PROF: per-plan counters on the plan's device
    const bool want_prof = prof != nullptr;
    auto kern = want_prof ? k_gather_i8<true> : k_gather_i8<false>;
    SGL_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(p.n_itiles, sms));
    kern<<<(unsigned)blocks, IT, sm, st>>>(p.dmap, p.itiles, p.n_itiles, p.inodes, p.wp, s0, s2, sA, gsh,
                                                  tsh, values, prof, &p.guard->fwd);
    if (want_prof) {
        std::vector<unsigned long long> h(4 * blocks);
        cudaMemcpyAsync(h.data(), prof, sizeof(unsigned long long) * 4 * blocks, cudaMemcpyDeviceToHost, st);
        cudaStreamSynchronize(st);
        double tot = 0, a = 0, b = 0, e = 0, mn = 1e300, mx = 0;
        for (int i = 0; i < blocks; ++i) {
            mn = std::min(mn, (double)h[4 * i]);
            mx = std::max(mx, (double)h[4 * i]);
            tot += h[4 * i];
            a += h[4 * i + 1];
            b += h[4 * i + 2];
            e += h[4 * i + 3];
        }
        fprintf(stderr,
                "i8 MMA warp: total %.0f cycles/CTA (min %.0f, max %.0f), wait fullA %.1f%%, fullB %.1f%%, tempty %.1f%%\n",
                tot / blocks, mn, mx, 100 * a / tot, 100 * b / tot, 100 * e / tot);
    }
    SGL_CUDA_CHECK(cudaGetLastError());
    return SGL_OK;
}

}  // namespace sgl
