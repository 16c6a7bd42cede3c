// Gaussian-window scatter (adjoint NFFT spreading, _gridding.py:77-95) on the
// int8 tensor cores (tcgen05.mma kind::i8) with FP64 results by the same
// exact byte-digit split as the gather (gather_i8.cu).  sm_100a.
//
// Per tile of <= 512 sorted nodes (one 8 x 16 pencil, consecutive in lo0) and
// its box of e0 x 40 x 48 cells, the spreading sum
//     G[a,b,c] += sum_n w0[n,a] w1[n,b] w2[n,c] v[n]
// is a GEMM with K = nodes: per M-block of 128 box cells (a, c),
//     D[(a,c), (b,re|im)] = sum_n W[(a,c), n] V[n, (b,re|im)],
//     W = w0 (x) w2 (weights, fixed point at the plan scale sA),
//     V = w1 v      (fixed point at a per-tile scale from the tile's max |v|),
// both split into 6 balanced bytes; the 21 digit pairs with p + q >= 5 in 9
// MMAs per K-step of 32 nodes (W digit p times V digits stacked along N),
// int32 diagonal accumulators in TMEM (6 x 80 columns).
//
// V does not depend on the M-block: two value-digit warps build a tile's
// digits once, one tile ahead, into the CTA's slot of a small ring in global
// memory (2 x 240 KB per CTA, L2-resident), already in the MN-major UMMA
// layout of a K-step (15 KB per 32 nodes), and a producer warp streams them
// into shared memory with 1-D bulk copies (cp.async.bulk) per M-block.  Only W is built on the fly, by 16 generator warps (node x
// 16-cell group, weights from per-node factors in shared memory), stored with
// st.async.  The epilogue converts an M-block to FP64 into a per-thread
// staging column, frees TMEM for the next block's MMAs and only then reduces
// the block into the halo-padded grid with RED.E.ADD.F64 (k_halo_fold folds
// the halo as for the FP64 scatter).  512-node tiles keep the REDs at ~300
// per node.
//
// CTA (one per SM, persistent, cluster of 1 for st.async): warp 0 MMA
// issuer, warp 1 value-digit producer, warps 2-17 weight-digit generators (two
// groups of 8 on alternating K-steps), warps 18-25 epilogue (two per TMEM lane
// quarter = cells, half the columns each), warps 26-27 value-digit generators.
#include <cuda_runtime.h>

#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "i8_common.cuh"
#include "sgl_internal.cuh"
#include "umma.cuh"

namespace sgl {
namespace {

using namespace i8;


static_assert(kI8SNodes <= 512, "combine6_i64 needs at most 512 nodes per tile");

constexpr int SN = kI8SNodes;            // nodes per tile (K)
constexpr int MR = 128;                  // box cells per M-block (MMA M)
constexpr int ROWS = 2 * kI8Box1;        // MMA N per digit: (b, re|im) = 80
constexpr int NGRP = 2;                  // generator groups, alternating K-steps (group = ring stage)
constexpr int NSTG = 3;                  // weight-digit ring (K-steps of 32 nodes): 1.5 stages per generator group
constexpr int NSTGB = 3;                 // value-digit ring
constexpr int KST = 32;                  // nodes per K-step
constexpr int A_DIGIT = (KST / 8) * 8 * 128;   // 4 node blocks x 8 cell blocks x 128 B (MN-major)
constexpr int A_STAGE = ND * A_DIGIT;
constexpr int B_KBLK = ND * (ROWS / 16) * 128;   // one 8-node block of all 6 value digits
constexpr int B_STAGE = (KST / 8) * B_KBLK;      // one K-step of value digits (global and smem layout)
constexpr int NWG = 8 * NGRP;            // weight generator warps (per group: 32 nodes x 8 cell groups)
constexpr int NEW = 8;                   // epilogue warps: EPW per TMEM lane quarter, 1/EPW of the columns each
constexpr int EPW = NEW / 4;
#ifndef SGL_NVW
#define SGL_NVW 2
#endif
constexpr int NVW = SGL_NVW;                   // value-digit generator warps (warp = K-step, lane = node)
constexpr int VSLOTS = 2;                // value-digit slots per CTA in global memory (tile parity)
constexpr int V_SLOT = (SN / KST) * B_STAGE;   // one tile's value digits (16 K-steps, 240 KB)
#ifndef SGL_VAHEAD
#define SGL_VAHEAD 7
#endif
constexpr int VAHEAD = SGL_VAHEAD;       // the next tile's value digits are built during the last VAHEAD M-blocks
constexpr int ST = (2 + NWG + NEW + NVW) * 32;

struct SSmem {
    uint8_t a[NSTG][A_STAGE];    // weight digits [digit][node/8][cell/16][node%8][cell%16]
    uint8_t b[NSTGB][B_STAGE];   // value digits  [node/8][digit][col/16][node%8][col%16]
    long long stage[ROWS - 4 * EPW][MR];   // epilogue: one M-block as exact int64 sums, [column][cell]; each
                                 // warp's last 4 columns stay in its registers
    double e2[CHUNKS][SN], f2[SN];   // W2 of chunk cc: w(cb + j) = e2[cc] (f2 kf[cc])^j exp(-h2 j^2)
    int win2[SN];                // axis-2 window relative to K column 0: lo | hi << 16 (signed)
    double w0t[4][SN];           // W0 of the current M-block's (<= 4) slabs, row = slab & 3
    uint64_t fullA[NSTG], emptyA[NSTG], fullB[NSTGB], emptyB[NSTGB];
    uint64_t tfull, tempty;
    uint64_t vready[VSLOTS], vfree[VSLOTS];   // a tile's value digits written / all its MMAs done
    uint64_t vgo;                             // the MMA warp is VAHEAD M-blocks from the tile's end
    uint32_t tbase;
};

struct K3 {
    double v[CHUNKS];   // exp(-32 h2 cc): chunk cc's ratio f2 of chunk 0's
};

struct G16 {
    double v[16];
    __device__ __forceinline__ double operator[](int j) const { return v[j]; }
};

__device__ __forceinline__ void gen_sync() { asm volatile("bar.sync 1, %0;\n" ::"n"(NWG * 32) : "memory"); }

__device__ __forceinline__ void red_add(double *addr, double v) {
    asm volatile("red.global.add.f64 [%0], %1;\n" ::"l"(addr), "d"(v) : "memory");
}


// SGL_FLAG_DETERMINISTIC: 64-bit fixed-point reduction (order-independent)
__device__ __forceinline__ void red_add_s64(double *addr, long long v) {
    asm volatile("red.global.add.u64 [%0], %1;\n" ::"l"(addr), "l"(v) : "memory");
}

// x 2^s rounded to an integer (s < 0: round half up by an arithmetic shift)
__device__ __forceinline__ long long fix_shift(long long x, int s) {
    if (s >= 0) return x << min(s, 62);
    if (s < -62) return 0;
    return (x + (1ll << (-s - 1))) >> (-s);
}

__device__ __forceinline__ void st_async_v4(void *dst, const uint32_t (&v)[4], uint64_t *bar) {
    asm volatile(
        "st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];\n" ::"r"(
            umma::smem_addr(dst)),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(umma::smem_addr(bar))
        : "memory");
}

// L2 policy of the value-digit ring (written once per tile, re-read per
// M-block): evict_last against the grid's RED stream, which otherwise pushes a
// tile's digits out to DRAM between their write and their reads (config 3:
// DRAM 3.3 + 4.6 GB per launch without the hint, 2.8 + 2.9 GB with it;
// evict_first on the REDs as well: no further gain)
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(p));
    return p;
}

__device__ __forceinline__ void bulk_load(void *dst, const void *src, uint32_t bytes, uint64_t *bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;\n" ::
            "r"(umma::smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(umma::smem_addr(bar)), "l"(pol)
        : "memory");
}

__device__ __forceinline__ void st_keep_v4(void *dst, uint32_t a, uint32_t b, uint32_t c, uint32_t d, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v4.b32 [%0], {%1, %2, %3, %4}, %5;\n" ::"l"(dst), "r"(a), "r"(b), "r"(c),
                 "r"(d), "l"(pol)
                 : "memory");
}

__device__ __forceinline__ int mblocks(const Tile &t) { return (t.e0 * CHUNKS * 16 + MR - 1) / MR; }
__device__ __forceinline__ int ksteps(const Tile &t) { return (t.count + KST - 1) / KST; }

// value digits of one K-step of a tile: lane = node of the K-step, walking all
// 40 axis-1 cells (the Gaussian recurrence runs on across the 5 16-column
// groups: one exp pair per node), written in the K-step's MN-major UMMA layout
__device__ __forceinline__ void vdigits_kstep(const Tile &t, int svt, int ks, int kl, const NodeSet &nodes,
                                              const WindowParams &wp, const double2 *__restrict__ values,
                                              uint8_t *__restrict__ blk, uint64_t pol) {
    // 2^svt as 2^min(svt, 960) on the digit split and the rest on the value
    // first: values below ~1e-290 need svt > 1023 (r02 fix: the one-factor
    // scale overflowed to Inf), and the pre-scaled value keeps w1 v normal
    const int svt1 = min(svt, 960);
    const double vsc = svt == NOSLAB ? 0.0 : ldexp(1.0, svt1);
    const double vsc2 = svt == NOSLAB ? 0.0 : ldexp(1.0, svt - svt1);
    const int kn = ks * KST + kl;
    const bool live = kn < t.count;
    const int64_t si = (int64_t)t.start + kn;
    const double u1 = live ? nodes.u1[si] : -1e9;
    SGL_DCHECK(!live || (si < nodes.n && nodes.perm[si] >= 0 && nodes.perm[si] < nodes.n));
    double2 vv = live ? values[nodes.perm[si]] : make_double2(0.0, 0.0);
    vv.x *= vsc2;
    vv.y *= vsc2;
    int lo1, hi1;
    window_cells(u1, wp.q, lo1, hi1);
    const int bf = max(0, lo1 - t.o1);   // first window cell, relative to the box
    const double d = u1 - (double)(t.o1 + bf);
    double w = wp.c1 * exp(-d * d * wp.h1), r = exp(wp.h1 * (2.0 * d - 1.0));
    uint8_t *dst = blk + (kl >> 3) * B_KBLK + (kl & 7) * 16;
#pragma unroll 1
    for (int vg = 0; vg < ROWS / 16; ++vg) {
        double wv[16];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int b = vg * 8 + j;
            const double w1 = (live && b >= bf && t.o1 + b <= hi1) ? w : 0.0;
            if (b >= bf) {
                w *= r;
                r *= wp.r1_1;
            }
            wv[2 * j] = w1 * vv.x;
            wv[2 * j + 1] = w1 * vv.y;
        }
        uint32_t dw[ND][4];
        digits16(vsc, wv, dw);
#pragma unroll
        for (int q = 0; q < ND; ++q)
            st_keep_v4(dst + vg * 128 + q * (ROWS / 16) * 128, dw[q][0], dw[q][1], dw[q][2], dw[q][3], pol);
    }
}

template <bool P>
__device__ __forceinline__ long long tick() {
    if constexpr (P) return clock64();
    else return 0;
}

// PROF: clock64 wait counters (SGL_FLAG_I8_PROF); compiled out otherwise.
// DET: SGL_FLAG_DETERMINISTIC -- the exact per-tile int64 sums are shifted to
// the call's fixed-point unit 2^-E (*det) and reduced as integers (determ.cu)
template <bool PROF, bool DET>
__global__ void __cluster_dims__(1, 1, 1) __launch_bounds__(ST, 1)
    k_scatter_i8(const Tile *__restrict__ tiles, int64_t ntiles, NodeSet nodes, WindowParams wp, double s0,
                 double s2, int sA, const int *__restrict__ tsv, const double2 *__restrict__ values,
                 uint8_t *__restrict__ vring, double *__restrict__ grid, const G16 g2, const K3 kf,
                 unsigned long long *__restrict__ prof, const int *__restrict__ skip,
                 const int *__restrict__ det) {
    if (*skip) return;   // non-finite values (guard.cu)
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    SSmem &S = *reinterpret_cast<SSmem *>(smem_raw);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

    if (tid == 0) {
        for (int s = 0; s < NSTG; ++s) {
            mbar_init(&S.fullA[s], 1);   // one expect_tx arrive + the st.async bytes
            mbar_init(&S.emptyA[s], 1);
        }
        for (int s = 0; s < NSTGB; ++s) {
            mbar_init(&S.fullB[s], 1);
            mbar_init(&S.emptyB[s], 1);
        }
        mbar_init(&S.tfull, 1);
        mbar_init(&S.tempty, NEW);
        for (int s = 0; s < VSLOTS; ++s) {
            mbar_init(&S.vready[s], NVW * 32);
            mbar_init(&S.vfree[s], 1);
        }
        mbar_init(&S.vgo, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (warp == 0) umma::tmem_alloc(&S.tbase, TCOLS);
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    const uint32_t tbase = S.tbase;

    if (warp == 0) {
        // ---- MMA issuer
        const uint64_t a0 = umma::desc_kmajor(umma::smem_addr(S.a[0]), 1024, 128);      // MN-major: LBO = node
        const uint64_t b0 = umma::desc_kmajor(umma::smem_addr(S.b[0]), B_KBLK, 128);    // block, SBO = 16 rows
        constexpr uint32_t MN = (1u << 15) | (1u << 16);                                // A, B MN-major
        uint32_t g = 0, mc = 0;
        int stgb = 0;            // value ring slot and phase, stepped (NSTGB is not a power of 2)
        uint32_t phb = 0;
        long long q0 = tick<PROF>(), qa = 0, qb = 0, qe = 0;
        uint32_t tj = 0;         // this CTA's tile counter (value-digit slot = tj % VSLOTS)
        for (int64_t ti = blockIdx.x; ti < ntiles; ti += gridDim.x, ++tj) {
            const Tile t = tiles[ti];
            const int nmb = mblocks(t), nks = ksteps(t);
            for (int mb = 0; mb < nmb; ++mb, ++mc) {
                long long x0 = tick<PROF>();
                if (mc) mbar_wait(&S.tempty, (mc - 1) & 1);
                qe += tick<PROF>() - x0;
                umma::fence_after();
                for (int ks = 0; ks < nks; ++ks, ++g) {
                    const int stg = (int)(g % NSTG);
                    long long x1 = tick<PROF>();
                    mbar_wait(&S.fullB[stgb], phb);
                    // start the value warps on the next tile's digits: late enough that
                    // the digits are still in L2 at their first read, early enough to be
                    // done.  After this tile's first value digits have arrived, i.e. after
                    // the value warps consumed the previous tile's vgo phase (short tiles
                    // trigger at M-block 0: an arrive before that wait could complete two
                    // phases ahead of the value warps' parity wait)
                    if (ks == 0 && mb == max(0, nmb - VAHEAD) && lane == 0) mbar_arrive(&S.vgo);
                    long long x2 = tick<PROF>();
                    mbar_wait(&S.fullA[stg], (g / NSTG) & 1);
                    qa += tick<PROF>() - x2;
                    qb += x2 - x1;
                    umma::fence_after();
                    if (umma::elect_one()) {
                        const uint64_t ad = a0 + (uint64_t)(stg * (A_STAGE >> 4));
                        const uint64_t bd = b0 + (uint64_t)(stgb * (B_STAGE >> 4));
                        const bool acc = ks > 0;
#define SGL_I8S_OP(P, Q0, NQ, ACC)                                                                         \
    umma::mma_i8(tbase + (uint32_t)(((P) + (Q0)-DMIN) * ROWS), ad + (uint64_t)((P)*A_DIGIT >> 4),         \
                 bd + (uint64_t)((Q0) * (ROWS / 16) * 128 >> 4), umma::idesc_i8(MR, (NQ)*ROWS, true, true) | MN, \
                 ACC)
                        // the two p = 5 MMAs cover every accumulator and carry the per-block reset
                        SGL_I8S_OP(5, 0, 3, acc);
                        SGL_I8S_OP(5, 3, 3, acc);
                        SGL_I8S_OP(4, 1, 3, true);
                        SGL_I8S_OP(4, 4, 2, true);
                        SGL_I8S_OP(3, 2, 3, true);
                        SGL_I8S_OP(3, 5, 1, true);
                        SGL_I8S_OP(2, 3, 3, true);
                        SGL_I8S_OP(1, 4, 2, true);
                        SGL_I8S_OP(0, 5, 1, true);
#undef SGL_I8S_OP
                        umma::commit(&S.emptyA[stg]);
                        umma::commit(&S.emptyB[stgb]);
                    }
                    __syncwarp();
                    if (++stgb == NSTGB) {
                        stgb = 0;
                        phb ^= 1;
                    }
                }
                if (umma::elect_one()) umma::commit(&S.tfull);
                __syncwarp();
            }
            // every bulk copy of the tile's value digits has landed and been read:
            // its slot may be overwritten (by the tile after next)
            if (umma::elect_one()) umma::commit(&S.vfree[tj % VSLOTS]);
            __syncwarp();
        }
        if (PROF && prof && lane == 0) {
            prof[blockIdx.x * 8 + 0] = tick<PROF>() - q0;
            prof[blockIdx.x * 8 + 1] = qa;
            prof[blockIdx.x * 8 + 2] = qb;
            prof[blockIdx.x * 8 + 3] = qe;
        }
    } else if (warp == 1) {
        // ---- value-digit producer: one bulk copy per K-step (re-read from L2 per M-block)
        if (lane == 0) {
            const uint64_t pol = policy_evict_last();
            uint32_t g = 0;
            int pstg = 0;        // ring slot and the phase of its current use
            uint32_t pph = 0;
            uint32_t tj = 0;
            for (int64_t ti = blockIdx.x; ti < ntiles; ti += gridDim.x, ++tj) {
                const Tile t = tiles[ti];
                const int nmb = mblocks(t), nks = ksteps(t);
                const int slot = (int)(tj % VSLOTS);
                const uint8_t *src = vring + ((size_t)blockIdx.x * VSLOTS + slot) * V_SLOT;
                mbar_wait(&S.vready[slot], (tj / VSLOTS) & 1);   // written + fenced by the value warps
                for (int mb = 0; mb < nmb; ++mb)
                    for (int ks = 0; ks < nks; ++ks, ++g) {
                        if (g >= (uint32_t)NSTGB) mbar_wait(&S.emptyB[pstg], pph ^ 1);   // its previous use
                        mbar_expect_tx(&S.fullB[pstg], B_STAGE);
                        bulk_load(S.b[pstg], src + ks * (int64_t)B_STAGE, B_STAGE, &S.fullB[pstg], pol);
                        if (++pstg == NSTGB) {
                            pstg = 0;
                            pph ^= 1;
                        }
                    }
            }
        }
    } else if (warp < 2 + NWG) {
        // ---- weight-digit generators: thread = (node of the K-step, 16-cell group);
        // lanes 0-7 take 8 consecutive nodes (each 16-byte store row of a warp
        // covers all 32 banks)
        const int gt = tid - 64, hg = gt >> 8, wi = (gt >> 5) & 7;
        const int kl = (wi & 3) * 8 + (lane & 7), grp = (wi >> 2) * 4 + (lane >> 3);
        uint32_t g = 0;
        long long q0 = tick<PROF>(), qe = 0, qt = 0, qw = 0;
        for (int64_t ti = blockIdx.x; ti < ntiles; ti += gridDim.x) {
            const Tile t = tiles[ti];
            const long long x0 = tick<PROF>();
            gen_sync();   // the previous tile's readers of the node tables are done
            const int kst = kstart2(t, wp) - wp.pad;   // cell of K-range column 0 (axis 2)
            const int kcount = ksteps(t) * KST;
            // axis-0 Gaussian walk of this thread's node (thread gt owns node gt: SN == NWG * 32):
            // W0 of its next slab, the ratio, its window in tile slabs (lo | hi << 16, signed)
            static_assert(SN <= NWG * 32, "one generator thread per node of the tile");
            double w0s = 0.0, r0s = 0.0;
            int win0 = 0x7fff | (-1 << 16);
            for (int i = gt; i < kcount; i += NWG * 32) {
                // per node: axis-0 coordinate, axis-2 window and the W2 factors of
                // the three 16-cell chunks (2 exps per chunk here, none per K-step);
                // the padding nodes of the last K-step get zero weights
                const bool live = i < t.count;
                const int64_t si = (int64_t)t.start + (live ? i : 0);
                const double u2 = nodes.u2[si];
                int lo2, hi2;
                window_cells(u2, wp.q, lo2, hi2);
                S.win2[i] = ((lo2 - kst) & 0xffff) | ((hi2 - kst) << 16);
                // W0 walk from the node's first window cell: w(c + 1) = w(c) r, r <- r e^{-2 h0}
                const double u0 = nodes.u0[si];
                int lo0, hi0;
                window_cells(u0, wp.q, lo0, hi0);
                lo0 = max(lo0, t.o0);   // (the box covers the window; kept for safety)
                const double d0 = u0 - (double)lo0;
                w0s = s0 * (wp.c0 * exp(-d0 * d0 * wp.h0));
                r0s = exp(wp.h0 * (2.0 * d0 - 1.0));
                if (live) win0 = ((lo0 - t.o0) & 0xffff) | ((hi0 - t.o0) << 16);
#pragma unroll
                for (int cc = 0; cc < CHUNKS; ++cc) {
                    const double d = u2 - (double)(kst + 16 * cc);
                    S.e2[cc][i] = live ? s2 * (wp.c2 * exp(-d * d * wp.h2)) : 0.0;
                }
                S.f2[i] = exp(2.0 * wp.h2 * (u2 - (double)kst));
            }
            gen_sync();
            qt += tick<PROF>() - x0;
            const int nmb = mblocks(t), nks = ksteps(t);
            int nxt = 0;   // next slab of the W0 walk
            for (int mb = 0; mb < nmb; ++mb) {
                const long long x1 = tick<PROF>();
                // W0 of the slabs this M-block adds (slabs a_mb .. a_mb + 3, each
                // computed once per tile, in order, by the walk; zero beyond e0)
                const int a_mb = (mb * 8) / CHUNKS;
                if (nxt <= a_mb + 3) {
                    gen_sync();   // the readers of the rows being replaced are done
                    for (int n = gt; n < kcount; n += NWG * 32) {
                        const int lo = (int)(short)(win0 & 0xffff), hi = win0 >> 16;
                        double w = w0s, r = r0s;
                        for (int x = nxt; x <= a_mb + 3; ++x) {
                            double v = 0.0;
                            if (x >= lo && x <= hi && x < t.e0) {
                                v = w;
                                w *= r;
                                r *= wp.r0_1;
                            }
                            S.w0t[x & 3][n] = v;
                        }
                        w0s = w;
                        r0s = r;
                    }
                    nxt = a_mb + 4;
                    gen_sync();
                }
                qw += tick<PROF>() - x1;
                const int cid = mb * 8 + grp, al = cid / CHUNKS, cc = cid - CHUNKS * al;
                // this thread's node tables for the M-block (padding nodes have e = 0)
                const double *w0p = S.w0t[al & 3] + kl, *e2p = S.e2[cc] + kl, *f2p = S.f2 + kl;
                const double kfc = kf.v[cc];
                const int *win2p = S.win2 + kl;
                // this group's K-steps of the M-block only (global K-step g0 + ks; a
                // strided loop instead of skipping the other group's: 29.19 -> 29.08 ms)
                const uint32_t g0 = g;
                g += nks;
                for (int ks = (int)(((uint32_t)hg + NGRP - g0 % NGRP) % NGRP); ks < nks; ks += NGRP) {
                    const uint32_t gk = g0 + ks;
                    const int stg = (int)(gk % NSTG);
                    const uint32_t use = gk / NSTG;
                    const int kn = ks * KST;
                    // W0 folded into the chunk factor: w0 w2(cb + j) = (w0 e) f^j g_j, so
                    // the g_j product is the digit FMA itself (one DMUL per entry fewer;
                    // scatter 29.67 -> 29.56 ms at config 3)
                    const double e = w0p[kn] * e2p[kn], f = f2p[kn] * kfc;
                    const int wn = win2p[kn], jlo = (int)(short)(wn & 0xffff) - 16 * cc, jhi = (wn >> 16) - 16 * cc;
                    // the node's window [jlo, jhi] inside this 16-cell chunk as an entry mask
                    const uint32_t mask = (jhi < 0 || jlo > 15)
                                              ? 0u
                                              : ((2u << min(15, jhi)) - 1u) & ~((1u << max(0, jlo)) - 1u);
                    uint32_t dw[ND][4];
                    // powers of f by a depth-4 product tree
                    double pw[16];
                    pw[0] = e;
                    pw[1] = e * f;
                    const double f2 = f * f, f4 = f2 * f2, f8 = f4 * f4;
                    pw[2] = e * f2;
                    pw[3] = pw[1] * f2;
                    pw[4] = e * f4;
                    pw[5] = pw[1] * f4;
                    pw[6] = pw[2] * f4;
                    pw[7] = pw[3] * f4;
#pragma unroll
                    for (int j = 8; j < 16; ++j) pw[j] = pw[j - 8] * f8;
                    digits16_masked(pw, g2.v, mask, dw);
                    const long long x2 = tick<PROF>();
                    if (use) mbar_wait(&S.emptyA[stg], (use - 1) & 1);
                    qe += tick<PROF>() - x2;
                    if ((gt & 255) == 0) mbar_expect_tx(&S.fullA[stg], A_STAGE);
                    uint8_t *dst = S.a[stg] + (kl >> 3) * 1024 + grp * 128 + (kl & 7) * 16;
#pragma unroll
                    for (int p = 0; p < ND; ++p) st_async_v4(dst + p * A_DIGIT, dw[p], &S.fullA[stg]);
                }
            }
        }
        if (PROF && prof && gt == 0) {
            prof[blockIdx.x * 8 + 4] = tick<PROF>() - q0;
            prof[blockIdx.x * 8 + 5] = qe;
            prof[blockIdx.x * 8 + 6] = qt;
            prof[blockIdx.x * 8 + 7] = qw;
        }
    } else if (warp >= 2 + NWG + NEW) {
        // ---- value-digit generators: V = w1 v does not depend on the M-block, so a
        // tile's digits are written once, during the previous tile's last M-blocks, into this CTA's slot of
        // an L2-resident ring in global memory (2 x 240 KB per CTA) and re-read
        // from there per M-block by the producer's bulk copies.  Generic-proxy
        // writes -> async-proxy reads: fence.proxy.async by every writer before
        // its arrive on vready.
        const int vw = warp - (2 + NWG + NEW);
        const uint64_t pol = policy_evict_last();
        uint32_t tj = 0;
        for (int64_t ti = blockIdx.x; ti < ntiles; ti += gridDim.x, ++tj) {
            const Tile t = tiles[ti];
            const int slot = (int)(tj % VSLOTS);
            if (tj >= 1) mbar_wait(&S.vgo, (tj - 1) & 1);   // one arrive per tile: tile tj - 1 is near its end
            if (tj >= (uint32_t)VSLOTS) mbar_wait(&S.vfree[slot], (tj / VSLOTS - 1) & 1);
            const int svt = __ldg(tsv + ti);
            uint8_t *dst = vring + ((size_t)blockIdx.x * VSLOTS + slot) * V_SLOT;
            for (int ks = vw; ks < ksteps(t); ks += NVW)
                vdigits_kstep(t, svt, ks, lane, nodes, wp, values, dst + (size_t)ks * B_STAGE, pol);
            asm volatile("fence.proxy.async;\n" ::: "memory");
            mbar_arrive(&S.vready[slot]);
            // the previous tile's digits are dead once all its MMAs are done: drop
            // their (dirty) L2 lines instead of letting them be written back to DRAM
            if (tj >= 1) {
                const int ps = (int)((tj - 1) % VSLOTS);
                mbar_wait(&S.vfree[ps], ((tj - 1) / VSLOTS) & 1);
                const Tile pt = tiles[ti - gridDim.x];
                uint8_t *old = vring + ((size_t)blockIdx.x * VSLOTS + ps) * V_SLOT;
                for (int o = (vw * 32 + lane) * 128; o < ksteps(pt) * B_STAGE; o += NVW * 32 * 128)
                    asm volatile("discard.global.L2 [%0], 128;\n" ::"l"(old + o) : "memory");
                // the next tile's digits go to the same slot, and a line is written by
                // other threads than the one that discards it: order every discard before
                // every such write (short tiles start them back to back; found by
                // tools/soak.py as 1e-2 errors on 2e5-node plans with q <= 8)
                __threadfence_block();
                asm volatile("bar.sync 2, %0;\n" ::"n"(NVW * 32) : "memory");
            }
        }
    } else {
        // ---- epilogue: thread = box cell of the M-block = TMEM lane
        const int quarter = warp & 3, m = quarter * 32 + lane, eh = (warp - 2 - NWG) >> 2;
        const uint32_t tl = tbase + ((uint32_t)(quarter * 32) << 16);
        uint32_t mc = 0;
        for (int64_t ti = blockIdx.x; ti < ntiles; ti += gridDim.x) {
            const Tile t = tiles[ti];
            const int nmb = mblocks(t);
            const int sv = __ldg(tsv + ti);
            const double unit = sv == NOSLAB ? 0.0 : ldexp(1.0, 8 * DMIN - sA - sv);
            // DET: this tile's shift to the call's unit (E == kDetOff cannot reach
            // here: non-finite values skip the kernel)
            const int dsh = DET ? 8 * DMIN - sA - sv + *det : 0;
            const int kst = kstart2(t, wp);   // padded axis-2 cell of K column 0
            const int c_in0 = t.o2 + wp.pad - kst, c_in1 = c_in0 + t.e2;
            for (int mb = 0; mb < nmb; ++mb, ++mc) {
                const int cell = mb * MR + m, al = cell / (CHUNKS * 16), cl = cell - al * CHUNKS * 16;
                const bool inbox = al < t.e0 && cl >= c_in0 && cl < c_in1;
                double *gp = grid + 2 * (((size_t)wrap1(t.o0 + (inbox ? al : 0), wp.N0) * wp.N1p + (t.o1 + wp.pad)) *
                                             wp.N2p + (kst + cl));
                mbar_wait(&S.tfull, mc & 1);
                umma::fence_after();
                // software-pipelined drain, 4 columns (2 axis-1 cells x re|im) per step:
                // the TMEM loads of step i+1 are in flight while step i converts
                constexpr int CB4 = ROWS / 4 / EPW;   // 4-column steps of this warp
                const int c0 = eh * CB4;
                constexpr int SROWS = (CB4 - 1) * 4;   // staged columns of this warp
                int32_t D[2][NBLK][4];
                long long keep[4];
                __syncwarp();   // tcgen05.ld is .sync.aligned
#pragma unroll
                for (int k = 0; k < NBLK; ++k) umma::tmem_ld4(tl + (uint32_t)(k * ROWS + c0 * 4), D[0][k]);
                umma::tmem_ld_wait();
#pragma unroll
                for (int i = 0; i < CB4; ++i) {
                    const int cur = i & 1;
                    if (i + 1 < CB4) {
#pragma unroll
                        for (int k = 0; k < NBLK; ++k)
                            umma::tmem_ld4(tl + (uint32_t)(k * ROWS + (c0 + i + 1) * 4), D[cur ^ 1][k]);
                    }
                    // the exact int64 only: its conversion to FP64 waits until after
                    // the TMEM release (scatter 29.73 -> 29.29 ms at config 3)
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const long long x = combine6_i64(D[cur][0][j], D[cur][1][j], D[cur][2][j], D[cur][3][j],
                                                         D[cur][4][j], D[cur][5][j]);
                        if (i + 1 < CB4) S.stage[eh * SROWS + i * 4 + j][m] = x;
                        else keep[j] = x;   // the last step stays in registers (8 KB of staging less)
                    }
                    umma::tmem_ld_wait();
                }
                umma::fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&S.tempty);   // TMEM free: the next block's MMAs overlap the REDs
                if (inbox) {
                    // one axis-1 cell (re, im) of this thread's grid column
                    auto emit = [&](int b, long long sre, long long sim) {
                        double *q = gp + 2 * (size_t)b * wp.N2p;
                        SGL_DCHECK(wrap1(t.o0 + al, wp.N0) < wp.N0 && t.o1 + wp.pad + b < wp.N1p &&
                                   kst + cl >= 0 && kst + cl < wp.N2p);
                        if (DET) {
                            if (sv == NOSLAB) return;
                            const long long xr = fix_shift(sre, dsh);
                            const long long xi = fix_shift(sim, dsh);
                            if (xr != 0) red_add_s64(q, xr);
                            if (xi != 0) red_add_s64(q + 1, xi);
                        } else {
                            const double re = (double)sre * unit;
                            const double im = (double)sim * unit;
                            if (re != 0.0) red_add(q, re);
                            if (im != 0.0) red_add(q + 1, im);
                        }
                    };
                    constexpr int BW = ROWS / 2 / EPW;   // axis-1 cells of this warp: BW - 2 staged, 2 in registers
                    const int b0 = eh * BW;
                    for (int lb = 0; lb < min(t.e1 - b0, BW - 2); ++lb)
                        emit(b0 + lb, S.stage[eh * SROWS + 2 * lb][m], S.stage[eh * SROWS + 2 * lb + 1][m]);
                    if (b0 + BW - 2 < t.e1) emit(b0 + BW - 2, keep[0], keep[1]);
                    if (b0 + BW - 1 < t.e1) emit(b0 + BW - 1, keep[2], keep[3]);
                }
            }
        }
    }

    umma::fence_before();
    __syncthreads();
    if (warp == 0) {
        __syncwarp();
        umma::fence_after();
        umma::tmem_free(tbase, TCOLS);
    }
}

// per tile: value scale from the tile's max |Re v|, |Im v| (|w1 v| 2^sV < 2^46, w1 <= c1)
__global__ void k_tile_vscale(const Tile *__restrict__ tiles, int64_t n, NodeSet nodes,
                              const double2 *__restrict__ values, double c1, int *__restrict__ tsv,
                              int *__restrict__ nonfinite) {
    const int64_t ti = blockIdx.x;
    if (ti >= n) return;
    const Tile t = tiles[ti];
    double m = 0.0;
    for (int i = threadIdx.x; i < t.count; i += blockDim.x) {
        const double2 v = values[nodes.perm[(int64_t)t.start + i]];
        m = fmax(m, cabsmax_naninf(v));   // NaN counts as +Inf
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    __shared__ double wm[8];
    if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = fmax(m, wm[w]);
        m = fmax(m, wm[0]) * c1;
        int ex;
        frexp(m, &ex);
        tsv[ti] = (m > 0.0 && isfinite(m)) ? 46 - ex : NOSLAB;
        if (!isfinite(m)) *nonfinite = 1;   // the FP64 scatter propagates NaN / Inf (guard.cu)
    }
}

}  // namespace

int setup_scatter_i8(Plan &p) {
    const WindowParams &w = p.wp;
    if (p.n_istiles > 0) {
        TileStats ts;
        const int rc = tile_stats(p.istiles, p.n_istiles, 2, w, nullptr, &ts);
        if (rc) return rc;
        if (ts.bad) {
            set_error("internal: int8 scatter tile outside its K range");
            return SGL_ECUDA;
        }
        p.i8_sksteps = ts.work;
    }
    // value-digit ring: VSLOTS tiles of digits per CTA (73 MB at 148 CTAs, L2-resident),
    // independent of the node count; on an allocation failure stay on the FP64 scatter
    const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(p.n_istiles, num_sms()));
    const size_t need = (size_t)blocks * VSLOTS * V_SLOT;
    if (cudaMalloc(&p.tsv, sizeof(int) * (p.n_istiles + 1)) != cudaSuccess ||
        cudaMalloc(&p.vdig, need) != cudaSuccess) {
        cudaGetLastError();
        for (void *b : {(void *)p.tsv, (void *)p.vdig, (void *)p.istiles})
            if (b) cudaFree(b);
        p.tsv = nullptr;
        p.vdig = nullptr;
        p.istiles = nullptr;
        p.n_istiles = 0;
        p.i8_sksteps = 0;
        p.i8s = false;   // FP64 scatter (as setup_i8 does for the gather)
        return SGL_OK;
    }
    return SGL_OK;
}

int launch_scatter_i8(const Plan &p, const double2 *values, double2 *grid, cudaStream_t st) {
    if (p.M == 0 || p.n_istiles == 0) return SGL_OK;
    int *skip = &p.guard->adj;
    k_tile_vscale<<<(unsigned)p.n_istiles, 256, 0, st>>>(p.istiles, p.n_istiles, p.inodes, values, p.wp.c1, p.tsv,
                                                         skip);
    SGL_CUDA_CHECK(cudaGetLastError());
    const int sms = num_sms();
    const int e = (int)std::ceil(std::log2(p.wp.c0 * p.wp.c2));
    const int sA = 46 - e, a0 = sA / 2;
    const size_t sm = sizeof(SSmem);
    unsigned long long *prof = p.prof;   // SGL_FLAG_I8_PROF: per-plan counters on the plan's device
    const bool want = prof != nullptr;
    const int *det = p.det_e();
    auto kern = want ? (det ? k_scatter_i8<true, true> : k_scatter_i8<true, false>)
                     : (det ? k_scatter_i8<false, true> : k_scatter_i8<false, false>);
    SGL_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(p.n_istiles, sms));
    G16 g2;
    for (int j = 0; j < 16; ++j) g2.v[j] = std::exp(-p.wp.h2 * (double)(j * j));
    K3 kf;
    for (int cc = 0; cc < CHUNKS; ++cc) kf.v[cc] = std::exp(-32.0 * p.wp.h2 * (double)cc);
    kern<<<(unsigned)blocks, ST, sm, st>>>(p.istiles, p.n_istiles, p.inodes, p.wp, std::ldexp(1.0, a0),
                                                  std::ldexp(1.0, sA - a0), sA, p.tsv, values, p.vdig,
                                                  reinterpret_cast<double *>(grid), g2, kf, prof, skip, det);
    SGL_CUDA_CHECK(cudaGetLastError());
    if (want) {   // SGL_I8_PROF=1: where the MMA warp waits (debug)
        std::vector<unsigned long long> h(8 * blocks);
        cudaMemcpyAsync(h.data(), prof, sizeof(unsigned long long) * 8 * blocks, cudaMemcpyDeviceToHost, st);
        cudaStreamSynchronize(st);
        double tot = 0, a = 0, b = 0, e = 0, gt = 0, ge = 0, gtab = 0, gw0 = 0;
        for (int64_t i = 0; i < blocks; ++i) {
            tot += h[8 * i];
            a += h[8 * i + 1];
            b += h[8 * i + 2];
            e += h[8 * i + 3];
            gt += h[8 * i + 4];
            ge += h[8 * i + 5];
            gtab += h[8 * i + 6];
            gw0 += h[8 * i + 7];
        }
        fprintf(stderr, "i8 scatter generator warp: %.0f cycles/CTA, wait emptyA %.1f%%, node tables %.1f%%, W0 %.1f%%\n",
                gt / blocks, 100 * ge / gt, 100 * gtab / gt, 100 * gw0 / gt);
        fprintf(stderr, "i8 scatter MMA warp: %.0f cycles/CTA, wait weights %.1f%%, values %.1f%%, TMEM drain %.1f%%\n",
                tot / blocks, 100 * a / tot, 100 * b / tot, 100 * e / tot);
    }
    return SGL_OK;
}

}  // namespace sgl
