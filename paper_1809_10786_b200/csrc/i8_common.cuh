// Device helpers shared by the int8 tensor-core window kernels (gather_i8.cu,
// scatter_i8.cu): mbarriers, TMA, digit constants, slab scales, K ranges.
#pragma once

#include <cuda.h>
#include <stdint.h>

#include "sgl_internal.cuh"
#include "umma.cuh"

namespace sgl {
namespace i8 {

constexpr int ND = 6;                     // byte digits per operand
constexpr int DMIN = 5;                   // kept digit diagonals p + q = DMIN .. 2 ND - 2
constexpr int NBLK = 2 * ND - 1 - DMIN;   // 6 TMEM accumulators
constexpr int CHUNKS = kI8Box2 / 16;      // 16-cell K-chunks per slab
constexpr uint32_t TCOLS = 512;
constexpr double MAGIC = 6755399441055744.0;   // 1.5 * 2^52: fma(x, y, MAGIC) rounds x y to an integer
// + 128 in each of the 6 digit bytes: the bytes of fma(x, y, MAGIC_BAL) are
// the balanced digits of rint(x y) (|.| < 2^46) offset by 128 (undone by ^ 0x80)
constexpr double MAGIC_BAL = 6755399441055744.0 + 141289400074368.0;
constexpr int NOSLAB = 4096;   // shift of an all-zero slab (never the tile minimum)

__device__ __forceinline__ int wrapi(int i, int n) {
    i %= n;
    return i < 0 ? i + n : i;
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(umma::smem_addr(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(umma::smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(umma::smem_addr(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity, int tag = 0) {
    (void)tag;
    uint32_t ok = 0, spins = 0;
    for (;;) {
        asm volatile(
            "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(ok)
            : "r"(umma::smem_addr(bar)), "r"(parity)
            : "memory");
        if (ok) return;
        if (++spins == (1u << 26)) __trap();   // lost phase: trap instead of hanging the GPU
    }
}
__device__ __forceinline__ void tma_load_4d(void *dst, const CUtensorMap *map, int c0, int c1, int c2, int c3,
                                            uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
        "[%6];\n" ::"r"(umma::smem_addr(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(umma::smem_addr(bar))
        : "memory");
}

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t s) {
    uint32_t r;
    asm("prmt.b32 %0, %1, %2, %3;\n" : "=r"(r) : "r"(a), "r"(b), "r"(s));
    return r;
}

// digit shift of a slab from its max |G| (bits of a non-negative double):
// |G| 2^sG < 2^46
__device__ __forceinline__ int slab_shift(unsigned long long bits) {
    const double m = __longlong_as_double((long long)bits);
    if (!(m > 0.0) || !isfinite(m)) return NOSLAB;
    int ex;
    frexp(m, &ex);   // m < 2^ex
    return 46 - ex;
}

// 2^e for e <= 0 (0 below 2^-1022)
__device__ __forceinline__ double pow2n(int e) {
    return e < -1022 ? 0.0 : __longlong_as_double((long long)(e + 1023) << 52);
}

// slab index modulo N0 for boxes that start at most one period out
__device__ __forceinline__ int wrap1(int a, int n) {
    a += a < 0 ? n : 0;
    return a >= n ? a - n : a;
}

// First padded axis-2 cell of a slab's K range: the TMA box start of the
// innermost dimension must be 16-byte aligned (measured: unaligned starts
// fault with an illegal instruction), so the 48-cell K range starts at the
// 16-aligned cell at or below the box origin; 16-aligned pencils with
// pad == q <= 16 keep every window inside it (checked at plan time).
__host__ __device__ __forceinline__ int kstart2(const Tile &t, const WindowParams &wp) {
    return (t.o2 + wp.pad) & ~15;
}


// 16 fixed-point entries y_e = fma(w0, w[e], MAGIC_BAL) -> their 6 balanced
// digit planes, 16 bytes each (4 words per digit: entries 4j .. 4j+3)
__device__ __forceinline__ void digits16(double w0, const double (&w)[16], uint32_t (&dw)[ND][4]) {
#pragma unroll
    for (int q4 = 0; q4 < 4; ++q4) {
        uint32_t L[4], H[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const double y = fma(w0, w[q4 * 4 + e], MAGIC_BAL);
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
}

// 16 entries y_e = fma(a[e], b[e], MAGIC_BAL) -> digit planes as digits16,
// with an entry mask (bit e: entry e inside the node's window): the bytes of
// masked-out entries are cleared with the same LOP3 that rebalances the
// digits, instead of a compare + select per entry on the FP64 inputs (outside
// the window the weights are finite, smaller than inside, and their digits
// are discarded)
__device__ __forceinline__ void digits16_masked(const double (&a)[16], const double (&b)[16], uint32_t mask16,
                                                uint32_t (&dw)[ND][4]) {
#pragma unroll
    for (int q4 = 0; q4 < 4; ++q4) {
        uint32_t L[4], H[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const double y = fma(a[q4 * 4 + e], b[q4 * 4 + e], MAGIC_BAL);
            L[e] = (uint32_t)__double2loint(y);
            H[e] = (uint32_t)__double2hiint(y);
        }
        const uint32_t bm = ((((mask16 >> (4 * q4)) & 0xfu) * 0x00204081u) & 0x01010101u) * 0xffu;
        const uint32_t t0 = prmt(L[0], L[1], 0x5140), t1 = prmt(L[2], L[3], 0x5140);
        const uint32_t t2 = prmt(L[0], L[1], 0x7362), t3 = prmt(L[2], L[3], 0x7362);
        const uint32_t h0 = prmt(H[0], H[1], 0x5140), h1 = prmt(H[2], H[3], 0x5140);
        dw[0][q4] = (prmt(t0, t1, 0x5410) ^ 0x80808080u) & bm;
        dw[1][q4] = (prmt(t0, t1, 0x7632) ^ 0x80808080u) & bm;
        dw[2][q4] = (prmt(t2, t3, 0x5410) ^ 0x80808080u) & bm;
        dw[3][q4] = (prmt(t2, t3, 0x7632) ^ 0x80808080u) & bm;
        dw[4][q4] = (prmt(h0, h1, 0x5410) ^ 0x80808080u) & bm;
        dw[5][q4] = (prmt(h0, h1, 0x7632) ^ 0x80808080u) & bm;
    }
}

// the 6 diagonal accumulators of one column, D_k weighted 256^k, as one exact
// int64 in units of 256^DMIN (converted once by the caller).  |operands| <
// 2^46 in balanced digits: the scatter's sums of <= 512 products are bounded
// by 2^(92 + 9 - 40) = 2^61; the gather's by 2^(92 + 10.1 - 40) since a node's
// weights are nonzero on at most (2q + 1)^2 <= 33^2 cells (q <= kMaxQTiled)
__device__ __forceinline__ long long combine6_i64(int32_t d0, int32_t d1, int32_t d2, int32_t d3, int32_t d4,
                                                  int32_t d5) {
    // the sum fits an int64, so wrapping arithmetic is exact: three
    // IMAD.WIDE for the low diagonals, d4 + 256 d5 added to the high word
    // modulo 2^32 (no carry chains)
    long long x = (long long)d0 + (long long)d1 * 256;
    x += (long long)d2 * 65536;
    x += (long long)d3 * 16777216;
    const uint32_t hadd = (uint32_t)d4 + ((uint32_t)d5 << 8);
    const uint32_t lo = (uint32_t)x, hi = (uint32_t)((unsigned long long)x >> 32) + hadd;
    return (long long)(((unsigned long long)hi << 32) | lo);
}

}  // namespace i8
}  // namespace sgl
