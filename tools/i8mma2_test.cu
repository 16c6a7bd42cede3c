// tcgen05.mma.cta_group::2 kind::i8 check and throughput probe (sm_100a): a CTA
// pair (cluster of 2) computes D[256 x N] = A[256 x K] * B[N x K]^T with A split
// by rows (CTA r holds rows 128 r ..) and B split by rows of B = columns of D
// (CTA r holds B rows r N/2 .. (r+1) N/2 - 1), both K-major interleave at the
// same shared-memory offsets; the leader CTA issues the MMA; each CTA reads its
// 128 x N half of D from its own TMEM.
//   1. correctness against a host int64 reference;
//   2. throughput: back-to-back MMAs (K = 32) on resident operands, every SM
//      pair, N in {80, 160, 240, 256}.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/i8mma2_test tools/i8mma2_test.cu
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <cuda_runtime.h>

#include "../paper_1809_10786_b200/csrc/umma.cuh"

using namespace sgl;

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(umma::smem_addr(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t ok = 0;
    while (!ok) {
        asm volatile(
            "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(ok)
            : "r"(umma::smem_addr(bar)), "r"(parity)
            : "memory");
    }
}
__device__ __forceinline__ uint32_t cta_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void mma2(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, bool acc) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"((uint32_t)acc));
}
__device__ __forceinline__ void commit2(uint64_t *bar) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
            umma::smem_addr(bar)),
        "h"((uint16_t)3)
        : "memory");
}
__device__ __forceinline__ void alloc2(uint32_t *dst, uint32_t cols) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(umma::smem_addr(dst)),
                 "r"(cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void free2(uint32_t base, uint32_t cols) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(base), "r"(cols) : "memory");
}

// A: 256 x K, B: N x K (row-major int8 in global); D: 256 x N int32
__global__ void __cluster_dims__(2, 1, 1) k_check2(const int8_t *A, const int8_t *B, int32_t *D, int K, int N,
                                                   int reps) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t rank = cta_rank();
    const int NH = N / 2;
    uint8_t *sA = sm;
    uint8_t *sB = sm + 128 * K;
    const uint32_t lboA = 128 * 16, lboB = NH * 16;
    for (int i = tid; i < 128 * K; i += blockDim.x) {
        int r = i / K, k = i % K;
        sA[(k / 16) * lboA + (r / 8) * 128 + (r % 8) * 16 + (k % 16)] = (uint8_t)A[(128 * rank + r) * K + k];
    }
    for (int i = tid; i < NH * K; i += blockDim.x) {
        int r = i / K, k = i % K;
        sB[(k / 16) * lboB + (r / 8) * 128 + (r % 8) * 16 + (k % 16)] = (uint8_t)B[(NH * rank + r) * K + k];
    }
    if (tid == 0) {
        mbar_init(&bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (warp == 0) alloc2(&tbase, 512);
    umma::fence_async_smem();
    umma::fence_before();
    __syncthreads();
    cluster_sync();   // both CTAs' operands written, barriers initialised
    umma::fence_after();
    const uint32_t td = tbase;
    long long t0 = clock64();
    if (rank == 0 && tid == 0) {
        const uint32_t id = umma::idesc_i8(256, N, true, true);
        if (reps == 1) {
            for (int kb = 0; kb < K / 32; ++kb) {
                uint64_t da = umma::desc_kmajor(umma::smem_addr(sA) + kb * 2 * lboA, lboA, 128);
                uint64_t db = umma::desc_kmajor(umma::smem_addr(sB) + kb * 2 * lboB, lboB, 128);
                mma2(td, da, db, id, kb > 0);
            }
        } else {   // rate: accumulate into two alternating D halves, 4 MMAs per iteration
            const uint64_t da = umma::desc_kmajor(umma::smem_addr(sA), lboA, 128);
            const uint64_t db = umma::desc_kmajor(umma::smem_addr(sB), lboB, 128);
            for (int r = 0; r < reps; r += 4) {
#pragma unroll
                for (int u = 0; u < 4; ++u) mma2(td + (u & 1) * 256, da, db, id, true);
            }
        }
        commit2(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    umma::fence_after();
    if (D) {
        for (int c = 0; c < N; c += 16) {
            int32_t v[16];
            umma::tmem_ld16(td + ((uint32_t)(warp * 32) << 16) + c, v);
            umma::tmem_ld_wait();
            for (int j = 0; j < 16; ++j)
                if (c + j < N) D[(128 * rank + warp * 32 + lane) * N + c + j] = v[j];
        }
    } else if (rank == 0 && tid == 0 && blockIdx.x == 0) {
        printf("N=%d: %.1f cycles per MMA (M=256 pair, K=32)\n", N, (double)(t1 - t0) / (reps * (K / 32)));
    }
    umma::fence_before();
    __syncthreads();
    cluster_sync();
    if (warp == 0) free2(td, 512);
}

int main() {
    const int K = 96;
    for (int N : {80, 160, 240, 256}) {
        std::vector<int8_t> A(256 * K), B(N * K);
        srand(1 + N);
        for (auto &x : A) x = (int8_t)(rand() % 256 - 128);
        for (auto &x : B) x = (int8_t)(rand() % 256 - 128);
        int8_t *dA, *dB;
        int32_t *dD;
        cudaMalloc(&dA, A.size());
        cudaMalloc(&dB, B.size());
        cudaMalloc(&dD, 256 * N * 4);
        cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
        cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
        const size_t sm = 128 * K + (N / 2) * K;
        cudaFuncSetAttribute(k_check2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        k_check2<<<2, 128, sm>>>(dA, dB, dD, K, N, 1);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<int32_t> D(256 * N);
        cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
        long bad = 0;
        for (int r = 0; r < 256; ++r)
            for (int c = 0; c < N; ++c) {
                long long s = 0;
                for (int k = 0; k < K; ++k) s += (long long)A[r * K + k] * B[c * K + k];
                if (s != D[r * N + c]) ++bad;
            }
        printf("check N=%d: %s, %ld mismatches of %d\n", N, cudaGetErrorString(e), bad, 256 * N);
        // throughput: every SM pair, operands resident, 4096 MMAs of K = 32
        const int Kt = 32;
        const size_t smt = 128 * Kt + (N / 2) * Kt;
        k_check2<<<148, 128, smt>>>(dA, dB, nullptr, Kt, N, 4096);
        e = cudaDeviceSynchronize();
        if (e != cudaSuccess) printf("throughput run: %s\n", cudaGetErrorString(e));
        cudaFree(dA);
        cudaFree(dB);
        cudaFree(dD);
    }
    return 0;
}
