// tcgen05.mma kind::i8 check and throughput probe (sm_100a).
//   1. correctness: D[128 x N] = A[128 x K] (u8 / s8) * B[N x K]^T (u8 / s8), K-major
//      interleave layouts built by threads, D read back from TMEM, compared on the host;
//   2. throughput: one CTA per SM issuing back-to-back MMAs on resident operands
//      (M = 128, N in {80, 256}, K = 32), int8 TOPS.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/i8mma_test tools/i8mma_test.cu
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

// A: 128 x K, B: N x K (row-major int8 in global); D: 128 x N int32
__global__ void k_check(const int8_t *A, const int8_t *B, int32_t *D, int K, int N, int as, int bs) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    uint8_t *sA = sm;
    uint8_t *sB = sm + 128 * K;
    const uint32_t lboA = 128 * 16, lboB = N * 16;
    for (int i = tid; i < 128 * K; i += blockDim.x) {
        int r = i / K, k = i % K;
        sA[(k / 16) * lboA + (r / 8) * 128 + (r % 8) * 16 + (k % 16)] = (uint8_t)A[i];
    }
    for (int i = tid; i < N * K; i += blockDim.x) {
        int r = i / K, k = i % K;
        sB[(k / 16) * lboB + (r / 8) * 128 + (r % 8) * 16 + (k % 16)] = (uint8_t)B[i];
    }
    if (tid == 0) {
        mbar_init(&bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (warp == 0) umma::tmem_alloc(&tbase, 256);
    umma::fence_async_smem();
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    const uint32_t td = tbase;
    if (tid == 0) {
        const uint32_t id = umma::idesc_i8(128, N, as != 0, bs != 0);
        for (int kb = 0; kb < K / 32; ++kb) {
            uint64_t da = umma::desc_kmajor(umma::smem_addr(sA) + kb * 2 * lboA, lboA, 128);
            uint64_t db = umma::desc_kmajor(umma::smem_addr(sB) + kb * 2 * lboB, lboB, 128);
            umma::mma_i8(td, da, db, id, kb > 0);
        }
        umma::commit(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    umma::fence_after();
    for (int c = 0; c < N; c += 16) {
        int32_t v[16];
        umma::tmem_ld16(td + ((uint32_t)(warp * 32) << 16) + c, v);
        umma::tmem_ld_wait();
        for (int j = 0; j < 16; ++j)
            if (c + j < N) D[(warp * 32 + lane) * N + c + j] = v[j];
    }
    umma::fence_before();
    __syncthreads();
    if (warp == 0) umma::tmem_free(td, 256);
}

// MN-major (no swizzle) operands: element (mn, k) at (mn / 16) * SBO + (k / 8) * LBO + (k % 8) * 16 + mn % 16
__global__ void k_check_mn(const int8_t *A, const int8_t *B, int32_t *D, int K, int N) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    uint8_t *sA = sm;
    uint8_t *sB = sm + 128 * K;
    // A: SBO = 128 B (next 16 rows), LBO = 16 * 128 = 2048 B (next 8 K)
    const uint32_t sboA = 128, lboA = 128 / 16 * 128, sboB = 128, lboB = N / 16 * 128;
    for (int i = tid; i < 128 * K; i += blockDim.x) {
        int r = i / K, k = i % K;
        sA[(r / 16) * sboA + (k / 8) * lboA + (k % 8) * 16 + r % 16] = (uint8_t)A[i];
    }
    for (int i = tid; i < N * K; i += blockDim.x) {
        int r = i / K, k = i % K;
        sB[(r / 16) * sboB + (k / 8) * lboB + (k % 8) * 16 + r % 16] = (uint8_t)B[i];
    }
    if (tid == 0) {
        mbar_init(&bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (warp == 0) umma::tmem_alloc(&tbase, 256);
    umma::fence_async_smem();
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    const uint32_t td = tbase;
    if (tid == 0) {
        const uint32_t id = umma::idesc_i8(128, N, true, true) | (1u << 15) | (1u << 16);   // A, B MN-major
        for (int kb = 0; kb < K / 32; ++kb) {
            uint64_t da = umma::desc_kmajor(umma::smem_addr(sA) + kb * 4 * lboA, lboA, sboA);
            uint64_t db = umma::desc_kmajor(umma::smem_addr(sB) + kb * 4 * lboB, lboB, sboB);
            umma::mma_i8(td, da, db, id, kb > 0);
        }
        umma::commit(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    umma::fence_after();
    for (int c = 0; c < N; c += 16) {
        int32_t v[16];
        umma::tmem_ld16(td + ((uint32_t)(warp * 32) << 16) + c, v);
        umma::tmem_ld_wait();
        for (int j = 0; j < 16; ++j)
            if (c + j < N) D[(warp * 32 + lane) * N + c + j] = v[j];
    }
    umma::fence_before();
    __syncthreads();
    if (warp == 0) umma::tmem_free(td, 256);
}

// A from TMEM: thread m writes its row (K bytes, 4 per 32-bit column) with
// tcgen05.st.32x32b.x8 (32 bytes = one K-step per store) at columns [col_a + 8 kb ...)
__global__ void k_check_ts(const int8_t *A, const int8_t *B, int32_t *D, int K, int N) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    uint8_t *sB = sm;
    const uint32_t lboB = N * 16;
    for (int i = tid; i < N * K; i += blockDim.x) {
        int r = i / K, k = i % K;
        sB[(k / 16) * lboB + (r / 8) * 128 + (r % 8) * 16 + (k % 16)] = (uint8_t)B[i];
    }
    if (tid == 0) {
        mbar_init(&bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (warp == 0) umma::tmem_alloc(&tbase, 512);
    umma::fence_async_smem();
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    const uint32_t td = tbase, ta = tbase + 256;
    // row m = tid: K bytes -> K / 4 words
    for (int kb = 0; kb < K / 32; ++kb) {
        uint32_t w[8];
        for (int j = 0; j < 8; ++j) {
            uint32_t x = 0;
            for (int b = 0; b < 4; ++b) x |= (uint32_t)(uint8_t)A[tid * K + kb * 32 + j * 4 + b] << (8 * b);
            w[j] = x;
        }
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(
                         ta + ((uint32_t)(warp * 32) << 16) + kb * 8),
                     "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7])
                     : "memory");
    }
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    if (tid == 0) {
        const uint32_t id = umma::idesc_i8(128, N, true, true);
        for (int kb = 0; kb < K / 32; ++kb) {
            uint64_t db = umma::desc_kmajor(umma::smem_addr(sB) + kb * 2 * lboB, lboB, 128);
            asm volatile(
                "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(td),
                "r"(ta + kb * 8), "l"(db), "r"(id), "r"((uint32_t)(kb > 0)));
        }
        umma::commit(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    umma::fence_after();
    for (int c = 0; c < N; c += 16) {
        int32_t v[16];
        umma::tmem_ld16(td + ((uint32_t)(warp * 32) << 16) + c, v);
        umma::tmem_ld_wait();
        for (int j = 0; j < 16; ++j)
            if (c + j < N) D[(warp * 32 + lane) * N + c + j] = v[j];
    }
    umma::fence_before();
    __syncthreads();
    if (warp == 0) umma::tmem_free(td, 512);
}

// throughput: each CTA issues iters x (K/32) MMAs on its resident operands
__global__ void k_rate(int K, int N, int iters, int32_t *sink) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < (128 + N) * K; i += blockDim.x) sm[i] = (uint8_t)(i * 7);
    if (tid == 0) {
        mbar_init(&bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (warp == 0) umma::tmem_alloc(&tbase, 512);
    umma::fence_async_smem();
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    const uint32_t td = tbase;
    const uint32_t lboA = 128 * 16, lboB = N * 16;
    if (tid == 0) {
        const uint32_t id = umma::idesc_i8(128, N, false, true);
        for (int it = 0; it < iters; ++it)
            for (int kb = 0; kb < K / 32; ++kb) {
                uint64_t da = umma::desc_kmajor(umma::smem_addr(sm) + kb * 2 * lboA, lboA, 128);
                uint64_t db = umma::desc_kmajor(umma::smem_addr(sm + 128 * K) + kb * 2 * lboB, lboB, 128);
                umma::mma_i8(td + (it & 1) * 256, da, db, id, true);
            }
        umma::commit(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    umma::fence_after();
    int32_t v[16];
    umma::tmem_ld16(td + ((uint32_t)(warp * 32) << 16), v);
    umma::tmem_ld_wait();
    if (v[0] == 12345) sink[tid] = v[1];
    umma::fence_before();
    __syncthreads();
    if (warp == 0) umma::tmem_free(td, 512);
}

// rate with a given descriptor layout: lay 0 = interleave (LBO = M*16), 1 = interleave with LBO + 16,
// 2 = SW128 K-major (SBO 1024, K advance 32 B), 3 = SW32 K-major (SBO 256)
__global__ void k_rate2(int N, int iters, int lay, int32_t *sink) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < 96 * 1024; i += blockDim.x) sm[i] = (uint8_t)(i * 7);
    if (tid == 0) {
        mbar_init(&bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (warp == 0) umma::tmem_alloc(&tbase, 512);
    umma::fence_async_smem();
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    const uint32_t td = tbase;
    const uint32_t sa = umma::smem_addr(sm), sb = umma::smem_addr(sm + 32768);
    if (tid == 0) {
        const uint32_t id = umma::idesc_i8(128, N, true, true);
        uint64_t da, db;
        uint32_t kadv_a, kadv_b;
        if (lay == 0 || lay == 1 || lay == 5) {
            const uint32_t ex = lay == 1 ? 16 : 0;
            da = umma::desc_kmajor(sa, 128 * 16 + ex, 128);
            db = umma::desc_kmajor(sb, N * 16 + ex, 128);
            kadv_a = 2 * (128 * 16 + ex);
            kadv_b = 2 * (N * 16 + ex);
        } else if (lay == 2) {
            da = umma::desc_kmajor(sa, 16, 1024) | ((uint64_t)2 << 61);
            db = umma::desc_kmajor(sb, 16, 1024) | ((uint64_t)2 << 61);
            kadv_a = kadv_b = 32;
        } else if (lay == 3) {
            da = umma::desc_kmajor(sa, 16, 256) | ((uint64_t)6 << 61);
            db = umma::desc_kmajor(sb, 16, 256) | ((uint64_t)6 << 61);
            kadv_a = 128 * 32;
            kadv_b = N * 32;
        } else {
            // MN-major interleave: SBO = 128 (next 16 MN), LBO = next 8 K
            da = umma::desc_kmajor(sa, 1024, 128);
            db = umma::desc_kmajor(sb, N / 16 * 128, 128);
            kadv_a = 4 * 1024;
            kadv_b = 4 * (N / 16 * 128);
        }
        const uint32_t idm = lay == 4 ? (id | (1u << 15) | (1u << 16)) : id;
        if (lay == 5) {   // A from TMEM (columns 256 + 8 kb), B interleave K-major
            for (int it = 0; it < iters; ++it)
#pragma unroll
                for (int kb = 0; kb < 4; ++kb)
                    umma::mma_i8_ts(td, td + 256 + 8 * kb, db + ((kb * kadv_b) >> 4), idm, true);
        } else
        for (int it = 0; it < iters; ++it)
#pragma unroll
            for (int kb = 0; kb < 4; ++kb)
                umma::mma_i8(td + (it & 1) * 256, da + ((kb * kadv_a) >> 4), db + ((kb * kadv_b) >> 4), idm, true);
        umma::commit(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    umma::fence_after();
    int32_t v[16];
    umma::tmem_ld16(td + ((uint32_t)(warp * 32) << 16), v);
    umma::tmem_ld_wait();
    if (v[0] == 12345) sink[tid] = v[1];
    umma::fence_before();
    __syncthreads();
    if (warp == 0) umma::tmem_free(td, 512);
}

int main() {
    int bad = 0;
    const int K = 96;
    for (int N : {80, 16, 256}) {
        for (int as = 0; as < 2; ++as)
            for (int bs = 0; bs < 2; ++bs) {
                std::vector<int8_t> A(128 * K), B(N * K);
                std::vector<int32_t> D(128 * N), R(128 * N);
                srand(1 + N + 2 * as + bs);
                for (auto &x : A) x = (int8_t)(rand() & 255);
                for (auto &x : B) x = (int8_t)(rand() & 255);
                for (int m = 0; m < 128; ++m)
                    for (int n = 0; n < N; ++n) {
                        long s = 0;
                        for (int k = 0; k < K; ++k) {
                            int a = as ? (int)A[m * K + k] : (int)(uint8_t)A[m * K + k];
                            int b = bs ? (int)B[n * K + k] : (int)(uint8_t)B[n * K + k];
                            s += a * b;
                        }
                        R[m * N + n] = (int32_t)s;
                    }
                int8_t *dA, *dB;
                int32_t *dD;
                cudaMalloc(&dA, A.size());
                cudaMalloc(&dB, B.size());
                cudaMalloc(&dD, D.size() * 4);
                cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
                cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
                cudaMemset(dD, 0, D.size() * 4);
                size_t smem = (128 + N) * K;
                cudaFuncSetAttribute(k_check, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                k_check<<<1, 128, smem>>>(dA, dB, dD, K, N, as, bs);
                cudaError_t e = cudaDeviceSynchronize();
                cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
                int nbad = 0;
                for (int i = 0; i < 128 * N; ++i) nbad += D[i] != R[i];
                printf("check N=%d a_signed=%d b_signed=%d: %s, %d mismatches (D[0]=%d ref %d)\n", N, as, bs,
                       cudaGetErrorString(e), nbad, D[0], R[0]);
                bad += nbad != 0 || e != cudaSuccess;
                cudaFree(dA);
                cudaFree(dB);
                cudaFree(dD);
            }
    }
    for (int N : {80, 160, 240}) {
        const int KK = 128;
        std::vector<int8_t> A(128 * KK), B(N * KK);
        std::vector<int32_t> D(128 * N), R(128 * N);
        srand(7 + N);
        for (auto &x : A) x = (int8_t)(rand() & 255);
        for (auto &x : B) x = (int8_t)(rand() & 255);
        for (int m = 0; m < 128; ++m)
            for (int n = 0; n < N; ++n) {
                long sacc = 0;
                for (int k = 0; k < KK; ++k) sacc += (int)A[m * KK + k] * (int)B[n * KK + k];
                R[m * N + n] = (int32_t)sacc;
            }
        int8_t *dA, *dB;
        int32_t *dD;
        cudaMalloc(&dA, A.size());
        cudaMalloc(&dB, B.size());
        cudaMalloc(&dD, D.size() * 4);
        cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
        cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
        size_t smem = (128 + N) * KK;
        cudaFuncSetAttribute(k_check_mn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_check_mn<<<1, 128, smem>>>(dA, dB, dD, KK, N);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
        int nbad = 0;
        for (int i = 0; i < 128 * N; ++i) nbad += D[i] != R[i];
        printf("check MN-major N=%d: %s, %d mismatches (D[0]=%d ref %d)\n", N, cudaGetErrorString(e), nbad, D[0], R[0]);
        bad += nbad != 0 || e != cudaSuccess;
    }
    for (int N : {64, 128, 256}) {
        const int KK = 96;
        std::vector<int8_t> A(128 * KK), B(N * KK);
        std::vector<int32_t> D(128 * N), R(128 * N);
        srand(17 + N);
        for (auto &x : A) x = (int8_t)(rand() & 255);
        for (auto &x : B) x = (int8_t)(rand() & 255);
        for (int m = 0; m < 128; ++m)
            for (int n = 0; n < N; ++n) {
                long sacc = 0;
                for (int k = 0; k < KK; ++k) sacc += (int)A[m * KK + k] * (int)B[n * KK + k];
                R[m * N + n] = (int32_t)sacc;
            }
        int8_t *dA, *dB;
        int32_t *dD;
        cudaMalloc(&dA, A.size());
        cudaMalloc(&dB, B.size());
        cudaMalloc(&dD, D.size() * 4);
        cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
        cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
        size_t smem = N * KK;
        cudaFuncSetAttribute(k_check_ts, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_check_ts<<<1, 128, smem>>>(dA, dB, dD, KK, N);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
        int nbad = 0;
        for (int i = 0; i < 128 * N; ++i) nbad += D[i] != R[i];
        printf("check A-in-TMEM N=%d: %s, %d mismatches (D[0]=%d ref %d)\n", N, cudaGetErrorString(e), nbad, D[0], R[0]);
        bad += nbad != 0 || e != cudaSuccess;
        if (e != cudaSuccess) return 1;
    }
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int32_t *sink;
    cudaMalloc(&sink, 4096);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int N : {80, 128, 256})
        for (int Kr : {32, 128}) {
            size_t smem = (128 + N) * Kr;
            cudaFuncSetAttribute(k_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            int iters = 20000 * 32 / Kr;
            k_rate<<<sms, 128, smem>>>(Kr, N, 100, sink);
            cudaEventRecord(e0);
            k_rate<<<sms, 128, smem>>>(Kr, N, iters, sink);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            double ops = 2.0 * 128 * N * Kr * (double)iters * sms;
            printf("rate M=128 N=%d K/issue-block=%d: %.1f int8 TOPS (%.3f ms) %s\n", N, Kr, ops / ms / 1e9, ms,
                   cudaGetErrorString(cudaGetLastError()));
        }
    for (int lay = 0; lay < 6; lay += (lay == 0 ? 4 : 1))
        for (int N : {80, 160, 240, 256}) {
            if (lay == 5 && N == 256) continue;   // D (N columns) + A (32 columns) within 512
            cudaFuncSetAttribute(k_rate2, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
            const int iters = 5000;
            k_rate2<<<sms, 128, 96 * 1024>>>(N, 100, lay, sink);
            cudaEventRecord(e0);
            k_rate2<<<sms, 128, 96 * 1024>>>(N, iters, lay, sink);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double mmas = 4.0 * iters;
            printf("layout %d N=%d: %.1f cycles/MMA at 1.9 GHz, %.0f TOPS %s\n", lay, N, ms * 1e-3 * 1.9e9 / mmas,
                   2.0 * 128 * N * 32 * mmas * sms / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
        }
    printf(bad ? "FAIL\n" : "PASS\n");
    return bad;
}
