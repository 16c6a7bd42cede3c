// Does tcgen05.st traffic from other warps slow concurrent tcgen05.mma?
// One thread issues MMAs (M=128, N=240, K=32 int8; A from smem or TMEM), while
// `stw` warps store to TMEM columns the MMAs do not touch (with or without
// tcgen05.wait::st after each store).  Prints cycles per MMA.
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_1809_10786_b200/csrc/i8_common.cuh"
using namespace sgl;
using namespace sgl::i8;

__global__ void k(int iters, int ts, int stw, int waitst, int32_t *sink, long long *cyc) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    __shared__ volatile int done;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int i = tid; i < 64 * 1024; i += blockDim.x) sm[i] = (uint8_t)(i * 7);
    if (tid == 0) { mbar_init(&bar, 1); done = 0; asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
    if (warp == 0) umma::tmem_alloc(&tbase, 512);
    umma::fence_async_smem();
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    const uint32_t td = tbase;
    const int N = 240;
    if (tid == 0) {
        const uint32_t id = umma::idesc_i8(128, N, true, true);
        const uint64_t da = umma::desc_kmajor(umma::smem_addr(sm), 128 * 16, 128);
        const uint64_t db = umma::desc_kmajor(umma::smem_addr(sm + 16384), N * 16, 128);
        long long c0 = clock64();
        for (int it = 0; it < iters; ++it) {
            if (ts) umma::mma_i8_ts(td, td + 480 + 8 * (it & 3), db, id, true);
            else umma::mma_i8(td, da, db, id, true);
        }
        umma::commit(&bar);
        mbar_wait(&bar, 0);
        cyc[blockIdx.x] = clock64() - c0;
        done = 1;
    } else if (warp >= 1 && warp <= stw) {
        // store warps: lane quarter warp % 4, columns 256 .. 479 (not read or written by the MMAs)
        const uint32_t ta = td + ((uint32_t)((warp & 3) * 32) << 16) + 256 + 8 * (warp >> 2);
        uint32_t v[4] = {1u, 2u, 3u, (uint32_t)lane};
        while (!done) {
            umma::tmem_st4(ta, v);
            if (waitst) umma::tmem_st_wait();
            v[0]++;
        }
    }
    __syncwarp();
    umma::fence_before();
    __syncthreads();
    if (warp == 0) umma::tmem_free(td, 512);
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int32_t *sink;
    long long *cyc;
    cudaMalloc(&sink, 4096);
    cudaMalloc(&cyc, 8 * sms);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    for (int ts = 0; ts < 2; ++ts)
        for (int stw : {0, 4, 12})
            for (int ws = 0; ws < 2; ++ws) {
                if (stw == 0 && ws) continue;
                const int iters = 20000;
                k<<<sms, 416, 64 * 1024>>>(iters, ts, stw, ws, sink, cyc);
                cudaError_t e = cudaDeviceSynchronize();
                long long h[256];
                cudaMemcpy(h, cyc, 8 * sms, cudaMemcpyDeviceToHost);
                double m = 0;
                for (int i = 0; i < sms; ++i) m += h[i];
                printf("A %s, %2d store warps%s: %.1f cycles per N=240 MMA (%s)\n", ts ? "TMEM" : "smem", stw,
                       ws ? " + wait::st" : "", m / sms / iters, cudaGetErrorString(e));
            }
    return 0;
}
