// tcgen05.ld throughput: W warps (W/4 per TMEM lane quarter) each read 480
// columns of their quarter `reps` times with 32x32b.xN loads (N = 4, 8, 16,
// 32), either waiting after every load (wait::ld) or after a batch of loads.
// Prints bytes read per SM-cycle.  The int8 window kernels' epilogues drain 6
// diagonals x 80 columns x 128 lanes = 240 KB per accumulator set.
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_1809_10786_b200/csrc/i8_common.cuh"
using namespace sgl;

template <int N>
__device__ __forceinline__ void ldN(uint32_t a, uint32_t (&v)[32]) {
    if constexpr (N == 4)
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];\n"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]) : "r"(a));
    else if constexpr (N == 8)
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                     : "r"(a));
    else if constexpr (N == 16)
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
            : "r"(a));
    else
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
              "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
              "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
            : "r"(a));
}

template <int N, int BATCH>
__global__ void k(int reps, uint32_t *sink, long long *cyc) {
    __shared__ uint32_t tbase;
    const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (warp == 0) umma::tmem_alloc(&tbase, 512);
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    const int quarter = warp & 3, part = warp >> 2, parts = nw / 4;
    const uint32_t ta = tbase + ((uint32_t)(quarter * 32) << 16);
    const int cols = 480 / parts, c0 = part * cols;   // this warp's share of the 480 columns
    uint32_t acc = 0, v[32];
    __syncthreads();
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        for (int c = 0; c + N * BATCH <= cols; c += N * BATCH) {
#pragma unroll
            for (int b = 0; b < BATCH; ++b) {
                ldN<N>(ta + c0 + c + b * N, v);
                if (b == BATCH - 1) umma::tmem_ld_wait();
#pragma unroll
                for (int j = 0; j < N; ++j) acc += v[j];
            }
        }
    }
    __syncthreads();
    long long t1 = clock64();
    if (acc == 12345) sink[threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    umma::fence_before();
    __syncthreads();
    if (warp == 0) umma::tmem_free(tbase, 512);
}

template <int N, int BATCH>
void run(int warps, uint32_t *sink, long long *cyc, int sms) {
    const int reps = 200;
    k<N, BATCH><<<sms, warps * 32>>>(reps, sink, cyc);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[256];
    cudaMemcpy(h, cyc, 8 * sms, cudaMemcpyDeviceToHost);
    double m = 0;
    for (int i = 0; i < sms; ++i) m += h[i];
    m /= sms;
    const int parts = warps / 4, cols = 480 / parts;
    const double bytes = (double)reps * 4 * parts * (cols / (N * BATCH)) * (N * BATCH) * 32 * 4;
    printf("x%-2d batch %d, %2d warps: %.1f B/cycle per SM (%.0f cycles per 240 KB drain) %s\n", N, BATCH, warps,
           bytes / m, 245760.0 / (bytes / m), cudaGetErrorString(e));
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint32_t *sink;
    long long *cyc;
    cudaMalloc(&sink, 4096 * 4);
    cudaMalloc(&cyc, 8 * sms);
    for (int w : {4, 8, 16}) {
        run<4, 1>(w, sink, cyc, sms);
        run<4, 6>(w, sink, cyc, sms);
        run<8, 1>(w, sink, cyc, sms);
        run<16, 1>(w, sink, cyc, sms);
        run<16, 2>(w, sink, cyc, sms);
        run<32, 1>(w, sink, cyc, sms);
    }
    return 0;
}
