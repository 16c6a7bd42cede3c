// Does ptxas' grouping of DMMA accumulation chains cost throughput?  The
// gather's per-slab fragment loop (9 N-tiles x 9 k-steps, chains grouped by
// ptxas) vs the same work with m16n8k4 (two interleaved 8x8 halves).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}
__global__ void __launch_bounds__(288, 2) grouped(const double* __restrict__ g, double* out, int n) {
    extern __shared__ double sl[];
    for (int i = threadIdx.x; i < 36*36*2*4; i += blockDim.x) sl[i] = g[i & 1023];
    __syncthreads();
    const int lane = threadIdx.x & 31, rb = lane >> 3, part = (lane >> 2) & 1, cc = lane & 3;
    double afr[9], w1r[9];
    for (int k = 0; k < 9; ++k) { afr[k] = g[k * 32 + lane]; w1r[k] = g[400 + k * 32 + lane]; }
    double s_re = 0, s_im = 0;
    for (int it = 0; it < n; ++it) {
      const double* s = sl + (it & 3) * 36 * 36 * 2;
#pragma unroll
      for (int nt0 = 0; nt0 < 9; nt0 += 3) {
        double d[3][2] = {{0,0},{0,0},{0,0}};
#pragma unroll
        for (int ks = 0; ks < 9; ++ks)
#pragma unroll
          for (int i = 0; i < 3; ++i) dmma(d[i], afr[ks], s[((nt0 + i) * 4 + rb) * 72 + (ks * 4 + cc) * 2 + part]);
#pragma unroll
        for (int i = 0; i < 3; ++i) { s_re = fma(w1r[nt0+i], d[i][0], s_re); s_im = fma(w1r[nt0+i], d[i][1], s_im); }
      }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s_re + s_im;
}
__global__ void __launch_bounds__(288, 2) m16(const double* __restrict__ g, double* out, int n) {
    extern __shared__ double sl[];
    for (int i = threadIdx.x; i < 36*36*2*4; i += blockDim.x) sl[i] = g[i & 1023];
    __syncthreads();
    const int lane = threadIdx.x & 31, gq = lane >> 2, cc = lane & 3;
    double afr[9], w1r[10];
    for (int k = 0; k < 9; ++k) afr[k] = g[k * 32 + lane];
    for (int k = 0; k < 10; ++k) w1r[k] = g[400 + k * 32 + lane];
    double s0 = 0, s1 = 0;
    for (int it = 0; it < n; ++it) {
      const double* s = sl + (it & 3) * 36 * 36 * 2;
#pragma unroll
      for (int mt = 0; mt < 5; ++mt) {
        double d[4] = {0, 0, 0, 0};
#pragma unroll
        for (int ks = 0; ks < 9; ++ks) {
          const int r0 = mt * 16 + gq, r1 = r0 + 8;
          const double a0 = s[(((r0 >> 1) % 36) * 36 + ks * 4 + cc) * 2 + (r0 & 1)];
          const double a1 = s[(((r1 >> 1) % 36) * 36 + ks * 4 + cc) * 2 + (r1 & 1)];
          asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                       : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3]) : "d"(a0), "d"(a1), "d"(afr[ks]));
        }
        s0 = fma(w1r[2 * mt], d[0], fma(w1r[2 * mt + 1], d[2], s0));
        s1 = fma(w1r[2 * mt], d[1], fma(w1r[2 * mt + 1], d[3], s1));
      }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s0 + s1;
}
int main() {
    double *g, *o; cudaMalloc(&g, 1 << 20); cudaMalloc(&o, 1 << 24); cudaMemset(g, 0, 1 << 20);
    const int smem = 36 * 36 * 2 * 4 * 8;
    cudaFuncSetAttribute(grouped, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(m16, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int warps : {8, 4}) {
      int threads = warps * 32, n = 2000, blocks = 148 * 2;
      float ms;
      grouped<<<blocks, threads, smem>>>(g, o, 10);
      cudaEventRecord(a); grouped<<<blocks, threads, smem>>>(g, o, n); cudaEventRecord(b); cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      double dm = (double)blocks * warps * n * 81;
      printf("grouped m8n8k4, %d warps/CTA x2: %.1f%% of DMMA peak (%.2f TF)\n", warps, 100 * dm * 16 / (ms * 1e-3 * 1.965e9 * 592), dm * 512 / ms / 1e9);
      m16<<<blocks, threads, smem>>>(g, o, 10);
      cudaEventRecord(a); m16<<<blocks, threads, smem>>>(g, o, n); cudaEventRecord(b); cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      dm = (double)blocks * warps * n * 90;
      printf("m16n8k4,         %d warps/CTA x2: %.1f%% of DMMA peak (%.2f TF)\n", warps, 100 * dm * 16 / (ms * 1e-3 * 1.965e9 * 592), dm * 512 / ms / 1e9);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
