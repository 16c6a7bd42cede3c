// RED.E.ADD.F64 throughput with the scatter's access pattern: each warp
// instruction covers 4 rows x 16 doubles (8 cols x re/im) of a large grid.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void red_pattern(double* grid, size_t pitch, int rows, int iters, int nplanes) {
  int lane = threadIdx.x & 31, warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int rb = lane >> 3, part = (lane >> 2) & 1, kk = lane & 3;
  for (int it = 0; it < iters; ++it) {
    size_t plane = (size_t)((warp * 7 + it * 13) % nplanes);
    for (int mt = 0; mt < 9; ++mt) {
      double* row = grid + (plane * rows + mt * 4 + rb) * pitch;
      #pragma unroll
      for (int ct = 0; ct < 5; ++ct)
        #pragma unroll
        for (int j = 0; j < 2; ++j)
          asm volatile("red.global.add.f64 [%0], %1;" :: "l"(row + 2 * (ct * 8 + 2 * kk + j) + part), "d"(1.0) : "memory");
    }
  }
}
int main() {
  size_t pitch = 2 * 288, rows = 544, nplanes = 512;
  double* g; cudaMalloc(&g, sizeof(double) * pitch * rows * nplanes);
  cudaMemset(g, 0, sizeof(double) * pitch * rows * nplanes);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int bps : {2, 4, 8}) {
    int blocks = 148 * bps, threads = 256, iters = 200;
    red_pattern<<<blocks, threads>>>(g, pitch, rows, 2, nplanes);
    cudaEventRecord(a); red_pattern<<<blocks, threads>>>(g, pitch, rows, iters, nplanes); cudaEventRecord(b);
    cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b);
    double ops = (double)blocks * threads * iters * 9 * 5 * 2;
    printf("blocks/SM=%d: %.3e RED lane-ops/s (%.2f per SM-cycle @1.965GHz)\n", bps, ops / ms * 1e3, ops / ms * 1e3 / 148 / 1.965e9);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
