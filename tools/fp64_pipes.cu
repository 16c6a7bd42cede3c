// DMMA latency / chain-count sweep and DMMA + DFMA co-issue test (sm_100a).
#include <cstdio>
#include <cuda_runtime.h>
template <int C>
__global__ void dmma_chains(double* out, double seed, int iters){
  double a=seed+threadIdx.x, b=seed-threadIdx.x;
  double c[C][2];
  #pragma unroll
  for(int j=0;j<C;j++){c[j][0]=0;c[j][1]=0;}
  for(int i=0;i<iters;i++){
    #pragma unroll
    for(int j=0;j<C;j++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
        : "+d"(c[j][0]),"+d"(c[j][1]) : "d"(a),"d"(b));
  }
  double s=0;
  #pragma unroll
  for(int j=0;j<C;j++) s+=c[j][0]+c[j][1];
  if(s==1234.5) out[threadIdx.x]=s;
}
template <int NF>
__global__ void mixed(double* out, double seed, int iters){
  double a=seed+threadIdx.x, b=seed-threadIdx.x;
  double c[8][2]; double x[8];
  #pragma unroll
  for(int j=0;j<8;j++){c[j][0]=0;c[j][1]=0;x[j]=seed+j;}
  for(int i=0;i<iters;i++){
    #pragma unroll
    for(int j=0;j<8;j++){
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
        : "+d"(c[j][0]),"+d"(c[j][1]) : "d"(a),"d"(b));
      #pragma unroll
      for(int k=0;k<NF;k++) x[(j+k)&7]=fma(x[(j+k)&7],0.999999,1e-7);
    }
  }
  double s=0;
  #pragma unroll
  for(int j=0;j<8;j++) s+=c[j][0]+c[j][1]+x[j];
  if(s==1234.5) out[threadIdx.x]=s;
}
template <typename K> float timeit(K k, int blocks, int threads, int iters, double* d){
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<<<blocks,threads>>>(d,1.0,10);
  cudaEventRecord(e0); k<<<blocks,threads>>>(d,1.0,iters); cudaEventRecord(e1);
  cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms,e0,e1); return ms;
}
int main(){
  double* d; cudaMalloc(&d, 1<<20);
  int sms=148; int it=4000;
  // one warp per SMSP: 148 blocks x 128 threads
  #define CH(C) { float ms=timeit(dmma_chains<C>, sms, 128, it, d); double fl=2.0*256*C*it*4.0*sms; \
     printf("DMMA chains=%d warps/SMSP=1: %.2f TFLOP/s, cycles/DMMA/SMSP=%.1f\n", C, fl/ms/1e9, ms*1e-3*1.965e9/(C*(double)it)); }
  CH(1) CH(2) CH(3) CH(4) CH(6) CH(8)
  #define MX(NF) { float ms=timeit(mixed<NF>, sms*2, 256, it, d); double fl=2.0*256*8*it*8.0*sms*2; double ff=2.0*NF*8*it*256.0*sms*2; \
     printf("mixed 8 DMMA + %d DFMA per warp-iter: DMMA %.2f TF + DFMA %.2f TF = %.2f TF\n", NF, fl/ms/1e9, ff/ms/1e9, (fl+ff)/ms/1e9); }
  MX(0) MX(1) MX(2) MX(4) MX(8)
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
