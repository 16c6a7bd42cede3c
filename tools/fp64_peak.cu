// FP64 peak microbenchmark: DFMA pipe and DMMA (mma.sync m8n8k4 f64) on sm_100a.
// Prints achieved TFLOP/s for each; used to set the FP64 roofline denominator.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_loop(double* out, double seed, int iters){
  double x[16];
  #pragma unroll
  for(int j=0;j<16;j++) x[j]=seed+threadIdx.x*1e-9+j;
  const double m=0.999999, a=1e-7;
  for(int i=0;i<iters;i++){
    #pragma unroll
    for(int j=0;j<16;j++) x[j]=fma(x[j],m,a);
  }
  double s=0;
  #pragma unroll
  for(int j=0;j<16;j++) s+=x[j];
  if(s==1234.5) out[threadIdx.x]=s;
}
__global__ void dmma_loop(double* out, double seed, int iters){
  double a=seed+threadIdx.x, b=seed-threadIdx.x;
  double c[8][2];
  #pragma unroll
  for(int j=0;j<8;j++){c[j][0]=0;c[j][1]=0;}
  for(int i=0;i<iters;i++){
    #pragma unroll
    for(int j=0;j<8;j++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
        : "+d"(c[j][0]),"+d"(c[j][1]) : "d"(a),"d"(b));
  }
  double s=0;
  #pragma unroll
  for(int j=0;j<8;j++) s+=c[j][0]+c[j][1];
  if(s==1234.5) out[threadIdx.x]=s;
}
int main(){
  double* d; cudaMalloc(&d, 1<<20);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int threads : {256, 512, 1024}) for (int bpsm : {1,2,4}) {
    int iters=20000; int blocks=sms*bpsm;
    dfma_loop<<<blocks,threads>>>(d,1.0,100);
    cudaEventRecord(e0); dfma_loop<<<blocks,threads>>>(d,1.0,iters); cudaEventRecord(e1);
    cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms,e0,e1);
    double fl=2.0*16*iters*(double)threads*blocks;
    printf("DFMA threads=%d blocks=%d: %.2f TFLOP/s (%.3f ms)\n",threads,blocks,fl/ms/1e9,ms);
  }
  for (int threads : {128, 256, 512, 1024}) for (int bpsm : {1,2,4}) {
    int iters=4000; int blocks=sms*bpsm;
    dmma_loop<<<blocks,threads>>>(d,1.0,10);
    cudaEventRecord(e0); dmma_loop<<<blocks,threads>>>(d,1.0,iters); cudaEventRecord(e1);
    cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms,e0,e1);
    double fl=2.0*256*8*iters*(double)(threads/32)*blocks;
    printf("DMMA threads=%d blocks=%d: %.2f TFLOP/s (%.3f ms)\n",threads,blocks,fl/ms/1e9,ms);
  }
  cudaError_t err=cudaGetLastError(); printf("err=%s\n",cudaGetErrorString(err));
  return 0;
}
