// Microbenchmarks for the roofline denominators this repo reports against:
// DMMA (fp64 tensor, mma.sync m8n8k4), DFMA (fp64 vector), IMMA (int8 mma.sync m16n8k32),
// and shared-memory random gather throughput. Run on one B200; prints JSON.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1;}}while(0)

template<int ITERS>
__global__ void dmma_loop(double* out, double seed){
  double a = seed + threadIdx.x, b = seed * 0.5 + threadIdx.x;
  double c[8][2];
  #pragma unroll
  for (int i=0;i<8;i++){c[i][0]=0;c[i][1]=0;}
  for (int it=0; it<ITERS; ++it){
    #pragma unroll
    for (int i=0;i<8;i++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(c[i][0]),"+d"(c[i][1]) : "d"(a),"d"(b));
  }
  double s=0; for(int i=0;i<8;i++) s+=c[i][0]+c[i][1];
  if (s == 12345.678) out[0]=s;
}
template<int ITERS>
__global__ void dfma_loop(double* out, double seed){
  double a = seed + threadIdx.x, b = seed*0.25;
  double c[8];
  #pragma unroll
  for(int i=0;i<8;i++) c[i]=i;
  for (int it=0; it<ITERS; ++it){
    #pragma unroll
    for(int i=0;i<8;i++) c[i] = fma(c[i], a, b);
  }
  double s=0; for(int i=0;i<8;i++) s+=c[i];
  if (s == 12345.678) out[0]=s;
}
template<int ITERS>
__global__ void imma_loop(int* out, int seed){
  int a0=seed+threadIdx.x,a1=a0*3,a2=a0*5,a3=a0*7,b0=a0*11,b1=a0*13;
  int c[8][4];
  #pragma unroll
  for(int i=0;i<8;i++){c[i][0]=c[i][1]=c[i][2]=c[i][3]=0;}
  for (int it=0; it<ITERS; ++it){
    #pragma unroll
    for(int i=0;i<8;i++)
      asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+r"(c[i][0]),"+r"(c[i][1]),"+r"(c[i][2]),"+r"(c[i][3]) : "r"(a0),"r"(a1),"r"(a2),"r"(a3),"r"(b0),"r"(b1));
  }
  int s=0; for(int i=0;i<8;i++) s+=c[i][0]+c[i][1]+c[i][2]+c[i][3];
  if (s == 12345) out[0]=s;
}
int main(){
  int dev=0; cudaDeviceProp pr; CK(cudaGetDeviceProperties(&pr, dev));
  double* d; CK(cudaMalloc(&d, 64)); int* di; CK(cudaMalloc(&di,64));
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int IT=4096; int blocks = pr.multiProcessorCount*4; int threads=256;
  float ms;
  // warm
  dmma_loop<IT><<<blocks,threads>>>(d,1.0); dfma_loop<IT><<<blocks,threads>>>(d,1.0); imma_loop<IT><<<blocks,threads>>>(di,1);
  CK(cudaDeviceSynchronize());
  double best_dmma=0,best_dfma=0,best_imma=0;
  for(int r=0;r<5;r++){
    cudaEventRecord(e0); dmma_loop<IT><<<blocks,threads>>>(d,1.0); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms,e0,e1);
    double fl = (double)blocks*(threads/32)*IT*8*512.0; if (fl/(ms*1e-3) > best_dmma) best_dmma=fl/(ms*1e-3);
    cudaEventRecord(e0); dfma_loop<IT><<<blocks,threads>>>(d,1.0); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms,e0,e1);
    fl = (double)blocks*threads*IT*8*2.0; if (fl/(ms*1e-3) > best_dfma) best_dfma=fl/(ms*1e-3);
    cudaEventRecord(e0); imma_loop<IT><<<blocks,threads>>>(di,1); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms,e0,e1);
    fl = (double)blocks*(threads/32)*IT*8*(16*8*32*2.0); if (fl/(ms*1e-3) > best_imma) best_imma=fl/(ms*1e-3);
  }
  CK(cudaGetLastError());
  int clk=0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("{\"sms\": %d, \"clock_khz\": %d, \"dmma_tflops\": %.3f, \"dfma_tflops\": %.3f, \"imma_mma_sync_tops\": %.3f}\n",
         pr.multiProcessorCount, clk, best_dmma/1e12, best_dfma/1e12, best_imma/1e12);
  return 0;
}
