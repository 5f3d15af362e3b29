// Micro-benchmark: FP32 issue/throughput of the dwell step (7 non-fused ops) written as
// (a) scalar, 1 orbit per thread; (b) scalar, 2 independent orbits per thread;
// (c) packed f32x2 (FFMA2(a,b,-0)/FADD2), 2 orbits per thread.  No escape test: a fixed
// number of steps from a non-escaping c (c = -1: period-2 cycle), so every lane works.
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 f2add(u64 a, u64 b){ u64 d; asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d;}
__device__ __forceinline__ u64 f2sub(u64 a, u64 b){ u64 d; asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d;}
__device__ __forceinline__ u64 f2mul(u64 a, u64 b, u64 nz){ u64 d; asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(nz)); return d;}
__device__ __forceinline__ u64 pk(float lo, float hi){ return (u64)__float_as_uint(lo) | ((u64)__float_as_uint(hi) << 32); }

__global__ void k_scalar1(float cr, float ci, int n, float *out){
  float x=0,y=0,x2=0,y2=0; cr += threadIdx.x*1e-9f;
  for(int i=0;i<n;++i){
#pragma unroll
    for(int k=0;k<8;++k){ float xy=__fmul_rn(x,y); x=__fadd_rn(__fsub_rn(x2,y2),cr); y=__fadd_rn(__fadd_rn(xy,xy),ci); x2=__fmul_rn(x,x); y2=__fmul_rn(y,y);} }
  out[blockIdx.x*blockDim.x+threadIdx.x]=x+y;
}
__global__ void k_scalar2(float cr, float ci, int n, float *out){
  float x=0,y=0,x2=0,y2=0, a=0,b=0,a2=0,b2=0; float cr2 = cr + threadIdx.x*1e-9f;
  for(int i=0;i<n;++i){
#pragma unroll
    for(int k=0;k<8;++k){ float xy=__fmul_rn(x,y); x=__fadd_rn(__fsub_rn(x2,y2),cr); y=__fadd_rn(__fadd_rn(xy,xy),ci); x2=__fmul_rn(x,x); y2=__fmul_rn(y,y);
      float ab=__fmul_rn(a,b); a=__fadd_rn(__fsub_rn(a2,b2),cr2); b=__fadd_rn(__fadd_rn(ab,ab),ci); a2=__fmul_rn(a,a); b2=__fmul_rn(b,b);} }
  out[blockIdx.x*blockDim.x+threadIdx.x]=x+y+a+b;
}
__global__ void k_pair(float cr, float ci, int n, float *out, u64 nz){
  u64 C=pk(cr, cr+threadIdx.x*1e-9f), CI=pk(ci,ci), x=0,y=0,x2=0,y2=0;
  for(int i=0;i<n;++i){
#pragma unroll
    for(int k=0;k<8;++k){ u64 xy=f2mul(x,y,nz); x=f2add(f2sub(x2,y2),C); y=f2add(f2add(xy,xy),CI); x2=f2mul(x,x,nz); y2=f2mul(y,y,nz);} }
  out[blockIdx.x*blockDim.x+threadIdx.x]=__uint_as_float((unsigned)(x^y))+__uint_as_float((unsigned)((x^y)>>32));
}
int main(){
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float *out; cudaMalloc(&out, 1<<26);
  const int tpb=256, blocks=sms*8*4, n=4096;
  cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b);
  u64 nz = 0x8000000080000000ull;
  for(int rep=0;rep<3;++rep){
    float ms; double ops;
    cudaEventRecord(a); k_scalar1<<<blocks,tpb>>>(-1.f,0.f,n,out); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b);
    ops=7.0*8*n*(double)blocks*tpb; printf("scalar1: %.3f ms  %.2f Tops/s\n", ms, ops/ms/1e9);
    cudaEventRecord(a); k_scalar2<<<blocks,tpb>>>(-1.f,0.f,n,out); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b);
    ops=2*7.0*8*n*(double)blocks*tpb; printf("scalar2: %.3f ms  %.2f Tops/s\n", ms, ops/ms/1e9);
    cudaEventRecord(a); k_pair<<<blocks,tpb>>>(-1.f,0.f,n,out,nz); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b);
    ops=2*7.0*8*n*(double)blocks*tpb; printf("pair   : %.3f ms  %.2f Tops/s\n", ms, ops/ms/1e9);
  }
  printf("sms=%d clk=%d kHz nominal 1-op/lane/clk peak=%.2f Tops/s\n", sms, clk, sms*128.0*clk/1e9);
  return 0;
}
