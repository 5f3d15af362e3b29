// Micro-benchmark: FP32 throughput of the dwell step (7 non-fused ops) vs warps per SM
// sub-partition, scalar vs packed f32x2 (FFMA2(a,b,-0) + FADD2), 1 or 2 packed chains per
// thread.  One block per SM (grid = #SMs), 32*4*W threads: W warps per sub-partition.
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__constant__ u64 c_nz = 0x8000000080000000ull;
__device__ __forceinline__ u64 f2add(u64 a, u64 b){ u64 d; asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d;}
__device__ __forceinline__ u64 f2sub(u64 a, u64 b){ u64 d; asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d;}
__device__ __forceinline__ u64 f2mul(u64 a, u64 b){ u64 d; asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c_nz)); return d;}
__device__ __forceinline__ u64 pk(float lo, float hi){ return (u64)__float_as_uint(lo) | ((u64)__float_as_uint(hi) << 32); }
#define STEP2(x,y,x2,y2,C,CI) { u64 xy=f2mul(x,y); x=f2add(f2sub(x2,y2),C); y=f2add(f2add(xy,xy),CI); x2=f2mul(x,x); y2=f2mul(y,y);}
__global__ void k_scalar(float cr, float ci, int n, float *out){
  float x=0,y=0,x2=0,y2=0; cr += threadIdx.x*1e-9f;
  for(int i=0;i<n;++i){
#pragma unroll
    for(int k=0;k<16;++k){ float xy=__fmul_rn(x,y); x=__fadd_rn(__fsub_rn(x2,y2),cr); y=__fadd_rn(__fadd_rn(xy,xy),ci); x2=__fmul_rn(x,x); y2=__fmul_rn(y,y);} }
  out[blockIdx.x*blockDim.x+threadIdx.x]=x+y;
}
__global__ void k_pair(float cr, float ci, int n, float *out){
  u64 C=pk(cr, cr+threadIdx.x*1e-9f), CI=pk(ci,ci), x=0,y=0,x2=0,y2=0;
  for(int i=0;i<n;++i){
#pragma unroll
    for(int k=0;k<16;++k) STEP2(x,y,x2,y2,C,CI) }
  out[blockIdx.x*blockDim.x+threadIdx.x]=__uint_as_float((unsigned)(x^y))+__uint_as_float((unsigned)((x^y)>>32));
}
__global__ void k_pair2(float cr, float ci, int n, float *out){
  u64 C=pk(cr, cr+threadIdx.x*1e-9f), D=pk(cr+1e-7f, cr-threadIdx.x*1e-9f), CI=pk(ci,ci), x=0,y=0,x2=0,y2=0, a=0,b=0,a2=0,b2=0;
  for(int i=0;i<n;++i){
#pragma unroll
    for(int k=0;k<8;++k){ STEP2(x,y,x2,y2,C,CI) STEP2(a,b,a2,b2,D,CI) } }
  out[blockIdx.x*blockDim.x+threadIdx.x]=__uint_as_float((unsigned)(x^y^a))+__uint_as_float((unsigned)((x^y^b)>>32));
}
int main(){
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float *out; cudaMalloc(&out, 1<<26);
  const int n=2048;
  cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b);
  double peak = sms*128.0*clk*1e3;
  int Ws[] = {1,2,3,4,6,8,12,16};
  for (int wi=0; wi<8; ++wi){
    int W=Ws[wi], tpb=128*W; if (tpb>1024){ tpb=1024; }
    int blocks = sms * (128*W/tpb);
    float ms; double ops;
    for(int rep=0;rep<2;++rep){
    cudaEventRecord(a); k_scalar<<<blocks,tpb>>>(-1.f,0.f,n,out); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b);}
    ops=7.0*16*n*(double)blocks*tpb; double s1=ops/ms/1e-3/peak;
    for(int rep=0;rep<2;++rep){
    cudaEventRecord(a); k_pair<<<blocks,tpb>>>(-1.f,0.f,n,out); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b);}
    ops=2*7.0*16*n*(double)blocks*tpb; double p1=ops/ms/1e-3/peak;
    for(int rep=0;rep<2;++rep){
    cudaEventRecord(a); k_pair2<<<blocks,tpb>>>(-1.f,0.f,n,out); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b);}
    ops=4*7.0*16*n*(double)blocks*tpb; double p2=ops/ms/1e-3/peak;
    printf("warps/SMSP=%2d  scalar %.3f  pair %.3f  pair2 %.3f  (fraction of %.2f T lane-ops/s)\n", W, s1, p1, p2, peak/1e12);
  }
  return 0;
}
