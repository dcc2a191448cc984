// Pipe-throughput microbenchmark for the pair kernel design (FFMA vs FFMA2,
// MUFU.RSQ, DFMA). Not part of the product; numbers go to profiles/.
#include <cstdio>
#include <cuda_runtime.h>
#define ITERS 4096
__global__ void k_ffma(float* out, float a, float b){
  float x0=threadIdx.x, x1=x0+1, x2=x0+2, x3=x0+3, x4=x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  #pragma unroll 16
  for(int i=0;i<ITERS;i++){
    x0=fmaf(x0,a,b); x1=fmaf(x1,a,b); x2=fmaf(x2,a,b); x3=fmaf(x3,a,b);
    x4=fmaf(x4,a,b); x5=fmaf(x5,a,b); x6=fmaf(x6,a,b); x7=fmaf(x7,a,b);
  }
  out[blockIdx.x*blockDim.x+threadIdx.x]=x0+x1+x2+x3+x4+x5+x6+x7;
}
__global__ void k_ffma_reg(float* out, float a0, float b0){
  // 3-register form: multiplier/addend in registers that vary per thread
  float a = a0 + threadIdx.x*1e-9f, b = b0 + threadIdx.x*1e-9f;
  float x0=threadIdx.x, x1=x0+1, x2=x0+2, x3=x0+3, x4=x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  #pragma unroll 16
  for(int i=0;i<ITERS;i++){
    x0=fmaf(x0,a,b); x1=fmaf(x1,a,b); x2=fmaf(x2,a,b); x3=fmaf(x3,a,b);
    x4=fmaf(x4,a,b); x5=fmaf(x5,a,b); x6=fmaf(x6,a,b); x7=fmaf(x7,a,b);
  }
  out[blockIdx.x*blockDim.x+threadIdx.x]=x0+x1+x2+x3+x4+x5+x6+x7;
}
__global__ void k_ffma2(float* out, float a0, float b0){
  float2 a = make_float2(a0 + threadIdx.x*1e-9f, a0), b = make_float2(b0, b0 + threadIdx.x*1e-9f);
  float2 x0=make_float2(threadIdx.x,1), x1=make_float2(2,3), x2=make_float2(4,5), x3=make_float2(6,7);
  float2 x4=make_float2(8,9), x5=make_float2(10,11), x6=make_float2(12,13), x7=make_float2(14,15);
  #pragma unroll 16
  for(int i=0;i<ITERS;i++){
    x0=__ffma2_rn(x0,a,b); x1=__ffma2_rn(x1,a,b); x2=__ffma2_rn(x2,a,b); x3=__ffma2_rn(x3,a,b);
    x4=__ffma2_rn(x4,a,b); x5=__ffma2_rn(x5,a,b); x6=__ffma2_rn(x6,a,b); x7=__ffma2_rn(x7,a,b);
  }
  out[blockIdx.x*blockDim.x+threadIdx.x]=x0.x+x1.x+x2.x+x3.x+x4.x+x5.x+x6.x+x7.x+x0.y+x1.y+x2.y+x3.y+x4.y+x5.y+x6.y+x7.y;
}
// FFMA2 with three distinct register-pair operands in every instruction
// (no operand reuse possible): tests register-bank read limits
__global__ void k_ffma2_distinct(float* out, float a0, float b0){
  float2 a[8], b[8], x[8];
  #pragma unroll
  for (int k = 0; k < 8; ++k) {
    a[k] = make_float2(a0 + (threadIdx.x + k) * 1e-9f, a0 - k * 1e-9f);
    b[k] = make_float2(b0 + k * 1e-9f, b0 + threadIdx.x * 1e-9f);
    x[k] = make_float2(threadIdx.x + k, k);
  }
  #pragma unroll 4
  for(int i=0;i<ITERS;i++){
    #pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = __ffma2_rn(x[k], a[k], b[k]);
  }
  float s = 0; for (int k = 0; k < 8; ++k) s += x[k].x + x[k].y;
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
__global__ void k_ffma_distinct(float* out, float a0, float b0){
  float a[8], b[8], x[8];
  #pragma unroll
  for (int k = 0; k < 8; ++k) { a[k] = a0 + (threadIdx.x + k) * 1e-9f; b[k] = b0 + k * 1e-9f; x[k] = threadIdx.x + k; }
  #pragma unroll 4
  for(int i=0;i<ITERS;i++){
    #pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = fmaf(x[k], a[k], b[k]);
  }
  float s = 0; for (int k = 0; k < 8; ++k) s += x[k];
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
__global__ void k_fmul2_distinct(float* out, float a0){
  float2 a[8], x[8];
  #pragma unroll
  for (int k = 0; k < 8; ++k) { a[k] = make_float2(1.0f + (threadIdx.x + k) * 1e-9f, 1.0f - k * 1e-9f); x[k] = make_float2(threadIdx.x + k, k); }
  #pragma unroll 4
  for(int i=0;i<ITERS;i++){
    #pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = __fmul2_rn(x[k], a[k]);
  }
  float s = 0; for (int k = 0; k < 8; ++k) s += x[k].x + x[k].y;
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
__global__ void k_rsqrt(float* out, float a){
  float x0=threadIdx.x+1, x1=x0+1, x2=x0+2, x3=x0+3, x4=x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  #pragma unroll 16
  for(int i=0;i<ITERS;i++){
    x0=rsqrtf(x0); x1=rsqrtf(x1); x2=rsqrtf(x2); x3=rsqrtf(x3);
    x4=rsqrtf(x4); x5=rsqrtf(x5); x6=rsqrtf(x6); x7=rsqrtf(x7);
  }
  out[blockIdx.x*blockDim.x+threadIdx.x]=x0+x1+x2+x3+x4+x5+x6+x7;
}
__global__ void k_dfma(double* out, double a0, double b0){
  double a = a0 + threadIdx.x*1e-12, b = b0;
  double x0=threadIdx.x, x1=x0+1, x2=x0+2, x3=x0+3, x4=x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  #pragma unroll 16
  for(int i=0;i<ITERS;i++){
    x0=fma(x0,a,b); x1=fma(x1,a,b); x2=fma(x2,a,b); x3=fma(x3,a,b);
    x4=fma(x4,a,b); x5=fma(x5,a,b); x6=fma(x6,a,b); x7=fma(x7,a,b);
  }
  out[blockIdx.x*blockDim.x+threadIdx.x]=x0+x1+x2+x3+x4+x5+x6+x7;
}
__global__ void k_shfl(float* out, float a){
  float x0=threadIdx.x, x1=x0+1, x2=x0+2, x3=x0+3;
  int l = (threadIdx.x+1)&31;
  #pragma unroll 16
  for(int i=0;i<ITERS;i++){
    x0=__shfl_sync(0xffffffff,x0,l); x1=__shfl_sync(0xffffffff,x1,l);
    x2=__shfl_sync(0xffffffff,x2,l); x3=__shfl_sync(0xffffffff,x3,l);
  }
  out[blockIdx.x*blockDim.x+threadIdx.x]=x0+x1+x2+x3;
}
int main(){
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  int blocks = sms*8, threads = 256;
  float* out; cudaMalloc(&out, sizeof(double)*blocks*threads);
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  double nthr = (double)blocks*threads;
  auto run = [&](const char* name, auto launch, double ops_per_thread, const char* unit){
    for(int w=0;w<3;w++) launch();
    cudaEventRecord(e0); for(int r=0;r<10;r++) launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms,e0,e1); ms/=10;
    double rate = nthr*ops_per_thread/(ms*1e-3);
    printf("%-10s %8.3f ms  %10.3f T%s/s  per-SM-per-clk(@%d MHz max)=%.1f\n", name, ms, rate/1e12, unit, clk/1000, rate/(sms*(clk*1e3)));
  };
  run("ffma_imm", [&]{k_ffma<<<blocks,threads>>>(out,1.0001f,0.5f);}, 8.0*ITERS, "FMA");
  run("ffma_reg", [&]{k_ffma_reg<<<blocks,threads>>>(out,1.0001f,0.5f);}, 8.0*ITERS, "FMA");
  run("ffma2", [&]{k_ffma2<<<blocks,threads>>>(out,1.0001f,0.5f);}, 16.0*ITERS, "FMA");
  run("ffma2_dist", [&]{k_ffma2_distinct<<<blocks,threads>>>(out,1.0f,0.5f);}, 16.0*ITERS, "FMA");
  run("ffma_dist", [&]{k_ffma_distinct<<<blocks,threads>>>(out,1.0f,0.5f);}, 8.0*ITERS, "FMA");
  run("fmul2_dist", [&]{k_fmul2_distinct<<<blocks,threads>>>(out,1.0f);}, 16.0*ITERS, "MUL");
  run("rsqrt", [&]{k_rsqrt<<<blocks,threads>>>(out,1.0f);}, 8.0*ITERS, "op");
  run("dfma", [&]{k_dfma<<<blocks,threads>>>((double*)out,1.0000001,0.5);}, 8.0*ITERS, "FMA");
  run("shfl", [&]{k_shfl<<<blocks,threads>>>(out,1.0f);}, 4.0*ITERS, "op");
  cudaError_t err = cudaGetLastError(); printf("status: %s\n", cudaGetErrorString(err));
  return err != cudaSuccess;
}
