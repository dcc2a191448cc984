// Instruction-mix ceiling of the FP32 pair loop (tuning aid, not product):
// warp_tile's per-pair arithmetic (ffm_tile.cuh, FP32, energy + gradient,
// 4 i-atoms per lane as two packed pairs) run on register / shared-memory
// data only, at the sweep's occupancy (8-warp CTAs, 2 per SM, 128 registers),
// to see how busy this mix can keep the FMA pipe by itself:
// (j-records from the doubled shared-memory block and the j-gradient column's
// three 64-bit lane shuffles per step, as in the real loop; without the
// shuffles ptxas hoists across the unrolled steps and spills)
// Reports pairs/s and FMA-pipe lane-ops (24 per pair in the sweep's SASS) as a
// fraction of 128 / clk / SM at the clock given on the command line.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include "../../paper_1810_03358_b200/csrc/ffm_common.cuh"
using namespace ffm;
using P = Pk<float>;
using V = P::V;
constexpr int kTiles = 256;  // tiles of 32 steps per warp

__global__ void __launch_bounds__(256, 2) k_pairs(float* out, float seed) {
  __shared__ float4 sj[8][64];
  __shared__ float2 sl[8][64];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float4 p = make_float4(-(lane * 0.37f + seed), -(lane * 0.11f), -(lane * 0.23f), 0.3f);
  float2 l = make_float2(1.1f + lane * 1e-3f, -0.9f);
  sj[w][lane] = p; sj[w][lane + 32] = p; sl[w][lane] = l; sl[w][lane + 32] = l;
  __syncwarp();
  V xi[2], yi[2], zi[2], qi[2], ai[2], bi[2], F[2][3];
  for (int pp = 0; pp < 2; ++pp) {
    xi[pp] = P::make(10.f + lane + pp, 11.f + lane); yi[pp] = P::make(3.f * pp, 1.f);
    zi[pp] = P::make(2.f, 5.f + pp); qi[pp] = P::make(0.2f, -0.3f);
    ai[pp] = P::make(6.f, 6.5f); bi[pp] = P::make(1.f, 1.2f);
    F[pp][0] = F[pp][1] = F[pp][2] = P::zero();
  }
  V ec2 = P::zero(), ev2 = P::zero();
  const float4* J = sj[w] + lane;
  const float2* L = sl[w] + lane;
  const int src = (lane + 1) & 31;
  for (int tile = 0; tile < kTiles; ++tile) {
    V gx = P::zero(), gy = P::zero(), gz = P::zero();
#pragma unroll
    for (int t = 0; t < 32; ++t) {
      float4 pj;
      float2 lj;
      pj = J[t];
      lj = L[t];
      V dx[2], dy[2], dz[2], r2[2], A[2], nB[2], Q[2], ri[2], i2[2];
#pragma unroll
      for (int pp = 0; pp < 2; ++pp) {
        dx[pp] = P::add(xi[pp], P::bc(pj.x)); dy[pp] = P::add(yi[pp], P::bc(pj.y));
        dz[pp] = P::add(zi[pp], P::bc(pj.z));
        r2[pp] = P::mul(dx[pp], dx[pp]); r2[pp] = P::fma(dy[pp], dy[pp], r2[pp]);
        r2[pp] = P::fma(dz[pp], dz[pp], r2[pp]);
      }
#pragma unroll
      for (int pp = 0; pp < 2; ++pp) {
        A[pp] = P::mul(ai[pp], P::bc(lj.x)); nB[pp] = P::mul(bi[pp], P::bc(lj.y));
        Q[pp] = P::mul(qi[pp], P::bc(pj.w));
        ri[pp] = P::rsqrt(r2[pp]); i2[pp] = P::rcp_or_sq(r2[pp], ri[pp]);
      }
#pragma unroll
      for (int pp = 0; pp < 2; ++pp) {
        const V i4 = P::mul(i2[pp], i2[pp]), i6 = P::mul(i4, i2[pp]);
        const V u = P::mul(A[pp], i6), v = P::add(u, nB[pp]), ecp = P::mul(Q[pp], ri[pp]);
        ec2 = P::add(ec2, ecp);
        const V pw = P::add(u, v);
        ev2 = P::fma(v, i6, ev2);
        const V g = P::mul(P::fma(pw, i6, ecp), i2[pp]);
        F[pp][0] = P::fma(g, dx[pp], F[pp][0]); F[pp][1] = P::fma(g, dy[pp], F[pp][1]);
        F[pp][2] = P::fma(g, dz[pp], F[pp][2]);
        gx = P::fma(g, dx[pp], gx); gy = P::fma(g, dy[pp], gy); gz = P::fma(g, dz[pp], gz);
      }
      {
        gx = __shfl_sync(0xffffffffu, gx, src); gy = __shfl_sync(0xffffffffu, gy, src);
        gz = __shfl_sync(0xffffffffu, gz, src);
      }
    }
    ec2 = P::add(ec2, P::add(gx, P::add(gy, gz)));
  }
  float s = P::lo(ec2) + P::hi(ev2);
  for (int pp = 0; pp < 2; ++pp) s += P::lo(F[pp][0]) + P::hi(F[pp][1]) + P::lo(F[pp][2]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main(int argc, char** argv) {
  const double mhz = argc > 1 ? atof(argv[1]) : 1965.0;
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 2 * 8, threads = 256;  // 8 waves of the 2-CTA/SM residency
  float* out;
  cudaMalloc(&out, sizeof(float) * blocks * threads);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const double pairs = (double)blocks * threads * 4 * 32 * kTiles;  // 4 i-atoms per lane
  auto run = [&](const char* name, auto launch) {
    for (int w = 0; w < 3; ++w) launch();
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= 5;
    const double rate = pairs / (ms * 1e-3);
    printf("%-6s %8.3f ms  %.4e pairs/s  FMA-pipe %5.1f%% of 128/clk/SM at %.0f MHz\n", name, ms,
           rate, 100.0 * rate * 24 / (128.0 * sms * mhz * 1e6), mhz);
  };
  run("pairmix", [&] { k_pairs<<<blocks, threads>>>(out, 0.5f); });
  cudaError_t err = cudaGetLastError();
  printf("status: %s\n", cudaGetErrorString(err));
  return err != cudaSuccess;
}
