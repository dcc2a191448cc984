// Instruction-mix ceiling of the pair loop (tuning aid, not product): the
// sweep's own warp_tile (ffm_tile.cuh, energy + gradient, unmasked, 4 i-atoms
// per lane) called tile after tile on a shared-memory j-block restaged per
// tile, at the
// sweep's occupancy (FP32: 8-warp CTAs, 2 per SM; FP64: 4-warp CTAs, 2 per
// SM) with no global memory traffic, masks, special-tile lookups, unit
// staging or cross-warp reductions.  Reports pairs/s and the pipe fraction
// it implies: FP32 24 FMA-pipe lane-ops per pair of 128 / clk / SM, FP64 32
// FP64-pipe ops per pair of 64 / clk / SM, at the clock given (MHz).
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include "../../paper_1810_03358_b200/csrc/ffm_tile.cuh"
using namespace ffm;
constexpr int kTiles = 256;  // tiles per warp

template <typename T, int NW, bool DBL = true>
__global__ void __launch_bounds__(NW * 32, 2) k_tiles(T* out, T seed) {
  using P = Pk<T>;
  using V = typename P::V;
  using V4 = typename Vec4T<T>::type;
  using V2 = typename Vec2T<T>::type;
  __shared__ V4 sj[NW][64];
  __shared__ V2 sl[NW][64];
  __shared__ T jacc[NW][3 * 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  V4 p;
  p.x = -(lane * T(0.37) + seed);
  p.y = -(lane * T(0.11));
  p.z = -(lane * T(0.23));
  p.w = T(0.3);
  V2 l;
  l.x = T(1.1) + lane * T(1e-3);
  l.y = T(-0.9);
  sj[w][lane] = p;
  sj[w][lane + 32] = p;
  sl[w][lane] = l;
  sl[w][lane + 32] = l;
  jacc[w][lane] = jacc[w][32 + lane] = jacc[w][64 + lane] = T(0);
  __syncwarp();
  V xi[2], yi[2], zi[2], qi[2], ai[2], bi[2], F[2][3];
  for (int pp = 0; pp < 2; ++pp) {
    xi[pp] = P::make(T(10) + lane + pp, T(11) + lane);
    yi[pp] = P::make(T(3) * pp, T(1));
    zi[pp] = P::make(T(2), T(5) + pp);
    qi[pp] = P::make(T(0.2), T(-0.3));
    ai[pp] = P::make(T(6), T(6.5));
    bi[pp] = P::make(T(1), T(1.2));
    F[pp][0] = F[pp][1] = F[pp][2] = P::zero();
  }
  const uint32_t mk[4] = {~0u, ~0u, ~0u, ~0u};
  T minr2 = T(1e30);
  double acc = 0.0;
  for (int tile = 0; tile < kTiles; ++tile) {
    // a new j-block every tile (as the sweep stages one): nothing of the
    // tile's arithmetic is loop-invariant for the compiler to hoist
    p.x -= T(1e-3);
    l.x += T(1e-6);
    __syncwarp();
    sj[w][lane] = p;
    sj[w][lane + 32] = p;
    sl[w][lane] = l;
    sl[w][lane + 32] = l;
    __syncwarp();
    V ec2 = P::zero(), ev2 = P::zero();
    warp_tile<T, true, false, false, 2, DBL>(sj[w], sl[w], lane, xi, yi, zi, qi, ai, bi, F, ec2,
                                             ev2, jacc[w], 32, mk, T(0), minr2);
    acc += double(P::lo(ec2)) + double(P::hi(ev2));
    __syncwarp();
  }
  T s = T(acc) + minr2;
  for (int pp = 0; pp < 2; ++pp) s += P::lo(F[pp][0]) + P::hi(F[pp][1]) + P::lo(F[pp][2]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + jacc[w][lane];
}

int main(int argc, char** argv) {
  const double mhz = argc > 1 ? atof(argv[1]) : 1965.0;
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, sizeof(double) * sms * 2 * 8 * 256);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char* name, int blocks, int threads, double ops, double lanes,
                 auto launch) {
    for (int w = 0; w < 3; ++w) launch();
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= 5;
    const double pairs = (double)blocks * threads * 4 * 32 * kTiles;
    const double rate = pairs / (ms * 1e-3);
    printf("%-5s %8.3f ms  %.4e pairs/s  pipe %5.1f%% of %.0f/clk/SM at %.0f MHz\n", name, ms,
           rate, 100.0 * rate * ops / (lanes * sms * mhz * 1e6), lanes, mhz);
  };
  const int b32 = sms * 2 * 8, b64 = sms * 2 * 8;
  run("fp32", b32, 256, 24, 128,
      [&] { k_tiles<float, 8><<<b32, 256>>>(reinterpret_cast<float*>(out), 0.5f); });
  run("fp64", b64, 128, 32, 64, [&] { k_tiles<double, 4><<<b64, 128>>>(out, 0.5); });
  // the same at the sweep's FP64 residency (two 4-warp CTAs per SM: extra
  // dynamic shared memory keeps a third out), doubled / single j-block copy
  int maxsm = 0;
  cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, 0);
  const int pad = maxsm / 2 - 20 * 1024;
  cudaFuncSetAttribute(k_tiles<double, 4, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, pad);
  cudaFuncSetAttribute(k_tiles<double, 4, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       pad);
  run("fp64/2", b64, 128, 32, 64,
      [&] { k_tiles<double, 4, true><<<b64, 128, pad>>>(out, 0.5); });
  run("fp64/2s", b64, 128, 32, 64,
      [&] { k_tiles<double, 4, false><<<b64, 128, pad>>>(out, 0.5); });
  cudaError_t err = cudaGetLastError();
  printf("status: %s\n", cudaGetErrorString(err));
  return err != cudaSuccess;
}
