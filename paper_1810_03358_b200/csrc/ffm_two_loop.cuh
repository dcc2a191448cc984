// ffm_two_loop.cuh -- the L-BFGS two-loop recursion (ffmin/optimizers/
// lbfgs.py:53-75, Algorithm 3) of a short vector by one block of 256
// threads: the ring pairs staged in shared memory once, q in registers, so
// its 2 m + 1 dependent phases cost block reductions instead of L2 round
// trips.  Element order, fma sequence and reductions are those of the
// multi-phase kernel (ffm_vec.cu two_loop_body) on one block: the same bits.
// Shared by the two-loop kernel (ffm_vec.cu) and the fused L-BFGS direction
// kernel (ffm_minimize.cu).
#pragma once
#include "ffm_kernels.h"

namespace ffm {

constexpr int kTwoLoopThreads = 256;
constexpr int kTwoLoopSmallE = 8;  // elements per thread: n <= 2048

// device-driven two-loop arguments (count / slots / rho / |g| in device memory)
struct TwoLoopDevArgs {
  int64_t n;
  const int* count;
  const int* idx;
  const double* rho;
  const double* gn;
  const double* S;
  const double* Y;
  const double* g;
  double* q;
  double* part;
};

// the block sum in every thread with one barrier: warp sums to sh (a buffer
// the previous call did not use), then every thread adds the eight of them
// in the same order as two_loop_block_sum's thread 0 -- the same bits
__device__ __forceinline__ double two_loop_allreduce(double v, double* sh) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < kTwoLoopThreads / 32; ++w) s += sh[w];
  return s;
}

__device__ __forceinline__ double two_loop_block_sum(double v, double* sh) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < kTwoLoopThreads / 32; ++w) s += sh[w];
  __syncthreads();
  return s;  // thread 0
}

// d = -H g into D.q and q[] (element t + 256 e of this thread); ring: dynamic
// shared memory of 2 * count * n doubles.  count = 0: the normalised
// antigradient (lbfgs.py:53-58), d = (1 / |g|) (-g), or -g when |g| = 0.
__device__ __forceinline__ void two_loop_small_body(const TwoLoopDevArgs& D, double* ring,
                                                    double (&q)[kTwoLoopSmallE]) {
  __shared__ double rho[kMaxLbfgsPairs], alpha[kMaxLbfgsPairs];
  const int count = *D.count;
  const int n = (int)D.n;
  const int t = threadIdx.x;
  if (count == 0) {
    const double gn = *D.gn;
    const double inv = 1.0 / gn;
#pragma unroll
    for (int e = 0; e < kTwoLoopSmallE; ++e) {
      const int i = t + e * kTwoLoopThreads;
      q[e] = 0.0;
      if (i < n) {
        const double v = -D.g[i];
        q[e] = gn == 0.0 ? v : inv * v;
        D.q[i] = q[e];
      }
    }
    return;
  }
  double* sS = ring;
  double* sY = ring + (size_t)count * n;
  for (int k = 0; k < count; ++k) {
    const double* s = D.S + (int64_t)D.idx[k] * n;
    const double* y = D.Y + (int64_t)D.idx[k] * n;
    for (int i = t; i < n; i += kTwoLoopThreads) {
      sS[(size_t)k * n + i] = s[i];
      sY[(size_t)k * n + i] = y[i];
    }
  }
  if (t < count) rho[t] = D.rho[t];
#pragma unroll
  for (int e = 0; e < kTwoLoopSmallE; ++e) {
    const int i = t + e * kTwoLoopThreads;
    q[e] = i < n ? D.g[i] : 0.0;
  }
  __syncthreads();
  double a = 0.0, b = 0.0, c = 0.0;
#pragma unroll
  for (int e = 0; e < kTwoLoopSmallE; ++e) {
    const int i = t + e * kTwoLoopThreads;
    if (i < n) {
      a = fma(sS[i], q[e], a);
      b = fma(sS[i], sY[i], b);
      c = fma(sY[i], sY[i], c);
    }
  }
  // (sums on alternating buffers: one barrier per phase, every thread holds
  // the sum, the scalars computed redundantly in each thread)
  __shared__ double shb[2][kTwoLoopThreads / 32];
  int pb = 0;
  a = two_loop_allreduce(a, shb[pb]);
  pb ^= 1;
  b = two_loop_allreduce(b, shb[pb]);
  pb ^= 1;
  c = two_loop_allreduce(c, shb[pb]);
  pb ^= 1;
  double prev_sum = a;
  const double gamma = (0.0 + b) / (0.0 + c);
  for (int k = 0; k < count; ++k) {
    // (explicit roundings: no contraction whatever the unit's -fmad, as in
    // the kernels whose bits this reproduces)
    const double al = __dmul_rn(rho[k], 0.0 + prev_sum);
    if (t == 0) alpha[k] = al;  // (read in the second loop, after barriers)
    const bool last = k + 1 == count;
    const double* y = sY + (size_t)k * n;
    const double* w = last ? sY + (size_t)(count - 1) * n : sS + (size_t)(k + 1) * n;
    double acc = 0.0;
#pragma unroll
    for (int e = 0; e < kTwoLoopSmallE; ++e) {
      const int i = t + e * kTwoLoopThreads;
      if (i < n) {
        double v = fma(-al, y[i], q[e]);
        if (last) v *= gamma;
        q[e] = v;
        acc = fma(w[i], v, acc);
      }
    }
    prev_sum = two_loop_allreduce(acc, shb[pb]);
    pb ^= 1;
  }
  for (int k = count - 1; k >= 0; --k) {
    const double coef = __dsub_rn(alpha[k], __dmul_rn(rho[k], 0.0 + prev_sum));
    const double* s = sS + (size_t)k * n;
    if (k == 0) {
#pragma unroll
      for (int e = 0; e < kTwoLoopSmallE; ++e) {
        const int i = t + e * kTwoLoopThreads;
        if (i < n) {
          q[e] = -fma(coef, s[i], q[e]);
          D.q[i] = q[e];
        }
      }
      break;
    }
    const double* y2 = sY + (size_t)(k - 1) * n;
    double acc = 0.0;
#pragma unroll
    for (int e = 0; e < kTwoLoopSmallE; ++e) {
      const int i = t + e * kTwoLoopThreads;
      if (i < n) {
        const double v = fma(coef, s[i], q[e]);
        q[e] = v;
        acc = fma(y2[i], v, acc);
      }
    }
    prev_sum = two_loop_allreduce(acc, shb[pb]);
    pb ^= 1;
  }
}

}  // namespace ffm
