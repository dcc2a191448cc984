// ffm_tile.cuh -- the 128 x 32 warp tile of the O(N^2) pair sweep
// (ffmin/kernels.py:285-356 restated), shared by the super-unit kernel and
// the small-system tile kernel (ffm_pairs.cu) and by the fused small-system
// evaluation (ffm_small.cu).  All arithmetic is explicit (packed f32x2 PTX,
// or __dmul_rn / __dadd_rn / __fma_rn in FP64), so every translation unit
// produces the same bits whatever its -fmad setting.
#pragma once
#include "ffm_plan.cuh"

namespace ffm {

#ifndef FFM_MINB64
#define FFM_MINB64 2  // FP64: two CTAs per SM (<= 128 registers)
#endif
#ifndef FFM_UNROLL
#define FFM_UNROLL 32
#endif
#ifndef FFM_UNROLL64
#define FFM_UNROLL64 0  // 0: 4 with gradient, 8 energy-only (measured best)
#endif
constexpr int kStepUnroll = FFM_UNROLL;  // steps of the 32-step tile loop unrolled
constexpr int kStepUnroll64 = FFM_UNROLL64;  // FP64 (register-bound at 2 CTAs/SM)
#ifndef FFM_F64FORM
#define FFM_F64FORM 2  // FP64 energy/gradient algebra variant (see warp_tile; 2 measured best)
#endif
#ifndef FFM_RCP
#define FFM_RCP 1  // FP32 r^-2 from MUFU.RCP instead of an FMA-pipe multiply
#endif

template <typename T>
__device__ __forceinline__ typename Pk<T>::V shfl_rot(typename Pk<T>::V v, int src);

template <>
__device__ __forceinline__ Pk<float>::V shfl_rot<float>(Pk<float>::V v, int src) {
  return __shfl_sync(0xffffffffu, v, src);
}
template <>
__device__ __forceinline__ Pk<double>::V shfl_rot<double>(Pk<double>::V v, int src) {
  return {__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src)};
}

// i-side pair loads: 64-bit (fp32 pair) / 128-bit (fp64 pair) straight into
// the packed registers
template <typename T>
__device__ __forceinline__ typename Pk<T>::V ld_pair(const T* __restrict__ base, int64_t r);
template <>
__device__ __forceinline__ Pk<float>::V ld_pair<float>(const float* __restrict__ base, int64_t r) {
  return __ldg(reinterpret_cast<const unsigned long long*>(base) + r);
}
template <>
__device__ __forceinline__ Pk<double>::V ld_pair<double>(const double* __restrict__ base,
                                                          int64_t r) {
  const double2 d = __ldg(reinterpret_cast<const double2*>(base) + r);
  return {d.x, d.y};
}

// i-atom pairs held per pass: FP32 keeps both packed pairs (4 i-atoms per
// lane) live; FP64 sweeps them one after the other so the kernel fits 128
// registers and two CTAs per SM
template <typename T> struct PairsPerPass { static constexpr int value = 2; };
template <> struct PairsPerPass<double> { static constexpr int value = 1; };

// One 128 x 32 warp tile.  J/L point at the doubled 64-entry copy of the
// j-block, so step t of lane l reads entry l + t (atom (l + t) mod 32) with
// an immediate offset.  MASKED tiles carry per-lane activity bitmasks
// (diagonal i < j condition and/or special pairs); inactive pairs are
// neutralised (r2 -> 1, coefficients -> 0) so they contribute exactly zero.
template <typename T, bool GRAD, bool CUTOFF, bool MASKED, int NP, bool DOUBLED = true>
__device__ __forceinline__ void warp_tile(
    const typename Vec4T<T>::type* __restrict__ J,
    const typename Vec2T<T>::type* __restrict__ L, int lane,
    const typename Pk<T>::V (&xi)[NP], const typename Pk<T>::V (&yi)[NP],
    const typename Pk<T>::V (&zi)[NP], const typename Pk<T>::V (&qi)[NP],
    const typename Pk<T>::V (&ai)[NP], const typename Pk<T>::V (&bi)[NP],
    typename Pk<T>::V (&F)[NP][3], typename Pk<T>::V& ec2,
    typename Pk<T>::V& ev2, T* __restrict__ jacc, int jacc_stride,
    const uint32_t (&mk)[2 * NP], T cut2, T& minr2) {
  using P = Pk<T>;
  using V = typename P::V;
  V gx = P::zero(), gy = P::zero(), gz = P::zero();
  const int src = (lane + 1) & 31;
  if (DOUBLED) {  // j-block stored twice: entry lane + t is an immediate offset
    J += lane;
    L += lane;
  }
#pragma unroll(sizeof(T) == 8 ? (kStepUnroll64 ? kStepUnroll64 : (GRAD ? 4 : 8)) : kStepUnroll)
  for (int t = 0; t < 32; ++t) {
    const int jt = DOUBLED ? t : ((lane + t) & 31);
    const auto pj = J[jt];  // (-x, -y, -z, q~) of atom (lane + t) mod 32
    const auto lj = L[jt];  // (a, -b)
    // phase-separated: both pairs' geometry first, the MUFU ops issued back
    // to back, coefficient products while they are in flight
    V dx[NP], dy[NP], dz[NP], r2[NP], A[NP], nB[NP], Q[NP], ri[NP], i2[NP];
#pragma unroll
    for (int pp = 0; pp < NP; ++pp) {
      dx[pp] = P::add(xi[pp], P::bc(pj.x));
      dy[pp] = P::add(yi[pp], P::bc(pj.y));
      dz[pp] = P::add(zi[pp], P::bc(pj.z));
      r2[pp] = P::mul(dx[pp], dx[pp]);
      r2[pp] = P::fma(dy[pp], dy[pp], r2[pp]);
      r2[pp] = P::fma(dz[pp], dz[pp], r2[pp]);
    }
#pragma unroll
    for (int pp = 0; pp < NP; ++pp) {
      A[pp] = P::mul(ai[pp], P::bc(lj.x));   // s A  (the i side carries s = LjIScale<T>)
      nB[pp] = P::mul(bi[pp], P::bc(lj.y));  // -s B
      Q[pp] = P::mul(qi[pp], P::bc(pj.w));
      if (MASKED) {
        const int jj = (lane + t) & 31;
        const bool a0 = (mk[2 * pp] >> jj) & 1u;
        const bool a1 = (mk[2 * pp + 1] >> jj) & 1u;
        r2[pp] = P::make(a0 ? P::lo(r2[pp]) : T(1), a1 ? P::hi(r2[pp]) : T(1));
        A[pp] = P::make(a0 ? P::lo(A[pp]) : T(0), a1 ? P::hi(A[pp]) : T(0));
        nB[pp] = P::make(a0 ? P::lo(nB[pp]) : T(0), a1 ? P::hi(nB[pp]) : T(0));
        Q[pp] = P::make(a0 ? P::lo(Q[pp]) : T(0), a1 ? P::hi(Q[pp]) : T(0));
      }
      if constexpr (sizeof(T) == 8) minr2 = fmin(minr2, fmin(P::lo(r2[pp]), P::hi(r2[pp])));
      if (CUTOFF) {
        const bool c0 = P::lo(r2[pp]) <= cut2;
        const bool c1 = P::hi(r2[pp]) <= cut2;
        A[pp] = P::make(c0 ? P::lo(A[pp]) : T(0), c1 ? P::hi(A[pp]) : T(0));
        nB[pp] = P::make(c0 ? P::lo(nB[pp]) : T(0), c1 ? P::hi(nB[pp]) : T(0));
        Q[pp] = P::make(c0 ? P::lo(Q[pp]) : T(0), c1 ? P::hi(Q[pp]) : T(0));
      }
      ri[pp] = P::rsqrt(r2[pp]);
      // FP32: r^-2 from MUFU.RCP (the FMA pipe is the bound, XU has slack)
      // (FP64 squares r^-1 in the consumer loop below)
      constexpr bool f32 = sizeof(T) == 4;
      if (f32 && (FFM_RCP == 1 || (FFM_RCP == 2 && pp == 0))) i2[pp] = P::rcp_or_sq(r2[pp], ri[pp]);
    }
#pragma unroll
    for (int pp = 0; pp < NP; ++pp) {
      constexpr bool f32 = sizeof(T) == 4;
      if (!f32 || FFM_RCP == 0 || (FFM_RCP == 2 && pp != 0)) i2[pp] = P::mul(ri[pp], ri[pp]);
      if (f32 && FFM_RCP == 3) i2[pp] = P::rcp_or_sq(r2[pp], ri[pp]);
      const V i4 = P::mul(i2[pp], i2[pp]);
      const V i6 = P::mul(i4, i2[pp]);
      V v, ecp, pw;
      if constexpr (sizeof(T) == 4 || FFM_F64FORM == 0) {
        const V u = P::mul(A[pp], i6);     // s A / r^6
        v = P::add(u, nB[pp]);             // s (A / r^6 - B)
        ecp = P::mul(Q[pp], ri[pp]);       // C q_i q_j / r
        ec2 = P::add(ec2, ecp);
        pw = P::add(u, v);                 // s (2 A / r^6 - B)
      } else {
        // FP64: A / r^6 folded into two FMAs (shorter dependency chains on
        // the FP64 pipe; no separate A / r^6 product)
        v = P::fma(A[pp], i6, nB[pp]);
        ecp = P::mul(Q[pp], ri[pp]);
        ec2 = (FFM_F64FORM == 2) ? P::fma(Q[pp], ri[pp], ec2) : P::add(ec2, ecp);
        pw = P::fma(A[pp], i6, v);
      }
      ev2 = P::fma(v, i6, ev2);            // s (A / r^12 - B / r^6)
      if (GRAD) {
        // g = -(dE/dr)/r = (C q q / r + 12 A / r^12 - 6 B / r^6) / r^2
        V w;
        if constexpr (sizeof(T) == 4) {
          w = P::fma(pw, i6, ecp);         // s = 6: no separate scaling multiply
        } else {                           // FP64 (s = 1): measured faster this way
          const V k = P::mul(pw, i6);
          w = P::fma(k, P::bc(T(6)), ecp);
        }
        const V g = P::mul(w, i2[pp]);
        // F_i = -grad_i = g (x_i - x_j);  grad_j += g (x_i - x_j)
#if defined(FFM_PAIRFMA) && FFM_PAIRFMA
        P::fma_pair(g, dx[pp], F[pp][0], gx);
        P::fma_pair(g, dy[pp], F[pp][1], gy);
        P::fma_pair(g, dz[pp], F[pp][2], gz);
#else
        F[pp][0] = P::fma(g, dx[pp], F[pp][0]);
        F[pp][1] = P::fma(g, dy[pp], F[pp][1]);
        F[pp][2] = P::fma(g, dz[pp], F[pp][2]);
        gx = P::fma(g, dx[pp], gx);
        gy = P::fma(g, dy[pp], gy);
        gz = P::fma(g, dz[pp], gz);
#endif
      }
    }
    if (GRAD) {  // the j column moves one lane down with its atom
      gx = shfl_rot<T>(gx, src);
      gy = shfl_rot<T>(gy, src);
      gz = shfl_rot<T>(gz, src);
    }
  }
  if (GRAD) {
    // after 32 rotations lane l holds the column of j = l again
    jacc[lane] += P::lo(gx) + P::hi(gx);
    jacc[jacc_stride + lane] += P::lo(gy) + P::hi(gy);
    jacc[2 * jacc_stride + lane] += P::lo(gz) + P::hi(gz);
  }
}


// ------------------------------------------------------- small systems
// One warp per 128 x 32 tile (i-sub-block kk, global j-block mg >= 4 kk): a
// system of a few thousand atoms has a handful of super-units, which would
// leave most SMs idle and run each unit's tiles back to back on one SM; in
// tile mode every tile of the triangle runs at once.  Partials per tile:
// i-rows [tile][3][128], j-columns [tile][3][32], energies
// [batch][tile][3]; the gather sums them in a fixed order.
//
// tile_warp evaluates launch slot `slot` of batch entry bidx with one warp;
// sj / sl / jacc are that warp's private shared-memory staging (2 x 32 j
// records, 2 x 32 LJ records, 3 x 32 column accumulators).
template <typename T, bool GRAD, bool CUTOFF>
__device__ __forceinline__ void tile_warp(const NbPlanDev& plan,
                                          const typename Vec4T<T>::type* __restrict__ pos,
                                          const typename Vec2T<T>::type* __restrict__ lj,
                                          const T* __restrict__ ipos, const T* __restrict__ ilj,
                                          T* __restrict__ ipart, T* __restrict__ jpart,
                                          double* __restrict__ epart, int slot, int bidx,
                                          typename Vec4T<T>::type* sj,
                                          typename Vec2T<T>::type* sl, T* jacc) {
  using P = Pk<T>;
  using V = typename P::V;
  using V4 = typename Vec4T<T>::type;
  using V2 = typename Vec2T<T>::type;
  const int lane = threadIdx.x & 31;
  const int t = plan.tile_list ? plan.tile_list[slot] : slot;
  __syncwarp();  // a warp running several tiles: the previous tile is done with sj / sl
  const int2 tk = plan.tiles[t];
  const int kk = tk.x, mg = tk.y;
  const int ib = kk * kIB, jb = mg * kJB;
  pos += (size_t)bidx * plan.np;
  ipos += (size_t)bidx * 4 * plan.np;
  const int64_t half = plan.np >> 1;
  {
    V4 p = pos[jb + lane];
    p.x = -p.x;
    p.y = -p.y;
    p.z = -p.z;
    sj[lane] = p;
    sj[lane + 32] = p;
    V2 l = lj[jb + lane];
    l.y = -l.y;
    sl[lane] = l;
    sl[lane + 32] = l;
    if (GRAD) jacc[lane] = jacc[32 + lane] = jacc[64 + lane] = T(0);
  }
  __syncwarp();
  constexpr int NP = PairsPerPass<T>::value;
  bool masked = jb < ib + kIB;  // straddles the diagonal
  uint32_t mk[4] = {~0u, ~0u, ~0u, ~0u};
  if (masked) {
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      const int d = ib + lane + 32 * p - jb;  // pair active iff jj > d
      mk[p] = d < 0 ? ~0u : (d >= 31 ? 0u : ~((2u << d) - 1u));
    }
  }
  for (int e = plan.spt_ptr[kk]; e < plan.spt_ptr[kk + 1]; ++e) {
    if (plan.spt_m[e] == mg) {
      masked = true;
#pragma unroll
      for (int p = 0; p < 4; ++p) mk[p] &= ~plan.spt_mask[(size_t)e * kIB + 32 * p + lane];
      break;
    }
  }
  const T cut2 = T(plan.cut2);
  T minr2 = T(1e30);
  double ec = 0.0, ev = 0.0;
  for (int p0 = 0; p0 < 2; p0 += NP) {
    V xi[NP], yi[NP], zi[NP], qi[NP], ai[NP], bi[NP];
#pragma unroll
    for (int pp = 0; pp < NP; ++pp) {
      const int64_t r = (int64_t)kk * 64 + (p0 + pp) * 32 + lane;
      xi[pp] = ld_pair<T>(ipos, r);
      yi[pp] = ld_pair<T>(ipos, half + r);
      zi[pp] = ld_pair<T>(ipos, 2 * half + r);
      qi[pp] = ld_pair<T>(ipos, 3 * half + r);
      ai[pp] = ld_pair<T>(ilj, r);
      bi[pp] = ld_pair<T>(ilj, half + r);
    }
    V F[NP][3];
#pragma unroll
    for (int pp = 0; pp < NP; ++pp) F[pp][0] = F[pp][1] = F[pp][2] = P::zero();
    V ec2 = P::zero(), ev2 = P::zero();
    uint32_t mkp[2 * NP];
#pragma unroll
    for (int q = 0; q < 2 * NP; ++q) mkp[q] = mk[2 * p0 + q];
    if (masked)
      warp_tile<T, GRAD, CUTOFF, true, NP>(sj, sl, lane, xi, yi, zi, qi, ai, bi, F,
                                           ec2, ev2, jacc, kJB, mkp, cut2, minr2);
    else
      warp_tile<T, GRAD, CUTOFF, false, NP>(sj, sl, lane, xi, yi, zi, qi, ai, bi, F,
                                            ec2, ev2, jacc, kJB, mkp, cut2, minr2);
    ec += double(P::lo(ec2)) + double(P::hi(ec2));
    ev += double(P::lo(ev2)) + double(P::hi(ev2));
    if (GRAD) {
      T* ip = ipart + (size_t)t * 3 * kIB;
#pragma unroll
      for (int pp = 0; pp < NP; ++pp)
#pragma unroll
        for (int c = 0; c < 3; ++c) {  // F = -gradient
          ip[c * kIB + lane + 64 * (p0 + pp)] = -P::lo(F[pp][c]);
          ip[c * kIB + lane + 64 * (p0 + pp) + 32] = -P::hi(F[pp][c]);
        }
    }
  }
  double mr = double(minr2);
  for (int o = 16; o > 0; o >>= 1) {
    ec += __shfl_xor_sync(0xffffffffu, ec, o);
    ev += __shfl_xor_sync(0xffffffffu, ev, o);
    mr = fmin(mr, __shfl_xor_sync(0xffffffffu, mr, o));
  }
  if (lane == 0) {
    double* e = epart + ((size_t)bidx * plan.ntiles + t) * 3;
    e[0] = ec;
    e[1] = ev / LjIScale<T>::value;
    e[2] = mr;
  }
  if (GRAD) {
    __syncwarp();
    T* jp = jpart + (size_t)t * 3 * kJB;
    for (int c = 0; c < 3; ++c) jp[c * kJB + lane] = jacc[c * kJB + lane];
  }
}

}  // namespace ffm
