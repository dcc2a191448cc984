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
#define FFM_MINB64 1  // FP64 8-warp CTAs (FFM_F64_WARPS=8 only): one per SM (~245 registers)
#endif
#ifndef FFM_UNROLL
#define FFM_UNROLL 32
#endif
#ifndef FFM_UNROLL64
#define FFM_UNROLL64 8  // FP64 steps unrolled (measured best with four i-atoms per lane)
#endif
constexpr int kStepUnroll = FFM_UNROLL;  // steps of the 32-step tile loop unrolled
constexpr int kStepUnroll64 = FFM_UNROLL64;  // FP64 (register-bound at 2 CTAs/SM)
#ifndef FFM_F64FORM
#define FFM_F64FORM 2  // FP64 energy/gradient algebra variant (see warp_tile; 2 measured best)
#endif
#ifndef FFM_RCP
#define FFM_RCP 1  // FP32 r^-2 from MUFU.RCP instead of an FMA-pipe multiply
#endif
#ifndef FFM_EFACTOR
#define FFM_EFACTOR 1  // energy-only tiles: i-side parameters factored out (warp_tile_energy)
#endif

// FP64 min r^2 of a tile (the close-contact flag that sends an evaluation
// to the exact finder).  FFM_F64IMIN: tracked on the high words of the
// non-negative doubles with integer min (ALU pipe, not the FP64 pipe); the
// result (low word 0) is <= the true minimum, so the flag stays conservative.
#ifndef FFM_F64IMIN
#define FFM_F64IMIN 1  // (FP64 100k energy-only sweep 6.50 -> 5.67 ms: the fmin pair was on the FP64 pipe)
#endif
__device__ __forceinline__ double min_r2_track(double m, double a, double b) {
#if FFM_F64IMIN
  const int h = min(min(__double2hiint(a), __double2hiint(b)), __double2hiint(m));
  return __hiloint2double(h, 0);
#else
  return fmin(m, fmin(a, b));
#endif
}

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

// i-atom pairs held per pass: both packed pairs (4 i-atoms per lane) live.
// FP64 then needs ~245 registers, i.e. eight warps per SM (two 4-warp
// CTAs: nb_warps), and the doubled independent work per step outruns two
// CTAs of two i-atoms per lane (100k atoms: 12.80 -> 11.71 ms with 8 steps
// unrolled, 11.43 ms as two 4-warp CTAs; tools/build_lib_variant.sh A/B:
// NP64, MINB64, UNROLL64)
template <typename T> struct PairsPerPass { static constexpr int value = 2; };
#ifndef FFM_NP64
#define FFM_NP64 2
#endif
template <> struct PairsPerPass<double> { static constexpr int value = FFM_NP64; };

// Energy-only 128 x 32 tile (line-search probes, batched candidates,
// energy_total): the i-side parameters are factored out of the pair sums,
//   E_coul(i) = q~_i sum_j q~_j / r,   s E_lj(i) = s a_i sum_j a_j / r^12 - s b_i sum_j b_j / r^6,
// so a pair costs the geometry, r^-1 (MUFU.RSQ), r^-2 = (r^-1)^2, r^-6,
// r^-12 and three accumulations with broadcast j operands: 13 FMA-pipe
// lane-ops and one MUFU instead of 15 and two, without the per-pair
// coefficient products (100k FP32 2.46 -> 2.19 ms, FP64 6.98 -> 6.47 ms;
// profiles/r02_energy_factor_ab.log).  Inactive pairs (mask, cutoff) get
// r^-1 = r^-2 = 0.  The three per-i-atom sums are folded into ec2 / ev2 at
// the end of the tile.
#ifndef FFM_ERCP
#define FFM_ERCP 0  // FP32 energy-only r^-2 via MUFU.RCP: 0 none (measured best), 1 all, 2 first pair
#endif
template <typename T, bool CUTOFF, bool MASKED, int NP, bool DOUBLED, int UNR, int NSTEP>
__device__ __forceinline__ void warp_tile_energy(
    const typename Vec4T<T>::type* __restrict__ J,
    const typename Vec2T<T>::type* __restrict__ L, int lane,
    const typename Pk<T>::V (&xi)[NP], const typename Pk<T>::V (&yi)[NP],
    const typename Pk<T>::V (&zi)[NP], const typename Pk<T>::V (&qi)[NP],
    const typename Pk<T>::V (&ai)[NP], const typename Pk<T>::V (&bi)[NP],
    typename Pk<T>::V& ec2, typename Pk<T>::V& ev2, const uint32_t (&mk)[2 * NP], T cut2,
    T& minr2, int t0) {
  using P = Pk<T>;
  using V = typename P::V;
  constexpr bool f32 = sizeof(T) == 4;
  V sc[NP], sa[NP], sb[NP];
#pragma unroll
  for (int pp = 0; pp < NP; ++pp) sc[pp] = sa[pp] = sb[pp] = P::zero();
  if (DOUBLED) {
    J += lane + t0;
    L += lane + t0;
  }
#pragma unroll(UNR ? UNR : sizeof(T) == 8 ? (kStepUnroll64 ? kStepUnroll64 : 8) : kStepUnroll)
  for (int ts = 0; ts < NSTEP; ++ts) {
    const int t = t0 + ts;
    const int jt = DOUBLED ? ts : ((lane + t) & 31);
    const auto pj = J[jt];  // (-x, -y, -z, q~) of atom (lane + t) mod 32
    const auto lj = L[jt];  // (a, -b)
    V r2[NP], ri[NP], i2[NP];
#pragma unroll
    for (int pp = 0; pp < NP; ++pp) {
      const V dx = P::add(xi[pp], P::bc(pj.x));
      const V dy = P::add(yi[pp], P::bc(pj.y));
      const V dz = P::add(zi[pp], P::bc(pj.z));
      r2[pp] = P::mul(dx, dx);
      r2[pp] = P::fma(dy, dy, r2[pp]);
      r2[pp] = P::fma(dz, dz, r2[pp]);
    }
#pragma unroll
    for (int pp = 0; pp < NP; ++pp) {
      bool a0 = true, a1 = true;
      if (MASKED) {
        const int jj = (lane + t) & 31;
        a0 = (mk[2 * pp] >> jj) & 1u;
        a1 = (mk[2 * pp + 1] >> jj) & 1u;
        r2[pp] = P::make(a0 ? P::lo(r2[pp]) : T(1), a1 ? P::hi(r2[pp]) : T(1));
      }
      if constexpr (sizeof(T) == 8) minr2 = min_r2_track(minr2, P::lo(r2[pp]), P::hi(r2[pp]));
      if (CUTOFF) {
        a0 = a0 && P::lo(r2[pp]) <= cut2;
        a1 = a1 && P::hi(r2[pp]) <= cut2;
      }
      ri[pp] = P::rsqrt_e(r2[pp]);
      const bool rcp = f32 && (FFM_ERCP == 1 || (FFM_ERCP == 2 && pp == 0));
      if (rcp) i2[pp] = P::rcp_or_sq(r2[pp], ri[pp]);
      if (MASKED || CUTOFF) {
        ri[pp] = P::make(a0 ? P::lo(ri[pp]) : T(0), a1 ? P::hi(ri[pp]) : T(0));
        if (rcp) i2[pp] = P::make(a0 ? P::lo(i2[pp]) : T(0), a1 ? P::hi(i2[pp]) : T(0));
      }
    }
#pragma unroll
    for (int pp = 0; pp < NP; ++pp) {
      const bool rcp = f32 && (FFM_ERCP == 1 || (FFM_ERCP == 2 && pp == 0));
      if (!rcp) i2[pp] = P::mul(ri[pp], ri[pp]);
      const V i4 = P::mul(i2[pp], i2[pp]);
      const V i6 = P::mul(i4, i2[pp]);
      const V i12 = P::mul(i6, i6);
      sc[pp] = P::fma(P::bc(pj.w), ri[pp], sc[pp]);   // sum q~_j / r
      sa[pp] = P::fma(P::bc(lj.x), i12, sa[pp]);      // sum a_j / r^12
      sb[pp] = P::fma(P::bc(lj.y), i6, sb[pp]);       // -sum b_j / r^6
    }
  }
#pragma unroll
  for (int pp = 0; pp < NP; ++pp) {
    ec2 = P::fma(qi[pp], sc[pp], ec2);
    ev2 = P::fma(ai[pp], sa[pp], ev2);
    ev2 = P::fma(bi[pp], sb[pp], ev2);
  }
}

// One 128 x 32 warp tile.  J/L point at the doubled 64-entry copy of the
// j-block, so step t of lane l reads entry l + t (atom (l + t) mod 32) with
// an immediate offset.  MASKED tiles carry per-lane activity bitmasks
// (diagonal i < j condition and/or special pairs); inactive pairs are
// neutralised (r2 -> 1, coefficients -> 0) so they contribute exactly zero.
//
// NSTEP < 32 evaluates only steps t0 .. t0 + NSTEP - 1 of the rotation (the
// small-system CTA tile splits one tile over four warps); the j-gradient
// column then ends in lane (j - t0 - NSTEP) mod 32 and is added to
// jacc[(lane + t0 + NSTEP) mod 32].
template <typename T, bool GRAD, bool CUTOFF, bool MASKED, int NP, bool DOUBLED = true,
          int UNR = 0, int NSTEP = 32>
__device__ __forceinline__ void warp_tile(
    const typename Vec4T<T>::type* __restrict__ J,
    const typename Vec2T<T>::type* __restrict__ L, int lane,
    const typename Pk<T>::V (&xi)[NP], const typename Pk<T>::V (&yi)[NP],
    const typename Pk<T>::V (&zi)[NP], const typename Pk<T>::V (&qi)[NP],
    const typename Pk<T>::V (&ai)[NP], const typename Pk<T>::V (&bi)[NP],
    typename Pk<T>::V (&F)[NP][3], typename Pk<T>::V& ec2,
    typename Pk<T>::V& ev2, T* __restrict__ jacc, int jacc_stride,
    const uint32_t (&mk)[2 * NP], T cut2, T& minr2, int t0 = 0) {
  using P = Pk<T>;
  using V = typename P::V;
#if FFM_EFACTOR
  if constexpr (!GRAD) {
    warp_tile_energy<T, CUTOFF, MASKED, NP, DOUBLED, UNR, NSTEP>(
        J, L, lane, xi, yi, zi, qi, ai, bi, ec2, ev2, mk, cut2, minr2, t0);
    return;
  }
#endif
  V gx = P::zero(), gy = P::zero(), gz = P::zero();
  const int src = (lane + 1) & 31;
  if (DOUBLED) {  // j-block stored twice: entry lane + t is an immediate offset
    J += lane + t0;
    L += lane + t0;
  }
#pragma unroll(UNR ? UNR : sizeof(T) == 8 ? (kStepUnroll64 ? kStepUnroll64 : (GRAD ? 4 : 8)) : kStepUnroll)
  for (int ts = 0; ts < NSTEP; ++ts) {
    const int t = t0 + ts;
    const int jt = DOUBLED ? ts : ((lane + t) & 31);
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
      if constexpr (sizeof(T) == 8) minr2 = min_r2_track(minr2, P::lo(r2[pp]), P::hi(r2[pp]));
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
        if constexpr (sizeof(T) == 4 || FFM_F64SCALE) {
          w = P::fma(pw, i6, ecp);         // s = 6: no separate scaling multiply
        } else {                           // FP64 with FFM_F64SCALE = 0 (s = 1)
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
    const int jl = NSTEP == 32 ? lane : ((lane + t0 + NSTEP) & 31);
    jacc[jl] += P::lo(gx) + P::hi(gx);
    jacc[jacc_stride + jl] += P::lo(gy) + P::hi(gy);
    jacc[2 * jacc_stride + jl] += P::lo(gz) + P::hi(gz);
  }
}


// ------------------------------------------------------- small systems
// One CTA of kTileWarps warps per 128 x 32 tile (i-sub-block kk, global
// j-block mg >= 4 kk).  A system of a few thousand atoms has a handful of
// super-units (most SMs idle) and, even in tiles, so few that each runs
// alone on its SM sub-partition: the tile's 32 rotation steps are then a
// latency chain.  Splitting them over the CTA's warps (warp q evaluates
// steps 8q .. 8q + 7 of the same tile) cuts that chain four-fold.  Warp
// partials (i-rows, j-columns, energies) are combined in a fixed order, so
// results are bit-identical run to run.  Partials per tile: i-rows
// [tile][3][128], j-columns [tile][3][32], energies [batch][tile][3]; the
// gather sums them in a fixed order.
constexpr int kTileWarps = 4;
constexpr int kTileSteps = 32 / kTileWarps;

template <typename T>
struct TileSmem {
  typename Vec4T<T>::type sj[2 * kJB];
  typename Vec2T<T>::type sl[2 * kJB];
  T jacc[kTileWarps][3 * kJB];
  T fred[kTileWarps][3 * kIB];
  double ered[kTileWarps][3];
};

// The compute and epilogue of one tile once the CTA has staged its j-block
// (sm.sj / sm.sl, negated, stored twice), zeroed sm.jacc and passed a
// barrier, with the lane's four i-atoms and masks in registers: warp q
// evaluates rotation steps 8q .. 8q + 7; warp partials are combined in warp
// order (block-uniform, contains __syncthreads).
template <typename T, bool GRAD, bool CUTOFF>
__device__ __forceinline__ void tile_body(const NbPlanDev& plan, TileSmem<T>& sm,
                                          const typename Pk<T>::V (&xi)[2],
                                          const typename Pk<T>::V (&yi)[2],
                                          const typename Pk<T>::V (&zi)[2],
                                          const typename Pk<T>::V (&qi)[2],
                                          const typename Pk<T>::V (&ai)[2],
                                          const typename Pk<T>::V (&bi)[2],
                                          const uint32_t (&mk)[4], bool masked, int t, int bidx,
                                          T* __restrict__ ipart, T* __restrict__ jpart,
                                          double* __restrict__ epart) {
  using P = Pk<T>;
  using V = typename P::V;
  constexpr int NP = 2;
  const int lane = threadIdx.x & 31, q = threadIdx.x >> 5;
  const T cut2 = T(plan.cut2);
  T minr2 = T(1e30);
  double ec = 0.0, ev = 0.0;
  T* jacc = sm.jacc[q];
  const int t0 = q * kTileSteps;
  {
    V F[NP][3];
#pragma unroll
    for (int pp = 0; pp < NP; ++pp) F[pp][0] = F[pp][1] = F[pp][2] = P::zero();
    V ec2 = P::zero(), ev2 = P::zero();
    if (masked)
      warp_tile<T, GRAD, CUTOFF, true, NP, true, kTileSteps, kTileSteps>(
          sm.sj, sm.sl, lane, xi, yi, zi, qi, ai, bi, F, ec2, ev2, jacc, kJB, mk, cut2, minr2,
          t0);
    else
      warp_tile<T, GRAD, CUTOFF, false, NP, true, kTileSteps, kTileSteps>(
          sm.sj, sm.sl, lane, xi, yi, zi, qi, ai, bi, F, ec2, ev2, jacc, kJB, mk, cut2, minr2,
          t0);
    ec += double(P::lo(ec2)) + double(P::hi(ec2));
    ev += double(P::lo(ev2)) + double(P::hi(ev2));
    if (GRAD) {
#pragma unroll
      for (int pp = 0; pp < NP; ++pp)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          sm.fred[q][c * kIB + lane + 64 * pp] = P::lo(F[pp][c]);
          sm.fred[q][c * kIB + lane + 64 * pp + 32] = P::hi(F[pp][c]);
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
    sm.ered[q][0] = ec;
    sm.ered[q][1] = ev;
    sm.ered[q][2] = mr;
  }
  __syncthreads();
  const int tid = threadIdx.x;
  if (tid == 0) {
    double e0 = 0.0, e1 = 0.0, e2 = sm.ered[0][2];
#pragma unroll
    for (int w = 0; w < kTileWarps; ++w) {
      e0 += sm.ered[w][0];
      e1 += sm.ered[w][1];
      e2 = fmin(e2, sm.ered[w][2]);
    }
    double* e = epart + ((size_t)bidx * plan.ntiles + t) * 3;
    e[0] = e0;
    e[1] = e1 / LjIScale<T>::value;
    e[2] = e2;
  }
  if (GRAD) {
    // F = -gradient; warp partials summed in warp order
    T* ip = ipart + (size_t)t * 3 * kIB;
    for (int x = tid; x < 3 * kIB; x += kTileWarps * 32) {
      T f = sm.fred[0][x];
#pragma unroll
      for (int w = 1; w < kTileWarps; ++w) f += sm.fred[w][x];
      ip[x] = -f;
    }
    T* jp = jpart + (size_t)t * 3 * kJB;
    if (tid < 3 * kJB) {
      T g = sm.jacc[0][tid];
#pragma unroll
      for (int w = 1; w < kTileWarps; ++w) g += sm.jacc[w][tid];
      jp[tid] = g;
    }
  }
}

// diagonal mask of a tile (pair (i, j) active iff j > i) for the lane's rows
__device__ __forceinline__ bool tile_diag_mask(int ib, int jb, int lane, uint32_t (&mk)[4]) {
  const bool masked = jb < ib + kIB;  // straddles the diagonal
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const int d = ib + lane + 32 * p - jb;  // pair active iff jj > d
    mk[p] = !masked || d < 0 ? ~0u : (d >= 31 ? 0u : ~((2u << d) - 1u));
  }
  return masked;
}

// The pair record of atom a straight from the evaluation's coordinates:
// the values the packing pass writes (pack_item / pad_kernel)
template <typename T>
__device__ __forceinline__ void atom_record(const CoordSrc& cs, const double* __restrict__ qt,
                                            int n, int a, T& x, T& y, T& z, T& w) {
  if (a < n) {
    x = T(cs.at(3 * (int64_t)a));
    y = T(cs.at(3 * (int64_t)a + 1));
    z = T(cs.at(3 * (int64_t)a + 2));
    w = T(qt[a]);
  } else {
    x = T(1.0e4 + 10.0 * (double)(a - n));
    y = T(1.0e4);
    z = T(1.0e4);
    w = T(0);
  }
}

// tile_cta evaluates launch slot `slot` of batch entry bidx with the whole
// CTA (kTileWarps warps; block-uniform call, contains __syncthreads).
// FROMX: positions and charges come straight from the coordinates (cs, qt)
// instead of the packed records pos / ipos (the fused evaluation of tiny
// systems, which so skips its packing pass and the barrier after it).
template <typename T, bool GRAD, bool CUTOFF, bool FROMX = false>
__device__ __forceinline__ void tile_cta(const NbPlanDev& plan,
                                         const typename Vec4T<T>::type* __restrict__ pos,
                                         const typename Vec2T<T>::type* __restrict__ lj,
                                         const T* __restrict__ ipos, const T* __restrict__ ilj,
                                         T* __restrict__ ipart, T* __restrict__ jpart,
                                         double* __restrict__ epart, int slot, int bidx,
                                         TileSmem<T>& sm, CoordSrc cs = {nullptr, nullptr, 0.0},
                                         const double* __restrict__ qt = nullptr) {
  using P = Pk<T>;
  using V = typename P::V;
  using V4 = typename Vec4T<T>::type;
  using V2 = typename Vec2T<T>::type;
  const int lane = threadIdx.x & 31, q = threadIdx.x >> 5;
  const int t = plan.tile_list ? plan.tile_list[slot] : slot;
  __syncthreads();  // a CTA running several tiles: the previous one is done with sm
  // a lone tile is latency-bound: one round trip for the tile record (its
  // special-pair mask entry resolved on the host), then every load the tile
  // needs -- j-block staging, the special-pair mask, the i-rows -- at once
  const int4 tk = plan.tiles[t];
  const int kk = tk.x, mg = tk.y, spe = tk.z;
  const int ib = kk * kIB, jb = mg * kJB;
  pos += (size_t)bidx * plan.np;
  ipos += (size_t)bidx * 4 * plan.np;
  const int64_t half = plan.np >> 1;
  if (q == 0) {
    V4 p;
    if constexpr (FROMX) atom_record<T>(cs, qt, plan.n, jb + lane, p.x, p.y, p.z, p.w);
    else p = pos[jb + lane];
    p.x = -p.x;
    p.y = -p.y;
    p.z = -p.z;
    sm.sj[lane] = p;
    sm.sj[lane + 32] = p;
  } else if (q == 1) {
    V2 l = lj[jb + lane];
    l.y = -l.y;
    sm.sl[lane] = l;
    sm.sl[lane + 32] = l;
  }
  static_assert(PairsPerPass<T>::value == 2, "a tile lane holds its four i-atoms in one pass");
  V xi[2], yi[2], zi[2], qi[2], ai[2], bi[2];
#pragma unroll
  for (int pp = 0; pp < 2; ++pp) {
    const int64_t r = (int64_t)kk * 64 + pp * 32 + lane;
    if constexpr (FROMX) {  // atoms (128 kk + 64 pp + lane, + 32): ipos_index's pair
      T x0, y0, z0, w0, x1, y1, z1, w1;
      const int a0 = ib + 64 * pp + lane;
      atom_record<T>(cs, qt, plan.n, a0, x0, y0, z0, w0);
      atom_record<T>(cs, qt, plan.n, a0 + 32, x1, y1, z1, w1);
      xi[pp] = P::make(x0, x1);
      yi[pp] = P::make(y0, y1);
      zi[pp] = P::make(z0, z1);
      qi[pp] = P::make(w0, w1);
    } else {
      xi[pp] = ld_pair<T>(ipos, r);
      yi[pp] = ld_pair<T>(ipos, half + r);
      zi[pp] = ld_pair<T>(ipos, 2 * half + r);
      qi[pp] = ld_pair<T>(ipos, 3 * half + r);
    }
    ai[pp] = ld_pair<T>(ilj, r);
    bi[pp] = ld_pair<T>(ilj, half + r);
  }
  uint32_t mk[4];
  bool masked = tile_diag_mask(ib, jb, lane, mk);
  if (spe >= 0) {  // this tile's special pairs (excluded / scaled)
    masked = true;
#pragma unroll
    for (int p = 0; p < 4; ++p) mk[p] &= ~plan.spt_mask[(size_t)spe * kIB + 32 * p + lane];
  }
  if (GRAD) sm.jacc[q][lane] = sm.jacc[q][32 + lane] = sm.jacc[q][64 + lane] = T(0);
  __syncthreads();  // sj / sl staged
  tile_body<T, GRAD, CUTOFF>(plan, sm, xi, yi, zi, qi, ai, bi, mk, masked, t, bidx, ipart, jpart,
                             epart);
}

}  // namespace ffm
