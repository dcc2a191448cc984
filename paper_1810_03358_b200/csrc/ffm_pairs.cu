// ffm_pairs.cu -- the O(N^2) nonbonded energy / gradient sweep.
//
// Restates ffmin/kernels.py:285-356 (_loop_nb_energy / _loop_nb_grad) for
// sm_100a.  Each unordered pair i < j is evaluated once (Newton's third law):
//
//   * a warp owns a 128 x 32 tile: every lane holds 4 i-atoms in registers
//     (two packed f32x2 pairs) and walks the 32 j-atoms of the tile along a
//     rotated diagonal, j = (lane + t) mod 32, reading them from shared memory
//     without bank conflicts; the j-gradient accumulator travels with j
//     through one lane shuffle per step, so no atomics are needed;
//   * a CTA (4 warps) owns an S x S super-unit of the upper triangle; its
//     i-gradient rows are reduced across warps in shared memory and its
//     j-gradient columns accumulate in shared memory, and both are written
//     once per unit to a partial buffer;
//   * a gather kernel (ffm_terms.cu) sums the partials of every atom in a
//     fixed order, so results are bit-identical run to run.
//
// Exclusions (1-2, 1-3) and scaled 1-4 pairs are removed from the dense sweep
// by per-tile bitmasks (only tiles near the diagonal of a chain carry any);
// the scaled ones are evaluated exactly by the sparse term kernel.
#include "ffm_kernels.h"
#include "ffm_tile.cuh"

namespace ffm {

// ------------------------------------------------ cutoff culling helpers
// boxes: [lo x, lo y, lo z, hi x, hi y, hi z] per 32-atom j-block; empty
// blocks (only padding atoms) hold +inf / -inf and never interact
template <typename T>
__device__ __forceinline__ T box_dist2(const T (&a)[6], const T (&b)[6]) {
  T d2 = T(0);
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const T gap = fmax(fmax(a[c] - b[3 + c], b[c] - a[3 + c]), T(0));
    d2 += gap * gap;
  }
  return d2 != d2 ? T(1e30) : d2;  // empty boxes give inf - inf = NaN
}

template <typename T>
__device__ __forceinline__ void box_union_seq(const T* __restrict__ bbox, int first, int count,
                                              T (&out)[6]) {
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    out[c] = T(INFINITY);
    out[3 + c] = T(-INFINITY);
  }
  for (int b = 0; b < count; ++b) {
    const T* q = bbox + (size_t)(first + b) * 6;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      out[c] = fmin(out[c], q[c]);
      out[3 + c] = fmax(out[3 + c], q[3 + c]);
    }
  }
}

template <typename T>
__device__ __forceinline__ void box_union_warp(const T* __restrict__ bbox, int first, int count,
                                               int lane, T (&out)[6]) {
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    out[c] = T(INFINITY);
    out[3 + c] = T(-INFINITY);
  }
  for (int b = lane; b < count; b += 32) {
    const T* q = bbox + (size_t)(first + b) * 6;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      out[c] = fmin(out[c], q[c]);
      out[3 + c] = fmax(out[3 + c], q[3 + c]);
    }
  }
#pragma unroll
  for (int c = 0; c < 3; ++c)
    for (int o = 16; o > 0; o >>= 1) {
      out[c] = fmin(out[c], __shfl_xor_sync(0xffffffffu, out[c], o));
      out[3 + c] = fmax(out[3 + c], __shfl_xor_sync(0xffffffffu, out[3 + c], o));
    }
}

template <typename T>
__global__ void bbox_kernel(int n, int np, int batch, const typename Vec4T<T>::type* __restrict__ pos,
                            T* __restrict__ bbox) {
  pdl_wait();
  pdl_launch_dependents();
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int nbox = np / kJB;
  if (w >= (int64_t)batch * nbox) return;
  const int64_t b = w / nbox;
  const int blk = (int)(w - b * nbox);
  const int a = blk * kJB + lane;
  const auto p = pos[b * np + a];
  const bool real = a < n;
  T lo[3] = {real ? p.x : T(INFINITY), real ? p.y : T(INFINITY), real ? p.z : T(INFINITY)};
  T hi[3] = {real ? p.x : T(-INFINITY), real ? p.y : T(-INFINITY), real ? p.z : T(-INFINITY)};
#pragma unroll
  for (int c = 0; c < 3; ++c)
    for (int o = 16; o > 0; o >>= 1) {
      lo[c] = fmin(lo[c], __shfl_xor_sync(0xffffffffu, lo[c], o));
      hi[c] = fmax(hi[c], __shfl_xor_sync(0xffffffffu, hi[c], o));
    }
  if (lane == 0) {
    T* q = bbox + (size_t)w * 6;
    q[0] = lo[0];
    q[1] = lo[1];
    q[2] = lo[2];
    q[3] = hi[0];
    q[4] = hi[1];
    q[5] = hi[2];
  }
}

cudaError_t launch_bbox(int n, int np, int batch, bool fp64, const void* pos, void* bbox,
                        cudaStream_t st) {
  const int64_t threads = (int64_t)batch * (np / kJB) * 32;
  const int blocks = (int)((threads + 255) / 256);
  count_launch();
  if (fp64)
    launch_k(bbox_kernel<double>, blocks, 256, 0, st, n, np, batch, static_cast<const double4*>(pos),
                                                static_cast<double*>(bbox));
  else
    launch_k(bbox_kernel<float>, blocks, 256, 0, st, n, np, batch, static_cast<const float4*>(pos),
                                               static_cast<float*>(bbox));
  return cudaGetLastError();
}

template <int NW>
__device__ __forceinline__ double block_sum(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < NW; ++w) s += red[w];
  return s;
}

template <int NW>
__device__ __forceinline__ double block_min(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = red[0];
  for (int w = 1; w < NW; ++w) s = fmin(s, red[w]);
  return s;
}

#ifdef FFM_UNIT_STAMPS
// tuning aid (variant builds only): globaltimer stamps of each CTA's phases
__device__ unsigned long long* g_unit_clock = nullptr;
#define FFM_STAMP(k)                                                              \
  do {                                                                            \
    if (g_unit_clock && threadIdx.x == 0 && blockIdx.y == 0) {                    \
      unsigned long long t_;                                                      \
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_));                       \
      g_unit_clock[(size_t)blockIdx.x * 16 + (k)] = t_;                           \
    }                                                                             \
  } while (0)
#else
#define FFM_STAMP(k) \
  do {               \
  } while (0)
#endif

// grid = (nunits, batch).  ipart/jpart: [nunits][3][S] gradient partials
// (GRAD only); epart: [batch][nunits][3] = (coulomb, vdw, min r^2).
#ifndef FFM_MINB
#define FFM_MINB 2
#endif
// NW warps per CTA: 8 for FP32 (two CTAs per SM), 4 for FP64 (two CTAs per
// SM, so one CTA's staging / reduction phases overlap the other's pair loop;
// one 8-warp FP64 CTA fills the register file alone -- measured 4 vs 8
// warps: 100k 11.72 -> 11.43 ms, 20k 571 -> 505 us, 10k 168 -> 159 us)
#ifndef FFM_MINB64E
#define FFM_MINB64E 3  // FP64 energy-only 4-warp CTAs per SM (no force accumulators)
#endif
// OCC > 0 overrides the CTAs per SM the registers are bounded for: FP32
// energy-only sweeps of units up to 512 atoms run three 8-warp CTAs per SM
// (79 registers, no spills; 10k atoms 45.6 -> 43.3 us, while at S = 1024
// the third CTA measured 1% slower: profiles/r01_energy_occupancy_ab.log)
template <typename T, bool GRAD, bool CUTOFF, int NW, int OCC = 0>
__global__ void __launch_bounds__(NW * 32, OCC > 0 ? OCC
                                  : sizeof(T) == 4 ? FFM_MINB * kWarps / NW
                                  : (NW == kWarps ? FFM_MINB64 : (GRAD ? 2 : FFM_MINB64E)))
nb_units_kernel(NbPlanDev plan, const typename Vec4T<T>::type* __restrict__ pos,
                const typename Vec2T<T>::type* __restrict__ lj, const T* __restrict__ ipos,
                const T* __restrict__ ilj, const T* __restrict__ bbox,
                T* __restrict__ ipart, T* __restrict__ jpart, double* __restrict__ epart) {
  pdl_wait();  // (no early pdl_launch_dependents: the dependents' waiting CTAs
               // measured 2% slower at 10k atoms than launching at completion)
  using P = Pk<T>;
  using V = typename P::V;
  using V4 = typename Vec4T<T>::type;
  using V2 = typename Vec2T<T>::type;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int kNT = NW * 32;
  __shared__ double red[NW];
  const int S = plan.S;
  V4* sj = reinterpret_cast<V4*>(smem_raw);   // [2S]: each j-block stored twice
  // FP32 stores each j-block twice (immediate-offset addressing in the hot
  // loop); FP64, bound by its pipe, stores it once so two CTAs fit an SM
  constexpr bool kDbl = sizeof(T) == 4;
  constexpr int kRep = kDbl ? 2 : 1;
  V2* sl = reinterpret_cast<V2*>(sj + kRep * S);  // [kRep S]
  T* jacc = reinterpret_cast<T*>(sl + kRep * S);  // [3][S]      (GRAD)
  T* ired = jacc + 3 * S;                      // [NW][3][kIB] (GRAD)

  FFM_STAMP(0);
  const int u = plan.unit_list ? plan.unit_list[blockIdx.x] : blockIdx.x;
  const int bidx = blockIdx.y;
  pos += (size_t)bidx * plan.np;
  ipos += (size_t)bidx * 4 * plan.np;
  const int64_t half = plan.np >> 1;
  const int2 rc = plan.unit_rc[u];
  const int i0 = rc.x * S, j0 = rc.y * S;
  const bool diag = rc.x == rc.y;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nbox = plan.np / kJB;
  if (CUTOFF) {
    // cutoff culling, unit level: if the bounding boxes of the row and
    // column blocks are farther apart than the cutoff no pair interacts;
    // the unit's partials are zeroed (the gather reads every unit)
    bbox += (size_t)bidx * nbox * 6;
    __shared__ int cull;
    if (warp == 0) {
      T r[6], c[6];
      box_union_warp<T>(bbox, i0 / kJB, S / kJB, lane, r);
      box_union_warp<T>(bbox, j0 / kJB, S / kJB, lane, c);
      if (lane == 0) cull = box_dist2<T>(r, c) > T(plan.cull2);
    }
    __syncthreads();
    if (cull) {
      if (GRAD)
        for (int x = tid; x < 3 * S; x += kNT) {
          ipart[(size_t)u * 3 * S + x] = T(0);
          jpart[(size_t)u * 3 * S + x] = T(0);
        }
      if (tid == 0) {
        double* e = epart + ((size_t)bidx * plan.nunits + u) * 3;
        e[0] = 0.0;
        e[1] = 0.0;
        e[2] = 1e30;
      }
      return;
    }
  }

  for (int e = tid; e < kRep * S; e += kNT) {
    const int a = kDbl ? j0 + (e >> 6) * kJB + (e & 31) : j0 + e;
    V4 p = pos[a];
    p.x = -p.x;
    p.y = -p.y;
    p.z = -p.z;
    sj[e] = p;
    V2 l = lj[a];
    l.y = -l.y;
    sl[e] = l;
  }
  if (GRAD)
    for (int a = tid; a < 3 * S; a += kNT) jacc[a] = T(0);
  __syncthreads();
  FFM_STAMP(1);

  double Ec = 0.0, Ev = 0.0;
  T minr2 = T(1e30);
  const T cut2 = T(plan.cut2);
  const int nsub = S / kIB, njb = S / kJB;
  constexpr int NP = PairsPerPass<T>::value;
  const int2 kr = plan.unit_ks ? plan.unit_ks[u] : make_int2(0, nsub);
  for (int ks = kr.x; ks < kr.y; ++ks) {
    const int ib = i0 + ks * kIB;
    const int kk = ib / kIB;
    const int e_beg = plan.spt_ptr[kk], e_end = plan.spt_ptr[kk + 1];
    // which j-blocks of this unit carry special pairs for these rows: one
    // bit per j-block (njb <= 32), so the tile loop tests a bit instead of
    // scanning the row's special-tile list
    uint32_t spbits = 0;
    for (int e = e_beg + lane; e < e_end; e += 32) {
      const int d = plan.spt_m[e] - j0 / kJB;
      if (d >= 0 && d < njb) spbits |= 1u << d;
    }
    spbits = __reduce_or_sync(0xffffffffu, spbits);
    T ibox[6];
    if (CUTOFF) box_union_seq<T>(bbox, ib / kJB, kIB / kJB, ibox);
    T* my = ired + warp * 3 * kIB;
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
    for (int m = warp; m < njb; m += NW) {
      const int jb = j0 + m * kJB;
      if (diag && jb + kJB <= ib) continue;  // whole tile has j < i
      if (CUTOFF) {  // tile-level culling
        T jbox[6];
        box_union_seq<T>(bbox, jb / kJB, 1, jbox);
        if (box_dist2<T>(ibox, jbox) > T(plan.cull2)) continue;
      }
      bool masked = diag && jb < ib + kIB;   // straddles the diagonal
      uint32_t mk[4] = {~0u, ~0u, ~0u, ~0u};
      if (masked) {
#pragma unroll
        for (int p = 0; p < 4; ++p) {
          const int d = ib + lane + 32 * p - jb;  // pair active iff jj > d
          mk[p] = d < 0 ? ~0u : (d >= 31 ? 0u : ~((2u << d) - 1u));
        }
      }
      const int mg = jb / kJB;
      if ((spbits >> m) & 1u) {
        for (int e = e_beg; e < e_end; ++e) {
          if (plan.spt_m[e] == mg) {
            masked = true;
#pragma unroll
            for (int p = 0; p < 4; ++p) mk[p] &= ~plan.spt_mask[(size_t)e * kIB + 32 * p + lane];
            break;
          }
        }
      }
      uint32_t mkp[2 * NP];
#pragma unroll
      for (int q = 0; q < 2 * NP; ++q) mkp[q] = mk[2 * p0 + q];
      T* jc = jacc + m * kJB;
      const V4* J = sj + m * kRep * kJB;
      const V2* L = sl + m * kRep * kJB;
      if (masked)
        warp_tile<T, GRAD, CUTOFF, true, NP, kDbl>(J, L, lane, xi, yi, zi, qi, ai, bi, F, ec2,
                                                   ev2, jc, S, mkp, cut2, minr2);
      else
        warp_tile<T, GRAD, CUTOFF, false, NP, kDbl>(J, L, lane, xi, yi, zi, qi, ai, bi, F, ec2,
                                                    ev2, jc, S, mkp, cut2, minr2);
      Ec += double(P::lo(ec2)) + double(P::hi(ec2));
      Ev += double(P::lo(ev2)) + double(P::hi(ev2));
      ec2 = P::zero();
      ev2 = P::zero();
      if (ks == 0 && m < 32) FFM_STAMP(10 + m / NW);
    }
    if (GRAD) {
#pragma unroll
      for (int pp = 0; pp < NP; ++pp) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          my[c * kIB + lane + 64 * (p0 + pp)] = P::lo(F[pp][c]);
          my[c * kIB + lane + 64 * (p0 + pp) + 32] = P::hi(F[pp][c]);
        }
      }
    }
    }  // p0
    if (ks < 8) FFM_STAMP(2 + ks);
    if (GRAD) {
      // cross-warp reduction of the i-rows of this sub-block (fixed order)
      __syncthreads();
      for (int x = tid; x < 3 * kIB; x += kNT) {
        const int c = x / kIB, a = x - c * kIB;
        T s = T(0);
#pragma unroll
        for (int w = 0; w < NW; ++w) s += ired[w * 3 * kIB + x];
        // F = -gradient
        ipart[((size_t)u * 3 + c) * S + ks * kIB + a] = -s;
      }
      __syncthreads();
    }
  }
  if (GRAD) {
    __syncthreads();
    for (int x = tid; x < 3 * S; x += kNT) jpart[(size_t)u * 3 * S + x] = jacc[x];
  }
  const double ec = block_sum<NW>(Ec, red);
  const double ev = block_sum<NW>(Ev, red) / LjIScale<T>::value;
  const double mr = block_min<NW>(double(minr2), red);
  if (tid == 0) {
    double* e = epart + ((size_t)bidx * plan.nunits + u) * 3;
    e[0] = ec;
    e[1] = ev;
    e[2] = mr;
  }
#ifdef FFM_UNIT_STAMPS
  if (g_unit_clock && tid == 0 && blockIdx.y == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
    g_unit_clock[(size_t)blockIdx.x * 16 + 15] = smid;
  }
#endif
  FFM_STAMP(14);
}

template <typename T, bool GRAD, bool CUTOFF>
__global__ void __launch_bounds__(kTileWarps * 32)
nb_tiles_kernel(NbPlanDev plan, const typename Vec4T<T>::type* __restrict__ pos,
                const typename Vec2T<T>::type* __restrict__ lj, const T* __restrict__ ipos,
                const T* __restrict__ ilj, T* __restrict__ ipart, T* __restrict__ jpart,
                double* __restrict__ epart) {
  pdl_wait();
  pdl_launch_dependents();
  __shared__ TileSmem<T> sm;
  tile_cta<T, GRAD, CUTOFF>(plan, pos, lj, ipos, ilj, ipart, jpart, epart, blockIdx.x, blockIdx.y,
                            sm);
}

template <typename T, bool GRAD, bool CUTOFF>
static cudaError_t launch_tiles_t(const NbPlanDev& plan, const void* pos, const void* lj,
                                  const void* ipos, const void* ilj, void* ipart, void* jpart,
                                  double* epart, int batch, cudaStream_t st) {
  if (plan.nlaunch == 0) return cudaSuccess;
  dim3 grid(plan.nlaunch, batch);  // one CTA per tile
  count_launch();
  launch_k(nb_tiles_kernel<T, GRAD, CUTOFF>, grid, kTileWarps * 32, 0, st, 
      plan, static_cast<const typename Vec4T<T>::type*>(pos),
      static_cast<const typename Vec2T<T>::type*>(lj), static_cast<const T*>(ipos),
      static_cast<const T*>(ilj), static_cast<T*>(ipart), static_cast<T*>(jpart), epart);
  return cudaGetLastError();
}

size_t nb_smem_bytes(int S, bool fp64, bool grad, int nw) {
  const size_t t = fp64 ? 8 : 4;
  size_t b = (size_t)(fp64 ? 1 : 2) * S * (4 * t + 2 * t);  // j-block copies, see nb_units_kernel
  if (grad) b += (size_t)3 * S * t + (size_t)nw * 3 * kIB * t;
  return b;
}

template <typename T, bool GRAD, bool CUTOFF, int NW, int OCC = 0>
static cudaError_t launch_nb_w(const NbPlanDev& plan, const void* pos, const void* lj,
                               const void* ipos, const void* ilj, const void* bbox,
                               void* ipart, void* jpart, double* epart, int batch,
                               cudaStream_t st) {
  const size_t smem = nb_smem_bytes(plan.S, sizeof(T) == 8, GRAD, NW);
  auto k = nb_units_kernel<T, GRAD, CUTOFF, NW, OCC>;
  // opt in once, for the largest super-unit (not a stream operation, so it
  // must not sit inside a graph capture)
  static int opted = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (opted != dev) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)nb_smem_bytes(1024, sizeof(T) == 8, GRAD, NW));
    if (e != cudaSuccess) return e;
    opted = dev;
  }
  if (plan.nlaunch == 0) return cudaSuccess;
  dim3 grid(plan.nlaunch, batch);
  count_launch(), launch_k(k, grid, NW * 32, smem, st, plan, static_cast<const typename Vec4T<T>::type*>(pos),
                                  static_cast<const typename Vec2T<T>::type*>(lj),
                                  static_cast<const T*>(ipos), static_cast<const T*>(ilj),
                                  static_cast<const T*>(bbox), static_cast<T*>(ipart),
                                  static_cast<T*>(jpart), epart);
  return cudaGetLastError();
}

// warps per CTA of a sweep of super-unit edge S and nlaunch units
// (FFM_F64_WARPS / FFM_F32_WARPS = 4 / 8 force one: tuning aid)
#ifndef FFM_F64_NW4_MAXS
#define FFM_F64_NW4_MAXS 1024
#endif
// FP32: 4-warp CTAs (four per SM) only for many 256-atom units -- measured
// (tools/mid_sweep.py, FFM_F32_WARPS A/B): 20k atoms (3160 units) 219 ->
// 205 us; 10k (820 units) and S = 512 (30k) unchanged or slower
int nb_warps(int S, bool fp64, int nlaunch) {
  if (!fp64) {
    static const int forced32 = [] {
      const char* f = getenv("FFM_F32_WARPS");
      return f ? atoi(f) : 0;
    }();
    if (forced32 == kWarps || (forced32 == 4 && S <= 512)) return forced32;
    if (S > 256) return kWarps;
    return nlaunch >= 2000 ? 4 : kWarps;
  }
  static const int forced = [] {
    const char* f = getenv("FFM_F64_WARPS");
    return f ? atoi(f) : 0;
  }();
  if (forced == 4 || forced == kWarps) return forced;
  return S <= FFM_F64_NW4_MAXS ? 4 : kWarps;
}

template <typename T, bool GRAD, bool CUTOFF>
static cudaError_t launch_nb_t(const NbPlanDev& plan, const void* pos, const void* lj,
                               const void* ipos, const void* ilj, const void* bbox,
                               void* ipart, void* jpart, double* epart, int batch,
                               cudaStream_t st) {
  if constexpr (sizeof(T) == 4 && !GRAD)
    if (plan.S <= 512)
      return launch_nb_w<T, GRAD, CUTOFF, kWarps, 3>(plan, pos, lj, ipos, ilj, bbox, ipart, jpart,
                                                     epart, batch, st);
  if (nb_warps(plan.S, sizeof(T) == 8, plan.nlaunch) == 4)
    return launch_nb_w<T, GRAD, CUTOFF, 4>(plan, pos, lj, ipos, ilj, bbox, ipart, jpart, epart,
                                           batch, st);
  return launch_nb_w<T, GRAD, CUTOFF, kWarps>(plan, pos, lj, ipos, ilj, bbox, ipart, jpart,
                                              epart, batch, st);
}

cudaError_t launch_nb(const NbPlanDev& plan, bool fp64, bool grad, const void* pos,
                      const void* lj, const void* ipos, const void* ilj, const void* bbox,
                      void* ipart, void* jpart, double* epart, int batch, cudaStream_t st) {
  const bool cut = plan.has_cutoff != 0;
  if (plan.ntiles > 0) {  // small system: tile-parallel sweep
#define FFM_NT(T, G, C) \
  return launch_tiles_t<T, G, C>(plan, pos, lj, ipos, ilj, ipart, jpart, epart, batch, st)
    if (fp64) {
      if (grad) { if (cut) FFM_NT(double, true, true); else FFM_NT(double, true, false); }
      else { if (cut) FFM_NT(double, false, true); else FFM_NT(double, false, false); }
    } else {
      if (grad) { if (cut) FFM_NT(float, true, true); else FFM_NT(float, true, false); }
      else { if (cut) FFM_NT(float, false, true); else FFM_NT(float, false, false); }
    }
#undef FFM_NT
  }
#define FFM_NB(T, G, C) \
  return launch_nb_t<T, G, C>(plan, pos, lj, ipos, ilj, bbox, ipart, jpart, epart, batch, st)
  if (fp64) {
    if (grad) { if (cut) FFM_NB(double, true, true); else FFM_NB(double, true, false); }
    else { if (cut) FFM_NB(double, false, true); else FFM_NB(double, false, false); }
  } else {
    if (grad) { if (cut) FFM_NB(float, true, true); else FFM_NB(float, true, false); }
    else { if (cut) FFM_NB(float, false, true); else FFM_NB(float, false, false); }
  }
#undef FFM_NB
}

}  // namespace ffm

#ifdef FFM_UNIT_STAMPS
extern "C" int ffm_debug_unit_clock(void* clock_d) {
  return (int)cudaMemcpyToSymbol(ffm::g_unit_clock, &clock_d, sizeof(void*));
}
#endif
