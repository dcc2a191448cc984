// ffm_device.cuh -- device-side bodies of the evaluation pipeline around the
// pair sweep (coordinate packing, bonded terms and scaled 1-4 pairs, the
// deterministic gradient gather, the energy reduction, the coincident-pair
// finder).  The stand-alone kernels of ffm_terms.cu and the fused small-system
// evaluation of ffm_small.cu run the same bodies, so both paths produce the
// same bits.  Every translation unit including this header is compiled with
// -fmad=false: the bonded-term degeneracy thresholds (ffmin/kernels.py:
// 130-140) see the same roundoff as the reference's CPU arithmetic.
#pragma once
#include <cfloat>
#include <climits>
#include "ffm_plan.cuh"

namespace ffm {

constexpr long long kSentinel = 0x7fffffffffffffffLL;

// ------------------------------------------------------------------ packing
// Two copies of the positions are written per evaluation:
//   pos  [batch][np]       Vec4 (x, y, z, q~)        -- j side, staged to smem
//   ipos [batch][4][np/2]  pairs (T, T) per component -- i side, loaded as
//        64/128-bit pairs straight into the packed registers of the pair
//        kernel: record r = k*64 + pp*32 + lane holds atoms
//        (128k + 64pp + lane, 128k + 64pp + lane + 32).
__device__ __forceinline__ int64_t ipos_index(int a, int np, int c) {
  const int k = a >> 7, i = a & 127;
  const int r = k * 64 + (i >> 6) * 32 + (i & 31);
  return ((int64_t)c * (np >> 1) + r) * 2 + ((i >> 5) & 1);
}

template <typename T>
__device__ __forceinline__ void put_atom(typename Vec4T<T>::type* pos, T* ipos, int np, int a,
                                         T x, T y, T z, T w) {
  typename Vec4T<T>::type p;
  p.x = x;
  p.y = y;
  p.z = z;
  p.w = w;
  pos[a] = p;
  ipos[ipos_index(a, np, 0)] = x;
  ipos[ipos_index(a, np, 1)] = y;
  ipos[ipos_index(a, np, 2)] = z;
  ipos[ipos_index(a, np, 3)] = w;
}

// one (batch entry, atom) item of the packing pass; item k < batch also
// resets that entry's status words
template <typename T>
__device__ __forceinline__ void pack_item(int64_t k, int n, int np, int batch,
                                          const double* __restrict__ coords,
                                          const double* __restrict__ qt,
                                          typename Vec4T<T>::type* __restrict__ pos,
                                          T* __restrict__ ipos, int64_t* __restrict__ status) {
  if (k < (int64_t)n * batch) {
    const int64_t b = k / n, a = k - b * n;
    const double* c = coords + 3 * k;
    put_atom<T>(pos + b * np, ipos + b * 4 * (int64_t)np, np, (int)a, T(c[0]), T(c[1]),
                T(c[2]), T(qt[a]));
  }
  if (status && k < batch) {
    int64_t* s = status + k * kStWords;
    s[kStNbBadI] = -1;
    s[kStNbBadJ] = -1;
    s[kStBond] = kSentinel;
    s[kStAngle] = kSentinel;
    s[kStDihedral] = kSentinel;
    s[kStNbSuspect] = 0;
    s[kStNbKey] = kSentinel;
    s[kStCount] = 0;
  }
}

// ------------------------------------------------------------- term physics
struct P3 {
  double x, y, z;
};
__device__ __forceinline__ P3 ld3(const double* c, int i) { return {c[3 * i], c[3 * i + 1], c[3 * i + 2]}; }
__device__ __forceinline__ P3 ld3(const CoordSrc& cs, int i) {
  return {cs.at(3 * (int64_t)i), cs.at(3 * (int64_t)i + 1), cs.at(3 * (int64_t)i + 2)};
}
__device__ __forceinline__ P3 sub(P3 a, P3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ __forceinline__ double dot(P3 a, P3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__device__ __forceinline__ P3 cross(P3 a, P3 b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
__device__ __forceinline__ void st3(double* f, P3 v) {
  f[0] = v.x;
  f[1] = v.y;
  f[2] = v.z;
}

// ffmin/kernels.py:52-86: K (r - r0)^2; grad variant checks r < RMIN.
__device__ inline bool bond_term(P3 ci, P3 cj, double K, double r0, bool grad, double* e, P3* gi) {
  const P3 d = sub(ci, cj);
  const double r = sqrt(dot(d, d));
  if (grad && r < kRmin) return false;
  const double dv = r - r0;
  *e = K * dv * dv;
  if (grad) {
    const double c = 2.0 * K * dv / r;
    *gi = {c * d.x, c * d.y, c * d.z};
  }
  return true;
}

// ffmin/kernels.py:89-161: K (theta - theta0)^2 at apex j.
__device__ inline bool angle_term(P3 ci, P3 cj, P3 ck, double K, double t0, bool grad, double* e,
                           P3* gi, P3* gk) {
  const P3 a = sub(ci, cj), b = sub(ck, cj);
  const double na = sqrt(dot(a, a)), nb = sqrt(dot(b, b));
  if (na < kDegenerateEps || nb < kDegenerateEps) return false;
  double u = dot(a, b) / (na * nb);
  u = u > 1.0 ? 1.0 : (u < -1.0 ? -1.0 : u);
  if (!grad) {
    const double d = acos(u) - t0;
    *e = K * d * d;
    return true;
  }
  const double sin_th = sqrt(1.0 - u * u);
  if (sin_th < kDegenerateEps) return false;
  const double d = acos(u) - t0;
  *e = K * d * d;
  const double pref = -2.0 * K * d / sin_th;
  const double nab = na * nb, naa = na * na, nbb = nb * nb;
  *gi = {pref * (b.x / nab - u * a.x / naa), pref * (b.y / nab - u * a.y / naa),
         pref * (b.z / nab - u * a.z / naa)};
  *gk = {pref * (a.x / nab - u * b.x / nbb), pref * (a.y / nab - u * b.y / nbb),
         pref * (a.z / nab - u * b.z / nbb)};
  return true;
}

// ffmin/kernels.py:164-282: OPLS cosine series on the atan2 dihedral.
__device__ inline bool dihedral_term(P3 ci, P3 cj, P3 ck, P3 cl, const double* V, bool grad,
                              double* e, P3* g) {
  const P3 b1 = sub(cj, ci), b2 = sub(ck, cj), b3 = sub(cl, ck);
  const P3 n1 = cross(b1, b2), n2 = cross(b2, b3);
  const double n1sq = dot(n1, n1), n2sq = dot(n2, n2);
  const double n1n = sqrt(n1sq), n2n = sqrt(n2sq);
  const double b2sq = dot(b2, b2), b2n = sqrt(b2sq);
  if (n1n < kDegenerateEps || n2n < kDegenerateEps || b2n < kDegenerateEps) return false;
  const P3 m = cross(n1, n2);
  const double y = dot(m, b2) / b2n;
  const double x = dot(n1, n2);
  // phi = atan2(y, x) in the reference; since m = n1 x n2 is parallel to b2,
  // x^2 + y^2 = |n1|^2 |n2|^2, so cos phi = x / (|n1| |n2|) and sin phi =
  // y / (|n1| |n2|) directly (no atan2 / sincos chains: the term blocks are
  // the latency-critical items of a small-system evaluation).  cos / sin of
  // 2 phi .. 4 phi by the angle-addition recurrences (eight libm calls in
  // the reference; they agree to a few ulp, far inside the FP64 tolerance)
  const double inv = 1.0 / (n1n * n2n);
  const double c1 = x * inv, s1 = y * inv;
  const double c2 = c1 * c1 - s1 * s1, s2 = 2.0 * s1 * c1;
  const double c3 = c2 * c1 - s2 * s1, s3 = s2 * c1 + c2 * s1;
  const double c4 = c2 * c2 - s2 * s2, s4 = 2.0 * s2 * c2;
  *e = 0.5 * (V[0] * (1.0 + c1) + V[1] * (1.0 - c2) + V[2] * (1.0 + c3) + V[3] * (1.0 - c4));
  if (!grad) return true;
  const double dedphi = 0.5 * (-V[0] * s1 + 2.0 * V[1] * s2 - 3.0 * V[2] * s3 + 4.0 * V[3] * s4);
  const P3 cI = {-(b2n / n1sq) * n1.x, -(b2n / n1sq) * n1.y, -(b2n / n1sq) * n1.z};
  const P3 cL = {(b2n / n2sq) * n2.x, (b2n / n2sq) * n2.y, (b2n / n2sq) * n2.z};
  const double p = dot(b1, b2) / b2sq;
  const double s = dot(b3, b2) / b2sq;
  const P3 cJ = {-(1.0 + p) * cI.x + s * cL.x, -(1.0 + p) * cI.y + s * cL.y,
                 -(1.0 + p) * cI.z + s * cL.z};
  const P3 cK = {-(1.0 + s) * cL.x + p * cI.x, -(1.0 + s) * cL.y + p * cI.y,
                 -(1.0 + s) * cL.z + p * cI.z};
  g[0] = {dedphi * cI.x, dedphi * cI.y, dedphi * cI.z};
  g[1] = {dedphi * cJ.x, dedphi * cJ.y, dedphi * cJ.z};
  g[2] = {dedphi * cK.x, dedphi * cK.y, dedphi * cK.z};
  g[3] = {dedphi * cL.x, dedphi * cL.y, dedphi * cL.z};
  return true;
}

// One scaled (0 < s < 1) nonbonded pair, ffmin/kernels.py:316-353 with the
// pair's own scale.  Returns false on coincidence.
__device__ inline bool scaled_pair(P3 ci, P3 cj, double qi, double qj, double sgi, double sgj,
                            double epi, double epj, double s, bool has_cut, double cutoff,
                            bool grad, double* ec, double* ev, P3* gi) {
  const P3 d = sub(ci, cj);
  const double r = sqrt(dot(d, d));
  *ec = 0.0;
  *ev = 0.0;
  *gi = {0.0, 0.0, 0.0};
  if (r < kRmin) return false;
  if (has_cut && r > cutoff) return true;
  const double qq = s * qi * qj;
  *ec = kCoulomb * qq / r;
  double dedr_over_r = -kCoulomb * qq / (r * r * r);
  const double eps_ij = sqrt(epi * epj);
  if (eps_ij > 0.0) {
    const double sig = sqrt(sgi * sgj);
    const double t = sig / r;
    const double t2 = t * t, x6 = t2 * (t2 * t2);  // numba lowers x**6 to powi
    *ev = 4.0 * s * eps_ij * (x6 * x6 - x6);
    dedr_over_r += 4.0 * s * eps_ij * (-12.0 * x6 * x6 + 6.0 * x6) / (r * r);
  }
  if (grad) *gi = {dedr_over_r * d.x, dedr_over_r * d.y, dedr_over_r * d.z};
  return true;
}

__device__ __forceinline__ void amin(int64_t* p, int64_t v) {
  atomicMin(reinterpret_cast<long long*>(p), (long long)v);
}

// ------------------------------------------------------------- term blocks
// one thread per term over [bonds | angles | dihedrals | scaled pairs]; the
// five energy sums leave as one fixed-order partial per (virtual) block of
// kTermThreads threads: block vb of nvb for batch entry b
constexpr int kTermThreads = 128;

__device__ __forceinline__ int term_block_count(const TermPlanDev& tp) {
  const int tot = tp.nbond + tp.nangle + tp.ndih + tp.nscaled;
  return (tot + kTermThreads - 1) / kTermThreads;
}

// One virtual block of kTermThreads bonded / scaled-pair terms.  Status:
// with warp_slots null the degenerate-term indices go straight into the
// status words (amin; the caller reset them beforehand); else each warp
// writes its own four words -- the first degenerate bond, angle and
// dihedral (kSentinel: none) and a scaled-pair coincidence flag -- to
// warp_slots[4 (kTermThreads / 32 vb + warp) ..], folded into the status
// words after a barrier (status_from_term_slots), so no reset has to
// precede the block (the fused small evaluation without a packing pass).
__device__ __forceinline__ void term_block(const TermPlanDev& tp, bool grad, CoordSrc cs,
                                           double* __restrict__ term_part,
                                           double* __restrict__ term_f,
                                           int64_t* __restrict__ status, int b, int vb, int nvb,
                                           double (*sh)[kTermThreads / 32],
                                           int64_t* __restrict__ warp_slots = nullptr) {
  cs.x += (size_t)b * tp.n * 3;
  status += (size_t)b * kStWords;
  double e5[5] = {0.0, 0.0, 0.0, 0.0, 0.0};  // stretch, bend, torsion, coulomb, vdw
  int bad_b = INT_MAX, bad_a = INT_MAX, bad_d = INT_MAX, bad_nb = 0;
  int t = vb * kTermThreads + threadIdx.x;
  if (t < tp.nbond) {
    const int i = tp.bond_idx[2 * t], j = tp.bond_idx[2 * t + 1];
    double e = 0.0;
    P3 gi = {0, 0, 0};
    if (!bond_term(ld3(cs, i), ld3(cs, j), tp.bond_K[t], tp.bond_r0[t], grad, &e, &gi))
      bad_b = t;
    e5[0] = e;
    if (grad) {
      st3(term_f + 3 * (2 * t), gi);
      st3(term_f + 3 * (2 * t + 1), {-gi.x, -gi.y, -gi.z});
    }
  } else if ((t -= tp.nbond) < tp.nangle) {
    const int i = tp.ang_idx[3 * t], j = tp.ang_idx[3 * t + 1], k = tp.ang_idx[3 * t + 2];
    double e = 0.0;
    P3 gi = {0, 0, 0}, gk = {0, 0, 0};
    if (!angle_term(ld3(cs, i), ld3(cs, j), ld3(cs, k), tp.ang_K[t], tp.ang_t0[t], grad, &e,
                    &gi, &gk)) {
      bad_a = t;
      e = 0.0;
      gi = gk = {0, 0, 0};
    }
    e5[1] = e;
    if (grad) {
      double* f = term_f + 3 * (tp.slot_angle0 + 3 * t);
      st3(f, gi);
      st3(f + 3, {-(gi.x + gk.x), -(gi.y + gk.y), -(gi.z + gk.z)});
      st3(f + 6, gk);
    }
  } else if ((t -= tp.nangle) < tp.ndih) {
    const int* id = tp.dih_idx + 4 * t;
    double e = 0.0;
    P3 g[4] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
    if (!dihedral_term(ld3(cs, id[0]), ld3(cs, id[1]), ld3(cs, id[2]), ld3(cs, id[3]),
                       tp.dih_V + 4 * t, grad, &e, g)) {
      bad_d = t;
      e = 0.0;
      g[0] = g[1] = g[2] = g[3] = {0, 0, 0};
    }
    e5[2] = e;
    if (grad) {
      double* f = term_f + 3 * (tp.slot_dih0 + 4 * t);
      for (int q = 0; q < 4; ++q) st3(f + 3 * q, g[q]);
    }
  } else if ((t -= tp.ndih) < tp.nscaled) {
    const int i = tp.sc_idx[2 * t], j = tp.sc_idx[2 * t + 1];
    double ec, ev;
    P3 gi;
    if (!scaled_pair(ld3(cs, i), ld3(cs, j), tp.q[i], tp.q[j], tp.sigma[i], tp.sigma[j],
                     tp.eps[i], tp.eps[j], tp.sc_s[t], tp.has_cutoff != 0, tp.cutoff, grad, &ec,
                     &ev, &gi))
      bad_nb = 1;
    e5[3] = ec;
    e5[4] = ev;
    if (grad) {
      double* f = term_f + 3 * (tp.slot_sc0 + 2 * t);
      st3(f, gi);
      st3(f + 3, {-gi.x, -gi.y, -gi.z});
    }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (warp_slots) {
    const unsigned mb = __reduce_min_sync(0xffffffffu, (unsigned)bad_b);
    const unsigned ma = __reduce_min_sync(0xffffffffu, (unsigned)bad_a);
    const unsigned md = __reduce_min_sync(0xffffffffu, (unsigned)bad_d);
    const bool fl = __any_sync(0xffffffffu, bad_nb);
    if (lane == 0) {
      int64_t* w = warp_slots + 4 * ((size_t)vb * (kTermThreads / 32) + warp);
      w[0] = mb == (unsigned)INT_MAX ? kSentinel : (int64_t)mb;
      w[1] = ma == (unsigned)INT_MAX ? kSentinel : (int64_t)ma;
      w[2] = md == (unsigned)INT_MAX ? kSentinel : (int64_t)md;
      w[3] = fl ? 1 : 0;
    }
  } else {
    if (bad_b != INT_MAX) amin(status + kStBond, bad_b);
    if (bad_a != INT_MAX) amin(status + kStAngle, bad_a);
    if (bad_d != INT_MAX) amin(status + kStDihedral, bad_d);
    if (bad_nb) status[kStNbSuspect] = 1;
  }
#pragma unroll
  for (int c = 0; c < 5; ++c) {
    double v = e5[c];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) sh[c][warp] = v;
  }
  __syncthreads();
  if (threadIdx.x < 5) {
    double v = 0.0;
    for (int w = 0; w < kTermThreads / 32; ++w) v += sh[threadIdx.x][w];
    term_part[((size_t)b * nvb + vb) * 5 + threadIdx.x] = v;
  }
  __syncthreads();  // sh is reused by the next virtual block
}

// The status words from the term blocks' warp slots (block-uniform: the
// threads scan shares of the slots, thread 0 writes when `write`); returns
// the scaled-pair coincidence flag to every thread.  st: the status words
// to fill (global or a shared copy).
__device__ __forceinline__ int status_from_term_slots(const int64_t* __restrict__ slots,
                                                      int nwarps, int64_t* st, bool write,
                                                      int64_t (*sh)[kTermThreads / 32]) {
  int64_t mb = kSentinel, ma = kSentinel, md = kSentinel;
  int fl = 0;
  for (int k = threadIdx.x; k < nwarps; k += blockDim.x) {
    const int64_t* w = slots + 4 * (size_t)k;
    mb = min(mb, w[0]);
    ma = min(ma, w[1]);
    md = min(md, w[2]);
    fl |= w[3] != 0;
  }
  fl = __syncthreads_or(fl);
  if (!write) return fl;
  for (int o = 16; o > 0; o >>= 1) {
    mb = min(mb, (int64_t)__shfl_xor_sync(0xffffffffu, (long long)mb, o));
    ma = min(ma, (int64_t)__shfl_xor_sync(0xffffffffu, (long long)ma, o));
    md = min(md, (int64_t)__shfl_xor_sync(0xffffffffu, (long long)md, o));
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
    sh[0][warp] = mb;
    sh[1][warp] = ma;
    sh[2][warp] = md;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      mb = min(mb, sh[0][w]);
      ma = min(ma, sh[1][w]);
      md = min(md, sh[2][w]);
    }
    st[kStBond] = mb;
    st[kStAngle] = ma;
    st[kStDihedral] = md;
  }
  __syncthreads();
  return fl;
}

// ---------------------------------------------------------- gradient gather
// The gather of one 32-atom group (atoms 32 g .. 32 g + 31; a group never
// straddles a super-block or a tile row) by the NW warps of a block
// (block-uniform call, contains __syncthreads).  The group's partial
// entries -- super-unit mode: the i-rows of units (b, b..nb-1) then the
// j-columns of units (0..b, b), from the plan's unit lists; tile mode: the i-rows of the tiles of its
// sub-block row, then the j-columns of the tiles of its j-block -- are dealt
// to the warps (entry k to warp k mod NW, 128-byte coalesced rows, all
// three components); the NW warp sums and the atom's term slots are then
// added in a fixed order.  part: NW x 3 x 32 doubles of shared memory.
template <typename T, int NW>
__device__ __forceinline__ void gather_group(int g, int n, int S, int nb,
                                             const int* __restrict__ unit_index,
                                             const int* __restrict__ trow_ptr,
                                             const int* __restrict__ tcol_ptr,
                                             const int* __restrict__ tcol_idx,
                                             const T* __restrict__ ipart,
                                             const T* __restrict__ jpart,
                                             const int* __restrict__ slot_ptr,
                                             const int* __restrict__ slot_idx,
                                             const double* __restrict__ term_f, int slot_sc0,
                                             bool use_nb, bool use_terms, bool use_sc,
                                             double* __restrict__ grad, double (*part)[3][32],
                                             int rank = 0, int nranks = 1) {
  // row-sharded plans (ffm_system_set_shard): unit / tile slot u belongs to
  // rank u % nranks, the slots of other ranks' ones hold exact zeros -- skip them
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int a0 = g << 5;
  double g0 = 0.0, g1 = 0.0, g2 = 0.0;
  if (use_nb && trow_ptr) {  // tile mode: [tile][3][128] rows, [tile][3][32] columns
    const int kk = a0 / kIB, mg = a0 / kJB, row = a0 - kk * kIB + lane;
    const int r0 = trow_ptr[kk], nr = trow_ptr[kk + 1] - r0;
    const int c0 = tcol_ptr[mg], nt = nr + tcol_ptr[mg + 1] - c0;
    // the warp's entries k = warp, warp + NW, ... in order: its rows, then
    // its columns, as two branch-free loops (with a per-entry branch -- row
    // or column, this rank's or not -- ptxas kept each entry's loads behind
    // the previous entry's sums; measured: no change in the evaluation time,
    // profiles/r02_small_tile_loads.log)
    int k = warp;
    if (nranks == 1) {
#pragma unroll 4
      for (; k < nr; k += NW) {
        const T* p = ipart + (size_t)(r0 + k) * 3 * kIB + row;
        g0 += (double)p[0];
        g1 += (double)p[kIB];
        g2 += (double)p[2 * kIB];
      }
#pragma unroll 4
      for (; k < nt; k += NW) {
        const T* p = jpart + (size_t)tcol_idx[c0 + k - nr] * 3 * kJB + lane;
        g0 += (double)p[0];
        g1 += (double)p[kJB];
        g2 += (double)p[2 * kJB];
      }
    } else {  // this rank's tiles only
      for (; k < nt; k += NW) {
        const bool isrow = k < nr;
        const int st = isrow ? kIB : kJB;
        const int t = isrow ? r0 + k : tcol_idx[c0 + k - nr];
        if (t % nranks != rank) continue;
        const T* p = isrow ? ipart + (size_t)t * 3 * kIB + row : jpart + (size_t)t * 3 * kJB + lane;
        g0 += (double)p[0];
        g1 += (double)p[st];
        g2 += (double)p[2 * st];
      }
    }
  } else if (use_nb) {  // super-unit mode: [unit][3][S] rows and columns
    // unit_index = [row lists' ptr (2 nb + 1) | column lists' ptr (nb + 1) |
    // row lists | column lists]: the units holding the rows of super-block
    // b's half h (units of the last wave come in halves), then the units
    // holding its columns (both halves of a split unit)
    const int* urow_ptr = unit_index;
    const int* ucol_ptr = unit_index + 2 * nb + 1;
    const int* urow_idx = unit_index + 3 * nb + 2;
    const int* ucol_idx = urow_idx + urow_ptr[2 * nb];
    const int b = a0 / S, offr = a0 - b * S, off = offr + lane;
    const int h = (offr / kIB) >= (S / kIB) / 2 ? 1 : 0;
    const int r0 = urow_ptr[2 * b + h], nr = urow_ptr[2 * b + h + 1] - r0;
    const int c0 = ucol_ptr[b], nt = nr + ucol_ptr[b + 1] - c0;
    if (nranks == 1) {
#pragma unroll 4
      for (int k = warp; k < nt; k += NW) {
        const T* p = k < nr ? ipart + (size_t)urow_idx[r0 + k] * 3 * S
                            : jpart + (size_t)ucol_idx[c0 + k - nr] * 3 * S;
        g0 += (double)p[off];
        g1 += (double)p[S + off];
        g2 += (double)p[2 * S + off];
      }
    } else {  // this rank's units only
      for (int k = warp; k < nt; k += NW) {
        const int u = k < nr ? urow_idx[r0 + k] : ucol_idx[c0 + k - nr];
        if (u % nranks != rank) continue;
        const T* p = (k < nr ? ipart : jpart) + (size_t)u * 3 * S;
        g0 += (double)p[off];
        g1 += (double)p[S + off];
        g2 += (double)p[2 * S + off];
      }
    }
  }
  part[warp][0][lane] = g0;
  part[warp][1][lane] = g1;
  part[warp][2][lane] = g2;
  __syncthreads();
  for (int x = threadIdx.x; x < 96; x += NW * 32) {
    // thread x writes grad[3 a0 + x]: coalesced
    const int l = x / 3, c = x - 3 * l, a = a0 + l;
    if (a < n) {
      double v = 0.0;
#pragma unroll
      for (int w = 0; w < NW; ++w) v += part[w][c][l];
      for (int s = slot_ptr[a]; s < slot_ptr[a + 1]; ++s) {
        const int k = slot_idx[s];
        if (k < slot_sc0 ? !use_terms : !use_sc) continue;
        v += term_f[3 * (size_t)k + c];
      }
      grad[3 * (size_t)a + c] = v;
    }
  }
  __syncthreads();  // part is reused by the block's next group
}

// Super-unit mode gather of a 128-atom span (one sub-block of one super-
// block: atoms 128 g .. 128 g + 127) by the NW warps of a block: the same
// entries and the same warp split as gather_group (entry k to warp k mod NW;
// per atom the warp sums in warp order, then the term slots), so identical
// bits -- but each warp reads 512 contiguous bytes per entry and component
// (four 128-byte rows) instead of 128, which the DRAM pages reward.
// part: NW x 3 x 128 doubles of shared memory.
template <typename T, int NW>
__device__ __forceinline__ void gather_span128(int g, int n, int S, int nb,
                                               const int* __restrict__ unit_index,
                                               const T* __restrict__ ipart,
                                               const T* __restrict__ jpart,
                                               const int* __restrict__ slot_ptr,
                                               const int* __restrict__ slot_idx,
                                               const double* __restrict__ term_f, int slot_sc0,
                                               bool use_nb, bool use_terms, bool use_sc,
                                               double* __restrict__ grad,
                                               double (*part)[3][128], int rank, int nranks) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int a0 = g * 128;
  double acc[4][3];
#pragma unroll
  for (int q = 0; q < 4; ++q) acc[q][0] = acc[q][1] = acc[q][2] = 0.0;
  if (use_nb) {
    const int* urow_ptr = unit_index;
    const int* ucol_ptr = unit_index + 2 * nb + 1;
    const int* urow_idx = unit_index + 3 * nb + 2;
    const int* ucol_idx = urow_idx + urow_ptr[2 * nb];
    const int b = a0 / S, offr = a0 - b * S;
    const int h = (offr / kIB) >= (S / kIB) / 2 ? 1 : 0;
    const int r0 = urow_ptr[2 * b + h], nr = urow_ptr[2 * b + h + 1] - r0;
    const int c0 = ucol_ptr[b], nt = nr + ucol_ptr[b + 1] - c0;
#pragma unroll 2
    for (int k = warp; k < nt; k += NW) {
      const int u = k < nr ? urow_idx[r0 + k] : ucol_idx[c0 + k - nr];
      if (nranks > 1 && u % nranks != rank) continue;
      const T* p = (k < nr ? ipart : jpart) + (size_t)u * 3 * S + offr + lane;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        acc[q][0] += (double)p[32 * q];
        acc[q][1] += (double)p[S + 32 * q];
        acc[q][2] += (double)p[2 * S + 32 * q];
      }
    }
  }
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int c = 0; c < 3; ++c) part[warp][c][32 * q + lane] = acc[q][c];
  __syncthreads();
  for (int x = threadIdx.x; x < 384; x += NW * 32) {
    const int l = x / 3, c = x - 3 * l, a = a0 + l;
    if (a < n) {
      double v = 0.0;
#pragma unroll
      for (int w = 0; w < NW; ++w) v += part[w][c][l];
      for (int s = slot_ptr[a]; s < slot_ptr[a + 1]; ++s) {
        const int k = slot_idx[s];
        if (k < slot_sc0 ? !use_terms : !use_sc) continue;
        v += term_f[3 * (size_t)k + c];
      }
      grad[3 * (size_t)a + c] = v;
    }
  }
  __syncthreads();
}

// status sentinels -> the reference's conventions (-1 = clean)
__device__ __forceinline__ void finalize_entry(int n, int64_t* s) {
  if (s[kStNbKey] != kSentinel) {
    s[kStNbBadI] = s[kStNbKey] / n;
    s[kStNbBadJ] = s[kStNbKey] % n;
  }
  for (int k = kStBond; k <= kStDihedral; ++k)
    if (s[k] == kSentinel) s[k] = -1;
}

// ---------------------------------------------------------- energy reduction
// one block of kRedThreads per batch entry; every partial summed in a fixed
// order (strided per thread, then a warp/block tree)
constexpr int kRedThreads = 128;

__device__ __forceinline__ double tree_sum(double v, double* sh) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x < 32) {
    s = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  }
  return s;  // valid in thread 0
}

__device__ __forceinline__ double tree_min(double v, double* sh) {
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = DBL_MAX;
  if (threadIdx.x < 32) {
    s = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : DBL_MAX;
    for (int o = 16; o > 0; o >>= 1) s = fmin(s, __shfl_xor_sync(0xffffffffu, s, o));
  }
  return s;
}

#ifndef FFM_RED_UNROLL
#define FFM_RED_UNROLL 2  // (8 changed the fused small kernel's register allocation: spills)
#endif
constexpr int kRedUnroll = FFM_RED_UNROLL;
constexpr int kRedUnroll4 = FFM_RED_UNROLL < 4 ? FFM_RED_UNROLL : 4;
// flag_suspect: mark a possible coincidence (non-finite sums, closest pair
// below RMIN) in the status words for the finder
__device__ __forceinline__ void reduce_entry(int nunits, int nterm_blocks,
                                             const double* __restrict__ epart,
                                             const double* __restrict__ term_part,
                                             double* __restrict__ energies,
                                             int64_t* __restrict__ status, int b, double* sh,
                                             bool flag_suspect = true, int finalize_n = -1) {
  epart += (size_t)b * nunits * 3;
  term_part += (size_t)b * nterm_blocks * 5;
  double ec = 0.0, ev = 0.0, mr = DBL_MAX, es = 0.0, eb = 0.0, et = 0.0;
  // (unrolled: a thread's partial loads are independent and go out
  // together; the sums keep their order)
#pragma unroll kRedUnroll
  for (int u = threadIdx.x; u < nunits; u += blockDim.x) {
    ec += epart[3 * u];
    ev += epart[3 * u + 1];
    mr = fmin(mr, epart[3 * u + 2]);
  }
#pragma unroll kRedUnroll4
  for (int k = threadIdx.x; k < nterm_blocks; k += blockDim.x) {
    const double* p = term_part + 5 * (size_t)k;
    es += p[0];
    eb += p[1];
    et += p[2];
    ec += p[3];
    ev += p[4];
  }
  ec = tree_sum(ec, sh);
  ev = tree_sum(ev, sh);
  es = tree_sum(es, sh);
  eb = tree_sum(eb, sh);
  et = tree_sum(et, sh);
  mr = tree_min(mr, sh);
  if (threadIdx.x == 0) {
    double* E = energies + 5 * (size_t)b;
    E[0] = es;
    E[1] = eb;
    E[2] = et;
    E[3] = ec;
    E[4] = ev;
    int64_t* s = status + (size_t)b * kStWords;
    if (flag_suspect && (!isfinite(ec) || !isfinite(ev) || mr < kRmin * kRmin))
      s[kStNbSuspect] = 1;
    // finalize_n >= 0: a clean entry (nothing for the finder, including
    // suspects flagged by the scaled-pair terms) is finalised here, so the
    // finder kernel exits at once and no separate finalize launch is needed
    if (finalize_n >= 0 && s[kStNbSuspect] == 0) finalize_entry(finalize_n, s);
  }
}

// The same reduction over many slots (a sharded or fine super-unit plan has
// tens of thousands) by `nparts` blocks: block `part` sums its contiguous
// slice of the slots into scratch[part]; the last block to finish (atomic
// counter, reset for the next evaluation) adds the parts in part order plus
// the term partials and writes energies / status exactly as reduce_entry
// does.  Fixed order throughout: bit-identical run to run.
__device__ __forceinline__ void reduce_split(int nunits, int nterm_blocks,
                                             const double* __restrict__ epart,
                                             const double* __restrict__ term_part,
                                             double* __restrict__ energies,
                                             int64_t* __restrict__ status, double* sh,
                                             double* scratch, unsigned* counter, int part,
                                             int nparts, int finalize_n) {
  __shared__ int last;
  const int chunk = (nunits + nparts - 1) / nparts;
  const int u0 = part * chunk, u1 = min(nunits, u0 + chunk);
  double ec = 0.0, ev = 0.0, mr = DBL_MAX;
  for (int u = u0 + threadIdx.x; u < u1; u += blockDim.x) {
    ec += epart[3 * u];
    ev += epart[3 * u + 1];
    mr = fmin(mr, epart[3 * u + 2]);
  }
  ec = tree_sum(ec, sh);
  ev = tree_sum(ev, sh);
  mr = tree_min(mr, sh);
  if (threadIdx.x == 0) {
    scratch[3 * part] = ec;
    scratch[3 * part + 1] = ev;
    scratch[3 * part + 2] = mr;
    __threadfence();
    last = atomicAdd(counter, 1u) == (unsigned)(nparts - 1);
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double es = 0.0, eb = 0.0, et = 0.0, tc = 0.0, tv = 0.0;
  for (int k = threadIdx.x; k < nterm_blocks; k += blockDim.x) {
    const double* p = term_part + 5 * (size_t)k;
    es += p[0];
    eb += p[1];
    et += p[2];
    tc += p[3];
    tv += p[4];
  }
  es = tree_sum(es, sh);
  eb = tree_sum(eb, sh);
  et = tree_sum(et, sh);
  tc = tree_sum(tc, sh);
  tv = tree_sum(tv, sh);
  if (threadIdx.x == 0) {
    double sc = 0.0, sv = 0.0, m = DBL_MAX;
    for (int q = 0; q < nparts; ++q) {
      sc += __ldcg(scratch + 3 * q);
      sv += __ldcg(scratch + 3 * q + 1);
      m = fmin(m, __ldcg(scratch + 3 * q + 2));
    }
    sc += tc;
    sv += tv;
    energies[0] = es;
    energies[1] = eb;
    energies[2] = et;
    energies[3] = sc;
    energies[4] = sv;
    if (!isfinite(sc) || !isfinite(sv) || m < kRmin * kRmin) status[kStNbSuspect] = 1;
    if (finalize_n >= 0 && status[kStNbSuspect] == 0) finalize_entry(finalize_n, status);
    *counter = 0u;
  }
}

// ------------------------------------------------------------ pair finder
// Exact restatement of the coincidence test of ffmin/kernels.py:294-302 for
// row i of the upper triangle (only run when the sweep flagged a suspect):
// the smallest key i * n + j of a coincident pair wins.
template <typename T>
__device__ __forceinline__ void finder_row(int i, int n, const typename Vec4T<T>::type* __restrict__ pos,
                                           const int* __restrict__ sp_ptr,
                                           const int* __restrict__ sp_j,
                                           const double* __restrict__ sp_s, int64_t* s) {
  const auto pi = pos[i];
  int cur = sp_ptr[i];
  const int end = sp_ptr[i + 1];
  for (int j = i + 1; j < n; ++j) {
    while (cur < end && sp_j[cur] < j) ++cur;
    if (cur < end && sp_j[cur] == j && sp_s[cur] == 0.0) continue;
    const auto pj = pos[j];
    const double dx = (double)pi.x - (double)pj.x, dy = (double)pi.y - (double)pj.y,
                 dz = (double)pi.z - (double)pj.z;
    if (sqrt(dx * dx + dy * dy + dz * dz) < kRmin) {
      amin(s + kStNbKey, (int64_t)i * n + j);
      break;
    }
  }
}


}  // namespace ffm
