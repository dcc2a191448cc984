// ffm_terms.cu -- everything around the pair sweep: coordinate packing,
// bonded terms and scaled 1-4 pairs (FP64), the deterministic gradient
// gather, the energy reduction, the coincident-pair finder and the exact
// single-atom move deltas used by the gradient-free method.  The per-item
// bodies live in ffm_device.cuh (shared with the fused small-system kernel).
#include "ffm_device.cuh"
#include "ffm_kernels.h"

namespace ffm {

// ------------------------------------------------------------------ packing
template <typename T>
__global__ void pack_kernel(int n, int np, int batch, const double* __restrict__ coords,
                            const double* __restrict__ qt,
                            typename Vec4T<T>::type* __restrict__ pos, T* __restrict__ ipos,
                            int64_t* __restrict__ status) {
  pdl_wait();
  pdl_launch_dependents();
  pack_item<T>((int64_t)blockIdx.x * blockDim.x + threadIdx.x, n, np, batch, coords, qt, pos,
               ipos, status);
}

template <typename T>
__global__ void pad_kernel(int n, int np, int batch, typename Vec4T<T>::type* __restrict__ pos,
                           T* __restrict__ ipos) {
  pdl_wait();
  pdl_launch_dependents();
  const int npad = np - n;
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= (int64_t)npad * batch) return;
  const int64_t b = k / npad, a = k - b * npad;
  // zero charge and LJ (set in lj/qt), far from everything and 10 A apart
  put_atom<T>(pos + b * np, ipos + b * 4 * (int64_t)np, np, n + (int)a,
              T(1.0e4 + 10.0 * (double)a), T(1.0e4), T(1.0e4), T(0));
}

cudaError_t launch_pack(int n, int np, int batch, bool fp64, const double* coords,
                        const double* qt, void* pos, void* ipos, int64_t* status,
                        cudaStream_t st) {
  const int64_t tot = (int64_t)n * batch > batch ? (int64_t)n * batch : batch;
  const int blocks = (int)((tot + 255) / 256);
  if (fp64)
    count_launch(), launch_k(pack_kernel<double>, blocks, 256, 0, st, n, np, batch, coords, qt,
                                                static_cast<double4*>(pos),
                                                static_cast<double*>(ipos), status);
  else
    count_launch(), launch_k(pack_kernel<float>, blocks, 256, 0, st, n, np, batch, coords, qt,
                                               static_cast<float4*>(pos),
                                               static_cast<float*>(ipos), status);
  return cudaGetLastError();
}

cudaError_t launch_pad(int n, int np, int batch, bool fp64, void* pos, void* ipos,
                       cudaStream_t st) {
  const int64_t tot = (int64_t)(np - n) * batch;
  if (tot <= 0) return cudaSuccess;
  const int blocks = (int)((tot + 255) / 256);
  if (fp64)
    count_launch(), launch_k(pad_kernel<double>, blocks, 256, 0, st, n, np, batch, static_cast<double4*>(pos),
                                               static_cast<double*>(ipos));
  else
    count_launch(), launch_k(pad_kernel<float>, blocks, 256, 0, st, n, np, batch, static_cast<float4*>(pos),
                                              static_cast<float*>(ipos));
  return cudaGetLastError();
}

// LJ (a, b) in the i-side pair layout, built once per system from the FP64
// records and scaled by LjIScale<T> (see ffm_common.cuh)
template <typename T>
__global__ void ilj_kernel(int np, const double2* __restrict__ lj64, T* __restrict__ ilj) {
  pdl_wait();
  pdl_launch_dependents();
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= np) return;
  ilj[ipos_index(a, np, 0)] = T(LjIScale<T>::value * lj64[a].x);
  ilj[ipos_index(a, np, 1)] = T(LjIScale<T>::value * lj64[a].y);
}

cudaError_t launch_ilj(int np, bool fp64, const void* lj64, void* ilj, cudaStream_t st) {
  const int blocks = (np + 255) / 256;
  const double2* src = static_cast<const double2*>(lj64);
  if (fp64)
    count_launch(), launch_k(ilj_kernel<double>, blocks, 256, 0, st, np, src, static_cast<double*>(ilj));
  else
    count_launch(), launch_k(ilj_kernel<float>, blocks, 256, 0, st, np, src, static_cast<float*>(ilj));
  return cudaGetLastError();
}

// ------------------------------------------------------------- term kernels
__global__ void __launch_bounds__(kTermThreads)
terms_kernel(TermPlanDev tp, bool grad, const double* __restrict__ coords,
             double* __restrict__ term_part, double* __restrict__ term_f,
             int64_t* __restrict__ status) {
  pdl_wait();
  pdl_launch_dependents();
  __shared__ double sh[5][kTermThreads / 32];
  term_block(tp, grad, CoordSrc{coords, nullptr, 0.0}, term_part, term_f, status, blockIdx.y,
             blockIdx.x, gridDim.x, sh);
}

int term_blocks(const TermPlanDev& tp) {
  const int tot = tp.nbond + tp.nangle + tp.ndih + tp.nscaled;
  return (tot + kTermThreads - 1) / kTermThreads;
}

cudaError_t launch_terms(const TermPlanDev& tp, bool grad, int batch, const double* coords,
                         double* term_part, double* term_f, int64_t* status, cudaStream_t st) {
  const int nblk = term_blocks(tp);
  if (nblk == 0) return cudaSuccess;
  dim3 grid(nblk, batch);
  count_launch();
  launch_k(terms_kernel, grid, kTermThreads, 0, st, tp, grad, coords, term_part, term_f, status);
  return cudaGetLastError();
}

// ---------------------------------------------------------- gradient gather
// Gather + energy reduction in one launch: block g < ngroups gathers atom
// group g (gather_group: NW warps, fixed order), the extra last block
// reduces the energies (reduce_entry), so results are bit-identical run to
// run.  Super-unit mode uses 8 warps per group, tile mode 4 (the same split
// as the fused small-system kernel, so both produce the same bits).
template <typename T, int NW, int SPAN>
__global__ void __launch_bounds__(NW * 32)
gather_reduce_kernel(int n, int S, int nb, const int* __restrict__ unit_index,
                     const int* __restrict__ trow_ptr, const int* __restrict__ tcol_ptr,
                     const int* __restrict__ tcol_idx, const T* __restrict__ ipart,
                     const T* __restrict__ jpart, const int* __restrict__ slot_ptr,
                     const int* __restrict__ slot_idx, const double* __restrict__ term_f,
                     int slot_sc0, bool use_nb, bool use_terms, bool use_sc,
                     double* __restrict__ grad, int nslots, int nterm_blocks,
                     const double* __restrict__ epart, const double* __restrict__ term_part,
                     double* __restrict__ energies, int64_t* __restrict__ status, int rank,
                     int nranks, double* __restrict__ escratch, unsigned* ecount, int nparts) {
  pdl_wait();
  pdl_launch_dependents();
  // 128-atom spans (gather_span128, super-unit mode, large systems) or
  // 32-atom groups (gather_group: more blocks in flight for smaller ones)
  constexpr int kSpan = SPAN;
  __shared__ double part[NW][3][kSpan];
  const int ngroups = (n + kSpan - 1) / kSpan;
  if ((int)blockIdx.x >= ngroups) {  // the energy reduction: nparts blocks
    if (nparts == 1)  // (the fused small-system kernel's order: identical bits)
      reduce_entry(nslots, nterm_blocks, epart, term_part, energies, status, 0, &part[0][0][0],
                   true, n);
    else
      reduce_split(nslots, nterm_blocks, epart, term_part, energies, status, &part[0][0][0],
                   escratch, ecount, blockIdx.x - ngroups, nparts, n);
    return;
  }
  if constexpr (kSpan == 128)
    gather_span128<T, NW>(blockIdx.x, n, S, nb, unit_index, ipart, jpart, slot_ptr, slot_idx,
                          term_f, slot_sc0, use_nb, use_terms, use_sc, grad, part, rank,
                          nranks);
  else
    gather_group<T, NW>(blockIdx.x, n, S, nb, unit_index, trow_ptr, tcol_ptr, tcol_idx, ipart,
                        jpart, slot_ptr, slot_idx, term_f, slot_sc0, use_nb, use_terms, use_sc,
                        grad, reinterpret_cast<double (*)[3][32]>(part), rank, nranks);
}

template <typename T>
static cudaError_t launch_gr_t(int n, int S, int nb, const int* unit_index, const int* trow_ptr,
                               const int* tcol_ptr, const int* tcol_idx, const void* ipart,
                               const void* jpart, const int* slot_ptr, const int* slot_idx,
                               const double* term_f, int slot_sc0, bool use_nb, bool use_terms,
                               bool use_sc, double* grad, int nslots, int nterm_blocks,
                               const double* epart, const double* term_part, double* energies,
                               int64_t* status, int rank, int nranks, double* escratch,
                               unsigned* ecount, cudaStream_t st) {
  const int nparts = energy_parts(nslots);
  // 128-atom spans from 40k atoms on (100k: 4479 -> 4467 us per evaluation;
  // at 10k the 4x fewer blocks cost 4 us: tools/mid_sweep.py A/B)
  const bool span = !trow_ptr && n >= 40000;
  const int blocks = (span ? (n + 127) / 128 : (n + 31) / 32) + nparts;
  const T* ip = static_cast<const T*>(ipart);
  const T* jp = static_cast<const T*>(jpart);
  count_launch();
  if (span)
    launch_k(gather_reduce_kernel<T, kGatherWarpsUnits, 128>, blocks, kGatherWarpsUnits * 32, 0, st, 
        n, S, nb, unit_index, trow_ptr, tcol_ptr, tcol_idx, ip, jp, slot_ptr, slot_idx, term_f,
        slot_sc0, use_nb, use_terms, use_sc, grad, nslots, nterm_blocks, epart, term_part,
        energies, status, rank, nranks, escratch, ecount, nparts);
  else if (trow_ptr)
    launch_k(gather_reduce_kernel<T, kGatherWarpsTiles, 32>, blocks, kGatherWarpsTiles * 32, 0, st, 
        n, S, nb, unit_index, trow_ptr, tcol_ptr, tcol_idx, ip, jp, slot_ptr, slot_idx, term_f,
        slot_sc0, use_nb, use_terms, use_sc, grad, nslots, nterm_blocks, epart, term_part,
        energies, status, rank, nranks, escratch, ecount, nparts);
  else
    launch_k(gather_reduce_kernel<T, kGatherWarpsUnits, 32>, blocks, kGatherWarpsUnits * 32, 0, st, 
        n, S, nb, unit_index, trow_ptr, tcol_ptr, tcol_idx, ip, jp, slot_ptr, slot_idx, term_f,
        slot_sc0, use_nb, use_terms, use_sc, grad, nslots, nterm_blocks, epart, term_part,
        energies, status, rank, nranks, escratch, ecount, nparts);
  return cudaGetLastError();
}

cudaError_t launch_gather_reduce(int n, int S, int nb, bool fp64, const int* unit_index,
                                 const int* trow_ptr, const int* tcol_ptr, const int* tcol_idx,
                                 const void* ipart, const void* jpart, const int* slot_ptr,
                                 const int* slot_idx, const double* term_f, int slot_sc0,
                                 bool use_nb, bool use_terms, bool use_sc, double* grad,
                                 int nslots, const TermPlanDev& tp, const double* epart,
                                 const double* term_part, double* energies, int64_t* status,
                                 int rank, int nranks, double* escratch, unsigned* ecount,
                                 cudaStream_t st) {
  if (fp64)
    return launch_gr_t<double>(n, S, nb, unit_index, trow_ptr, tcol_ptr, tcol_idx, ipart, jpart,
                               slot_ptr, slot_idx, term_f, slot_sc0, use_nb, use_terms, use_sc,
                               grad, nslots, term_blocks(tp), epart, term_part, energies, status,
                               rank, nranks, escratch, ecount, st);
  return launch_gr_t<float>(n, S, nb, unit_index, trow_ptr, tcol_ptr, tcol_idx, ipart, jpart,
                            slot_ptr, slot_idx, term_f, slot_sc0, use_nb, use_terms, use_sc, grad,
                            nslots, term_blocks(tp), epart, term_part, energies, status, rank,
                            nranks, escratch, ecount, st);
}

// ---------------------------------------------------------- energy reduction
__global__ void __launch_bounds__(kRedThreads)
reduce_kernel(int nunits, int nterm_blocks, const double* __restrict__ epart,
              const double* __restrict__ term_part, double* __restrict__ energies,
              int64_t* __restrict__ status, int n) {
  pdl_wait();
  pdl_launch_dependents();
  __shared__ double sh[32];
  reduce_entry(nunits, nterm_blocks, epart, term_part, energies, status, blockIdx.x, sh, true,
               n);
}

__global__ void __launch_bounds__(kRedThreads)
reduce_split_kernel(int nunits, int nterm_blocks, const double* __restrict__ epart,
                    const double* __restrict__ term_part, double* __restrict__ energies,
                    int64_t* __restrict__ status, int n, double* escratch, unsigned* ecount) {
  pdl_wait();
  pdl_launch_dependents();
  __shared__ double sh[32];
  reduce_split(nunits, nterm_blocks, epart, term_part, energies, status, sh, escratch, ecount,
               blockIdx.x, gridDim.x, n);
}

int energy_parts(int nslots) {
  const int p = (nslots + kEnergySlotsPerPart - 1) / kEnergySlotsPerPart;
  return p < 1 ? 1 : (p > kMaxEnergyParts ? kMaxEnergyParts : p);
}

cudaError_t launch_reduce(int nunits, const TermPlanDev& tp, int batch, const double* epart,
                          const double* term_part, double* energies, int64_t* status, int n,
                          double* escratch, unsigned* ecount, cudaStream_t st) {
  count_launch();
  if (batch == 1 && escratch && energy_parts(nunits) > 1)
    launch_k(reduce_split_kernel, energy_parts(nunits), kRedThreads, 0, st, 
        nunits, term_blocks(tp), epart, term_part, energies, status, n, escratch, ecount);
  else
    launch_k(reduce_kernel, batch, kRedThreads, 0, st, nunits, term_blocks(tp), epart, term_part,
                                                  energies, status, n);
  return cudaGetLastError();
}

// ------------------------------------------------------------ pair finder
template <typename T>
__global__ void finder_kernel(int n, int np, const typename Vec4T<T>::type* __restrict__ pos,
                              const int* __restrict__ sp_ptr, const int* __restrict__ sp_j,
                              const double* __restrict__ sp_s, int64_t* __restrict__ status) {
  pdl_wait();
  pdl_launch_dependents();
  const int b = blockIdx.y;
  int64_t* s = status + (size_t)b * kStWords;
  // clean entries were finalised by the reduction (reduce_entry)
  if (*(volatile int64_t*)(s + kStNbSuspect) == 0) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) finder_row<T>(i, n, pos + (size_t)b * np, sp_ptr, sp_j, sp_s, s);
  // the entry's last finder block converts the sentinels (status word
  // kStCount counts finished blocks; reset for the next evaluation)
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    unsigned long long* cnt = reinterpret_cast<unsigned long long*>(s + kStCount);
    if (atomicAdd(cnt, 1ull) == gridDim.x - 1) {
      __threadfence();
      finalize_entry(n, s);
      *cnt = 0;
    }
  }
}

cudaError_t launch_finder(int n, int np, int batch, bool fp64, const void* pos,
                          const int* sp_ptr, const int* sp_j, const double* sp_s,
                          int64_t* status, cudaStream_t st) {
  dim3 grid((n + 127) / 128, batch);
  if (n == 0) return cudaSuccess;  // nothing to find; the reduction finalised
  if (fp64)
    count_launch(), launch_k(finder_kernel<double>, grid, 128, 0, st, n, np, static_cast<const double4*>(pos),
                                                sp_ptr, sp_j, sp_s, status);
  else
    count_launch(), launch_k(finder_kernel<float>, grid, 128, 0, st, n, np, static_cast<const float4*>(pos), sp_ptr,
                                               sp_j, sp_s, status);
  return cudaGetLastError();
}

// -------------------------------------------------------- single-atom moves
constexpr int kDeltaThreads = 256;

__device__ __forceinline__ P3 pick(const double* c, int atom, P3 np, int i) {
  return i == atom ? np : ld3(c, i);
}

// delta_blocks(n) blocks per candidate move (the partner range split
// between them, the first also takes the bonded terms; the last block to
// finish adds the blocks' partial sums in block order: deterministic).
// One block per candidate left the FP64 pair arithmetic of a 10k-atom
// system on 6 SMs (71 us per wiggle probe launch).  Nonbonded part restates
// ffmin/kernels.py:419-454 (_loop_nb_atom_delta), bonded parts 457-593.
#ifndef FFM_DELTA_PARTNERS
#define FFM_DELTA_PARTNERS 512  // partners per block (tuning aid)
#endif
#ifndef FFM_DELTA_MAXBLK
#define FFM_DELTA_MAXBLK 32
#endif
int delta_blocks(int n) {
  const int b = (n + FFM_DELTA_PARTNERS - 1) / FFM_DELTA_PARTNERS;
  return b < 1 ? 1 : (b > FFM_DELTA_MAXBLK ? FFM_DELTA_MAXBLK : b);
}

__global__ void __launch_bounds__(kDeltaThreads)
atom_delta_kernel(TermPlanDev tp, const double* __restrict__ coords,
                  const int* __restrict__ fsp_ptr, const int* __restrict__ fsp_j,
                  const double* __restrict__ fsp_s, const int* __restrict__ aterm_ptr,
                  const int* __restrict__ aterm_idx, const int* __restrict__ atoms,
                  const double* __restrict__ newpos, double lin_cutoff,
                  double* __restrict__ out, int64_t* __restrict__ status, int nblk,
                  double* __restrict__ part, long long* __restrict__ part_bad,
                  unsigned* __restrict__ count) {
  pdl_wait();
  pdl_launch_dependents();
  __shared__ double sh[32];
  __shared__ long long bad[3];
  __shared__ bool last_s;
  const int k = blockIdx.x / nblk, blk = blockIdx.x - k * nblk;
  const int a = atoms[k];
  const P3 np = {newpos[3 * k], newpos[3 * k + 1], newpos[3 * k + 2]};
  const P3 ca = ld3(coords, a);
  if (threadIdx.x < 3) bad[threadIdx.x] = kSentinel;
  __syncthreads();
  const int sb = fsp_ptr[a], se = fsp_ptr[a + 1];
  const bool lin = lin_cutoff > 0.0;
  const P3 dl = sub(np, ca);
  double dec = 0.0, dev = 0.0, far = 0.0;
  for (int j = blk * kDeltaThreads + threadIdx.x; j < tp.n; j += nblk * kDeltaThreads) {
    if (j == a) continue;
    // binary search of the (short, sorted) special row of atom a
    double s = 1.0;
    int lo = sb, hi = se;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (fsp_j[mid] < j) lo = mid + 1; else hi = mid;
    }
    if (lo < se && fsp_j[lo] == j) s = fsp_s[lo];
    const P3 cj = ld3(coords, j);
    const P3 o = sub(ca, cj);
    if (lin) {
      // far-field linearisation (ffmin/kernels.py:359-416): excluded / 1-4
      // partners and everything within the cutoff are treated exactly, the
      // far Coulomb sum by its gradient at the current position
      const double ro = sqrt(dot(o, o));
      if (!(ro <= lin_cutoff || s != 1.0)) {
        const double qq = tp.q[a] * tp.q[j];
        far += -kCoulomb * qq / (ro * ro * ro) * dot(o, dl);
        continue;
      }
      if (s == 0.0) continue;
      const P3 nn = sub(np, cj);
      const double rn = sqrt(dot(nn, nn));
      if (ro < kRmin || rn < kRmin) {
        atomicMin(&bad[0], (long long)j);
        continue;
      }
      const double qq = s * tp.q[a] * tp.q[j];
      dec += kCoulomb * qq * (1.0 / rn - 1.0 / ro);
      const double eps_ij = sqrt(tp.eps[a] * tp.eps[j]);
      if (eps_ij > 0.0) {
        const double sig = sqrt(tp.sigma[a] * tp.sigma[j]);
        const double to = sig / ro, to2 = to * to, xo = to2 * (to2 * to2);
        const double tn = sig / rn, tn2 = tn * tn, xn = tn2 * (tn2 * tn2);
        dev += 4.0 * s * eps_ij * ((xn * xn - xn) - (xo * xo - xo));
      }
      continue;
    }
    if (s == 0.0) continue;
    const P3 nn = sub(np, cj);
    const double ro = sqrt(dot(o, o)), rn = sqrt(dot(nn, nn));
    if (ro < kRmin || rn < kRmin) {
      atomicMin(&bad[0], (long long)j);
      continue;
    }
    const double qq = s * tp.q[a] * tp.q[j];
    const double eps_ij = sqrt(tp.eps[a] * tp.eps[j]);
    const double sig = sqrt(tp.sigma[a] * tp.sigma[j]);
    const bool in_old = !tp.has_cutoff || ro <= tp.cutoff;
    const bool in_new = !tp.has_cutoff || rn <= tp.cutoff;
    if (in_old) {
      dec -= kCoulomb * qq / ro;
      if (eps_ij > 0.0) {
        const double t = sig / ro, t2 = t * t, x = t2 * (t2 * t2);
        dev -= 4.0 * s * eps_ij * (x * x - x);
      }
    }
    if (in_new) {
      dec += kCoulomb * qq / rn;
      if (eps_ij > 0.0) {
        const double t = sig / rn, t2 = t * t, x = t2 * (t2 * t2);
        dev += 4.0 * s * eps_ij * (x * x - x);
      }
    }
  }
  // bonded terms touching the atom
  double db = 0.0, da = 0.0, dd = 0.0;
  for (int q = aterm_ptr[a] + threadIdx.x; blk == 0 && q < aterm_ptr[a + 1]; q += kDeltaThreads) {
    int t = aterm_idx[q];
    if (t < tp.nbond) {
      const int i = tp.bond_idx[2 * t], j = tp.bond_idx[2 * t + 1];
      P3 d = sub(ld3(coords, i), ld3(coords, j));
      const double dold = sqrt(dot(d, d)) - tp.bond_r0[t];
      d = sub(pick(coords, a, np, i), pick(coords, a, np, j));
      const double dnew = sqrt(dot(d, d)) - tp.bond_r0[t];
      db += tp.bond_K[t] * (dnew * dnew - dold * dold);
      continue;
    }
    t -= tp.nbond;
    if (t < tp.nangle) {
      const int i = tp.ang_idx[3 * t], j = tp.ang_idx[3 * t + 1], kk = tp.ang_idx[3 * t + 2];
      double eo, en;
      P3 g0, g1;
      if (!angle_term(ld3(coords, i), ld3(coords, j), ld3(coords, kk), tp.ang_K[t],
                      tp.ang_t0[t], false, &eo, &g0, &g1) ||
          !angle_term(pick(coords, a, np, i), pick(coords, a, np, j),
                      pick(coords, a, np, kk), tp.ang_K[t], tp.ang_t0[t], false, &en, &g0,
                      &g1)) {
        atomicMin(&bad[1], (long long)t);
        continue;
      }
      da += en - eo;
      continue;
    }
    t -= tp.nangle;
    const int* id = tp.dih_idx + 4 * t;
    double eo, en;
    P3 g[4];
    if (!dihedral_term(ld3(coords, id[0]), ld3(coords, id[1]), ld3(coords, id[2]),
                       ld3(coords, id[3]), tp.dih_V + 4 * t, false, &eo, g) ||
        !dihedral_term(pick(coords, a, np, id[0]), pick(coords, a, np, id[1]),
                       pick(coords, a, np, id[2]), pick(coords, a, np, id[3]),
                       tp.dih_V + 4 * t, false, &en, g)) {
      atomicMin(&bad[2], (long long)t);
      continue;
    }
    dd += en - eo;
  }
  dec = tree_sum(dec, sh);
  dev = tree_sum(dev, sh);
  db = tree_sum(db, sh);
  da = tree_sum(da, sh);
  dd = tree_sum(dd, sh);
  far = tree_sum(far, sh);
  double v[6] = {dec, dev, db, da, dd, far};
  long long bv[3] = {bad[0], bad[1], bad[2]};
  if (nblk > 1) {  // partials of this block; the last block of the candidate adds them
    if (threadIdx.x == 0) {
      double* p = part + 6 * ((size_t)k * nblk + blk);
      for (int q = 0; q < 6; ++q) p[q] = v[q];
      long long* pb = part_bad + 3 * ((size_t)k * nblk + blk);
      for (int q = 0; q < 3; ++q) pb[q] = bv[q];
      __threadfence();
      last_s = atomicAdd(count + k, 1u) == (unsigned)(nblk - 1);
    }
    __syncthreads();
    if (!last_s) return;
    if (threadIdx.x == 0) {
      __threadfence();
      for (int q = 0; q < 6; ++q) {
        double acc = 0.0;
        for (int b2 = 0; b2 < nblk; ++b2)
          acc += __ldcg(part + 6 * ((size_t)k * nblk + b2) + q);
        v[q] = acc;
      }
      for (int q = 0; q < 3; ++q) {
        long long m = kSentinel;
        for (int b2 = 0; b2 < nblk; ++b2) {
          const long long x = __ldcg(part_bad + 3 * ((size_t)k * nblk + b2) + q);
          m = x < m ? x : m;
        }
        bv[q] = m;
      }
      count[k] = 0;  // ready for the next launch
    }
  }
  if (threadIdx.x == 0) {
    const int w = lin ? 6 : 5;
    double* o = out + w * (size_t)k;
    o[0] = v[0];
    o[1] = v[1];
    o[2] = v[2];
    o[3] = v[3];
    o[4] = v[4];
    if (lin) o[5] = v[5];
    int64_t* s = status + 3 * (size_t)k;
    for (int q = 0; q < 3; ++q) s[q] = bv[q] == kSentinel ? -1 : (int64_t)bv[q];
  }
}

cudaError_t launch_atom_delta(const TermPlanDev& tp, const double* coords,
                              const int* fsp_ptr, const int* fsp_j, const double* fsp_s,
                              const int* aterm_ptr, const int* aterm_idx, int ncand,
                              const int* atoms, const double* newpos, double lin_cutoff,
                              double* out, int64_t* status, double* part,
                              long long* part_bad, unsigned* count, cudaStream_t st) {
  if (ncand <= 0) return cudaSuccess;
  const int nblk = part ? delta_blocks(tp.n) : 1;
  count_launch(), launch_k(atom_delta_kernel, ncand * nblk, kDeltaThreads, 0, st, tp, coords,
                           fsp_ptr, fsp_j, fsp_s, aterm_ptr, aterm_idx, atoms, newpos, lin_cutoff,
                           out, status, nblk, part, part_bad, count);
  return cudaGetLastError();
}

// ffmin/kernels.py:359-387 (_loop_farfield_build): far-field Coulomb energy of
// one atom and its gradient, and the exact near set; one block.
__global__ void __launch_bounds__(kDeltaThreads)
farfield_kernel(TermPlanDev tp, const double* __restrict__ coords,
                const int* __restrict__ fsp_ptr, const int* __restrict__ fsp_j,
                const double* __restrict__ fsp_s, int a, double cutoff,
                double* __restrict__ e0_coef, uint8_t* __restrict__ near_mask,
                int64_t* __restrict__ bad) {
  pdl_wait();
  pdl_launch_dependents();
  __shared__ double sh[32];
  __shared__ long long first_bad;
  if (threadIdx.x == 0) first_bad = kSentinel;
  __syncthreads();
  const P3 ca = ld3(coords, a);
  const int sb = fsp_ptr[a], se = fsp_ptr[a + 1];
  double e0 = 0.0, cx = 0.0, cy = 0.0, cz = 0.0;
  for (int j = threadIdx.x; j < tp.n; j += kDeltaThreads) {
    uint8_t near = 0;
    if (j != a) {
      double s = 1.0;
      int lo = sb, hi = se;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (fsp_j[mid] < j) lo = mid + 1; else hi = mid;
      }
      if (lo < se && fsp_j[lo] == j) s = fsp_s[lo];
      const P3 d = sub(ca, ld3(coords, j));
      const double r = sqrt(dot(d, d));
      if (r <= cutoff || s != 1.0) {
        near = 1;
      } else if (r < kRmin) {
        atomicMin(&first_bad, (long long)j);
      } else {
        const double qq = tp.q[a] * tp.q[j];
        e0 += kCoulomb * qq / r;
        const double g = -kCoulomb * qq / (r * r * r);
        cx += g * d.x;
        cy += g * d.y;
        cz += g * d.z;
      }
    }
    near_mask[j] = near;
  }
  e0 = tree_sum(e0, sh);
  cx = tree_sum(cx, sh);
  cy = tree_sum(cy, sh);
  cz = tree_sum(cz, sh);
  if (threadIdx.x == 0) {
    e0_coef[0] = e0;
    e0_coef[1] = cx;
    e0_coef[2] = cy;
    e0_coef[3] = cz;
    *bad = first_bad == kSentinel ? -1 : (int64_t)first_bad;
  }
}

cudaError_t launch_farfield(const TermPlanDev& tp, const double* coords, const int* fsp_ptr,
                            const int* fsp_j, const double* fsp_s, int atom, double cutoff,
                            double* e0_coef, uint8_t* near_mask, int64_t* bad,
                            cudaStream_t st) {
  count_launch();
  launch_k(farfield_kernel, 1, kDeltaThreads, 0, st, tp, coords, fsp_ptr, fsp_j, fsp_s, atom, cutoff,
                                               e0_coef, near_mask, bad);
  return cudaGetLastError();
}

}  // namespace ffm
