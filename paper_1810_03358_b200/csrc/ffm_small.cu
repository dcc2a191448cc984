// ffm_small.cu -- one-launch evaluation of a small system (tile mode).
//
// A system of up to a few thousand atoms costs ~2-20 us of pair work, less
// than the launch chain around it (pack, pair tiles, bonded terms, gather,
// reduction, finder: seven dependent kernels, ~40 us per evaluation inside
// an L-BFGS line search).  This cooperative kernel runs the same per-item
// bodies (ffm_device.cuh, ffm_tile.cuh) in phases separated by grid-wide
// barriers, so it produces the same bits as the kernel chain:
//
//   P0  pack coordinates into the pair records, reset the status words
//   P1  bonded / scaled-pair term blocks (CTA items) and 128 x 32 pair tiles
//       (warp items)
//   P2  gradient gather (thread items); energy reduction (CTA 0); every CTA
//       decides from the same data whether a coincidence is possible
//   P3  only then: the exact first-coincident-pair finder, and the status
//       conventions (CTA 0)
//
// Compiled with -fmad=false like ffm_terms.cu (the bonded terms need it; the
// pair tile arithmetic is explicit and flag-independent).
#include <algorithm>
#include <cstdlib>

#include <cooperative_groups.h>

#include "ffm_device.cuh"
#include "ffm_kernels.h"
#include "ffm_min_dev.cuh"
#include "ffm_tile.cuh"

namespace ffm {

namespace cg = cooperative_groups;

constexpr int kSmallThreads = 128;  // = kTermThreads = kRedThreads = 4 tile warps
static_assert(kSmallThreads == kTermThreads && kSmallThreads == kRedThreads, "block shape");
static_assert(kTermSlotsPerBlock == kTermThreads / 32, "term status slots: one per warp");

// FROMX (tiny systems, small_fromx): no packing pass and no barrier after
// P0 -- the pair tiles read positions and charges straight from the
// coordinates, line-search trial points are formed on the fly by every
// reader with the trial buffer's fma, and the term blocks leave their status
// in per-warp slots folded after P1; the same arithmetic, so the same bits.
template <typename T, bool GRAD, bool CUTOFF, bool FROMX>
__global__ void __launch_bounds__(kSmallThreads)
small_eval_kernel(SmallEvalArgs a) {
  using V4 = typename Vec4T<T>::type;
  using V2 = typename Vec2T<T>::type;
  __shared__ TileSmem<T> tsm;
  __shared__ double gpart[kGatherWarpsTiles][3][32];
  __shared__ double sh[5][kTermThreads / 32];
  __shared__ double red[32];
  __shared__ MinState ms;  // the probe controller's copy of the driver state
  __shared__ int64_t st_s[kStWords];
  __shared__ double en_s[5];  // stretch, bend, torsion, coulomb, vdw
  __shared__ int64_t shs[3][kTermThreads / 32];
  cg::grid_group grid = cg::this_grid();
  const NbPlanDev& plan = a.plan;
  const int n = plan.n;
  const int64_t gt = (int64_t)blockIdx.x * kSmallThreads + threadIdx.x;
  const int64_t gs = (int64_t)gridDim.x * kSmallThreads;
  V4* pos = static_cast<V4*>(a.pos);
  T* ipos = static_cast<T*>(a.ipos);
  T* ipart = static_cast<T*>(a.ipart);
  T* jpart = static_cast<T*>(a.jpart);
  // optional phase clock (tools/time_small_phases.py): [CTA][8] globaltimer
  // stamps (slots 0-5 used)
  unsigned long long* clk = a.phase_clock ? a.phase_clock + 8 * blockIdx.x : nullptr;
  auto stamp = [&](int k) {
    if (clk && threadIdx.x == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
      clk[k] = t;
    }
  };
  stamp(0);
  FFM_MSTAMP(4);
  // the probe controller (the last CTA, every pass) works on a shared-memory
  // copy of the driver state, read once per launch: its scalar logic is a
  // chain of dependent reads and writes (~4 us per probe as L2 round trips);
  // nothing else writes the state during the launch, and every pass writes
  // the copy back for the other CTAs (h_trial, ls_more) and the graph
  constexpr int kW = (int)(sizeof(MinState) / sizeof(unsigned long long));
  static_assert(sizeof(MinState) % sizeof(unsigned long long) == 0, "MinState words");
  unsigned long long* gw = reinterpret_cast<unsigned long long*>(a.ls_state);
  unsigned long long* sw = reinterpret_cast<unsigned long long*>(&ms);
  if (a.ls_state && blockIdx.x == gridDim.x - 1)
    for (int w = threadIdx.x; w < kW; w += kSmallThreads) sw[w] = gw[w];  // (synced below)

  // a line-search trial repeats the whole evaluation for every probe the
  // controller asks for (one launch per search instead of one per probe:
  // each probe would cost a conditional-node relaunch and a cooperative
  // launch, ~6 us, on systems whose evaluation takes ~10 us)
  for (;;) {
    // P0 (a line-search trial first forms its point x_t = lincomb(1, x, h, r),
    // the axpby of the host-driven loop, into the trial buffer)
    const double* coords = a.trial_out ? a.trial_out : a.coords;
    const double th = a.trial_out ? *(volatile const double*)a.trial_h : 0.0;
    // FROMX readers form x_t themselves; the others read the trial buffer
    const CoordSrc cs = FROMX && a.trial_out ? CoordSrc{a.trial_x, a.trial_r, th}
                                             : CoordSrc{coords, nullptr, 0.0};
    if constexpr (FROMX) {
      if (gt == 0) {
        int64_t* st = a.status;
        st[kStNbBadI] = -1;
        st[kStNbBadJ] = -1;
        st[kStBond] = kSentinel;
        st[kStAngle] = kSentinel;
        st[kStDihedral] = kSentinel;
        st[kStNbSuspect] = 0;
        st[kStNbKey] = kSentinel;
        st[kStCount] = 0;
      }
      if (a.trial_out)
        for (int64_t q = gt; q < 3 * (int64_t)n; q += gs) a.trial_out[q] = cs.at(q);
    } else {
      for (int64_t k = gt; k < (n > 1 ? n : 1); k += gs) {
        if (a.trial_out && k < n)
          for (int c = 0; c < 3; ++c) {
            const int64_t q = 3 * k + c;
            a.trial_out[q] = fma(th, a.trial_r[q], 1.0 * a.trial_x[q]);
          }
        pack_item<T>(k, n, plan.np, 1, coords, a.qt, pos, ipos, a.status);
      }
      grid.sync();
    }
    stamp(1);
    FFM_MSTAMP(10);

    // P1: CTA items -- the pair tiles (one CTA each, the longer items, first)
    // and the bonded / scaled-pair term blocks, dealt round-robin so a CTA
    // with a tile does not also run a term block when the grid covers both
    // (a cp.async double-buffered variant that fetched a CTA's next tile
    // during the current one measured no faster: a tile's loads are not its
    // critical path, profiles/r02_small_tile_loads.log)
    const int nitems = plan.nlaunch + a.nterm_blocks;
    for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
      if (it < plan.nlaunch)
        tile_cta<T, GRAD, CUTOFF, FROMX>(plan, pos, static_cast<const V2*>(a.lj), ipos,
                                         static_cast<const T*>(a.ilj), ipart, jpart, a.epart, it,
                                         0, tsm, cs, a.qt);
      else
        term_block(a.tp, GRAD, cs, a.term_part, a.term_f, a.status, 0, it - plan.nlaunch,
                   a.nterm_blocks, sh, FROMX ? a.term_st : nullptr);
    }
    __syncthreads();
    stamp(2);
    grid.sync();
    stamp(3);
    FFM_MSTAMP(11);

    // P2: the finder decision, made identically by every CTA: a coincident
    // pair shows as a non-finite tile partial (FP32) or a closest-pair r^2
    // below RMIN^2 (FP64), or was flagged by the scaled-pair terms.  Each
    // thread tests its tiles without an early exit, so its partial loads go
    // out together (the early-exit scan was ~ntiles / 128 dependent L2 round
    // trips per CTA: 6.7 us of the 3000-atom evaluation)
    int bad = FROMX ? 0 : *(volatile const int64_t*)(a.status + kStNbSuspect) != 0;
#pragma unroll 8
    for (int t = threadIdx.x; t < plan.ntiles; t += kSmallThreads) {
      const double* e = a.epart + 3 * (size_t)t;
      bad |= !isfinite(e[0]) | !isfinite(e[1]) | (e[2] < kRmin * kRmin);
    }
    int suspect = __syncthreads_or(bad);
    if constexpr (FROMX)  // the term blocks' slots (the last CTA also writes the status words)
      suspect |= status_from_term_slots(a.term_st, a.nterm_blocks * kTermSlotsPerBlock, a.status,
                                        blockIdx.x == gridDim.x - 1, shs);
    if (GRAD)  // 32-atom groups, the same 4-warp split as the chain's gather
      for (int g = blockIdx.x; g < ((n + 31) >> 5); g += gridDim.x)
        gather_group<T, kGatherWarpsTiles>(g, n, plan.S, plan.nb, nullptr, a.trow_ptr, a.tcol_ptr,
                                           a.tcol_idx, ipart, jpart, a.slot_ptr, a.slot_idx,
                                           a.term_f, a.tp.slot_sc0, true, true, true, a.grad,
                                           gpart);
    if (blockIdx.x == gridDim.x - 1)  // the gather groups fill the first CTAs
      reduce_entry(plan.ntiles, a.nterm_blocks, a.epart, a.term_part, a.energies, a.status, 0, red,
                   false);
    __syncthreads();
    stamp(4);
    if (suspect) {  // P3 (uniform across the grid)
      grid.sync();
      if constexpr (FROMX) {  // the finder reads packed positions: pack them now
        for (int64_t i = gt; i < n; i += gs) {
          V4 p;
          atom_record<T>(cs, a.qt, n, (int)i, p.x, p.y, p.z, p.w);
          pos[i] = p;
        }
        grid.sync();
      }
      for (int64_t i = gt; i < n; i += gs)
        finder_row<T>((int)i, n, pos, a.sp_ptr, a.sp_j, a.sp_s, a.status);
      grid.sync();
      if (blockIdx.x == 0 && threadIdx.x == 0) a.status[kStNbSuspect] = 1;  // as the chain leaves it
    }
    // the CTA that reduced the energies finalises the status words and, for a
    // line-search trial, runs the probe controller (ffm_min_dev.cuh)
    FFM_MSTAMP_LAST(12);
    if (blockIdx.x == gridDim.x - 1) {
      // (the status words and energies likewise: every input is read in one
      // round trip, the outputs written back together)
      if (threadIdx.x < kStWords) st_s[threadIdx.x] = a.status[threadIdx.x];
      else if (threadIdx.x < kStWords + 5) en_s[threadIdx.x - kStWords] = a.energies[threadIdx.x - kStWords];
      __syncthreads();
      FFM_MSTAMP_LAST(15);
      if (threadIdx.x == 0) {
        finalize_entry(n, st_s);
        if (a.ls_state) mindev::ls_step(&ms, en_s, st_s, a.ls_loop);
      }
      FFM_MSTAMP_LAST(16);
      __syncthreads();
      if (a.ls_state)
        for (int w = threadIdx.x; w < kW; w += kSmallThreads) gw[w] = sw[w];
      if (threadIdx.x < kStWords) a.status[threadIdx.x] = st_s[threadIdx.x];
    }
    FFM_MSTAMP_LAST(13);
    stamp(5);
    FFM_MSTAMP(5);
    if (!a.ls_state) break;
    grid.sync();  // the controller's decision and next step are visible to all CTAs
    FFM_MSTAMP(14);
    if (!*(volatile int*)&a.ls_state->ls_more) break;
  }
}

template <typename T, bool GRAD, bool CUTOFF>
static void* small_kernel_ptr(bool fromx) {
  return fromx ? reinterpret_cast<void*>(&small_eval_kernel<T, GRAD, CUTOFF, true>)
               : reinterpret_cast<void*>(&small_eval_kernel<T, GRAD, CUTOFF, false>);
}

static void* small_kernel(bool fp64, bool grad, bool cut, bool fromx) {
  if (fp64) {
    if (grad) return cut ? small_kernel_ptr<double, true, true>(fromx) : small_kernel_ptr<double, true, false>(fromx);
    return cut ? small_kernel_ptr<double, false, true>(fromx) : small_kernel_ptr<double, false, false>(fromx);
  }
  if (grad) return cut ? small_kernel_ptr<float, true, true>(fromx) : small_kernel_ptr<float, true, false>(fromx);
  return cut ? small_kernel_ptr<float, false, true>(fromx) : small_kernel_ptr<float, false, false>(fromx);
}

// The FROMX variant (small_eval_kernel) where it measured faster (one B200,
// profiles/r02_small_tile_loads.log): FP32 evaluations up to 1500 atoms
// (500 atoms 16.5 -> 14.6 us, 1500 18.1 -> 16.9 us) and line-search trials
// in both precisions (FP64 L-BFGS, 500 atoms 0.179 -> 0.174 ms per
// iteration); a single FP64 evaluation keeps the packing pass (500 atoms
// 13.1 vs 14.6 us).
#ifndef FFM_SMALL_FROMX_MAXN
#define FFM_SMALL_FROMX_MAXN 1500
#endif
bool small_fromx(const SmallEvalArgs& a, bool fp64) {
  // tuning / test overrides, read per call (a launch is captured once per graph)
  const char* fm = getenv("FFM_SMALL_FROMX_MAXN");
  const int maxn = fm ? atoi(fm) : FFM_SMALL_FROMX_MAXN;
  const char* ff = getenv("FFM_SMALL_FROMX_F64");  // FP64 single evaluations too
  const bool f64_all = ff && atoi(ff) != 0;
  return a.plan.n <= maxn && a.term_st != nullptr && (!fp64 || f64_all || a.ls_state != nullptr);
}

int small_eval_grid(const SmallEvalArgs& a, bool fp64, bool grad, int device) {
  const bool cut = a.plan.has_cutoff != 0;
  int sms = 0, per_sm = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(
          &per_sm, small_kernel(fp64, grad, cut, small_fromx(a, fp64)), kSmallThreads, 0) !=
          cudaSuccess)
    return 0;
  int64_t want = 1;
  want = std::max<int64_t>(want, (int64_t)a.plan.nlaunch + a.nterm_blocks);
  want = std::max<int64_t>(want, (3 * (int64_t)a.plan.n + kSmallThreads - 1) / kSmallThreads);
  return (int)std::min<int64_t>(want, (int64_t)sms * per_sm);
}

cudaError_t launch_small_eval(const SmallEvalArgs& a, bool fp64, bool grad, int grid,
                              cudaStream_t st) {
  if (grid < 1) return cudaErrorInvalidConfiguration;
  SmallEvalArgs args = a;
  void* params[] = {&args};
  count_launch();
  return cudaLaunchCooperativeKernel(small_kernel(fp64, grad, a.plan.has_cutoff != 0, small_fromx(a, fp64)),
                                     dim3(grid), dim3(kSmallThreads), params, 0, st);
}

}  // namespace ffm

#ifdef FFM_MIN_STAMPS
extern "C" int ffm_debug_min_clock_small(void* clock_d) {
  return (int)cudaMemcpyToSymbol(ffm::g_mclk, &clock_d, sizeof(void*));
}
#endif
