// ffm_kernels.h -- host-side launch wrappers shared by the C-ABI layer.
#pragma once
#include "ffm_common.cuh"
#include "ffm_plan.cuh"

#include <atomic>
#include <cstdlib>
#include <utility>

namespace ffm {

// every kernel launch of the engine, for the benchmark's gpu_launches claim
extern std::atomic<long long> g_launch_count;
inline void count_launch(long long k = 1) { g_launch_count.fetch_add(k, std::memory_order_relaxed); }

// Kernel launch with programmatic stream serialization (PDL): the next
// kernel of a dependent chain is scheduled onto SMs freed by its
// predecessor's last wave and starts the moment the predecessor completes
// (pdl_wait, ffm_common.cuh), instead of after a full launch latency --
// inside the captured evaluation / minimiser graphs too.  FFM_PDL=0 turns
// it off (plain launches).
inline bool pdl_enabled() {
  static const bool on = [] {
    const char* f = getenv("FFM_PDL");
    return f ? atoi(f) != 0 : true;
  }();
  return on;
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                            cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

size_t nb_smem_bytes(int S, bool fp64, bool grad, int nw);
int nb_warps(int S, bool fp64, int nlaunch);  // warps per CTA of the super-unit sweep

// all-pairs sweep over every super-unit; batch > 1 only without GRAD.
// pos/lj: j-side records; ipos/ilj: the same data in the i-side pair layout
// bbox: per 32-atom block bounding boxes (cutoff culling), null without cutoff
cudaError_t launch_nb(const NbPlanDev& plan, bool fp64, bool grad, const void* pos,
                      const void* lj, const void* ipos, const void* ilj, const void* bbox,
                      void* ipart, void* jpart, double* epart, int batch, cudaStream_t st);
cudaError_t launch_bbox(int n, int np, int batch, bool fp64, const void* pos, void* bbox,
                        cudaStream_t st);

// coords (fp64, [batch][n][3]) -> padded pos / ipos records of the chosen
// precision; also resets the status words of every batch entry.
cudaError_t launch_pack(int n, int np, int batch, bool fp64, const double* coords,
                        const double* qt, void* pos, void* ipos, int64_t* status,
                        cudaStream_t st);

// fills the padding atoms (zero charge / LJ, far apart) once per buffer
cudaError_t launch_pad(int n, int np, int batch, bool fp64, void* pos, void* ipos,
                       cudaStream_t st);

// LJ (a, b) records -> i-side pair layout (once per system)
// ilj from the FP64 (a, b) records, scaled by LjIScale<T>
cudaError_t launch_ilj(int np, bool fp64, const void* lj64, void* ilj, cudaStream_t st);

// bonded + scaled-pair terms in FP64; writes per-block energy partials
// term_part[batch][term_blocks(tp)][5] and slot forces
int term_blocks(const TermPlanDev& tp);
cudaError_t launch_terms(const TermPlanDev& tp, bool grad, int batch, const double* coords,
                         double* term_part, double* term_f, int64_t* status, cudaStream_t st);

// energies[batch][5] = (stretch, bend, torsion, coulomb, vdw); flags suspect
// coincidences for the finder
// (clean entries are finalised here: sentinels -> -1; n = atoms)
// batch 1 with escratch: split over energy_parts(nunits) blocks (reduce_split)
cudaError_t launch_reduce(int nunits, const TermPlanDev& tp, int batch, const double* epart,
                          const double* term_part, double* energies, int64_t* status, int n,
                          double* escratch, unsigned* ecount, cudaStream_t st);
// blocks of the split energy reduction: one per kEnergySlotsPerPart slots;
// escratch holds kMaxEnergyParts x 3 doubles, ecount one counter (zeroed)
constexpr int kEnergySlotsPerPart = 2048;
constexpr int kMaxEnergyParts = 64;
int energy_parts(int nslots);

// batch 1: the gradient gather (gather_group, ffm_device.cuh: tile mode
// when trow_ptr is set, else super-unit mode) and the energy reduction in
// one launch
constexpr int kGatherWarpsUnits = 8;
constexpr int kGatherWarpsTiles = 4;
cudaError_t launch_gather_reduce(int n, int S, int nb, bool fp64, const int* unit_index,
                                 const int* trow_ptr, const int* tcol_ptr, const int* tcol_idx,
                                 const void* ipart, const void* jpart, const int* slot_ptr,
                                 const int* slot_idx, const double* term_f, int slot_sc0,
                                 bool use_nb, bool use_terms, bool use_sc, double* grad,
                                 int nslots, const TermPlanDev& tp, const double* epart,
                                 const double* term_part, double* energies, int64_t* status,
                                 int rank, int nranks, double* escratch, unsigned* ecount,
                                 cudaStream_t st);

// exact first coincident pair (reference loop order), only when flagged;
// the last block then converts the status sentinels to -1.
cudaError_t launch_finder(int n, int np, int batch, bool fp64, const void* pos,
                          const int* sp_ptr, const int* sp_j, const double* sp_s,
                          int64_t* status, cudaStream_t st);

// exact single-atom move deltas (ffmin/energy.py:284-313) for a batch of
// candidate moves: out[k][5] = (coulomb, vdw, stretch, bend, torsion) deltas;
// status[k][3] = (bad nonbonded partner j, bad angle row, bad dihedral row)
cudaError_t launch_atom_delta(const TermPlanDev& tp, const double* coords,
                              const int* fsp_ptr, const int* fsp_j, const double* fsp_s,
                              const int* aterm_ptr, const int* aterm_idx, int ncand,
                              const int* atoms, const double* newpos, double lin_cutoff,
                              double* out, int64_t* status, double* part, long long* part_bad,
                              unsigned* count, cudaStream_t st);
// blocks per candidate of launch_atom_delta (with scratch: part [ncand *
// blocks][6], part_bad [ncand * blocks][3], count [ncand] zeroed; null part:
// one block per candidate)
int delta_blocks(int n);

// far-field linearisation of one atom: e0_coef[4] = (E_far, dE/dx, dE/dy,
// dE/dz), near_mask[n], bad = first coincident far partner or -1
cudaError_t launch_farfield(const TermPlanDev& tp, const double* coords, const int* fsp_ptr,
                            const int* fsp_j, const double* fsp_s, int atom, double cutoff,
                            double* e0_coef, uint8_t* near_mask, int64_t* bad,
                            cudaStream_t st);

// ---- fused small-system evaluation (ffm_small.cu) ----
// One cooperative launch = pack + term blocks + pair tiles + gather +
// reduction (+ finder when flagged) for a tile-mode system evaluated whole
// (batch 1, unsharded, all terms), same bits as the kernel chain.
// term status slots per term block (one per warp of its kTermThreads)
constexpr int kTermSlotsPerBlock = 4;
struct SmallEvalArgs {
  NbPlanDev plan;
  TermPlanDev tp;
  int nterm_blocks;
  const double* coords;
  const double* qt;
  void* pos;
  void* ipos;
  const void* lj;
  const void* ilj;
  void* ipart;
  void* jpart;
  double* epart;
  double* term_part;
  double* term_f;
  int64_t* term_st;  // [nterm_blocks * kTermSlotsPerBlock][4] term status slots (tiny systems)
  const int* trow_ptr;
  const int* tcol_ptr;
  const int* tcol_idx;
  const int* slot_ptr;
  const int* slot_idx;
  const int* sp_ptr;
  const int* sp_j;
  const double* sp_s;
  double* grad;
  double* energies;
  int64_t* status;
  unsigned long long* phase_clock;  // null, or [grid][8] timestamps (tuning aid)
  // line-search trial of a graph-resident driver (null trial_out: a plain
  // evaluation of coords): the point x_t = lincomb(1, trial_x, *trial_h,
  // trial_r) is formed into trial_out and evaluated, then the probe
  // controller runs on ls_state and sets the probe loop's condition ls_loop
  double* trial_out;
  const double* trial_x;
  const double* trial_r;
  const double* trial_h;
  struct MinState* ls_state;
  cudaGraphConditionalHandle ls_loop;
};
// grid size (co-resident CTAs, at most what the work needs) of the kernel
// variant this call selects (small_fromx); 0 on error
int small_eval_grid(const SmallEvalArgs& a, bool fp64, bool grad, int device);
bool small_fromx(const SmallEvalArgs& a, bool fp64);
cudaError_t launch_small_eval(const SmallEvalArgs& a, bool fp64, bool grad, int grid,
                              cudaStream_t st);

// ---- sharded evaluations completed on the device (ffm_vec.cu): pack the
// rank's partial [gradient | energies | error words] into buf (3n + 13
// doubles; grad null: the 13-word tail only), and unpack the all-reduced sums
cudaError_t launch_combine_encode(int64_t natoms, const double* grad, const double* energies,
                                  const int64_t* status, double* buf, cudaStream_t st);
cudaError_t launch_combine_decode(int64_t natoms, const double* buf, double* grad,
                                  double* energies, int64_t* status, cudaStream_t st);

// ---- vector algebra (ffm_vec.cu) ----
int vec_reduce_blocks();
cudaError_t launch_dot(int64_t n, const double* x, const double* y, double* part,
                       double* out, cudaStream_t st);
cudaError_t launch_dots(int64_t n, int k, const double* const* x, const double* const* y,
                        double* part, double* out, cudaStream_t st);
cudaError_t launch_axpby(int64_t n, const double* a_dev, double a_host, double sa,
                         const double* x, const double* b_dev, double b_host,
                         const double* y, double* z, cudaStream_t st);
constexpr int kMaxLbfgsPairs = 32;
size_t two_loop_scratch_doubles();
cudaError_t launch_lbfgs_two_loop(int64_t n, int count, const int* idx, const double* rho,
                                  const double* S, const double* Y, const double* g,
                                  double* q, double* scratch, cudaStream_t st);
// the same with count / slots / rho / |g| read from device memory
// m: the ring capacity (sizes the short-vector variant's shared staging)
cudaError_t launch_lbfgs_two_loop_dev(int64_t n, int m, const int* count, const int* idx,
                                      const double* rho, const double* gn, const double* S,
                                      const double* Y, const double* g, double* q,
                                      double* scratch, cudaStream_t st);
cudaError_t two_loop_small_prepare();  // once, outside graph capture

// ---- device-resident L-BFGS controllers (ffm_minimize.cu, state in ffm_min.cuh) ----
struct MinState;
cudaError_t launch_min_launch_begin(MinState* S, cudaStream_t st);
cudaError_t launch_min_it_begin(MinState* S, cudaGraphConditionalHandle hdir,
                                cudaGraphConditionalHandle hls, cudaGraphConditionalHandle hacc,
                                cudaStream_t st);
cudaError_t launch_min_dir(MinState* S, cudaGraphConditionalHandle hls, cudaStream_t st);
cudaError_t launch_min_ls_init(MinState* S, cudaGraphConditionalHandle hloop, cudaStream_t st);
cudaError_t launch_min_ls_step(MinState* S, const double* en, const int64_t* stw,
                               cudaGraphConditionalHandle hloop, cudaStream_t st);
cudaError_t launch_min_ls_post(MinState* S, double* rec, cudaGraphConditionalHandle hacc,
                               cudaStream_t st);
cudaError_t launch_min_acc_check(MinState* S, const int64_t* stw, cudaStream_t st);
cudaError_t launch_min_commit(MinState* S, cudaStream_t st);
// nonlinear CG: beta from S->cgd, p+ in place, descent check, p <- -src when S->cg_reset
cudaError_t launch_min_cg_beta(MinState* S, cudaStream_t st);
cudaError_t launch_cg_update(MinState* S, int64_t n, const double* g_new, double* p,
                             cudaStream_t st);
cudaError_t launch_min_cg_check(MinState* S, cudaStream_t st);
cudaError_t launch_select_neg(MinState* S, int64_t n, const double* src, double* dst,
                              cudaStream_t st);
// FGM: theta / beta (heval = evaluate at w when k > 0), checks and |g_w| after
// the evaluation, the accepted step, and the end-of-iteration vector shift
cudaError_t launch_fgm_pre(MinState* S, cudaGraphConditionalHandle heval, cudaStream_t st);
cudaError_t launch_fgm_post_eval(MinState* S, const double* en, const int64_t* stw,
                                 cudaGraphConditionalHandle hls, cudaStream_t st);
cudaError_t launch_fgm_accept(MinState* S, double* rec, cudaStream_t st);
// fixed-step family: momentum coefficient (heval = gradient at w), the
// check after grad f(w), and the bookkeeping after the evaluation at x+
cudaError_t launch_mom_pre(MinState* S, cudaGraphConditionalHandle heval, int has_eval,
                           cudaStream_t st);
cudaError_t launch_mom_wcheck(MinState* S, const int64_t* stw, cudaStream_t st);
cudaError_t launch_mom_post(MinState* S, const double* en, const int64_t* stw, double* rec,
                            cudaStream_t st);
// OFGM (Eq. (12)): schedule coefficients, the dn == 0 / search split, value
// and gradient bookkeeping, the search result, x from y, end of iteration
cudaError_t launch_ofgm_pre(MinState* S, cudaStream_t st);
cudaError_t launch_ofgm_dir(MinState* S, cudaGraphConditionalHandle hz,
                            cudaGraphConditionalHandle hnz, cudaStream_t st);
cudaError_t launch_ofgm_value(MinState* S, const double* en, const int64_t* stw, int which,
                              cudaStream_t st);
cudaError_t launch_ofgm_gcheck(MinState* S, const int64_t* stw, cudaStream_t st);
cudaError_t launch_ofgm_ls_post(MinState* S, cudaStream_t st);
cudaError_t launch_ofgm_x(MinState* S, int64_t n, const double* y, const double* r, double* x,
                          int from_ls, cudaStream_t st);
cudaError_t launch_ofgm_post(MinState* S, const double* en, const int64_t* stw, double* rec,
                             int from_en, cudaStream_t st);
// gradient-free wiggle (ffmin/optimizers/wiggle.py): probe positions, the
// three decisions (vertex probe hv, exact check hx, epoch re-evaluation he)
cudaError_t launch_wig_prep(MinState* S, const double* coords, int* atoms6, double* newpos6,
                            cudaStream_t st);
cudaError_t launch_wig_ctrl1(MinState* S, const double* out, const int64_t* stw, int* atoms1,
                             cudaGraphConditionalHandle hv, cudaStream_t st);
cudaError_t launch_wig_pos(MinState* S, const double* coords, double* newpos1, int which,
                           cudaStream_t st);
cudaError_t launch_wig_ctrl_v(MinState* S, const double* out, const int64_t* stw,
                              cudaStream_t st);
cudaError_t launch_wig_ctrl2(MinState* S, cudaGraphConditionalHandle hx, cudaStream_t st);
cudaError_t launch_wig_ctrl3(MinState* S, const double* out, const int64_t* stw, double* coords,
                             cudaStream_t st);
cudaError_t launch_wig_end(MinState* S, cudaGraphConditionalHandle he, cudaStream_t st);
cudaError_t launch_wig_epoch(MinState* S, const double* en, const int64_t* stw, cudaStream_t st);
cudaError_t launch_wig_record(MinState* S, double* rec, cudaStream_t st);
cudaError_t launch_fgm_shift(MinState* S, int64_t n, double* x, double* x_prev, const double* w,
                             const double* x_new, double* best, cudaStream_t st);
cudaError_t launch_min_store(MinState* S, int64_t n, const double* s_tmp, const double* y_tmp,
                             double* ring_s, double* ring_y, const double* x_new,
                             const double* g_new, double* x, double* g, cudaStream_t st);
cudaError_t launch_min_iter_end(MinState* S, double* rec, cudaStream_t st);
// the L-BFGS direction of a short vector in one launch (two-loop, <d,d>,
// min_dir, r = d / |d|, <g,r>); _prepare once outside graph capture
bool lbfgs_dir_small_applies(int64_t n, int m);
cudaError_t lbfgs_dir_small_prepare();
cudaError_t launch_lbfgs_dir_small(MinState* S, int64_t n, int m, double* d, double* r,
                                   const double* S_ring, const double* Y_ring, const double* g,
                                   cudaGraphConditionalHandle hls, cudaStream_t st);
// the L-BFGS acceptance tail of a short vector in one launch (n <= kAcceptSmallN)
constexpr int64_t kAcceptSmallN = 3072;  // (2000 atoms: one block measured slower than the chain)
cudaError_t launch_lbfgs_accept_small(MinState* S, int64_t n, const int64_t* stw,
                                      const double* x_new, const double* g_new, double* x,
                                      double* g, double* s_tmp, double* y_tmp, double* ring_s,
                                      double* ring_y, double* rec, cudaStream_t st);
cudaError_t launch_min_it_end(MinState* S, cudaGraphConditionalHandle hout, cudaStream_t st);

}  // namespace ffm
