// ffm_min.cuh -- state of a device-resident L-BFGS run (ffm_lbfgs_*).
//
// The reference drives L-BFGS from Python: every line-search probe, every
// curvature dot product and every convergence test is a host decision
// (ffmin/optimizers/lbfgs.py:93-128, ffmin/linesearch.py, ffmin/optimizers/
// common.py).  Here the whole iteration runs as one CUDA graph with
// conditional nodes: single-thread controller kernels replay the reference's
// scalar logic on this struct (same IEEE double operations in the same
// order, compiled without FMA contraction), so no value leaves the device
// between iterations.  The host polls it once per chunk of iterations.
#pragma once
#include "ffm_kernels.h"

namespace ffm {

constexpr int kLsMaxPoints = 24;  // ls_par keeps <= K + 2 points per attempt

struct MinConfig {
  int m;                  // memory depth
  int ls_kind;            // 0 = ls_h, 1 = ls_par
  int K;                  // ls_par refinement budget
  int use_gs;             // ls_par: seed with the directional derivative
  int stop_on_ls_failure;
  int chunk;              // iterations per graph launch
  long long max_iter;     // -1: no bound
  long long max_calls;    // -1: no bound (value + gradient calls)
  double thr;             // gradient-norm threshold
  double h0, eps_h, k_plus, k_minus, trust;
  int method;          // kMethodLbfgs / kMethodCg / kMethodSd / kMethodFgm / kMethodFixed
  int cg_kind;         // 0..6: fr, prp, prp+, hs, cd, ls, dy
  int restart_period;  // CG: restart p <- -g every restart_period iterations
  int momentum_kind;   // fixed-step family: 0 GD, 1 heavy ball, 2 NAG, 3 NAG-SC
  double fixed_step, momentum;
  // OFGM: horizon N and the schedule t[0..N] (device array, ffm_lbfgs_set_schedule);
  // fixed_step > 0 selects the 1/L variant, else the line-searched one
  long long horizon;
  const double* sched;
  int ls_needs_grad;   // the line search seeds from the slope (ls_par + gradient start)
  int wig_epoch;       // wiggle: exact re-evaluation period (incremental probes)
  double wig_h, wig_cutoff;  // wiggle: probe step, linearisation cutoff (0: exact probes)
  const int* wig_atoms;      // wiggle: the atom of each iteration of a launch
};

enum : int { kMethodLbfgs = 0, kMethodCg = 1, kMethodSd = 2, kMethodFgm = 3, kMethodFixed = 4,
             kMethodOfgm = 5, kMethodWiggle = 6 };

// run status codes (host maps them to the reference's strings)
enum : int { kMinNone = 0, kMinConverged = 1, kMinIterBudget = 2, kMinLsFailure = 3,
             kMinOracleBudget = 4, kMinHorizon = 5 };
// error kinds
enum : int { kMinErrNone = 0, kMinErrEval = 1, kMinErrDiverged = 2 };

constexpr int kMinRecWidth = 8;  // k, f, |g|, step, value calls, grad calls, t (ns), best f

struct MinState {
  MinConfig c;
  // run
  long long k, vcalls, gcalls, nrec, iters_launch;
  int status, done, pause, cleared, err, err_grad;
  long long err_st[8];
  double f, gn;
  unsigned long long t_launch;
  // direction and the dot products the controllers consume
  double dd, dn, inv_dn, slope, gg, sy, ss, yy;
  // L-BFGS memory: ring slots of the m most recent pairs, oldest first,
  // and the free slots (LbfgsMemory._free); newest-first copies feed the
  // two-loop kernel
  int count, nfree, store_slot, pad0;
  int order[kMaxLbfgsPairs + 1];
  int freel[kMaxLbfgsPairs + 1];
  double rho[kMaxLbfgsPairs];
  int idx_nf[kMaxLbfgsPairs];
  double rho_nf[kMaxLbfgsPairs];
  // line search (LineSearcher warm start + one attempt's state)
  double warm;
  int attempt, stage, nref, np;
  double a_h0, lo, hi, f0;
  double ph[kLsMaxPoints], pf[kLsMaxPoints];
  double h_trial;
  double h_keep, f_keep;  // ls_h: first accepted probe
  int found, pad1;
  double res_h, res_f;
  // CG (ffmin/optimizers/cg.py): the running direction p lives in the
  // direction buffer; cgd = <g+,g+>, <g+,y>, <g,g>, <p,y>, <p,g>; pg = <p+,g+>
  int since_restart, failures, cg_reset, cg_else;
  double beta, cgd[5], pg;
  // best point so far (OptimizationRun.update_best) and FGM (ffmin/
  // optimizers/fgm.py): theta schedule, f at the extrapolated point w, the
  // end-of-iteration vector shift (1: x_prev <- x, x <- w; 2: x <- x+) and
  // which vector becomes the best point (1: w, 2: x+)
  double best_f, theta_prev, theta, fw;
  int fgm_mode, best_src;
  double f_init;  // f(x0): the fixed-step divergence test
  // OFGM: t_k, 1 - 1/t_{k+1}, 2/t_{k+1}, 1/t_{k+1}; the iteration's step
  double oc[4], step;
  // wiggle (ffmin/optimizers/wiggle.py): the iteration's atom, its six axis
  // probe values, vertex probe, chosen move and outcome
  int wig_atom, wig_vtx, wig_best, wig_moved;
  int ls_more, pad3;  // the probe controller's loop decision (small-system probe loop)
  double wig_pv[6], wig_vertex[3], wig_dv, wig_delta[3], wig_est;
};

}  // namespace ffm
