// ffm_minimize.cu -- controller kernels of the graph-resident L-BFGS.
//
// Each controller is a single-thread kernel that advances the scalar part of
// the reference's L-BFGS iteration on MinState (ffm_min.cuh) and steers the
// CUDA graph through conditional handles; the vector work (two-loop
// recursion, dot products, axpby, energy/gradient evaluations) stays in the
// engine's own kernels.  The scalar logic restates, operation for operation:
//   ffmin/optimizers/lbfgs.py:93-128   iteration, memory clear-and-retry
//   ffmin/optimizers/lbfgs.py:20-50    curvature guard, ring of m pairs
//   ffmin/linesearch.py (ls_h, ls_par) one-dimensional searches
//   ffmin/optimizers/common.py         LineSearcher warm start and retry,
//                                      budget checks, trace records
// This file is compiled with -fmad=false: every product and sum rounds
// separately, as in the reference's Python float arithmetic.
#include "ffm_min_dev.cuh"
#include "ffm_two_loop.cuh"

namespace ffm {

namespace {

using namespace mindev;

__global__ void min_launch_begin_kernel(MinState* S) {
  pdl_wait();
  pdl_launch_dependents();
  S->iters_launch = 0;
  S->pause = 0;
  S->nrec = 0;
  S->t_launch = globaltimer();
}

__global__ void min_it_begin_kernel(MinState* S, cudaGraphConditionalHandle hdir,
                                    cudaGraphConditionalHandle hls,
                                    cudaGraphConditionalHandle hacc) {
  pdl_wait();
  FFM_MSTAMP(1);
  pdl_launch_dependents();
  cudaGraphSetConditional(hls, 0);
  cudaGraphSetConditional(hacc, 0);
  unsigned go = 0;
  const MinConfig& c = S->c;
  if (!S->done) {
    // Run.budget_status order: iterations, (wall time: host, per chunk), calls
    if (c.method == kMethodOfgm && S->k >= c.horizon) {  // fgm.py: checked first
      S->status = kMinHorizon;
      S->done = 1;
    } else if (c.max_iter >= 0 && S->k >= c.max_iter) {
      S->status = kMinIterBudget;
      S->done = 1;
    } else if (c.max_calls >= 0 && S->vcalls + S->gcalls >= c.max_calls) {
      S->status = kMinOracleBudget;
      S->done = 1;
    } else if (S->iters_launch >= c.chunk) {
      S->pause = 1;
    } else {
      S->iters_launch++;
      go = 1;
    }
  }
  cudaGraphSetConditional(hdir, go);
}

// after d (two-loop or antigradient) and <d, d>
__global__ void min_dir_kernel(MinState* S, cudaGraphConditionalHandle hls) {
  pdl_wait();
  FFM_MSTAMP(2);
  pdl_launch_dependents();
  if (S->c.method == kMethodSd) {
    // r = div(lincomb(-1, g), |g|)  (ffmin/optimizers/gradient.py, Eq. (4))
    S->dn = S->gn;
    S->inv_dn = 1.0 / S->gn;
    cudaGraphSetConditional(hls, 1);
    return;
  }
  if (S->c.method == kMethodCg) {
    // pn = |p|; a zero p restarts along the antigradient with pn = |g|
    // (ffmin/optimizers/cg.py:107-110)
    double pn = sqrt(S->dd);
    S->cg_reset = 0;
    if (pn == 0.0) {
      S->cg_reset = 1;  // p <- -g (select_neg_kernel)
      pn = S->gn;
      S->since_restart = 0;
    }
    S->dn = pn;
    S->inv_dn = 1.0 / pn;
    cudaGraphSetConditional(hls, 1);
    return;
  }
  const double dn = sqrt(S->dd);
  S->dn = dn;
  if (dn == 0.0) {
    S->status = kMinConverged;
    S->done = 1;
    cudaGraphSetConditional(hls, 0);
    return;
  }
  S->inv_dn = 1.0 / dn;  // ops.div(d, dn) = lincomb(1 / dn, d)
  cudaGraphSetConditional(hls, 1);
}

// after r = d / |d| and slope = <g, r>: LineSearcher.search, first attempt
__global__ void min_ls_init_kernel(MinState* S, cudaGraphConditionalHandle hloop) {
  pdl_wait();
  FFM_MSTAMP(3);
  pdl_launch_dependents();
  if (S->err) {  // an evaluation before the search failed (OFGM: value(y))
    cudaGraphSetConditional(hloop, 0);
    return;
  }
  // FGM searches from w, OFGM from y
  S->f0 = (S->c.method == kMethodFgm || S->c.method == kMethodOfgm) ? S->fw : S->f;
  S->attempt = 0;
  ls_start(S, S->warm);
  cudaGraphSetConditional(hloop, 1);
}

__global__ void min_ls_step_kernel(MinState* S, const double* en, const int64_t* stw,
                                   cudaGraphConditionalHandle hloop) {
  pdl_wait();
  pdl_launch_dependents();
  ls_step(S, en, stw, hloop);
}

// lbfgs.py: what a line-search result does to the iteration
__global__ void min_ls_post_kernel(MinState* S, double* rec, cudaGraphConditionalHandle hacc) {
  pdl_wait();
  FFM_MSTAMP(7);
  pdl_launch_dependents();
  unsigned acc = 0;
  if (!S->err && S->c.method == kMethodFgm) {
    // ffmin/optimizers/fgm.py: a failed search stops the run, or records an
    // idle iteration and moves x to w
    if (!S->found) {
      if (S->c.stop_on_ls_failure) {
        S->status = kMinLsFailure;
        S->done = 1;
      } else {
        S->k++;
        const double f = S->f;
        S->f = S->fw;  // record(k, f_w, gn, 0.0)
        record(S, rec, 0.0);
        S->f = f;
        S->fgm_mode = 1;
        S->theta_prev = S->theta;
      }
    } else {
      acc = 1;
    }
    cudaGraphSetConditional(hacc, acc);
    return;
  }
  if (!S->err && S->c.method == kMethodCg) {
    // ffmin/optimizers/cg.py:112-124: a second consecutive failure ends the
    // run (or records an idle iteration); every failure restarts p <- -g
    S->cg_reset = 0;
    if (!S->found) {
      S->failures++;
      if (S->failures >= 2) {
        if (S->c.stop_on_ls_failure) {
          S->status = kMinLsFailure;
          S->done = 1;
          cudaGraphSetConditional(hacc, 0);
          return;
        }
        S->k++;
        record(S, rec, 0.0);
        S->failures = 0;
      }
      S->cg_reset = 1;
      S->since_restart = 0;
    } else {
      S->failures = 0;
      acc = 1;
    }
    cudaGraphSetConditional(hacc, acc);
    return;
  }
  if (!S->err) {
    if (!S->found) {
      if (S->count > 0 && !S->cleared) {
        memory_clear(S);  // stale metric: drop it, retry along the antigradient
        S->cleared = 1;
      } else if (S->c.stop_on_ls_failure) {
        S->status = kMinLsFailure;
        S->done = 1;
      } else {
        S->k++;
        record(S, rec, 0.0);
        S->cleared = 0;
      }
    } else {
      S->cleared = 0;
      acc = 1;
    }
  }
  cudaGraphSetConditional(hacc, acc);
}

// after the gradient at x_new and <g_new, g_new>
__device__ inline void acc_check(MinState* S, const int64_t* stw) {
  S->gcalls++;
  if (bad_status(stw, true)) {
    set_err(S, kMinErrEval, stw, true);
    return;
  }
  if (!isfinite(S->res_f) || !isfinite(S->gg)) set_err(S, kMinErrDiverged, nullptr, true);
}

__global__ void min_acc_check_kernel(MinState* S, const int64_t* stw) {
  pdl_wait();
  pdl_launch_dependents();
  acc_check(S, stw);
}

// after <s,y>, <s,s>, <y,y>: LbfgsMemory._commit
__device__ inline void commit(MinState* S) {
  S->store_slot = -1;
  if (S->err) return;
  const double sy = S->sy, ss = S->ss, yy = S->yy;
  if (!(sy > 1e-12 * sqrt(ss) * sqrt(yy))) return;  // curvature guard
  const int m = S->c.m;
  const int slot = S->freel[0];
  for (int q = 1; q < S->nfree; ++q) S->freel[q - 1] = S->freel[q];
  S->nfree--;
  if (S->count == m) {  // evict the oldest pair, its slot becomes free
    S->freel[S->nfree++] = S->order[0];
    for (int q = 1; q < m; ++q) {
      S->order[q - 1] = S->order[q];
      S->rho[q - 1] = S->rho[q];
    }
    S->count--;
  }
  S->order[S->count] = slot;
  S->rho[S->count] = 1.0 / sy;
  S->count++;
  for (int q = 0; q < S->count; ++q) {  // newest first for the two-loop kernel
    S->idx_nf[q] = S->order[S->count - 1 - q];
    S->rho_nf[q] = S->rho[S->count - 1 - q];
  }
  S->store_slot = slot;
}

__global__ void min_commit_kernel(MinState* S) {
  pdl_wait();
  FFM_MSTAMP(8);
  pdl_launch_dependents();
  commit(S);
}

__global__ void min_store_kernel(const MinState* S, int64_t n, const double* __restrict__ s_tmp,
                                 const double* __restrict__ y_tmp, double* __restrict__ ring_s,
                                 double* __restrict__ ring_y, const double* __restrict__ x_new,
                                 const double* __restrict__ g_new, double* __restrict__ x,
                                 double* __restrict__ g) {
  pdl_wait();
  pdl_launch_dependents();
  if (S->err) return;
  const int slot = S->store_slot;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (slot >= 0) {
      ring_s[(int64_t)slot * n + i] = s_tmp[i];
      ring_y[(int64_t)slot * n + i] = y_tmp[i];
    }
    x[i] = x_new[i];
    g[i] = g_new[i];
  }
}

// ---- nonlinear CG (ffmin/optimizers/cg.py:125-145), after the five dot
// products <g+,g+>, <g+,y>, <g,g>, <p,y>, <p,g> (y = g+ - g)
__device__ double cg_beta_of(int kind, const double* d) {
  const double gg_new = d[0], gy = d[1], gg_old = d[2], py = d[3], pg = d[4];
  double num, den;
  switch (kind) {
    case 0: num = gg_new; den = gg_old; break;                // fr
    case 1: num = gy; den = gg_old; break;                    // prp
    case 2: num = (0.0 > gy) ? 0.0 : gy; den = gg_old; break;  // prp+: max(gy, 0.0)
    case 3: num = gy; den = py; break;                        // hs
    case 4: num = gg_new; den = -pg; break;                   // cd
    case 5: num = gy; den = -pg; break;                       // ls
    default: num = gg_new; den = py; break;                   // dy
  }
  return den == 0.0 ? (double)NAN : num / den;
}

__global__ void min_cg_beta_kernel(MinState* S) {
  pdl_wait();
  pdl_launch_dependents();
  if (S->err) return;
  S->since_restart++;
  if (S->since_restart >= S->c.restart_period) {
    S->cg_else = 0;  // periodic restart: p+ = -g+
    S->since_restart = 0;
    S->beta = 0.0;
  } else {
    S->cg_else = 1;
    S->beta = cg_beta_of(S->c.cg_kind, S->cgd);
  }
}

// p+ = lincomb(-1, g+, beta, p) for a finite beta, else lincomb(-1, g+);
// in place (each element reads its old p first)
__global__ void cg_update_kernel(const MinState* S, int64_t n, const double* __restrict__ g_new,
                                 double* __restrict__ p) {
  pdl_wait();
  pdl_launch_dependents();
  if (S->err) return;
  const double beta = S->beta;
  const bool use_beta = S->cg_else && isfinite(beta);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double v = -1.0 * g_new[i];
    p[i] = use_beta ? fma(beta, p[i], v) : v;
  }
}

// descent test dot(p+, -g+) <= 0 (= -<p+, g+>, the negation is exact) or a
// non-finite beta: restart p+ = -g+
__global__ void min_cg_check_kernel(MinState* S) {
  pdl_wait();
  pdl_launch_dependents();
  S->cg_reset = 0;
  if (S->err || !S->cg_else) return;
  if (!isfinite(S->beta) || -S->pg <= 0.0) {
    S->cg_reset = 1;
    S->since_restart = 0;
  }
}

// dst = lincomb(-1, src) when *flag (device-decided restarts)
__global__ void select_neg_kernel(const int* flag, const int* err, int64_t n,
                                  const double* __restrict__ src, double* __restrict__ dst) {
  pdl_wait();
  pdl_launch_dependents();
  if (!*flag || *err) return;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = -1.0 * src[i];
}

// ---- FGM (ffmin/optimizers/fgm.py, Algorithm 1)
// theta_k and beta_k from theta_{k-1}; the caller then forms
// w = lincomb(1, x, beta, lincomb(1, x, -1, x_prev))
__global__ void fgm_pre_kernel(MinState* S, cudaGraphConditionalHandle heval) {
  pdl_wait();
  pdl_launch_dependents();
  const double tp = S->theta_prev;
  const double theta = 0.5 * tp * (sqrt(tp * tp + 4.0) - tp);
  S->theta = theta;
  S->beta = tp * (1.0 - tp) / (tp * tp + theta);
  S->fgm_mode = 0;
  S->best_src = 0;
  cudaGraphSetConditional(heval, S->k > 0 ? 1u : 0u);  // k == 0: f_w, g_w = f, g
}

// after f(w), grad f(w) (k > 0) and <g_w, g_w>: finiteness, best point,
// |g_w| and the convergence test, then the search direction scale
__global__ void fgm_post_eval_kernel(MinState* S, const double* en, const int64_t* stw,
                                     cudaGraphConditionalHandle hls) {
  pdl_wait();
  pdl_launch_dependents();
  cudaGraphSetConditional(hls, 0);
  if (S->k > 0) {
    S->vcalls++;
    S->gcalls++;
    if (bad_status(stw, true)) {
      set_err(S, kMinErrEval, stw, true);
      return;
    }
    S->fw = en[0] + en[1] + en[2] + en[3] + en[4];
  } else {
    S->fw = S->f;
  }
  if (!isfinite(S->fw) || !isfinite(S->gg)) {
    set_err(S, kMinErrDiverged, nullptr, true);
    return;
  }
  if (S->fw < S->best_f) {
    S->best_f = S->fw;
    S->best_src = 1;
  }
  S->gn = sqrt(S->gg);
  if (S->gn <= S->c.thr) {
    S->status = kMinConverged;
    S->done = 1;
    return;
  }
  S->dn = S->gn;
  S->inv_dn = 1.0 / S->gn;  // r = div(lincomb(-1, g_w), |g_w|)
  cudaGraphSetConditional(hls, 1);
}

__global__ void fgm_accept_kernel(MinState* S, double* rec) {
  pdl_wait();
  pdl_launch_dependents();
  S->f = S->res_f;
  S->theta_prev = S->theta;
  S->k++;
  if (S->f < S->best_f) {
    S->best_f = S->f;
    S->best_src = 2;
  }
  record(S, rec, S->res_h);
  S->fgm_mode = 2;
}

// end of an FGM iteration: best point copy, then x_prev <- x, x <- w or x+
__global__ void fgm_shift_kernel(const MinState* S, int64_t n, double* __restrict__ x,
                                 double* __restrict__ x_prev, const double* __restrict__ w,
                                 const double* __restrict__ x_new, double* __restrict__ best) {
  pdl_wait();
  pdl_launch_dependents();
  if (S->err) return;
  const int mode = S->fgm_mode, bs = S->best_src;
  if (mode == 0 && bs == 0) return;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (bs) best[i] = bs == 1 ? w[i] : x_new[i];
    if (mode) {
      x_prev[i] = x[i];
      x[i] = mode == 1 ? w[i] : x_new[i];
    }
  }
}

// ---- fixed-step family (ffmin/optimizers/gradient.py): GD, heavy ball,
// Nesterov (NAG, NAG-SC).  coef(k) and whether the gradient at w is needed
__global__ void mom_pre_kernel(MinState* S, cudaGraphConditionalHandle heval, int has_eval) {
  pdl_wait();
  pdl_launch_dependents();
  const int kind = S->c.momentum_kind;
  const double k = (double)S->k;
  S->beta = kind == 2 ? (k - 1.0) / (k + 2.0) : S->c.momentum;
  S->fgm_mode = 2;  // x_prev <- x, x <- x+ (fgm_shift_kernel)
  S->best_src = 0;
  if (has_eval) cudaGraphSetConditional(heval, (kind >= 2 && S->k > 0) ? 1u : 0u);
}

// after grad f(w) (Nesterov schemes, k > 0): oracle.gradient(w)
__global__ void mom_wcheck_kernel(MinState* S, const int64_t* stw) {
  pdl_wait();
  pdl_launch_dependents();
  S->gcalls++;
  if (bad_status(stw, true)) set_err(S, kMinErrEval, stw, true);
}

// after f (and grad f) at x+ and <g, g>: call counts, error / divergence
// tests, record, convergence
__global__ void mom_post_kernel(MinState* S, const double* en, const int64_t* stw, double* rec) {
  pdl_wait();
  pdl_launch_dependents();
  if (S->err) return;
  const int kind = S->c.momentum_kind;
  const bool wform = kind >= 2;
  S->vcalls++;
  if (!wform) S->gcalls++;  // value_and_gradient(x+)
  if (bad_status(stw, !wform)) {
    set_err(S, kMinErrEval, stw, !wform);
    return;
  }
  const double f = en[0] + en[1] + en[2] + en[3] + en[4];
  const double af0 = fabs(S->f_init);
  const bool diverged = !isfinite(f) || (kind > 0 && f > 1e3 * (af0 > 1.0 ? af0 : 1.0));
  S->f = f;
  if (diverged || !isfinite(S->gg)) {
    set_err(S, kMinErrDiverged, nullptr, true);
    return;
  }
  S->gn = sqrt(S->gg);
  S->k++;
  if (f < S->best_f) S->best_f = f;
  record(S, rec, S->c.fixed_step);
  if (S->gn <= S->c.thr) {
    S->status = kMinConverged;
    S->done = 1;
  }
}

// ---- OFGM (ffmin/optimizers/fgm.py, Eq. (12))
// the schedule coefficients of iteration k (host arithmetic: 1.0 - 1.0 / t,
// 2.0 / t, 1.0 / t)
__global__ void ofgm_pre_kernel(MinState* S) {
  pdl_wait();
  pdl_launch_dependents();
  const double tk = S->c.sched[S->k], tk1 = S->c.sched[S->k + 1];
  S->oc[0] = tk;
  S->oc[1] = 1.0 - 1.0 / tk1;
  S->oc[2] = 2.0 / tk1;
  S->oc[3] = 1.0 / tk1;
  S->step = S->c.fixed_step;
  S->fgm_mode = 0;
  S->best_src = 0;
}

// line-searched variant, after <d, d>: dn == 0 takes x = y (hz), else the
// search along -d / |d| from y (hnz)
__global__ void ofgm_dir_kernel(MinState* S, cudaGraphConditionalHandle hz,
                                cudaGraphConditionalHandle hnz) {
  pdl_wait();
  pdl_launch_dependents();
  const double dn = sqrt(S->dd);
  S->dn = dn;
  if (dn == 0.0) {
    S->step = 0.0;
    cudaGraphSetConditional(hz, 1);
    cudaGraphSetConditional(hnz, 0);
  } else {
    S->inv_dn = 1.0 / dn;
    cudaGraphSetConditional(hz, 0);
    cudaGraphSetConditional(hnz, 1);
  }
}

// after an energy-only evaluation: value(y) (which = 0: f_y, seeds the
// search) or value(x) with x = y (which = 1: f)
__global__ void ofgm_value_kernel(MinState* S, const double* en, const int64_t* stw, int which) {
  pdl_wait();
  pdl_launch_dependents();
  if (S->err) return;
  S->vcalls++;
  if (bad_status(stw, false)) {
    set_err(S, kMinErrEval, stw, false);
    return;
  }
  const double f = en[0] + en[1] + en[2] + en[3] + en[4];
  if (which == 0) S->fw = f; else S->f = f;
}

// after a gradient evaluation (gradient(y) for the slope, gradient(x))
__global__ void ofgm_gcheck_kernel(MinState* S, const int64_t* stw) {
  pdl_wait();
  pdl_launch_dependents();
  if (S->err) return;
  S->gcalls++;
  if (bad_status(stw, true)) set_err(S, kMinErrEval, stw, true);
}

// the search result: x = lincomb(1, y, h, r) when found, else x = y with f_y
__global__ void ofgm_ls_post_kernel(MinState* S) {
  pdl_wait();
  pdl_launch_dependents();
  if (S->err) return;
  if (S->found) {
    S->step = S->res_h;
    S->f = S->res_f;
  } else {
    S->step = 0.0;
    S->f = S->fw;
  }
}

__global__ void ofgm_x_kernel(const MinState* S, int64_t n, const double* __restrict__ y,
                              const double* __restrict__ r, double* __restrict__ x, int from_ls) {
  pdl_wait();
  pdl_launch_dependents();
  if (S->err) return;
  const bool move = from_ls && S->found;
  const double h = S->res_h;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    x[i] = move ? fma(h, r[i], 1.0 * y[i]) : y[i];
}

// end of an OFGM iteration, after grad f(x) and <g, g> (from_en: the 1/L
// variant's value_and_gradient(x) supplies f and both call counts)
__global__ void ofgm_post_kernel(MinState* S, const double* en, const int64_t* stw, double* rec,
                                 int from_en) {
  pdl_wait();
  pdl_launch_dependents();
  if (S->err) return;
  if (from_en) {
    S->vcalls++;
    S->gcalls++;
    if (bad_status(stw, true)) {
      set_err(S, kMinErrEval, stw, true);
      return;
    }
    S->f = en[0] + en[1] + en[2] + en[3] + en[4];
  }
  const double f = S->f;
  const double af0 = fabs(S->f_init);
  if (!isfinite(f) || f > 1e3 * (af0 > 1.0 ? af0 : 1.0) || !isfinite(S->gg)) {
    set_err(S, kMinErrDiverged, nullptr, true);
    return;
  }
  S->gn = sqrt(S->gg);
  S->k++;
  if (f < S->best_f) S->best_f = f;
  record(S, rec, S->step);
  if (S->gn <= S->c.thr) {
    S->status = kMinConverged;
    S->done = 1;
  }
}

// ---- gradient-free atom wiggle (ffmin/optimizers/wiggle.py)
constexpr double kWigAcceptMargin = 1e-9;  // wiggle.py ACCEPT_MARGIN

// a probe's energy change (out row of atom_delta_kernel); +inf when the move
// hit degenerate geometry (the reference catches the evaluation error)
__device__ inline double wig_value(const double* o, const int64_t* st, bool lin) {
  if (st[0] >= 0 || st[1] >= 0 || st[2] >= 0) return (double)INFINITY;
  double v = o[2] + o[3] + o[4] + o[0] + o[1];  // float(o[2]) + ... left to right
  if (lin) v += o[5];
  return v;
}

// the iteration's atom and its six axis probes (+-h along x, y, z)
__global__ void wig_prep_kernel(MinState* S, const double* __restrict__ coords,
                                int* __restrict__ atoms6, double* __restrict__ newpos6) {
  pdl_wait();
  pdl_launch_dependents();
  const int a = S->c.wig_atoms[S->iters_launch - 1];
  S->wig_atom = a;
  const double h = S->c.wig_h;
  for (int i = 0; i < 6; ++i) {
    const int axis = i >> 1;
    const double step = (i & 1) ? 1.0 * h : -1.0 * h;
    atoms6[i] = a;
    for (int c = 0; c < 3; ++c) newpos6[3 * i + c] = coords[3 * a + c] + (c == axis ? step : 0.0);
  }
}

// the six probe values -> per-axis parabola vertex (fit_parabola through
// (-h, dm), (0, 0), (h, dp); without an interior minimum the best probe
// offset); a non-zero vertex is probed next (hv)
__global__ void wig_ctrl1_kernel(MinState* S, const double* __restrict__ out,
                                 const int64_t* __restrict__ st, int* __restrict__ atoms1,
                                 cudaGraphConditionalHandle hv) {
  pdl_wait();
  pdl_launch_dependents();
  const bool lin = S->c.wig_cutoff > 0.0;
  const int w = lin ? 6 : 5;
  const double h = S->c.wig_h;
  for (int i = 0; i < 6; ++i) S->wig_pv[i] = wig_value(out + w * i, st + 3 * i, lin);
  S->vcalls += 6;
  bool any = false;
  for (int axis = 0; axis < 3; ++axis) {
    const double dm = S->wig_pv[2 * axis], dp = S->wig_pv[2 * axis + 1];
    bool have = false;
    double v = 0.0;
    if (isfinite(dm) && isfinite(dp)) {
      const double x0 = -h, x1 = 0.0, x2 = h, f0 = dm, f1 = 0.0, f2 = dp;
      const double s01 = (f1 - f0) / (x1 - x0);
      const double s12 = (f2 - f1) / (x2 - x1);
      const double curv = (s12 - s01) / (x2 - x0);
      double mx = fabs(f0);
      if (fabs(f1) > mx) mx = fabs(f1);
      if (fabs(f2) > mx) mx = fabs(f2);
      const bool degenerate = fabs(curv) < 1e-12 * mx;
      if (!(curv <= 0.0 || degenerate)) {
        have = true;
        v = 0.5 * (x0 + x1) - s01 / (2.0 * curv);
      }
    }
    double vx;
    if (!have) {  // min(choices): (value, offset) tuples, lexicographic
      double bv = 0.0, bo = 0.0;
      if (isfinite(dm) && (dm < bv || (dm == bv && -h < bo))) bv = dm, bo = -h;
      if (isfinite(dp) && (dp < bv || (dp == bv && h < bo))) bv = dp, bo = h;
      vx = bo;
    } else {  // min(max(v, -10 h), 10 h), Python's first-maximum semantics
      const double lo = -10.0 * h, hi = 10.0 * h;
      const double t = lo > v ? lo : v;
      vx = hi < t ? hi : t;
    }
    S->wig_vertex[axis] = vx;
    any = any || vx != 0.0;
  }
  S->wig_vtx = any ? 1 : 0;
  S->wig_dv = (double)INFINITY;
  atoms1[0] = S->wig_atom;  // the single-candidate probes (vertex, exact)
  cudaGraphSetConditional(hv, any ? 1u : 0u);
}

// newpos1 = coords[atom] + (vertex | delta)  (which = 0: vertex, 1: delta)
__global__ void wig_pos_kernel(const MinState* S, const double* __restrict__ coords,
                               double* __restrict__ newpos1, int which) {
  pdl_wait();
  pdl_launch_dependents();
  const int a = S->wig_atom;
  const double* d = which ? S->wig_delta : S->wig_vertex;
  for (int c = 0; c < 3; ++c) newpos1[c] = coords[3 * a + c] + d[c];
}

__global__ void wig_ctrl_v_kernel(MinState* S, const double* __restrict__ out,
                                  const int64_t* __restrict__ st) {
  pdl_wait();
  pdl_launch_dependents();
  S->wig_dv = wig_value(out, st, S->c.wig_cutoff > 0.0);
  S->vcalls++;
}

// the candidate of least estimated change (axis probes in order, then the
// vertex; first minimum as min(..., key=...)); a clear decrease is checked
// exactly next (hx)
__global__ void wig_ctrl2_kernel(MinState* S, cudaGraphConditionalHandle hx) {
  pdl_wait();
  pdl_launch_dependents();
  const double h = S->c.wig_h;
  int best = -1;
  double bv = 0.0;
  for (int i = 0; i < 6; ++i)
    if (isfinite(S->wig_pv[i]) && (best < 0 || S->wig_pv[i] < bv)) best = i, bv = S->wig_pv[i];
  if (S->wig_vtx && isfinite(S->wig_dv) && (best < 0 || S->wig_dv < bv)) best = 6, bv = S->wig_dv;
  S->wig_best = best;
  S->wig_moved = 0;
  unsigned go = 0;
  if (best >= 0) {
    for (int c = 0; c < 3; ++c)
      S->wig_delta[c] = best == 6 ? S->wig_vertex[c]
                                  : (c == (best >> 1) ? ((best & 1) ? 1.0 * h : -1.0 * h) : 0.0);
    S->wig_est = bv;
    go = bv < -kWigAcceptMargin ? 1u : 0u;
  }
  cudaGraphSetConditional(hx, go);
}

// the exact change decides: coords[atom] += delta, e += exact
__global__ void wig_ctrl3_kernel(MinState* S, const double* __restrict__ out,
                                 const int64_t* __restrict__ st, double* __restrict__ coords) {
  pdl_wait();
  pdl_launch_dependents();
  const double exact = wig_value(out, st, false);
  if (isfinite(exact)) S->vcalls++;
  if (exact < -kWigAcceptMargin) {
    const int a = S->wig_atom;
    for (int c = 0; c < 3; ++c) coords[3 * a + c] = coords[3 * a + c] + S->wig_delta[c];
    S->f = S->f + exact;
    S->wig_moved = 1;
  }
}

// end of an iteration: k, the epoch re-evaluation (he), then the record
__global__ void wig_end_kernel(MinState* S, cudaGraphConditionalHandle he) {
  pdl_wait();
  pdl_launch_dependents();
  S->k++;
  const bool epoch = S->c.wig_cutoff > 0.0 && S->k % S->c.wig_epoch == 0;
  cudaGraphSetConditional(he, epoch ? 1u : 0u);
}

__global__ void wig_epoch_kernel(MinState* S, const double* en, const int64_t* stw) {
  pdl_wait();
  pdl_launch_dependents();
  if (bad_status(stw, false)) {
    set_err(S, kMinErrEval, stw, false);
    return;
  }
  S->f = en[0] + en[1] + en[2] + en[3] + en[4];
  S->vcalls++;
}

// record (k, e, -, step, calls, -, t, best): the move's components ride in
// columns 2, 3, 5 (NaN in 2 when nothing moved); the host takes the norm
__global__ void wig_record_kernel(MinState* S, double* rec) {
  pdl_wait();
  pdl_launch_dependents();
  if (S->err) return;
  if (S->f < S->best_f) S->best_f = S->f;
  double* r = rec + S->nrec * kMinRecWidth;
  const bool m = S->wig_moved != 0;
  r[0] = (double)S->k;
  r[1] = S->f;
  r[2] = m ? S->wig_delta[0] : (double)NAN;
  r[3] = m ? S->wig_delta[1] : 0.0;
  r[4] = (double)S->vcalls;
  r[5] = m ? S->wig_delta[2] : 0.0;
  r[6] = (double)(globaltimer() - S->t_launch);
  r[7] = S->best_f;
  S->nrec++;
}

__device__ inline void iter_end(MinState* S, double* rec) {
  if (S->err) return;
  S->f = S->res_f;
  S->gn = sqrt(S->gg);
  S->k++;
  if (S->f < S->best_f) S->best_f = S->f;
  record(S, rec, S->res_h);
  if (S->gn <= S->c.thr) {
    S->status = kMinConverged;
    S->done = 1;
  }
}

__global__ void min_iter_end_kernel(MinState* S, double* rec) {
  pdl_wait();
  pdl_launch_dependents();
  iter_end(S, rec);
}

// The L-BFGS direction of a short vector (n <= 256 kTwoLoopSmallE) as one
// block: the two-loop d (two_loop_small_body, written to D.q), <d, d>, the
// min_dir step (|d|, 1 / |d|, the line-search condition) and, when the
// search runs, r = d / |d| and its slope <g, r> -- five graph nodes (the
// two-loop, two dot launches, min_dir, the search's axpby) in one, each
// step with the arithmetic and reduction order of its own kernel: the same
// bits.
__global__ void __launch_bounds__(kTwoLoopThreads)
lbfgs_dir_small_kernel(MinState* S, TwoLoopDevArgs D, double* __restrict__ r,
                       cudaGraphConditionalHandle hls) {
  pdl_wait();
  pdl_launch_dependents();
  extern __shared__ double ring[];
  __shared__ double sh2[kTwoLoopThreads / 32];
  __shared__ double inv_s;
  __shared__ int go_s;
  const int t = threadIdx.x;
  const int n = (int)D.n;
  double q[kTwoLoopSmallE];
  two_loop_small_body(D, ring, q);
  double acc = 0.0;  // <d, d> (dots_small_kernel order)
#pragma unroll
  for (int e = 0; e < kTwoLoopSmallE; ++e)
    if (t + e * kTwoLoopThreads < n) acc = fma(q[e], q[e], acc);
  acc = two_loop_block_sum(acc, sh2);
  if (t == 0) {  // min_dir_kernel, L-BFGS branch
    S->dd = acc;
    const double dn = sqrt(S->dd);
    S->dn = dn;
    int go = 1;
    if (dn == 0.0) {
      S->status = kMinConverged;
      S->done = 1;
      go = 0;
    } else {
      S->inv_dn = 1.0 / dn;  // ops.div(d, dn) = lincomb(1 / dn, d)
    }
    cudaGraphSetConditional(hls, go ? 1u : 0u);
    inv_s = go ? S->inv_dn : 0.0;
    go_s = go;
  }
  __syncthreads();
  if (!go_s) return;
  // r = (1 / |d|) d (axpby_kernel: v = a x; z = 1 v) and <g, r>
  double sl = 0.0;
#pragma unroll
  for (int e = 0; e < kTwoLoopSmallE; ++e) {
    const int i = t + e * kTwoLoopThreads;
    if (i < n) {
      const double v = 1.0 * (inv_s * q[e]);
      r[i] = v;
      sl = fma(D.g[i], v, sl);
    }
  }
  sl = two_loop_block_sum(sl, sh2);
  if (t == 0) S->slope = sl;
}

// The L-BFGS acceptance tail of a short vector (n <= kAcceptSmallN) as one
// block: <g+,g+>, the acceptance checks, s = x+ - x, y = g+ - g, <s,y>,
// <s,s>, <y,y>, the memory commit, the ring store and the iteration record
// -- eight graph nodes in one, each step with the arithmetic and reduction
// order of its own kernel (axpby_kernel, dots_small_kernel: one block,
// per-thread strides of 256, then the block sum), so the same bits.  The
// scalar steps run on a shared copy of the driver state.
constexpr int kAcceptThreads = 256;
__device__ __forceinline__ double block_sum_accept(double v, double* sh) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < kAcceptThreads / 32; ++w) t += sh[w];
  __syncthreads();
  return t;  // thread 0
}

__global__ void __launch_bounds__(kAcceptThreads)
lbfgs_accept_small_kernel(MinState* S, int64_t n, const int64_t* __restrict__ stw,
                          const double* __restrict__ x_new, const double* __restrict__ g_new,
                          double* __restrict__ x, double* __restrict__ g, double* __restrict__ st,
                          double* __restrict__ yt, double* __restrict__ ring_s,
                          double* __restrict__ ring_y, double* rec) {
  pdl_wait();
  pdl_launch_dependents();
  __shared__ MinState ms;
  __shared__ double sh[kAcceptThreads / 32];
  constexpr int kW = (int)(sizeof(MinState) / sizeof(unsigned long long));
  unsigned long long* gw = reinterpret_cast<unsigned long long*>(S);
  unsigned long long* sw = reinterpret_cast<unsigned long long*>(&ms);
  const int t = threadIdx.x;
  for (int w = t; w < kW; w += kAcceptThreads) sw[w] = gw[w];
  // <g+, g+> (launch_dots, one product)
  double acc = 0.0;
  for (int64_t i = t; i < n; i += kAcceptThreads) acc = fma(g_new[i], g_new[i], acc);
  acc = block_sum_accept(acc, sh);  // (its barriers also publish ms)
  if (t == 0) {
    ms.gg = acc;
    acc_check(&ms, stw);
  }
  // s = x+ - x, y = g+ - g (axpby_kernel: v = 1 x+; v = fma(-1, x, v); z = 1 v)
  for (int64_t i = t; i < n; i += kAcceptThreads) {
    double v = 1.0 * x_new[i];
    v = fma(-1.0, x[i], v);
    st[i] = 1.0 * v;
    double w = 1.0 * g_new[i];
    w = fma(-1.0, g[i], w);
    yt[i] = 1.0 * w;
  }
  __syncthreads();
  // <s,y>, <s,s>, <y,y>
  const double* xa[3] = {st, st, yt};
  const double* ya[3] = {yt, st, yt};
  double d3[3];
  for (int q = 0; q < 3; ++q) {
    double a = 0.0;
    for (int64_t i = t; i < n; i += kAcceptThreads) a = fma(xa[q][i], ya[q][i], a);
    d3[q] = block_sum_accept(a, sh);
  }
  __shared__ int slot_s, err_s;
  if (t == 0) {
    ms.sy = d3[0];
    ms.ss = d3[1];
    ms.yy = d3[2];
    commit(&ms);
    slot_s = ms.store_slot;
    err_s = ms.err;
  }
  __syncthreads();
  // the ring store and x <- x+, g <- g+ (min_store_kernel)
  if (!err_s) {
    const int slot = slot_s;
    for (int64_t i = t; i < n; i += kAcceptThreads) {
      if (slot >= 0) {
        ring_s[(int64_t)slot * n + i] = st[i];
        ring_y[(int64_t)slot * n + i] = yt[i];
      }
      x[i] = x_new[i];
      g[i] = g_new[i];
    }
  }
  if (t == 0) iter_end(&ms, rec);
  __syncthreads();
  for (int w = t; w < kW; w += kAcceptThreads) gw[w] = sw[w];
}

__global__ void min_it_end_kernel(MinState* S, cudaGraphConditionalHandle hout) {
  pdl_wait();
  FFM_MSTAMP(9);
  pdl_launch_dependents();
  S->fgm_mode = 0;  // consumed by fgm_shift_kernel
  S->best_src = 0;
  cudaGraphSetConditional(hout, (!S->done && !S->pause) ? 1u : 0u);
}

}  // namespace

#define FFM_ONE(kern, ...)                   \
  do {                                       \
    count_launch();                          \
    launch_k(kern, 1, 1, 0, st, __VA_ARGS__);      \
    return cudaGetLastError();               \
  } while (0)

cudaError_t launch_min_launch_begin(MinState* S, cudaStream_t st) {
  FFM_ONE(min_launch_begin_kernel, S);
}
cudaError_t launch_min_it_begin(MinState* S, cudaGraphConditionalHandle hdir,
                                cudaGraphConditionalHandle hls, cudaGraphConditionalHandle hacc,
                                cudaStream_t st) {
  FFM_ONE(min_it_begin_kernel, S, hdir, hls, hacc);
}
cudaError_t launch_min_dir(MinState* S, cudaGraphConditionalHandle hls, cudaStream_t st) {
  FFM_ONE(min_dir_kernel, S, hls);
}
cudaError_t launch_min_ls_init(MinState* S, cudaGraphConditionalHandle hloop, cudaStream_t st) {
  FFM_ONE(min_ls_init_kernel, S, hloop);
}
cudaError_t launch_min_ls_step(MinState* S, const double* en, const int64_t* stw,
                               cudaGraphConditionalHandle hloop, cudaStream_t st) {
  FFM_ONE(min_ls_step_kernel, S, en, stw, hloop);
}
cudaError_t launch_min_ls_post(MinState* S, double* rec, cudaGraphConditionalHandle hacc,
                               cudaStream_t st) {
  FFM_ONE(min_ls_post_kernel, S, rec, hacc);
}
cudaError_t launch_min_acc_check(MinState* S, const int64_t* stw, cudaStream_t st) {
  FFM_ONE(min_acc_check_kernel, S, stw);
}
cudaError_t launch_min_commit(MinState* S, cudaStream_t st) { FFM_ONE(min_commit_kernel, S); }
cudaError_t launch_min_cg_beta(MinState* S, cudaStream_t st) { FFM_ONE(min_cg_beta_kernel, S); }
cudaError_t launch_fgm_pre(MinState* S, cudaGraphConditionalHandle heval, cudaStream_t st) {
  FFM_ONE(fgm_pre_kernel, S, heval);
}
cudaError_t launch_fgm_post_eval(MinState* S, const double* en, const int64_t* stw,
                                 cudaGraphConditionalHandle hls, cudaStream_t st) {
  FFM_ONE(fgm_post_eval_kernel, S, en, stw, hls);
}
cudaError_t launch_fgm_accept(MinState* S, double* rec, cudaStream_t st) {
  FFM_ONE(fgm_accept_kernel, S, rec);
}
cudaError_t launch_ofgm_pre(MinState* S, cudaStream_t st) { FFM_ONE(ofgm_pre_kernel, S); }
cudaError_t launch_wig_prep(MinState* S, const double* coords, int* atoms6, double* newpos6,
                            cudaStream_t st) {
  FFM_ONE(wig_prep_kernel, S, coords, atoms6, newpos6);
}
cudaError_t launch_wig_ctrl1(MinState* S, const double* out, const int64_t* stw, int* atoms1,
                             cudaGraphConditionalHandle hv, cudaStream_t st) {
  FFM_ONE(wig_ctrl1_kernel, S, out, stw, atoms1, hv);
}
cudaError_t launch_wig_pos(MinState* S, const double* coords, double* newpos1, int which,
                           cudaStream_t st) {
  FFM_ONE(wig_pos_kernel, S, coords, newpos1, which);
}
cudaError_t launch_wig_ctrl_v(MinState* S, const double* out, const int64_t* stw,
                              cudaStream_t st) {
  FFM_ONE(wig_ctrl_v_kernel, S, out, stw);
}
cudaError_t launch_wig_ctrl2(MinState* S, cudaGraphConditionalHandle hx, cudaStream_t st) {
  FFM_ONE(wig_ctrl2_kernel, S, hx);
}
cudaError_t launch_wig_ctrl3(MinState* S, const double* out, const int64_t* stw, double* coords,
                             cudaStream_t st) {
  FFM_ONE(wig_ctrl3_kernel, S, out, stw, coords);
}
cudaError_t launch_wig_end(MinState* S, cudaGraphConditionalHandle he, cudaStream_t st) {
  FFM_ONE(wig_end_kernel, S, he);
}
cudaError_t launch_wig_epoch(MinState* S, const double* en, const int64_t* stw, cudaStream_t st) {
  FFM_ONE(wig_epoch_kernel, S, en, stw);
}
cudaError_t launch_wig_record(MinState* S, double* rec, cudaStream_t st) {
  FFM_ONE(wig_record_kernel, S, rec);
}
cudaError_t launch_ofgm_dir(MinState* S, cudaGraphConditionalHandle hz,
                            cudaGraphConditionalHandle hnz, cudaStream_t st) {
  FFM_ONE(ofgm_dir_kernel, S, hz, hnz);
}
cudaError_t launch_ofgm_value(MinState* S, const double* en, const int64_t* stw, int which,
                              cudaStream_t st) {
  FFM_ONE(ofgm_value_kernel, S, en, stw, which);
}
cudaError_t launch_ofgm_gcheck(MinState* S, const int64_t* stw, cudaStream_t st) {
  FFM_ONE(ofgm_gcheck_kernel, S, stw);
}
cudaError_t launch_ofgm_ls_post(MinState* S, cudaStream_t st) { FFM_ONE(ofgm_ls_post_kernel, S); }
cudaError_t launch_ofgm_post(MinState* S, const double* en, const int64_t* stw, double* rec,
                             int from_en, cudaStream_t st) {
  FFM_ONE(ofgm_post_kernel, S, en, stw, rec, from_en);
}
cudaError_t launch_mom_pre(MinState* S, cudaGraphConditionalHandle heval, int has_eval,
                           cudaStream_t st) {
  FFM_ONE(mom_pre_kernel, S, heval, has_eval);
}
cudaError_t launch_mom_wcheck(MinState* S, const int64_t* stw, cudaStream_t st) {
  FFM_ONE(mom_wcheck_kernel, S, stw);
}
cudaError_t launch_mom_post(MinState* S, const double* en, const int64_t* stw, double* rec,
                            cudaStream_t st) {
  FFM_ONE(mom_post_kernel, S, en, stw, rec);
}
cudaError_t launch_min_cg_check(MinState* S, cudaStream_t st) { FFM_ONE(min_cg_check_kernel, S); }
cudaError_t launch_min_iter_end(MinState* S, double* rec, cudaStream_t st) {
  FFM_ONE(min_iter_end_kernel, S, rec);
}
constexpr size_t kDirSmallSmem = 200 * 1024;
bool lbfgs_dir_small_applies(int64_t n, int m) {
  return n <= (int64_t)kTwoLoopSmallE * kTwoLoopThreads && m <= kMaxLbfgsPairs &&
         (size_t)2 * m * n * sizeof(double) <= kDirSmallSmem;
}
cudaError_t lbfgs_dir_small_prepare() {
  return cudaFuncSetAttribute(lbfgs_dir_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)kDirSmallSmem);
}
cudaError_t launch_lbfgs_dir_small(MinState* S, int64_t n, int m, double* d, double* r,
                                   const double* S_ring, const double* Y_ring, const double* g,
                                   cudaGraphConditionalHandle hls, cudaStream_t st) {
  TwoLoopDevArgs D{n, &S->count, S->idx_nf, S->rho_nf, &S->gn, S_ring, Y_ring, g, d, nullptr};
  count_launch();
  launch_k(lbfgs_dir_small_kernel, 1, kTwoLoopThreads, (size_t)2 * m * n * sizeof(double), st, S,
           D, r, hls);
  return cudaGetLastError();
}

cudaError_t launch_lbfgs_accept_small(MinState* S, int64_t n, const int64_t* stw,
                                      const double* x_new, const double* g_new, double* x,
                                      double* g, double* s_tmp, double* y_tmp, double* ring_s,
                                      double* ring_y, double* rec, cudaStream_t st) {
  count_launch();
  launch_k(lbfgs_accept_small_kernel, 1, kAcceptThreads, 0, st, S, n, stw, x_new, g_new, x, g,
           s_tmp, y_tmp, ring_s, ring_y, rec);
  return cudaGetLastError();
}
cudaError_t launch_min_it_end(MinState* S, cudaGraphConditionalHandle hout, cudaStream_t st) {
  FFM_ONE(min_it_end_kernel, S, hout);
}
#undef FFM_ONE

static int vec_blocks(int64_t n) {
  int64_t blocks = (n + 255) / 256;
  if (blocks > 1184) blocks = 1184;
  return blocks < 1 ? 1 : (int)blocks;
}

cudaError_t launch_cg_update(MinState* S, int64_t n, const double* g_new, double* p,
                             cudaStream_t st) {
  count_launch();
  launch_k(cg_update_kernel, vec_blocks(n), 256, 0, st, S, n, g_new, p);
  return cudaGetLastError();
}

cudaError_t launch_ofgm_x(MinState* S, int64_t n, const double* y, const double* r, double* x,
                          int from_ls, cudaStream_t st) {
  count_launch();
  launch_k(ofgm_x_kernel, vec_blocks(n), 256, 0, st, S, n, y, r, x, from_ls);
  return cudaGetLastError();
}

cudaError_t launch_fgm_shift(MinState* S, int64_t n, double* x, double* x_prev, const double* w,
                             const double* x_new, double* best, cudaStream_t st) {
  count_launch();
  launch_k(fgm_shift_kernel, vec_blocks(n), 256, 0, st, S, n, x, x_prev, w, x_new, best);
  return cudaGetLastError();
}

cudaError_t launch_select_neg(MinState* S, int64_t n, const double* src, double* dst,
                              cudaStream_t st) {
  count_launch();
  launch_k(select_neg_kernel, vec_blocks(n), 256, 0, st, &S->cg_reset, &S->err, n, src, dst);
  return cudaGetLastError();
}

cudaError_t launch_min_store(MinState* S, int64_t n, const double* s_tmp, const double* y_tmp,
                             double* ring_s, double* ring_y, const double* x_new,
                             const double* g_new, double* x, double* g, cudaStream_t st) {
  int64_t blocks = (n + 255) / 256;
  if (blocks > 1184) blocks = 1184;
  if (blocks < 1) blocks = 1;
  count_launch();
  launch_k(min_store_kernel, (int)blocks, 256, 0, st, S, n, s_tmp, y_tmp, ring_s, ring_y, x_new, g_new,
                                                x, g);
  return cudaGetLastError();
}

}  // namespace ffm

#ifdef FFM_MIN_STAMPS
extern "C" int ffm_debug_min_clock_minimize(void* clock_d) {
  return (int)cudaMemcpyToSymbol(ffm::g_mclk, &clock_d, sizeof(void*));
}
#endif
