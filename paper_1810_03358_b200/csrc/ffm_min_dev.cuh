// ffm_min_dev.cuh -- the scalar controller logic of the graph-resident
// drivers (MinState, ffm_min.cuh) as device functions: the line searches
// (ffmin/linesearch.py ls_h / ls_par, common.py LineSearcher warm start and
// retry), trace records and status checks.  Included by ffm_minimize.cu
// (the controller kernels) and ffm_small.cu (a small-system line-search
// trial runs the step controller at the end of its fused evaluation); both
// are compiled with -fmad=false, so every product and sum rounds separately,
// as in the reference's Python float arithmetic.
#pragma once
#include <cfloat>
#include "ffm_min.cuh"

namespace ffm {
namespace mindev {

__device__ inline unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// raise_status (energy.py): energy-only evaluations report coincident
// nonbonded pairs, angles and dihedrals; gradient evaluations also bonds
__device__ inline bool bad_status(const int64_t* stw, bool grad) {
  return stw[kStNbBadI] >= 0 || stw[kStAngle] >= 0 || stw[kStDihedral] >= 0 ||
         (grad && stw[kStBond] >= 0);
}

__device__ inline void set_err(MinState* S, int kind, const int64_t* stw, bool grad) {
  S->err = kind;
  S->err_grad = grad ? 1 : 0;
  if (stw)
    for (int q = 0; q < 8; ++q) S->err_st[q] = stw[q];
  S->done = 1;
}

__device__ inline void record(MinState* S, double* rec, double step) {
  double* r = rec + S->nrec * kMinRecWidth;
  r[0] = (double)S->k;
  r[1] = S->f;
  r[2] = S->gn;
  r[3] = step;
  r[4] = (double)S->vcalls;
  r[5] = (double)S->gcalls;
  r[6] = (double)(globaltimer() - S->t_launch);
  r[7] = S->best_f;
  S->nrec++;
}

__device__ inline void memory_clear(MinState* S) {
  S->count = 0;
  S->nfree = S->c.m + 1;
  for (int q = 0; q <= S->c.m; ++q) S->freel[q] = q;
}

// --------------------------------------------------------- line searches
__device__ inline bool rank_less(double fa, double ha, double fb, double hb) {
  // Python tuple order of (f, |h|)
  return fa < fb || (fa == fb && fabs(ha) < fabs(hb));
}

// _accept_vertex (linesearch.py): finite, clamped to [lo, hi], not a
// duplicate of a sampled abscissa
__device__ inline bool accept_vertex(const MinState* S, double& v) {
  if (!isfinite(v)) return false;
  if (S->lo > v) v = S->lo;  // max(v, lo)
  if (S->hi < v) v = S->hi;  // min(v, hi)
  const double av = fabs(v);
  const double scale = av > 1.0 ? av : 1.0;
  for (int q = 0; q < S->np; ++q) {
    const double ah = fabs(S->ph[q]);
    const double m = ah > scale ? ah : scale;
    if (fabs(v - S->ph[q]) <= 1e-13 * m) return false;
  }
  return true;
}

__device__ inline void ls_start(MinState* S, double h0) {
  const MinConfig& c = S->c;
  S->a_h0 = h0;
  S->np = 0;
  S->nref = 0;
  S->found = 0;
  if (c.ls_kind == 1) {
    S->hi = c.trust * h0;
    S->lo = c.use_gs ? 0.0 : -S->hi;
    S->ph[0] = 0.0;
    S->pf[0] = S->f0;
    S->np = 1;
    if (c.use_gs) {
      S->stage = 10;
      S->h_trial = h0;
    } else {
      S->stage = 20;
      S->h_trial = -0.5 * h0;
    }
  } else {
    S->stage = 1;
    S->h_trial = h0;
  }
}

__device__ inline void ls_finish(MinState* S, bool found, double h, double f) {
  S->found = found ? 1 : 0;
  S->res_h = found ? h : 0.0;
  S->res_f = found ? f : S->f0;
}

// ls_par: the remaining refinement steps (at most K - 1)
__device__ inline bool ls_par_refine(MinState* S) {
  if (S->nref >= S->c.K - 1 || S->np < 3) return false;
  // sorted(pts, key=(f, |h|))[:3] -- a stable selection of the three best
  int b[3] = {-1, -1, -1};
  for (int q = 0; q < S->np; ++q) {
    int pos = 3;
    for (int t = 2; t >= 0; --t)
      if (b[t] < 0 || rank_less(S->pf[q], S->ph[q], S->pf[b[t]], S->ph[b[t]])) pos = t;
    if (pos < 3) {
      for (int t = 2; t > pos; --t) b[t] = b[t - 1];
      b[pos] = q;
    }
  }
  const double x0 = S->ph[b[0]], x1 = S->ph[b[1]], x2 = S->ph[b[2]];
  const double f0 = S->pf[b[0]], f1 = S->pf[b[1]], f2 = S->pf[b[2]];
  if (x0 == x1 || x0 == x2 || x1 == x2) return false;
  // fit_parabola: divided differences
  const double s01 = (f1 - f0) / (x1 - x0);
  const double s12 = (f2 - f1) / (x2 - x1);
  const double curv = (s12 - s01) / (x2 - x0);
  double mx = fabs(f0);
  if (fabs(f1) > mx) mx = fabs(f1);
  if (fabs(f2) > mx) mx = fabs(f2);
  const bool degenerate = fabs(curv) < 1e-12 * mx;
  if (curv <= 0.0 || degenerate) return false;
  double v = 0.5 * (x0 + x1) - s01 / (2.0 * curv);
  if (!accept_vertex(S, v)) return false;
  S->nref++;
  S->h_trial = v;
  return true;
}

__device__ inline void ls_par_finish(MinState* S) {
  int bi = 0;  // min(pts, key=rank): the first minimal point
  for (int q = 1; q < S->np; ++q)
    if (rank_less(S->pf[q], S->ph[q], S->pf[bi], S->ph[bi])) bi = q;
  const double hb = S->ph[bi], fb = S->pf[bi];
  ls_finish(S, hb != 0.0 && fb < S->f0, hb, fb);
}

// consume phi(h_trial) = f; true while the attempt wants another probe
__device__ inline bool ls_on_value(MinState* S, double f) {
  const MinConfig& c = S->c;
  if (c.ls_kind == 1) {
    S->ph[S->np] = S->h_trial;
    S->pf[S->np] = f;
    S->np++;
    switch (S->stage) {
      case 10: {  // seeded by the slope at 0 and phi(h0)
        const double h0 = S->a_h0, f0 = S->f0, f1 = f;
        const double curv = (f1 - f0 - S->slope * h0) / (h0 * h0);
        const double mx = fabs(f0) > fabs(f1) ? fabs(f0) : fabs(f1);
        if (curv <= 0.0 || fabs(curv) < 1e-12 * mx) break;  // ok = False
        double v = -S->slope / (2.0 * curv);
        if (!accept_vertex(S, v)) break;
        S->stage = 11;
        S->h_trial = v;
        return true;
      }
      case 20:
        S->stage = 21;
        S->h_trial = 0.5 * S->a_h0;
        return true;
      default:  // 11, 21: initial points complete; 30: a refinement probe
        S->stage = 30;
        if (ls_par_refine(S)) return true;
        break;
    }
    ls_par_finish(S);
    return false;
  }
  // ls_h
  switch (S->stage) {
    case 1:
      if (f < S->f0) {
        S->h_keep = S->h_trial;
        S->f_keep = f;
        S->stage = 2;
        S->h_trial = c.k_plus * S->h_trial;
        return true;
      }
      S->stage = 3;
      S->h_trial = c.k_minus * S->a_h0;
      return true;
    case 2:
      if (f < S->f_keep) ls_finish(S, true, S->h_trial, f);
      else ls_finish(S, true, S->h_keep, S->f_keep);
      return false;
    default: {  // 3: contraction
      if (f < S->f0) {
        ls_finish(S, true, S->h_trial, f);
        return false;
      }
      const double h = c.k_minus * S->h_trial;
      if (h <= c.eps_h) {
        ls_finish(S, false, 0.0, S->f0);
        return false;
      }
      S->h_trial = h;
      return true;
    }
  }
}

// ------------------------------------------------------------ kernels

// one line-search probe value: LineSearcher / ls_h / ls_par bookkeeping and
// the loop condition of the probe WHILE node
__device__ inline void ls_step(MinState* S, const double* en, const int64_t* stw,
                               cudaGraphConditionalHandle hloop) {
  S->vcalls++;
  S->ls_more = 0;
  if (bad_status(stw, false)) {
    set_err(S, kMinErrEval, stw, false);
    cudaGraphSetConditional(hloop, 0);
    return;
  }
  const double f = en[0] + en[1] + en[2] + en[3] + en[4];  // EnergyBreakdown.total order
  bool more = ls_on_value(S, f);
  if (!more) {
    // LineSearcher: one retry from the configured h0 after a warm-started miss
    if (!S->found && S->attempt == 0 && S->warm != S->c.h0) {
      S->attempt = 1;
      ls_start(S, S->c.h0);
      more = true;
    } else {
      S->warm = S->found ? fabs(S->res_h) : S->c.h0;
    }
  }
  S->ls_more = more ? 1 : 0;
  // the loop condition is 1 from ls_init on: only its end needs a write
  if (!more) cudaGraphSetConditional(hloop, 0u);
}

}  // namespace mindev
}  // namespace ffm
