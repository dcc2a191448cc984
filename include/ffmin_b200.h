/*
 * ffmin_b200.h -- C ABI of the B200 force-field energy / gradient engine.
 *
 * This is the drop-in boundary for the reference's hot path.  The reference
 * (ffmin, pure Python + NumPy/numba) reaches its kernels through
 * `KernelBackend` objects (ffmin/kernels.py:984-1024) whose functions the
 * energy layer calls once per oracle evaluation (ffmin/energy.py:114-174,
 * 284-313).  Every entry point below replaces one of those calls; the
 * Python host package paper_1810_03358_b200 binds them with ctypes and
 * passes PyTorch / NumPy buffers as plain pointers.
 *
 * Conventions
 *   - plain pointers and sizes only; `stream` is a cudaStream_t (NULL =
 *     legacy default stream) passed as void*;
 *   - pointers named *_d are device (HBM) pointers, *_h host pointers;
 *   - coordinates are float64 (n, 3) row-major, as MolecularSystem.coords
 *     (ffmin/model.py:224-231); gradients come back in the same layout;
 *   - every function returns 0 on success and a negative FFM_E* code on
 *     failure; ffm_last_error() describes the last failure of the calling
 *     thread.  Geometry problems are NOT errors at this level: like the
 *     reference kernels (ffmin/kernels.py:11-14) they are reported through
 *     status words (index of the first bad term / pair, -1 when clean) and
 *     the host layer raises EnergyEvaluationError.
 */
#ifndef FFMIN_B200_H
#define FFMIN_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FFM_OK 0
#define FFM_EINVAL (-1)   /* bad argument / validation failure */
#define FFM_ECUDA (-2)    /* CUDA runtime error */
#define FFM_ENOMEM (-3)   /* device allocation failed */

/* kernel precision: ffmin's dtype argument (ffmin/energy.py:90-179) */
#define FFM_F64 0  /* all arithmetic in FP64 */
#define FFM_F32 1  /* pair arithmetic in FP32, accumulation in FP64 */

/* evaluation flags */
#define FFM_ENERGY 1
#define FFM_GRAD 2
#define FFM_NO_NB 4     /* skip the nonbonded terms (all pairs + scaled 1-4) */
#define FFM_NO_TERMS 8  /* skip the bonded terms (stretch, bend, torsion)    */
#define FFM_TIME_NB 16  /* record CUDA events around the pair sweep          */
#define FFM_NO_GRAPH 32 /* issue the kernels directly instead of replaying a
                         * captured CUDA graph of the same call              */
#define FFM_NO_FUSE 64  /* small systems: run the kernel chain instead of the
                         * one-launch fused evaluation (same bits; tests)    */

/* status words (int64[8] per evaluation) */
#define FFM_ST_NB_BAD_I 0   /* first coincident nonbonded pair, -1 clean */
#define FFM_ST_NB_BAD_J 1
#define FFM_ST_BOND 2       /* first degenerate bond term (grad only)   */
#define FFM_ST_ANGLE 3      /* first degenerate angle term              */
#define FFM_ST_DIHEDRAL 4   /* first degenerate dihedral term           */
#define FFM_STATUS_WORDS 8

/* energies: double[5] = stretch, bend, torsion, coulomb, vdw (kJ/mol),
 * the fields of ffmin.energy.EnergyBreakdown (ffmin/energy.py:30-41). */
#define FFM_NTERMS 5

typedef struct ffm_system ffm_system_t;

const char* ffm_version(void);
const char* ffm_last_error(void);

/* Upload one molecular system (parameters + topology) to `device`.
 * Replaces MolecularSystem.arrays() (ffmin/model.py:259-319): q/sigma/eps
 * per atom, and the nonbonded policy as a sparse list of the pairs whose
 * scale is not 1 (excluded pairs with s = 0, 1-4 pairs with s = s14) instead
 * of the dense (n, n) matrix.  cutoff <= 0 means no cutoff. */
int ffm_system_create(ffm_system_t** out, int device, int64_t n, const double* q_h,
                      const double* sigma_h, const double* eps_h, int64_t nspecial,
                      const int64_t* special_i_h, const int64_t* special_j_h,
                      const double* special_s_h, double cutoff);

/* Bonded term tables, as MolecularSystem.arrays() bond_idx/bond_K/bond_r0,
 * ang_idx/ang_K/ang_t0 (radians), dih_idx/dih_V (ffmin/model.py:273-288). */
int ffm_system_set_terms(ffm_system_t* sys, int64_t nbond, const int64_t* bond_idx_h,
                         const double* bond_K_h, const double* bond_r0_h, int64_t nangle,
                         const int64_t* ang_idx_h, const double* ang_K_h,
                         const double* ang_t0_h, int64_t ndih, const int64_t* dih_idx_h,
                         const double* dih_V_h);

int ffm_system_destroy(ffm_system_t* sys);

/* Row sharding over `nranks` GPUs (one process per GPU): this handle then
 * evaluates only its share of the S x S super-units of the pair triangle
 * (units dealt heaviest first to the least-loaded rank, rank 0 counted with
 * its O(N) work) and, on rank 0 only, the O(N) bonded / 1-4 terms.  Gradients and energies of an evaluation are partial
 * sums; the caller all-reduces them (NCCL over NVLink in
 * paper_1810_03358_b200.parallel).  nranks = 1 restores the full sweep. */
int ffm_system_set_shard(ffm_system_t* sys, int rank, int nranks);

/* Super-unit edge S of the pair sweep's plan (units mode only: a multiple
 * of 128 in [128, 1024] dividing the padded atom count; FFM_EINVAL in tile
 * mode).  ffm_preferred_edge gives the edge an n-atom system evaluated
 * mostly in `precision` runs best with (0: tile mode): the creation default,
 * except 128 for FP64 mid-size systems.  No reference counterpart (tuning of
 * this engine's plan); paper_1810_03358_b200.engine.engine_for applies it. */
int ffm_preferred_edge(int64_t n, int precision, int* edge);
int ffm_system_set_edge(ffm_system_t* sys, int S);

/* The NCCL communicator (ncclComm_t, e.g. torch's ProcessGroupNCCL
 * _comm_ptr()) of a sharded system's ranks.  With it attached, every
 * ffm_eval / ffm_eval_host of the sharded system -- and every evaluation
 * inside the graph-resident drivers, which then accept sharded systems --
 * completes on the device with one all-reduce of [gradient | energies |
 * error words] on the evaluation's stream (what parallel.ShardCombiner does
 * from Python; capturable in CUDA graphs), so it returns global values.
 * ffm_eval_batch keeps returning the rank's partial energies.  The library
 * resolves ncclAllReduce from the libnccl.so.2 already loaded in the
 * process.  NULL detaches. */
int ffm_system_set_comm(ffm_system_t* sys, void* nccl_comm);

/* Device time of the pair sweep of the last FFM_TIME_NB evaluation
 * (CUDA events on the evaluation's stream; synchronises on them). */
int ffm_system_nb_ms(ffm_system_t* sys, float* ms_h);

/* Number of kernels this library has launched in the process. */
long long ffm_launch_count(void);

/* Tuning aid: the fused small-system evaluation (FFM_NO_FUSE clears it)
 * writes 6 globaltimer stamps per CTA into clock_d ([grid][6] uint64, or
 * NULL to stop) at its phase boundaries; grids_h[4] receives the
 * cooperative grid sizes [precision][grad] chosen so far (0 = not yet). */
int ffm_debug_phase_clock(ffm_system_t* sys, void* clock_d, int* grids_h);

/* info[0..7] = n, padded n, super-unit S, blocks, units, special tiles,
 * scaled pairs, device */
int ffm_system_info(const ffm_system_t* sys, int64_t* info_h);

/* Full evaluation on device buffers (no host synchronisation).  The first
 * call with a given (precision, flags, buffer addresses) captures its seven
 * kernels into a CUDA graph; later identical calls replay it with one
 * launch (keep input/output buffers fixed to benefit).
 * replaces energy_total / energy_and_gradient (ffmin/energy.py:133-174) and
 * the KernelBackend nb_energy / nb_grad / *_grad calls they make.
 * grad_d (n*3, overwritten) may be NULL without FFM_GRAD. */
int ffm_eval(ffm_system_t* sys, int precision, int flags, const double* coords_d,
             double* grad_d, double* energies_d, int64_t* status_d, void* stream);

/* Same, through host buffers: copies in, evaluates, copies out and
 * synchronises -- the reference-facing call a NumPy caller makes. */
int ffm_eval_host(ffm_system_t* sys, int precision, int flags, const double* coords_h,
                  double* grad_h, double* energies_h, int64_t* status_h);

/* Energies of `batch` candidate geometries of the same system
 * (coords_d: [batch][n][3]); energies_d: [batch][5]; status_d: [batch][8].
 * The batched form of energy_total (ffmin/energy.py:133-141) that
 * probe_full (ffmin/optimizers/wiggle.py:118-127) calls once per candidate:
 * B full geometries per launch (BASELINE configs[3], finite-difference
 * gradients).  The atom-wiggle driver itself probes with exact single-atom
 * deltas (ffm_atom_delta below), which equal probe_full's
 * energy_total(moved) - e_run up to that difference's roundoff. */
int ffm_eval_batch(ffm_system_t* sys, int precision, int64_t batch, const double* coords_d,
                   double* energies_d, int64_t* status_d, void* stream);

/* Exact energy change of `ncand` single-atom moves of the current geometry
 * (ffmin/energy.py:284-313, exact_delta_atom_move): atoms_d[k] moves to
 * newpos_d[k][3].  out_d[k][5] = (coulomb, vdw, stretch, bend, torsion)
 * deltas, status_d[k][3] = (first coincident partner j, first degenerate
 * angle row, first degenerate dihedral row), -1 when clean.  Batches of
 * fewer than 148 candidates split each candidate's partners over several
 * blocks and add the partial sums in a fixed order (deterministic; sums of
 * the same terms in another order than a larger batch's, so the two agree
 * to rounding).  Not reentrant across streams for such batches (one
 * scratch per system). */
int ffm_atom_delta(ffm_system_t* sys, const double* coords_d, int64_t ncand,
                   const int32_t* atoms_d, const double* newpos_d, double* out_d,
                   int64_t* status_d, void* stream);

/* Far-field linearised single-atom move deltas (ffmin/energy.py:215-281,
 * linearize_farfield_coulomb + delta_energy_atom_move, the incremental mode
 * of the gradient-free method, paper section 3): partners within lin_cutoff
 * of the atom's current position, and every excluded / 1-4 partner, are
 * treated exactly; the far Coulomb sum by its first-order Taylor term; far
 * vdW is neglected.  out_d[k][6] = (near coulomb, near vdw, stretch, bend,
 * torsion, far linear term); status_d as ffm_atom_delta.  Requires a
 * system without a nonbonded cutoff. */
int ffm_atom_delta_lin(ffm_system_t* sys, const double* coords_d, int64_t ncand,
                       const int32_t* atoms_d, const double* newpos_d, double lin_cutoff,
                       double* out_d, int64_t* status_d, void* stream);

/* ffmin/energy.py:215-240 linearize_farfield_coulomb (kernels.py:359-387):
 * e0_coef_d[4] = (far-field Coulomb energy of `atom`, its gradient x/y/z),
 * near_mask_d[n] = 1 for the exact near set, bad_d[0] = first coincident far
 * partner or -1. */
int ffm_farfield_build(ffm_system_t* sys, const double* coords_d, int64_t atom, double cutoff,
                       double* e0_coef_d, uint8_t* near_mask_d, int64_t* bad_d, void* stream);

/* ---- optimiser vector algebra on device vectors (ffmin/optimizers) ---- */

/* out_d[0] = <x, y>, deterministic fixed-order reduction.  scratch_d holds
 * ffm_vec_scratch_doubles() doubles. */
int64_t ffm_vec_scratch_doubles(void);
int ffm_dot(int64_t n, const double* x_d, const double* y_d, double* out_d,
            double* scratch_d, void* stream);

/* out_d[q] = <xs_h[q], ys_h[q]> for q < k <= 8 in one pass (host arrays of
 * device pointers), same fixed-order reduction as ffm_dot. */
int ffm_dots(int64_t n, int k, const double* const* xs_h, const double* const* ys_h,
             double* out_d, double* scratch_d, void* stream);

/* z = sa * (a * x + b * y); a/b read from a_d/b_d when non-NULL, else a_h/b_h;
 * y_d may be NULL. */
int ffm_axpby(int64_t n, const double* a_d, double a_h, double sa, const double* x_d,
              const double* b_d, double b_h, const double* y_d, double* z_d, void* stream);

/* L-BFGS two-loop recursion (ffmin/optimizers/lbfgs.py:53-75) in one
 * cooperative kernel.  S_d/Y_d: ring buffers [m][n]; order_h[count] ring
 * slots newest first; rho_h[count] = 1/<s,y> in the same order.  d_d gets
 * the raw direction -H g (count >= 1; count = 0 is the caller's normalised
 * antigradient). */
int ffm_lbfgs_two_loop(int64_t n, int count, const int32_t* order_h, const double* rho_h,
                       const double* S_d, const double* Y_d, const double* g_d, double* d_d,
                       double* scratch_d, void* stream);

/* ---- graph-resident minimisers (ffmin/optimizers/*.py) ----
 *
 * The whole iteration of a driver -- for L-BFGS (ffmin/optimizers/lbfgs.py:
 * 93-128) the direction (two-loop recursion), the line search (ls_par /
 * ls_h with the LineSearcher warm start and retry, ffmin/linesearch.py,
 * ffmin/optimizers/common.py), the gradient at the new point, the
 * curvature-guarded memory update and the convergence test; likewise for
 * nonlinear CG, steepest descent, FGM, OFGM, the fixed-step family and the
 * gradient-free wiggle (cfg.method) -- runs as one CUDA graph with
 * conditional nodes; no value crosses to the host between iterations.  The
 * host launches chunks of iterations and reads the trace records after each
 * chunk.  Unsharded systems, or sharded ones with a communicator
 * (ffm_system_set_comm).  The "lbfgs" in the names is historical. */
typedef struct ffm_lbfgs ffm_lbfgs_t;

typedef struct {
  int32_t m;                   /* memory depth, 1..32 */
  int32_t ls_kind;             /* 0 = ls_h, 1 = ls_par */
  int32_t K;                   /* ls_par refinement budget, 2..22 */
  int32_t use_gradient_start;  /* ls_par seed */
  int32_t stop_on_linesearch_failure;
  int32_t chunk;               /* iterations per ffm_lbfgs_run launch, >= 1 */
  int64_t max_iterations;      /* -1: unbounded */
  int64_t max_oracle_calls;    /* -1: unbounded (value + gradient calls) */
  double threshold;            /* stop when |g| <= threshold */
  double h0, eps_h, k_plus, k_minus, trust;  /* line-search configuration */
  /* the search-direction method run by the same graph (appended fields):
   * 0 = L-BFGS (ffmin/optimizers/lbfgs.py:93-128), 1 = nonlinear conjugate
   * gradients (ffmin/optimizers/cg.py:95-152; cg_kind 0..6 = fr, prp, prp+,
   * hs, cd, ls, dy; restart every restart_period iterations), 2 = steepest
   * descent (ffmin/optimizers/gradient.py, Eq. (4)), 3 = FGM with the theta
   * schedule and best-point tracking (ffmin/optimizers/fgm.py, Algorithm 1).
   * m is ignored (but must be in range) for methods 1..6 (5 = OFGM, see
   * ffm_lbfgs_set_schedule; 6 = wiggle, below). */
  int32_t method;
  int32_t cg_kind;
  int32_t restart_period;
  int32_t reserved;
  /* method 4 = fixed-step family (ffmin/optimizers/gradient.py): momentum_kind
   * 0 = gradient descent x+ = x - step g (Eq. (2)), 1 = heavy ball with
   * constant momentum (Eq. (9)), 2 = Nesterov with (k-1)/(k+2) and the
   * gradient at the extrapolated point (Eq. (10)), 3 = the strongly convex
   * Nesterov scheme with constant momentum (Eq. (11)); no line search. */
  double fixed_step;
  double momentum;
  int32_t momentum_kind;
  int32_t reserved2;
  /* method 6 = gradient-free atom wiggle (ffmin/optimizers/wiggle.py): probe
   * step h, far-field linearisation cutoff (0 = exact probes), exact
   * re-evaluation every epoch_iterations iterations (incremental mode); the
   * atom of each iteration comes from ffm_lbfgs_set_atoms. */
  double wiggle_h;
  double wiggle_cutoff;
  int32_t wiggle_epoch;
  int32_t reserved3;
} ffm_lbfgs_config;

int ffm_lbfgs_create(ffm_system_t* sys, int precision, const ffm_lbfgs_config* cfg,
                     ffm_lbfgs_t** out);
/* change the run-time fields of a run's configuration (budgets, threshold,
 * line-search constants, CG variant, momentum) so the captured graph is
 * reused; m, chunk, method, momentum_kind, fixed_step and whether ls_par
 * seeds from the slope shape the graph and must match (FFM_EINVAL). */
int ffm_lbfgs_configure(ffm_lbfgs_t* run, const ffm_lbfgs_config* cfg);
/* start point: x_d, g_d device (3n) float64; f, |g| as computed by the
 * caller; warm_h = the line searcher's current warm-start step */
int ffm_lbfgs_start(ffm_lbfgs_t* run, const double* x_d, const double* g_d, double f,
                    double gnorm, double warm_h, void* stream);
/* one chunk of up to cfg.chunk iterations (asynchronous) */
int ffm_lbfgs_run(ffm_lbfgs_t* run, void* stream);
/* synchronise and read the run state.  ints[8] = (iterations, status
 * 0 none / 1 converged / 2 iteration budget / 3 line-search failure /
 * 4 oracle budget / 5 horizon complete, done, error 0 none / 1 evaluation / 2 divergence,
 * error came from a gradient evaluation, value calls, gradient calls,
 * memory pairs); dbls[4] = (f, |g|, warm-start step, best f so far);
 * rec_h[cap][8] receives the chunk's trace records (iteration, f, |g|, step,
 * value calls, gradient calls, ns since the chunk started, best f),
 * *nrec their number; err_status_h[8] the status words of a failed
 * evaluation. */
int ffm_lbfgs_poll(ffm_lbfgs_t* run, int64_t* ints, double* dbls, double* rec_h, int64_t cap,
                   int64_t* nrec, int64_t* err_status_h);
/* copy the current iterate and gradient out (device pointers, 3n) */
int ffm_lbfgs_result(ffm_lbfgs_t* run, double* x_d, double* g_d, void* stream);
/* OFGM (method 5, ffmin/optimizers/fgm.py Eq. (12)): the schedule t[0..N]
 * (len = N + 1, ofgm_schedule), before ffm_lbfgs_start; fixed_step = 1/L
 * selects the fixed-step variant, 0 the line-searched one */
int ffm_lbfgs_set_schedule(ffm_lbfgs_t* run, const double* t_h, int64_t len);
/* wiggle (method 6): the atoms of the next ffm_lbfgs_run launch, one per
 * iteration (count >= cfg.chunk; drawn by the caller's generator) */
int ffm_lbfgs_set_atoms(ffm_lbfgs_t* run, const int32_t* atoms_h, int64_t count);
/* copy the best point seen so far out (device pointer, 3n; FGM's result
 * unless the run converged -- OptimizationRun.finish_best) */
int ffm_lbfgs_best(ffm_lbfgs_t* run, double* x_d, void* stream);
int ffm_lbfgs_destroy(ffm_lbfgs_t* run);

#ifdef __cplusplus
}
#endif
#endif /* FFMIN_B200_H */
