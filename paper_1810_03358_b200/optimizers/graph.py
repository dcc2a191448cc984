"""Graph-resident drivers: L-BFGS, nonlinear CG, steepest descent and FGM with
the whole iteration on the device (include/ffmin_b200.h ffm_lbfgs_*,
csrc/ffm_minimize.cu).

The reference decides every line-search probe, curvature / beta dot product
and convergence test in Python (ffmin/optimizers/lbfgs.py:93-128,
cg.py:95-152, gradient.py, fgm.py; linesearch.py).  Here one CUDA graph with
conditional nodes runs up to GRAPH_CHUNK iterations per launch: single-thread
controller kernels replay the drivers' scalar logic in IEEE double, vectors
go through the same kernels as the host-driven loop, so the traces are
bit-identical to it.  The host polls once per chunk to append trace records
and check the wall clock.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

LBFGS, CG, SD, FGM, FIXED, OFGM = 0, 1, 2, 3, 4, 5
# fixed-step family (method FIXED): momentum_kind
GD, HEAVY_BALL, NAG, NAG_SC = 0, 1, 2, 3
GRAPH_CHUNK = 32  # iterations per graph launch between host polls


def eligible_fixed(oracle, ops) -> bool:
    """The device molecular oracle (and FFMIN_B200_HOST_LOOP unset): the
    fixed-step drivers run in the graph."""
    from ..oracle import MolecularOracle
    from ..parallel import ShardedMolecularOracle

    if os.environ.get("FFMIN_B200_HOST_LOOP"):
        return False
    if ops.space != "device":
        return False
    # a row-sharded oracle qualifies when its evaluations complete on the
    # device (NCCL communicator attached): the all-reduce is captured too
    return type(oracle) is MolecularOracle or (
        type(oracle) is ShardedMolecularOracle and oracle.native)


def eligible(oracle, ops, linesearch, m: int = 1) -> bool:
    """The device molecular oracle with a built-in line searcher (and
    FFMIN_B200_HOST_LOOP unset): the graph path applies."""
    from .common import LineSearcher

    if not eligible_fixed(oracle, ops):
        return False
    if not isinstance(linesearch, LineSearcher) or not 1 <= m <= 32:
        return False
    c = linesearch.config
    return linesearch.kind == "h" or 2 <= c.K <= 22


class _GraphRun:
    """An ffm_lbfgs handle (include/ffmin_b200.h) with its engine kept alive."""

    def __init__(self, engine, precision, cfg):
        from .. import _native as N

        self.N, self.lib, self.engine = N, N.load(), engine
        h = C.c_void_p()
        N.check(self.lib.ffm_lbfgs_create(engine.handle, precision, C.byref(cfg), C.byref(h)),
                "ffm_lbfgs_create")
        self.handle = h
        self.cap = int(cfg.chunk) + 1

    def __del__(self):
        try:
            if self.handle:
                self.lib.ffm_lbfgs_destroy(self.handle)
                self.handle = None
        except Exception:
            pass


def run_graph(run, oracle, x, f, g, gn, linesearch, method, m=1, cg_kind="prp",
              restart_period=100, step=0.0, momentum=0.0, momentum_kind=GD,
              diverge_msg=None, schedule=None):
    """Run the iterations of `method` on the device from (x, f, g, |g|) and
    finish `run` like the host loop would.  linesearch is None for the
    fixed-step family (method FIXED: step, momentum, momentum_kind;
    diverge_msg formats its divergence error with k, f and f0) and for
    OFGM with a fixed step (schedule = ofgm_schedule's t, step = 1/L)."""
    import torch

    from .. import _native as N
    from ..energy import raise_status
    from .common import TIME_BUDGET, DivergenceError, TraceRecord

    stop = run.stop
    if linesearch is None:  # fixed-step family: the line-search fields are unused
        from ..linesearch import LsParConfig

        c, kind, warm = LsParConfig(), 1, 1.0
    else:
        c = linesearch.config
        kind = 1 if linesearch.kind == "par" else 0
        warm = float(linesearch.h)
    calls0 = (oracle.value_calls, oracle.grad_calls)
    chunk = 4 if stop.max_wall_time is not None else GRAPH_CHUNK
    cfg = N.LbfgsConfig(
        m=m, ls_kind=kind, K=c.K if kind else 2,
        use_gradient_start=int(c.use_gradient_start) if kind else 0,
        stop_on_linesearch_failure=int(stop.stop_on_linesearch_failure), chunk=chunk,
        max_iterations=-1 if stop.max_iterations is None else int(stop.max_iterations),
        max_oracle_calls=-1 if stop.max_oracle_calls is None
        else max(0, int(stop.max_oracle_calls) - calls0[0] - calls0[1]),
        threshold=run.threshold, h0=c.h0, eps_h=0.0 if kind else c.eps_h,
        k_plus=0.0 if kind else c.k_plus, k_minus=0.0 if kind else c.k_minus,
        trust=c.trust if kind else 0.0, method=method,
        cg_kind=N.CG_KINDS.index(cg_kind) if method == CG else 0,
        restart_period=int(restart_period) if method == CG else 1, reserved=0,
        fixed_step=float(step) if method in (FIXED, OFGM) else 0.0,
        momentum=float(momentum) if method == FIXED else 0.0,
        momentum_kind=int(momentum_kind) if method == FIXED else 0, reserved2=0)
    # one captured graph per structure (ffm_lbfgs_configure: budgets,
    # tolerances and line-search constants are run-time state)
    key = (cfg.m, cfg.chunk, cfg.method, cfg.momentum_kind, cfg.fixed_step,
           int(cfg.ls_kind == 1 and cfg.use_gradient_start))
    cache = oracle.__dict__.setdefault("_graph_runs", {})
    gr = cache.get(key)
    if gr is None:
        gr = cache[key] = _GraphRun(oracle.engine, oracle.precision, cfg)
    lib, h = gr.lib, gr.handle
    N.check(lib.ffm_lbfgs_configure(h, C.byref(cfg)), "ffm_lbfgs_configure")
    if method == OFGM:
        t = np.ascontiguousarray(schedule, dtype=np.float64)
        N.check(lib.ffm_lbfgs_set_schedule(h, t.ctypes.data, len(t)), "ffm_lbfgs_set_schedule")
    stream = C.c_void_p(torch.cuda.current_stream(oracle.device).cuda_stream)
    N.check(lib.ffm_lbfgs_start(h, C.c_void_p(x.data_ptr()), C.c_void_p(g.data_ptr()), f, gn,
                                warm, stream), "ffm_lbfgs_start")
    ints = np.zeros(8, np.int64)
    dbls = np.zeros(4)
    recs = np.zeros((gr.cap, N.LBFGS_REC_WIDTH))
    nrec = np.zeros(1, np.int64)
    errst = np.zeros(8, np.int64)
    status = None
    while True:
        t_launch = run.elapsed()
        N.check(lib.ffm_lbfgs_run(h, stream), "ffm_lbfgs_run")
        N.check(lib.ffm_lbfgs_poll(h, ints.ctypes.data, dbls.ctypes.data, recs.ctypes.data,
                                   gr.cap, nrec.ctypes.data, errst.ctypes.data),
                "ffm_lbfgs_poll")
        for r in recs[:int(nrec[0])]:
            run.trace.append(TraceRecord(
                iteration=int(r[0]), f=float(r[1]), grad_norm=float(r[2]), step=float(r[3]),
                value_calls=calls0[0] + int(r[4]), grad_calls=calls0[1] + int(r[5]),
                wall_seconds=t_launch + float(r[6]) * 1e-9, best_f=float(r[7])))
        oracle.value_calls = calls0[0] + int(ints[5])
        oracle.grad_calls = calls0[1] + int(ints[6])
        if ints[3] == 1:
            raise_status(oracle.system, errst, grad=bool(ints[4]))
        if ints[3] == 2:
            if diverge_msg is not None:
                raise DivergenceError(diverge_msg.format(k=int(ints[0]) + 1, f=float(dbls[0]),
                                                         f0=f))
            raise DivergenceError(f"non-finite objective or gradient at iteration "
                                  f"{int(ints[0]) + 1}")
        if ints[2]:
            status = N.LBFGS_STATUS[int(ints[1])]
            break
        if run.wall_time_reached():
            status = TIME_BUDGET
            break
    if linesearch is not None:
        linesearch.h = float(dbls[2])
    x_out = torch.empty_like(x)
    g_out = torch.empty_like(g)
    N.check(lib.ffm_lbfgs_result(h, C.c_void_p(x_out.data_ptr()), C.c_void_p(g_out.data_ptr()),
                                 stream), "ffm_lbfgs_result")
    f_out, gn_out = float(dbls[0]), float(dbls[1])
    if method == FGM:  # the extrapolated points can be the best ones
        best = torch.empty_like(x)
        N.check(lib.ffm_lbfgs_best(h, C.c_void_p(best.data_ptr()), stream), "ffm_lbfgs_best")
        run.best_f, run.best_x = float(dbls[3]), best
    else:  # every accepted step strictly lowers f: the iterate is the best point
        run.best_f, run.best_x = f_out, x_out
    return run.finish_best(status, x_out, f_out, gn_out)
