"""Fixed-step descent, steepest descent and momentum methods
(mirrors ffmin/optimizers/gradient.py: Eq. (2), (4), (9), (10), (11)).

All vector updates go through the run's vector space (vecops).  With the
molecular oracle every driver here runs its iterations as one conditional
CUDA graph (optimizers/graph.py): no value reaches the host between polls;
the loops below are the graph's bit-exact specification and serve other
oracles.
"""

from __future__ import annotations

import math

from . import graph
from .common import (
    CONVERGED,
    DIVERGENCE_FACTOR,
    LINESEARCH_FAILURE,
    NO_RELAXATION,
    DivergenceError,
    OptimizeResult,
    check_finite,
    search,
    start,
)


def _diverged(f, f0):
    return not math.isfinite(f) or f > DIVERGENCE_FACTOR * max(1.0, abs(f0))


def gradient_descent_fixed(oracle, x0, L, stop=None) -> OptimizeResult:
    """x_{k+1} = x_k - (1/L) grad f(x_k)."""
    if not L > 0:
        raise ValueError("L must be positive")
    run, ops, x, f, g, gn = start(oracle, x0, stop, {"method": "gd", "L": L})
    status = CONVERGED if gn <= run.threshold else None
    step = 1.0 / L
    if status is None and graph.eligible_fixed(oracle, ops):
        # the whole iteration on the device (optimizers/graph.py)
        return graph.run_graph(run, oracle, x, f, g, gn, None, graph.FIXED, step=step,
                               momentum_kind=graph.GD)
    k = 0
    while status is None:
        status = run.budget_status(k)
        if status:
            break
        x = ops.lincomb(1.0, x, -step, g)
        f, g = oracle.value_and_gradient(x)
        check_finite(ops, f, g, f"iteration {k + 1}")
        gn = ops.norm(g)
        k += 1
        run.update_best(x, f)
        run.record(k, f, gn, step)
        if gn <= run.threshold:
            status = CONVERGED
    return run.finish(status, x, f, gn)


def steepest_descent(oracle, x0, linesearch, stop=None) -> OptimizeResult:
    """Line search along the normalised antigradient (Eq. (4))."""
    run, ops, x, f, g, gn = start(oracle, x0, stop,
                                  {"method": "sd", "linesearch": linesearch.describe()})
    status = CONVERGED if gn <= run.threshold else None
    if status is None and graph.eligible(oracle, ops, linesearch):
        # the whole iteration on the device (optimizers/graph.py)
        return graph.run_graph(run, oracle, x, f, g, gn, linesearch, graph.SD)
    k = 0
    while status is None:
        status = run.budget_status(k)
        if status:
            break
        r = ops.div(ops.lincomb(-1.0, g), gn)
        res = search(linesearch, oracle, x, r, f, g, ops)
        if res.status == NO_RELAXATION:
            if run.stop.stop_on_linesearch_failure:
                status = LINESEARCH_FAILURE
                break
            k += 1
            run.record(k, f, gn, 0.0)
            continue
        x = ops.lincomb(1.0, x, res.h, r)
        f = res.f_at_step
        g = oracle.gradient(x)
        check_finite(ops, f, g, f"iteration {k + 1}")
        gn = ops.norm(g)
        k += 1
        run.update_best(x, f)
        run.record(k, f, gn, res.h)
        if gn <= run.threshold:
            status = CONVERGED
    return run.finish_best(status, x, f, gn)


def _momentum_run(oracle, x0, stop, meta, step, coef, use_w_gradient, kind=None, m=0.0):
    """Shared loop of heavy ball (gradient at x) and the Nesterov schemes
    (gradient at the extrapolated point w).  kind / m: the graph path's
    momentum_kind and constant momentum (optimizers/graph.py)."""
    run, ops, x, f, g, gn = start(oracle, x0, stop, meta)
    f0 = f
    if gn > run.threshold and kind is not None and graph.eligible_fixed(oracle, ops):
        # the whole iteration on the device
        msg = run.trace.meta.pop("_diverge", None)
        return graph.run_graph(run, oracle, x, f, g, gn, None, graph.FIXED, step=step,
                               momentum=m, momentum_kind=kind, diverge_msg=msg)
    x_prev = ops.copy(x)
    status = CONVERGED if gn <= run.threshold else None
    k = 0
    while status is None:
        status = run.budget_status(k)
        if status:
            break
        m = coef(k)
        if use_w_gradient:
            w = ops.lincomb(1.0, x, m, ops.lincomb(1.0, x, -1.0, x_prev))
            gw = g if k == 0 else oracle.gradient(w)
            x_prev = x
            x = ops.lincomb(1.0, w, -step, gw)
            f = oracle.value(x)
            bad = _diverged(f, f0) or not ops.all_finite(gw)
            gn = ops.norm(gw)
        else:
            x_new = ops.lincomb(1.0, ops.lincomb(1.0, x, -step, g), m,
                                ops.lincomb(1.0, x, -1.0, x_prev))
            x_prev, x = x, x_new
            f, g = oracle.value_and_gradient(x)
            bad = _diverged(f, f0) or not ops.all_finite(g)
            gn = ops.norm(g)
        if bad:
            raise DivergenceError(meta["_diverge"].format(k=k + 1, f=f, f0=f0))
        k += 1
        run.update_best(x, f)
        run.record(k, f, gn, step)
        if gn <= run.threshold:
            status = CONVERGED
    run.trace.meta.pop("_diverge", None)
    return run.finish(status, x, f, gn)


def heavy_ball(oracle, x0, alpha, beta, stop=None) -> OptimizeResult:
    """Polyak momentum (Eq. (9)): x+ = x - alpha g + beta (x - x_prev)."""
    if not alpha > 0:
        raise ValueError("alpha must be positive")
    if not 0.0 <= beta < 1.0:
        raise ValueError("beta must lie in [0, 1)")
    meta = {"method": "hb", "alpha": alpha, "beta": beta,
            "_diverge": "heavy ball diverged at iteration {k}: f={f!r} (start f={f0!r}); "
                        "reduce alpha or beta"}
    return _momentum_run(oracle, x0, stop, meta, alpha, lambda k: beta, False,
                         graph.HEAVY_BALL, beta)


def nesterov_momentum(oracle, x0, L, stop=None) -> OptimizeResult:
    """Eq. (10): extrapolation (k-1)/(k+2), gradient at the extrapolated
    point; the trace's grad_norm reports |grad f(w_k)|."""
    if not L > 0:
        raise ValueError("L must be positive")
    meta = {"method": "nag", "L": L,
            "_diverge": "nesterov momentum diverged at iteration {k}: f={f!r}"}
    return _momentum_run(oracle, x0, stop, meta, 1.0 / L, lambda k: (k - 1.0) / (k + 2.0), True,
                         graph.NAG)


def nesterov_strongly_convex(oracle, x0, L, mu, stop=None) -> OptimizeResult:
    """Eq. (11): constant momentum (sqrt L - sqrt mu)/(sqrt L + sqrt mu)."""
    if not L > 0 or not mu > 0:
        raise ValueError("L and mu must be positive")
    if mu > L:
        raise ValueError("mu must not exceed L")
    m = (math.sqrt(L) - math.sqrt(mu)) / (math.sqrt(L) + math.sqrt(mu))
    meta = {"method": "nag-sc", "L": L, "mu": mu,
            "_diverge": "strongly convex nesterov diverged at iteration {k}: f={f!r}"}
    return _momentum_run(oracle, x0, stop, meta, 1.0 / L, lambda k: m, True, graph.NAG_SC, m)
