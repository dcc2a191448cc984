"""NumPy restatement of the reference L-BFGS driver -- TEST INFRASTRUCTURE.

Follows ffmin/optimizers/lbfgs.py:78-128 (driver), :53-75 (two-loop),
:18-50 (memory with curvature guard), ffmin/optimizers/common.py:195-240
(warm-started LineSearcher) and ffmin/linesearch.py:154-227 (ls_par with a
gradient start), evaluated with the C oracle.  Used to check the device
L-BFGS trace on sizes the reference itself cannot be run at, and as the
timed CPU baseline of the minimiser.
"""

from __future__ import annotations

import math

import numpy as np

from . import Arrays, energy_and_gradient

_DUP_TOL = 1e-13
CURVATURE_RTOL = 1e-12


class _Oracle:
    def __init__(self, A: Arrays, threads=1):
        self.A = A
        self.threads = threads
        self.value_calls = 0
        self.grad_calls = 0

    def _eval(self, x, grad):
        e, g, err = energy_and_gradient(self.A, x.reshape(-1, 3), grad, self.threads)
        if err is not None:
            raise ValueError(f"degenerate geometry: {err}")
        return e[0] + e[1] + e[2] + e[3] + e[4], g

    def value(self, x):
        self.value_calls += 1
        return self._eval(x, False)[0]

    def gradient(self, x):
        self.grad_calls += 1
        return self._eval(x, True)[1]

    def value_and_gradient(self, x):
        self.value_calls += 1
        self.grad_calls += 1
        return self._eval(x, True)


def _fit(points):
    (x0, f0), (x1, f1), (x2, f2) = points
    d01 = (f1 - f0) / (x1 - x0)
    d12 = (f2 - f1) / (x2 - x1)
    a = (d12 - d01) / (x2 - x0)
    tol = 1e-12 * max(abs(f0), abs(f1), abs(f2))
    if a <= 0.0 or abs(a) < tol:
        return None
    return (x0 + x1) / 2.0 - d01 / (2.0 * a)


def _clamp(v, lo, hi, points):
    if not math.isfinite(v):
        return None
    v = min(max(v, lo), hi)
    scale = max(1.0, abs(v))
    for h, _ in points:
        if abs(v - h) <= _DUP_TOL * max(scale, abs(h)):
            return None
    return v


def ls_par(oracle, x0, r, h0, f0, g0, K=6, trust=10.0):
    """ffmin/linesearch.py:154-215 with use_gradient_start=True."""
    phi = lambda h: oracle.value(x0 + h * r)
    lo, hi = 0.0, trust * h0
    points = [(0.0, f0)]
    failed = False
    slope = float(np.dot(g0, r))
    f1 = phi(h0)
    points.append((h0, f1))
    a = (f1 - f0 - slope * h0) / (h0 * h0)
    tol = 1e-12 * max(abs(f0), abs(f1))
    if a <= 0.0 or abs(a) < tol:
        failed = True
    else:
        v = _clamp(-slope / (2.0 * a), lo, hi, points)
        if v is None:
            failed = True
        else:
            points.append((v, phi(v)))
    if not failed:
        for _ in range(2, K + 1):
            best3 = sorted(points, key=lambda p: (p[1], abs(p[0])))[:3]
            if len({p[0] for p in best3}) < 3:
                break
            v = _fit(best3)
            if v is None:
                break
            v = _clamp(v, lo, hi, points)
            if v is None:
                break
            points.append((v, phi(v)))
    h_best, f_best = min(points, key=lambda p: (p[1], abs(p[0])))
    if h_best != 0.0 and f_best < f0:
        return h_best, f_best, True
    return 0.0, f0, False


def lbfgs(A: Arrays, x0, m=3, max_iterations=10_000, gtol=0.0, rtol=0.0, h0=1.0, K=6,
          threads=1):
    """Returns dict(x, f, grad_norm, iterations, status, f_trace, calls)."""
    orc = _Oracle(A, threads)
    x = np.array(x0, dtype=np.float64).reshape(-1)
    f, g = orc.value_and_gradient(x)
    gn = float(np.linalg.norm(g))
    thr = max(gtol, rtol * max(1.0, gn))
    f_trace = [f]
    calls = [(orc.value_calls, orc.grad_calls)]
    S, Y, RHO = [], [], []
    h_warm = h0
    status = "converged" if gn <= thr else None
    cleared = False
    k = 0
    while status is None:
        if k >= max_iterations:
            status = "iteration_budget"
            break
        if not S:
            d = -g / gn if gn > 0 else -g
        else:
            q = g.copy()
            al = [0.0] * len(S)
            for i in range(len(S) - 1, -1, -1):
                al[i] = RHO[i] * float(S[i] @ q)
                q -= al[i] * Y[i]
            q *= float(S[-1] @ Y[-1]) / float(Y[-1] @ Y[-1])
            for i in range(len(S)):
                b = RHO[i] * float(Y[i] @ q)
                q += (al[i] - b) * S[i]
            d = -q
        dn = float(np.linalg.norm(d))
        if dn == 0.0:
            status = "converged"
            break
        r = d / dn
        h, fs, ok = ls_par(orc, x, r, h_warm, f, g, K)
        if not ok and h_warm != h0:
            h, fs, ok = ls_par(orc, x, r, h0, f, g, K)
        if ok:
            h_warm = abs(h)
        else:
            h_warm = h0
        if not ok:
            if S and not cleared:
                S.clear(), Y.clear(), RHO.clear()
                cleared = True
                continue
            status = "linesearch_failure"
            break
        cleared = False
        x_new = x + h * r
        g_new = orc.gradient(x_new)
        s, y = x_new - x, g_new - g
        sy = float(s @ y)
        if sy > CURVATURE_RTOL * float(np.linalg.norm(s)) * float(np.linalg.norm(y)):
            if len(S) == m:
                S.pop(0), Y.pop(0), RHO.pop(0)
            S.append(s), Y.append(y), RHO.append(1.0 / sy)
        x, f, g = x_new, fs, g_new
        gn = float(np.linalg.norm(g))
        k += 1
        f_trace.append(f)
        calls.append((orc.value_calls, orc.grad_calls))
        if gn <= thr:
            status = "converged"
    return dict(x=x, f=f, grad_norm=gn, iterations=k, status=status, f_trace=f_trace,
                calls=calls)
