"""Inexact one-dimensional searches (mirrors ffmin/linesearch.py).

Same two procedures, configurations, results and call budgets as the
reference (Algorithms 5 and 6 of the paper):

  ls_h    probe h0; expand once by k_plus if it relaxes, else contract by
          k_minus until a strictly relaxing step or h <= eps_h;
  ls_par  parabolic interpolation seeded either by the directional
          derivative at h = 0 (G0) or by samples at +-h0/2, at most K + 2
          oracle calls.

Trial points x0 + h r are formed in the oracle's own vector space
(vecops), so on the device path the only traffic per probe is the energy
scalar coming back.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

from .vecops import ops_for

FOUND = "found"
NO_RELAXATION = "no_relaxation"

# a vertex within this relative distance of a sampled abscissa would only
# reproduce the same parabola (ffmin/linesearch.py:26-28)
_DUP_TOL = 1e-13


@dataclass(frozen=True)
class LsHConfig:
    h0: float = 1.0
    eps_h: float = 1e-12
    k_plus: float = 2.0
    k_minus: float = 0.5

    def __post_init__(self):
        if not self.h0 > 0:
            raise ValueError(f"h0 must be > 0, got {self.h0}")
        if not 0 < self.eps_h < 1:
            raise ValueError(f"eps_h must be in (0,1), got {self.eps_h}")
        if not self.k_plus > 1:
            raise ValueError(f"k_plus must be > 1, got {self.k_plus}")
        if not 0 < self.k_minus < 1:
            raise ValueError(f"k_minus must be in (0,1), got {self.k_minus}")


@dataclass(frozen=True)
class LsParConfig:
    h0: float = 1.0
    K: int = 6
    use_gradient_start: bool = True
    trust: float = 10.0  # vertex steps clamped to trust * h0

    def __post_init__(self):
        if not self.h0 > 0:
            raise ValueError(f"h0 must be > 0, got {self.h0}")
        if self.K < 2:
            raise ValueError(f"K must be >= 2, got {self.K}")
        if not self.trust > 0:
            raise ValueError(f"trust must be > 0, got {self.trust}")


@dataclass(frozen=True)
class LineSearchResult:
    h: float
    f_at_step: float
    oracle_calls: int
    status: str

    def __post_init__(self):
        if self.status not in (FOUND, NO_RELAXATION):
            raise ValueError(f"bad status {self.status!r}")
        if self.status == NO_RELAXATION and self.h != 0.0:
            raise ValueError("no_relaxation implies h = 0")


@dataclass(frozen=True)
class ParabolaFit:
    points: tuple
    vertex: float | None
    curvature_positive: bool


def fit_parabola(points) -> ParabolaFit:
    """Interpolating parabola through three points (divided differences)."""
    (x0, f0), (x1, f1), (x2, f2) = points
    if x0 == x1 or x0 == x2 or x1 == x2:
        raise ValueError("parabola fit needs pairwise distinct abscissae")
    s01 = (f1 - f0) / (x1 - x0)
    s12 = (f2 - f1) / (x2 - x1)
    curv = (s12 - s01) / (x2 - x0)  # half the second derivative
    degenerate = abs(curv) < 1e-12 * max(abs(f0), abs(f1), abs(f2))
    if curv <= 0.0 or degenerate:
        return ParabolaFit(tuple(points), None, curv > 0.0)
    return ParabolaFit(tuple(points), 0.5 * (x0 + x1) - s01 / (2.0 * curv), True)


def parabola_min(points):
    """Vertex abscissa of the interpolating parabola, None on failure."""
    return fit_parabola(points).vertex


class _Probe:
    """phi(h) = f(x0 + h r) with a call counter, in the oracle's space."""

    def __init__(self, oracle, x0, r, ops):
        self.oracle, self.x0, self.r, self.ops = oracle, x0, r, ops
        self.calls = 0

    def __call__(self, h):
        self.calls += 1
        return self.oracle.value(self.ops.lincomb(1.0, self.x0, h, self.r))


def _unit(ops, r):
    nrm = ops.norm(r)
    if abs(nrm - 1.0) > 1e-8:
        raise ValueError(f"direction must be unit length, got norm {nrm}")


def ls_h(oracle, x0, r, config: LsHConfig, f0: float, ops=None, _checked=False) -> LineSearchResult:
    """Algorithm 5: probe, one expansion, or contraction to eps_h."""
    ops = ops or ops_for(oracle)
    if not _checked:
        x0, r = ops.asvec(x0), ops.asvec(r)
        _unit(ops, r)
    phi = _Probe(oracle, x0, r, ops)
    h = config.h0
    fh = phi(h)
    if fh < f0:
        h2 = config.k_plus * h
        f2 = phi(h2)
        if f2 < fh:
            return LineSearchResult(h2, f2, phi.calls, FOUND)
        return LineSearchResult(h, fh, phi.calls, FOUND)
    h = config.k_minus * config.h0
    fh = phi(h)
    while not fh < f0:  # relaxation must be strict
        h = config.k_minus * h
        if h <= config.eps_h:
            return LineSearchResult(0.0, f0, phi.calls, NO_RELAXATION)
        fh = phi(h)
    return LineSearchResult(h, fh, phi.calls, FOUND)


def _accept_vertex(v, lo, hi, points):
    if not math.isfinite(v):
        return None
    v = min(max(v, lo), hi)
    scale = max(1.0, abs(v))
    if any(abs(v - h) <= _DUP_TOL * max(scale, abs(h)) for h, _ in points):
        return None
    return v


def _rank(p):
    return (p[1], abs(p[0]))


def ls_par(oracle, x0, r, config: LsParConfig, f0: float, g0=None, ops=None,
           _checked=False, slope=None) -> LineSearchResult:
    """Algorithm 6: parabolic refinement, at most K + 2 oracle calls."""
    ops = ops or ops_for(oracle)
    if not _checked:
        x0, r = ops.asvec(x0), ops.asvec(r)
        _unit(ops, r)
    phi = _Probe(oracle, x0, r, ops)
    h0 = config.h0
    hi = config.trust * h0
    lo = 0.0 if config.use_gradient_start else -hi
    pts = [(0.0, f0)]
    ok = True
    if config.use_gradient_start:
        if g0 is None and slope is None:
            raise ValueError("use_gradient_start requires g0")
        if slope is None:
            slope = ops.dot(g0 if _checked else ops.asvec(g0), r)
        f1 = phi(h0)
        pts.append((h0, f1))
        # quadratic through (0, f0) with slope `slope`, and (h0, f1)
        curv = (f1 - f0 - slope * h0) / (h0 * h0)
        if curv <= 0.0 or abs(curv) < 1e-12 * max(abs(f0), abs(f1)):
            ok = False
        else:
            v = _accept_vertex(-slope / (2.0 * curv), lo, hi, pts)
            if v is None:
                ok = False
            else:
                pts.append((v, phi(v)))
    else:
        for h in (-0.5 * h0, 0.5 * h0):
            pts.append((h, phi(h)))
    if ok:
        for _ in range(config.K - 1):
            best = sorted(pts, key=_rank)[:3]
            if len({h for h, _ in best}) < 3:
                break
            v = fit_parabola(best).vertex
            v = None if v is None else _accept_vertex(v, lo, hi, pts)
            if v is None:
                break
            pts.append((v, phi(v)))
    hb, fb = min(pts, key=_rank)
    if hb != 0.0 and fb < f0:
        return LineSearchResult(hb, fb, phi.calls, FOUND)
    return LineSearchResult(0.0, f0, phi.calls, NO_RELAXATION)
