"""Host-side optimiser logic, checked bit for bit against the reference run
recorded in the golden file (the driver is the same code the device path
runs; only the vector space differs).  CPU only."""

import math

import numpy as np
import pytest

import oracle as O
from conftest import oracle_arrays
from paper_1810_03358_b200.linesearch import (
    FOUND, NO_RELAXATION, LsHConfig, LsParConfig, fit_parabola, ls_h, ls_par, parabola_min)
from paper_1810_03358_b200.oracle import FunctionOracle
from paper_1810_03358_b200.optimizers import (
    LINESEARCH_FAILURE, LbfgsMemory, StopCriteria, lbfgs, lbfgs_direction, make_linesearch)


def c_oracle(A):
    def ev(x, grad):
        e, g, err = O.energy_and_gradient(A, np.asarray(x).reshape(-1, 3), grad)
        assert err is None
        return e[0] + e[1] + e[2] + e[3] + e[4], g
    return FunctionOracle(3 * A.n, lambda x: ev(x, False)[0], lambda x: ev(x, True)[1],
                          lambda x: ev(x, True))


def test_lbfgs_driver_reproduces_reference_run_bit_for_bit(golden):
    A, c = oracle_arrays(golden, "lbfgs500")
    stop = StopCriteria(max_iterations=300, gradient_norm_tol=1e-3, gradient_norm_rtol=0.0)
    res = lbfgs(c_oracle(A), c.reshape(-1), m=3, linesearch=make_linesearch("par"), stop=stop)
    f = np.array([r.f for r in res.trace.records])
    calls = np.array([[r.value_calls, r.grad_calls] for r in res.trace.records])
    assert np.array_equal(f, golden["lbfgs500/f_trace"])
    assert np.array_equal(calls, golden["lbfgs500/calls"])
    assert np.array_equal(res.x, golden["lbfgs500/x"])
    assert res.status == str(golden["lbfgs500/status"])


def test_parabola_hand_cases():
    assert parabola_min([(0, 1), (1, 0), (2, 1)]) == pytest.approx(1.0)
    assert parabola_min([(0, 0), (1, 1), (2, 2)]) is None
    with pytest.raises(ValueError):
        fit_parabola([(0, 0), (0, 1), (2, 2)])
    v = 0.37
    pts = [(x, 2.5 * (x - v) ** 2 + 1.0) for x in (-1.0, 0.2, 1.3)]
    assert parabola_min(pts) == pytest.approx(v, abs=1e-12)


def quad1d(center=0.0):
    return FunctionOracle(1, lambda x: float((x[0] - center) ** 2),
                          lambda x: np.array([2.0 * (x[0] - center)]))


def test_ls_h_hand_trace():
    # f = x^2 at 1, r = -1, h0 = 0.5: f(0.5) relaxes, expansion to h = 1 gives 0
    res = ls_h(quad1d(), np.array([1.0]), np.array([-1.0]), LsHConfig(h0=0.5), 1.0)
    assert (res.h, res.f_at_step, res.status, res.oracle_calls) == (1.0, 0.0, FOUND, 2)
    # increasing along r: no relaxation, call budget 2 + ceil(log2(h0 / eps))
    cfg = LsHConfig(h0=1.0, eps_h=1e-3)
    res = ls_h(quad1d(), np.array([0.0]), np.array([1.0]), cfg, 0.0)
    assert res.status == NO_RELAXATION and res.h == 0.0
    assert res.oracle_calls <= 2 + math.ceil(math.log(cfg.h0 / cfg.eps_h, 2))


def test_ls_par_exact_on_quadratics():
    orc = quad1d(center=0.7)
    x0 = np.array([0.0])
    res = ls_par(orc, x0, np.array([1.0]), LsParConfig(h0=0.25), orc.value(x0),
                 orc.gradient(x0))
    assert res.status == FOUND and res.h == pytest.approx(0.7, rel=1e-10)
    # no gradient start: samples at +-h0/2 then the vertex (spec hand trace)
    orc = quad1d(center=1.0)
    res = ls_par(orc, x0, np.array([1.0]), LsParConfig(h0=1.0, K=2, use_gradient_start=False),
                 orc.value(x0))
    assert res.h == pytest.approx(1.0) and res.f_at_step == pytest.approx(0.0)
    assert res.oracle_calls <= 2 + 2


def test_direction_must_be_unit():
    with pytest.raises(ValueError, match="unit"):
        ls_h(quad1d(), np.array([1.0]), np.array([-2.0]), LsHConfig(), 1.0)


def test_memory_semantics():
    mem = LbfgsMemory(2)
    s = np.array([1.0, 0.0])
    assert not mem.push(s, np.array([0.0, 1.0]))
    assert not mem.push(s, np.array([-1.0, 0.0]))
    assert len(mem) == 0
    assert np.array_equal(lbfgs_direction(mem, np.array([3.0, 4.0])), np.array([-0.6, -0.8]))
    v = np.array([1.0, 2.0])
    assert mem.push(v, v)
    g = np.array([0.3, -1.1])
    assert np.allclose(lbfgs_direction(mem, g), -g, atol=1e-15)
    with pytest.raises(ValueError):
        LbfgsMemory(0)


def test_two_loop_matches_dense_bfgs():
    rng = np.random.default_rng(1)
    mem = LbfgsMemory(5)
    pairs = []
    for _ in range(4):
        s = rng.standard_normal(6)
        y = s + 0.3 * rng.standard_normal(6)
        if s @ y > 0 and mem.push(s, y):
            pairs.append((s, y))
    g = rng.standard_normal(6)
    gamma = pairs[-1][0] @ pairs[-1][1] / (pairs[-1][1] @ pairs[-1][1])
    H = gamma * np.eye(6)
    for s, y in pairs:
        rho = 1.0 / (s @ y)
        V = np.eye(6) - rho * np.outer(y, s)
        H = V.T @ H @ V + rho * np.outer(s, s)
    assert np.allclose(lbfgs_direction(mem, g), -H @ g, rtol=1e-12, atol=1e-12)


def test_lbfgs_clears_memory_once_then_fails():
    class Flaky:
        def __init__(self):
            self.calls = 0

        def describe(self):
            return {"kind": "stub"}

        def search(self, oracle, x, r, f0, g0=None):
            from paper_1810_03358_b200.linesearch import LineSearchResult
            self.calls += 1
            if self.calls == 1:
                return LineSearchResult(0.5, oracle.value(x + 0.5 * r), 1, FOUND)
            return LineSearchResult(0.0, f0, 1, NO_RELAXATION)

    A = np.diag([1.0, 5.0, 10.0])
    orc = FunctionOracle(3, lambda x: 0.5 * x @ A @ x, lambda x: A @ x)
    stub = Flaky()
    res = lbfgs(orc, np.ones(3), m=3, linesearch=stub)
    assert res.status == LINESEARCH_FAILURE and res.iterations == 1 and stub.calls == 3


DRIVERS = ["sd_h", "sd_par", "gd", "hb", "nag", "nagsc", "fgm", "ofgm_L", "ofgm_ls", "lbfgs",
           "cg_fr", "cg_prp", "cg_prp+", "cg_hs", "cg_cd", "cg_ls", "cg_dy"]


@pytest.mark.parametrize("name", DRIVERS)
def test_every_driver_reproduces_reference_trace(golden, name):
    """Host vector space + C oracle: each driver's 40-iteration trace on the
    30-atom chain equals the reference's bit for bit."""
    from drivers_common import driver_runs, trace

    A, c = oracle_arrays(golden, "drv30")
    res = driver_runs(c.reshape(-1))[name](c_oracle(A))
    f, calls = trace(res)
    assert np.array_equal(f, golden[f"drv30/{name}/f"])
    assert np.array_equal(calls, golden[f"drv30/{name}/calls"])
    assert np.array_equal(res.x, golden[f"drv30/{name}/x"])
    assert res.status == str(golden[f"drv30/{name}/status"])


def test_wall_time_budget_uses_the_agreed_elapsed_time():
    """A row-sharded oracle runs the same driver on every rank and every
    evaluation ends in a collective, so the max_wall_time test must use the
    ranks' agreed (MAX) elapsed time (ShardedMolecularOracle.agreed_elapsed):
    an oracle whose agreement reports an expired budget stops the run at the
    next budget check even though the local clock has not run out, and one
    that reports none lets it run to its iteration budget."""
    from paper_1810_03358_b200.optimizers.common import TIME_BUDGET

    class Agreeing(FunctionOracle):
        def __init__(self, remote):  # Rosenbrock: no line-search failure in 3 steps
            super().__init__(
                2, lambda x: float((1 - x[0]) ** 2 + 100 * (x[1] - x[0] ** 2) ** 2),
                lambda x: np.array([-2 * (1 - x[0]) - 400 * x[0] * (x[1] - x[0] ** 2),
                                    200 * (x[1] - x[0] ** 2)]))
            self.remote = remote
            self.asked = 0

        def agreed_elapsed(self, t):
            self.asked += 1
            return max(t, self.remote)

    for remote, want in ((1e9, TIME_BUDGET), (0.0, "iteration_budget")):
        o = Agreeing(remote)
        res = lbfgs(o, np.array([-1.2, 1.0]), m=2, linesearch=make_linesearch("par"),
                    stop=StopCriteria(max_iterations=3, max_wall_time=60.0,
                                      gradient_norm_rtol=0.0, gradient_norm_tol=0.0))
        assert res.status == want and o.asked >= 1
        assert res.iterations == (0 if remote else 3)
