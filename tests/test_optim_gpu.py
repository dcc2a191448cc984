"""Device-resident optimiser algebra and the L-BFGS driver on the B200.
GPU only (-m gpu)."""

import numpy as np
import pytest

from conftest import golden_system

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dops():
    from paper_1810_03358_b200.vecops import DeviceOps

    return DeviceOps()


def test_dot_and_axpby_kernels(dops):
    import torch

    rng = np.random.default_rng(0)
    for n in (1, 1000, 300_000):
        a, b = rng.standard_normal(n), rng.standard_normal(n)
        ta, tb = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
        d = dops.dot(ta, tb)
        assert d == pytest.approx(float(a @ b), rel=1e-12, abs=1e-12)
        assert dops.dot(ta, tb) == d  # deterministic, bit for bit
        z = dops.lincomb(0.5, ta, -2.0, tb).cpu().numpy()
        assert np.allclose(z, 0.5 * a - 2.0 * b, rtol=1e-15, atol=1e-15)


@pytest.mark.parametrize("n,m", [(3000, 3), (300_000, 5), (999, 1)])
def test_two_loop_kernel_matches_host(dops, n, m):
    import torch

    from paper_1810_03358_b200.optimizers import LbfgsMemory, lbfgs_direction
    from paper_1810_03358_b200.vecops import HostOps

    rng = np.random.default_rng(n + m)
    hmem, dmem = LbfgsMemory(m, HostOps()), LbfgsMemory(m, dops)
    for _ in range(m + 2):  # wraps the ring
        s = rng.standard_normal(n)
        y = s + 0.2 * rng.standard_normal(n)
        assert hmem.push(s, y) == dmem.push(torch.from_numpy(s).cuda(), torch.from_numpy(y).cuda())
    g = rng.standard_normal(n)
    want = lbfgs_direction(hmem, g)
    got = lbfgs_direction(dmem, torch.from_numpy(g).cuda(), dops).cpu().numpy()
    assert np.max(np.abs(got - want)) <= 1e-11 * np.max(np.abs(want))


def test_device_lbfgs_follows_reference_trace(golden):
    """500-atom chain, FP64: the device run tracks the reference run of the
    golden file iteration by iteration until roundoff differences (1e-14
    per evaluation) are amplified by the nonconvex landscape."""
    from paper_1810_03358_b200.oracle import MolecularOracle
    from paper_1810_03358_b200.optimizers import StopCriteria, lbfgs, make_linesearch

    s = golden_system(golden, "lbfgs500")
    stop = StopCriteria(max_iterations=25, gradient_norm_tol=1e-3, gradient_norm_rtol=0.0)
    res = lbfgs(MolecularOracle(s), s.coords.ravel(), m=3, linesearch=make_linesearch("par"),
                stop=stop)
    f = np.array([r.f for r in res.trace.records])
    ref = golden["lbfgs500/f_trace"][: len(f)]
    np.testing.assert_allclose(f, ref, rtol=1e-7)
    # gradient calls are one per iteration in both; a line search may take
    # one probe more or less when two probe energies tie to roundoff
    calls = np.array([[r.value_calls, r.grad_calls] for r in res.trace.records])
    ref_calls = golden["lbfgs500/calls"][: len(f)]
    assert np.array_equal(calls[:, 1], ref_calls[:, 1])
    assert np.max(np.abs(calls[:, 0] - ref_calls[:, 0])) <= 3


def test_device_lbfgs_horizon_at_least_references_own(golden):
    """configs[0], the bounded 300-iteration run: how long the device trace
    stays within 1e-8 of the reference's (numba) trace must be at least how
    long the reference's numpy backend stays within 1e-8 of its numba
    backend (lbfgs500/self_horizon, tests/golden/make_golden_r2.py) -- the
    basin the unconverged run ends in is decided by roundoff in both."""
    from paper_1810_03358_b200.oracle import MolecularOracle
    from paper_1810_03358_b200.optimizers import StopCriteria, lbfgs, make_linesearch

    s = golden_system(golden, "lbfgs500")
    stop = StopCriteria(max_iterations=300, gradient_norm_tol=1e-3, gradient_norm_rtol=0.0)
    res = lbfgs(MolecularOracle(s), s.coords.ravel(), m=3, linesearch=make_linesearch("par"),
                stop=stop)
    f = np.array([r.f for r in res.trace.records])
    ref = golden["lbfgs500/f_trace"]
    k = min(len(f), len(ref))
    bad = np.nonzero(np.abs(f[:k] - ref[:k]) > 1e-8 * np.abs(ref[:k]))[0]
    horizon = int(bad[0]) if len(bad) else k
    assert horizon >= int(golden["lbfgs500/self_horizon"]) > 0


@pytest.mark.parametrize("name,m", [("conv10", 5), ("conv60", 5), ("conv200", 5),
                                    ("conv500", 5)])
def test_device_lbfgs_reaches_reference_minimum(golden, name, m):
    """Run to the precision limit like the reference; final energies agree
    to 1e-9 relative (north star: 1e-6), both in FP64 and FP32 modes."""
    from paper_1810_03358_b200.oracle import MolecularOracle
    from paper_1810_03358_b200.optimizers import StopCriteria, lbfgs, make_linesearch

    s = golden_system(golden, name)
    ref_f, _, _, tol = golden[f"{name}/final"]
    stop = StopCriteria(max_iterations=20000, gradient_norm_tol=tol, gradient_norm_rtol=0.0)
    res = lbfgs(MolecularOracle(s), s.coords.ravel(), m=m, linesearch=make_linesearch("par"),
                stop=stop)
    assert res.f == pytest.approx(ref_f, rel=1e-9)
    assert np.max(np.abs(res.x - golden[f"{name}/x"])) < 1e-3
    best = [r.best_f for r in res.trace.records]
    assert all(b2 <= b1 for b1, b2 in zip(best, best[1:]))
    res32 = lbfgs(MolecularOracle(s, dtype=np.float32), s.coords.ravel(), m=m,
                  linesearch=make_linesearch("par"),
                  stop=StopCriteria(max_iterations=20000, gradient_norm_tol=1e-2,
                                    gradient_norm_rtol=0.0))
    from paper_1810_03358_b200.energy import energy_total
    f32_in_f64 = energy_total(s.with_coords(res32.x.reshape(-1, 3))).total
    assert f32_in_f64 == pytest.approx(ref_f, rel=1e-4)


@pytest.mark.parametrize("n,iters", [(10000, 8), (100000, 1)])
def test_device_lbfgs_at_benchmark_sizes_tracks_oracle(n, iters):
    """configs[2] / configs[4] sizes: the graph-resident FP64 L-BFGS on the
    10k / 100k-atom globules of bench.py against oracle/optim.py (the
    reference driver restated, lbfgs.py:78-128, on the threaded C oracle):
    same f trace (1e-7 relative), gradient calls, value calls within a
    probe or so, iterate within 1e-4 A."""
    import oracle as O
    import oracle.optim as OO
    from paper_1810_03358_b200.oracle import MolecularOracle
    from paper_1810_03358_b200.optimizers import StopCriteria, lbfgs, make_linesearch
    from paper_1810_03358_b200.synth import make_globule_system

    s = make_globule_system(n, seed=1)
    res = lbfgs(MolecularOracle(s), s.coords.ravel(), m=5, linesearch=make_linesearch("par"),
                stop=StopCriteria(max_iterations=iters, gradient_norm_rtol=0.0))
    ref = OO.lbfgs(O.Arrays.from_system(s), s.coords.ravel(), m=5, max_iterations=iters,
                   threads=O.host_threads())
    f = np.array([r.f for r in res.trace.records])
    assert len(f) == len(ref["f_trace"]) == iters + 1
    # roundoff of two summation orders, amplified by the strained start's
    # steep descent (measured 2.4e-9 after 7 iterations at 10k)
    np.testing.assert_allclose(f, ref["f_trace"], rtol=1e-7, atol=0)
    calls = np.array([(r.value_calls, r.grad_calls) for r in res.trace.records])
    ref_calls = np.array(ref["calls"])
    assert np.array_equal(calls[:, 1], ref_calls[:, 1])
    assert np.max(np.abs(calls[:, 0] - ref_calls[:, 0])) <= 3  # a probe more or less on ties
    assert np.max(np.abs(res.x - ref["x"])) <= 1e-4


def test_device_results_stay_on_device():
    import torch

    from paper_1810_03358_b200.oracle import MolecularOracle
    from paper_1810_03358_b200.optimizers import StopCriteria, lbfgs, make_linesearch
    from paper_1810_03358_b200.synth import make_globule_system

    s = make_globule_system(3000, seed=3)
    orc = MolecularOracle(s)
    x0 = orc.initial_point()
    res = lbfgs(orc, x0, m=3, linesearch=make_linesearch("par"),
                stop=StopCriteria(max_iterations=20, gradient_norm_rtol=0.0))
    assert isinstance(res.x, torch.Tensor) and res.x.is_cuda
    assert res.f < res.trace.records[0].f


DRIVERS = ["sd_h", "sd_par", "gd", "hb", "nag", "nagsc", "fgm", "ofgm_L", "ofgm_ls", "lbfgs",
           "cg_fr", "cg_prp", "cg_prp+", "cg_hs", "cg_cd", "cg_ls", "cg_dy"]
FIXED_STEP = {"gd", "hb", "nag", "nagsc", "ofgm_L"}


@pytest.mark.parametrize("name", DRIVERS)
def test_every_driver_on_device_tracks_reference(golden, name):
    """The same drivers with x, g and directions in HBM (FP64): traces agree
    with the reference to 1e-7 -- all 40 iterations for the fixed-step
    methods, the first 10 for line-searched ones (a line search may take a
    different branch once two probe energies tie to roundoff)."""
    from drivers_common import driver_runs, trace

    from paper_1810_03358_b200.oracle import MolecularOracle

    s = golden_system(golden, "drv30")
    res = driver_runs(s.coords.ravel())[name](MolecularOracle(s))
    f, _ = trace(res)
    ref = golden[f"drv30/{name}/f"]
    k = len(ref) if name in FIXED_STEP else 11
    np.testing.assert_allclose(f[:k], ref[:k], rtol=1e-7)
    assert res.status == str(golden[f"drv30/{name}/status"])


def _run_lbfgs(s, host_loop, monkeypatch, kind, m, stop, dtype=np.float64, **ls):
    from paper_1810_03358_b200.oracle import MolecularOracle
    from paper_1810_03358_b200.optimizers import lbfgs, make_linesearch

    if host_loop:
        monkeypatch.setenv("FFMIN_B200_HOST_LOOP", "1")
    else:
        monkeypatch.delenv("FFMIN_B200_HOST_LOOP", raising=False)
    o = MolecularOracle(s, dtype=dtype)
    res = lbfgs(o, s.coords.ravel(), m=m, linesearch=make_linesearch(kind, **ls), stop=stop)
    return res, o


@pytest.mark.parametrize("case", [
    ("conv60", "par", 5, {}), ("conv200", "par", 3, {}), ("conv200", "h", 5, {}),
    ("lbfgs500", "par", 3, {"use_gradient_start": False}), ("globule", "par", 5, {}),
    ("globule32", "par", 5, {})])
def test_graph_lbfgs_equals_host_driven_loop(golden, monkeypatch, case):
    """The graph-resident iteration (conditional CUDA graph, csrc/
    ffm_minimize.cu) makes the same decisions with the same arithmetic as
    the host-driven loop: identical trace records, iterate and status."""
    from paper_1810_03358_b200.optimizers import StopCriteria
    from paper_1810_03358_b200.synth import make_globule_system

    name, kind, m, ls = case
    dtype = np.float32 if name == "globule32" else np.float64
    if name.startswith("globule"):
        s = make_globule_system(1500, seed=3)
        stop = StopCriteria(max_iterations=60, gradient_norm_rtol=1e-4)
    else:
        s = golden_system(golden, name)
        stop = StopCriteria(max_iterations=400, gradient_norm_tol=1e-6, gradient_norm_rtol=0.0)
    a, oa = _run_lbfgs(s, True, monkeypatch, kind, m, stop, dtype, **ls)
    b, ob = _run_lbfgs(s, False, monkeypatch, kind, m, stop, dtype, **ls)
    ra = [(r.iteration, r.f, r.grad_norm, r.step, r.value_calls, r.grad_calls, r.best_f)
          for r in a.trace.records]
    rb = [(r.iteration, r.f, r.grad_norm, r.step, r.value_calls, r.grad_calls, r.best_f)
          for r in b.trace.records]
    assert len(ra) == len(rb)
    assert ra == rb
    assert a.status == b.status and a.f == b.f and a.grad_norm == b.grad_norm
    assert np.array_equal(a.x, b.x)
    assert (oa.value_calls, oa.grad_calls) == (ob.value_calls, ob.grad_calls)


@pytest.mark.parametrize("natoms,m", [(682, 5), (683, 5), (1024, 5), (1025, 3), (1500, 7),
                                     (2048, 5), (2049, 5)])
def test_graph_lbfgs_equals_host_loop_at_size_boundaries(monkeypatch, natoms, m):
    """Bit-identical graph-resident and host-driven L-BFGS on both sides of
    the short-vector thresholds: the fused direction (n <= 2048, shared-memory
    ring), the fused acceptance tail (n <= 3072), the fused evaluation without
    its packing pass (<= 1500 atoms) and the one-block two-loop (n <= 6144)."""
    from paper_1810_03358_b200.optimizers import StopCriteria
    from paper_1810_03358_b200.synth import make_globule_system

    s = make_globule_system(natoms, seed=natoms % 13)
    stop = StopCriteria(max_iterations=12, gradient_norm_rtol=0.0)
    a, oa = _run_lbfgs(s, True, monkeypatch, "par", m, stop)
    b, ob = _run_lbfgs(s, False, monkeypatch, "par", m, stop)
    ra = [(r.iteration, r.f, r.grad_norm, r.step, r.value_calls, r.grad_calls, r.best_f)
          for r in a.trace.records]
    rb = [(r.iteration, r.f, r.grad_norm, r.step, r.value_calls, r.grad_calls, r.best_f)
          for r in b.trace.records]
    assert ra == rb
    assert a.status == b.status and np.array_equal(a.x, b.x)


def test_graph_lbfgs_budgets(golden, monkeypatch):
    """Iteration and oracle-call budgets stop the graph run where the host
    loop stops."""
    from paper_1810_03358_b200.optimizers import StopCriteria

    s = golden_system(golden, "conv200")
    for stop in (StopCriteria(max_iterations=7, gradient_norm_rtol=0.0),
                 StopCriteria(max_iterations=None, max_oracle_calls=41, gradient_norm_rtol=0.0)):
        a, _ = _run_lbfgs(s, True, monkeypatch, "par", 5, stop)
        b, _ = _run_lbfgs(s, False, monkeypatch, "par", 5, stop)
        assert a.status == b.status and a.iterations == b.iterations and a.f == b.f


def _run_method(s, host_loop, monkeypatch, method, stop, dtype=np.float64, kind="par", **kw):
    from paper_1810_03358_b200.oracle import MolecularOracle
    from paper_1810_03358_b200.optimizers import cg, fgm, make_linesearch, steepest_descent

    if host_loop:
        monkeypatch.setenv("FFMIN_B200_HOST_LOOP", "1")
    else:
        monkeypatch.delenv("FFMIN_B200_HOST_LOOP", raising=False)
    o = MolecularOracle(s, dtype=dtype)
    ls = make_linesearch(kind)
    if method == "sd":
        res = steepest_descent(o, s.coords.ravel(), ls, stop)
    elif method == "fgm":
        res = fgm(o, s.coords.ravel(), ls, stop)
    else:
        from paper_1810_03358_b200.optimizers.cg import CgVariant

        res = cg(o, s.coords.ravel(), CgVariant(kind=method, **kw), ls, stop)
    return res, o


@pytest.mark.parametrize("case", [
    ("sd", "conv60", "par", {}), ("sd", "conv200", "h", {}),
    ("fr", "conv200", "par", {}), ("prp", "conv200", "par", {}), ("prp+", "conv200", "h", {}),
    ("hs", "conv60", "par", {}), ("cd", "conv60", "par", {}), ("ls", "conv200", "par", {}),
    ("dy", "conv200", "par", {}), ("prp+", "conv200", "par", {"restart_period": 7}),
    ("prp+", "globule", "par", {}), ("fr", "globule32", "par", {}),
    ("sd", "globule32", "par", {}), ("fgm", "conv200", "par", {}), ("fgm", "conv60", "h", {}),
    ("fgm", "conv60", "par", {}), ("fgm", "globule", "par", {}), ("fgm", "globule32", "h", {})])
def test_graph_cg_sd_equal_host_driven_loop(golden, monkeypatch, case):
    """Nonlinear CG (all seven betas, periodic and descent restarts, the
    two-failure rule), steepest descent and FGM (theta schedule, search from
    the extrapolated point, best-point tracking) run as the same conditional
    CUDA graph as L-BFGS: identical trace records (best f included),
    iterate, status and call counts to the host-driven loop."""
    from paper_1810_03358_b200.optimizers import StopCriteria
    from paper_1810_03358_b200.synth import make_globule_system

    method, name, kind, kw = case
    dtype = np.float32 if name == "globule32" else np.float64
    if name.startswith("globule"):
        s = make_globule_system(1500, seed=3)
        stop = StopCriteria(max_iterations=60, gradient_norm_rtol=1e-4)
    else:
        s = golden_system(golden, name)
        stop = StopCriteria(max_iterations=300, gradient_norm_tol=1e-6, gradient_norm_rtol=0.0,
                            stop_on_linesearch_failure=(name != "conv60"))
    a, oa = _run_method(s, True, monkeypatch, method, stop, dtype, kind, **kw)
    b, ob = _run_method(s, False, monkeypatch, method, stop, dtype, kind, **kw)
    assert "_graph_runs" not in oa.__dict__ and "_graph_runs" in ob.__dict__  # paths taken
    ra = [(r.iteration, r.f, r.grad_norm, r.step, r.value_calls, r.grad_calls, r.best_f)
          for r in a.trace.records]
    rb = [(r.iteration, r.f, r.grad_norm, r.step, r.value_calls, r.grad_calls, r.best_f)
          for r in b.trace.records]
    assert len(ra) == len(rb)
    assert ra == rb
    assert a.status == b.status and a.f == b.f and a.grad_norm == b.grad_norm
    assert np.array_equal(a.x, b.x)
    assert (oa.value_calls, oa.grad_calls) == (ob.value_calls, ob.grad_calls)


@pytest.mark.parametrize("name", ["gd", "hb", "nag", "nagsc", "sd_h", "fgm", "lbfgs", "cg_prp+",
                                  "ofgm_L", "ofgm_ls"])
@pytest.mark.parametrize("system", ["drv30", "globule"])
def test_graph_drivers_equal_host_loop_table(golden, monkeypatch, name, system):
    """Every graph-resident driver of the golden driver table (fixed-step GD,
    heavy ball, both Nesterov schemes, and the line-searched ones) against
    the host-driven loop on the same oracle: identical records and iterate."""
    from drivers_common import driver_runs

    from paper_1810_03358_b200.oracle import MolecularOracle
    from paper_1810_03358_b200.synth import make_globule_system

    s = golden_system(golden, "drv30") if system == "drv30" else make_globule_system(1200, seed=5)
    out = []
    for host in (True, False):
        if host:
            monkeypatch.setenv("FFMIN_B200_HOST_LOOP", "1")
        else:
            monkeypatch.delenv("FFMIN_B200_HOST_LOOP", raising=False)
        o = MolecularOracle(s)
        res = driver_runs(s.coords.ravel())[name](o)
        out.append((res, o))
    (a, oa), (b, ob) = out
    assert "_graph_runs" not in oa.__dict__ and "_graph_runs" in ob.__dict__
    ra = [(r.iteration, r.f, r.grad_norm, r.step, r.value_calls, r.grad_calls, r.best_f)
          for r in a.trace.records]
    rb = [(r.iteration, r.f, r.grad_norm, r.step, r.value_calls, r.grad_calls, r.best_f)
          for r in b.trace.records]
    assert ra == rb
    assert a.status == b.status and a.f == b.f and a.grad_norm == b.grad_norm
    assert np.array_equal(a.x, b.x)
    assert a.trace.meta == b.trace.meta


@pytest.mark.parametrize("driver", ["gd", "hb", "nag"])
def test_graph_fixed_step_divergence_matches_host(golden, monkeypatch, driver):
    """A step far too long diverges: the graph raises the host loop's
    DivergenceError, message included."""
    from paper_1810_03358_b200.optimizers import (
        DivergenceError, StopCriteria, gradient_descent_fixed, heavy_ball, nesterov_momentum)
    from paper_1810_03358_b200.oracle import MolecularOracle

    s = golden_system(golden, "drv30")
    stop = StopCriteria(max_iterations=200, gradient_norm_rtol=0.0)
    run = {"gd": lambda o: gradient_descent_fixed(o, s.coords.ravel(), 0.5, stop),
           "hb": lambda o: heavy_ball(o, s.coords.ravel(), 2.0, 0.9, stop),
           "nag": lambda o: nesterov_momentum(o, s.coords.ravel(), 0.5, stop)}[driver]
    msgs = []
    for host in (True, False):
        if host:
            monkeypatch.setenv("FFMIN_B200_HOST_LOOP", "1")
        else:
            monkeypatch.delenv("FFMIN_B200_HOST_LOOP", raising=False)
        o = MolecularOracle(s)
        with pytest.raises(Exception) as ei:
            run(o)
        msgs.append((type(ei.value).__name__, str(ei.value), o.value_calls, o.grad_calls))
    assert msgs[0] == msgs[1]


@pytest.mark.parametrize("ls", ["par", "par_nogs", "h"])
def test_graph_ofgm_line_search_variants(golden, monkeypatch, ls):
    """OFGM along -d from y with every line search (ls_par seeded by the
    slope needs grad f(y): one more gradient call per iteration), a horizon
    shorter than the budget: identical to the host loop, horizon status."""
    from paper_1810_03358_b200.optimizers import StopCriteria, make_linesearch, ofgm
    from paper_1810_03358_b200.oracle import MolecularOracle

    s = golden_system(golden, "conv200")
    out = []
    for host in (True, False):
        if host:
            monkeypatch.setenv("FFMIN_B200_HOST_LOOP", "1")
        else:
            monkeypatch.delenv("FFMIN_B200_HOST_LOOP", raising=False)
        o = MolecularOracle(s)
        lsr = make_linesearch("h") if ls == "h" else make_linesearch(
            "par", use_gradient_start=(ls == "par"))
        res = ofgm(o, s.coords.ravel(), 25, linesearch=lsr,
                   stop=StopCriteria(max_iterations=100, gradient_norm_rtol=0.0))
        out.append((res, o))
    (a, oa), (b, ob) = out
    assert "_graph_runs" in ob.__dict__
    ra = [(r.iteration, r.f, r.grad_norm, r.step, r.value_calls, r.grad_calls, r.best_f)
          for r in a.trace.records]
    rb = [(r.iteration, r.f, r.grad_norm, r.step, r.value_calls, r.grad_calls, r.best_f)
          for r in b.trace.records]
    assert ra == rb
    assert a.status == b.status == "horizon_complete"
    assert a.f == b.f and np.array_equal(a.x, b.x)


def test_graph_reused_across_stop_criteria(golden, monkeypatch):
    """A captured graph is reused for runs that differ only in run-time
    configuration (budgets, tolerances, CG variant): results equal those of
    a fresh capture, and only one graph is built per structure."""
    from paper_1810_03358_b200.optimizers import StopCriteria, cg, lbfgs, make_linesearch
    from paper_1810_03358_b200.oracle import MolecularOracle

    monkeypatch.delenv("FFMIN_B200_HOST_LOOP", raising=False)
    s = golden_system(golden, "conv200")
    x0 = s.coords.ravel()
    o = MolecularOracle(s)
    lbfgs(o, x0, m=5, linesearch=make_linesearch("par"),
          stop=StopCriteria(max_iterations=4, gradient_norm_rtol=0.0))
    cg(o, x0, "fr", make_linesearch("par"), StopCriteria(max_iterations=3, gradient_norm_rtol=0.0))
    stop = StopCriteria(max_iterations=40, gradient_norm_tol=1e-3, gradient_norm_rtol=0.0)
    a = lbfgs(o, x0, m=5, linesearch=make_linesearch("par"), stop=stop)
    c = cg(o, x0, "prp+", make_linesearch("par"), stop)
    assert len(o._graph_runs) == 2
    b = lbfgs(MolecularOracle(s), x0, m=5, linesearch=make_linesearch("par"), stop=stop)
    d = cg(MolecularOracle(s), x0, "prp+", make_linesearch("par"), stop)
    for u, v in ((a, b), (c, d)):
        assert [(r.f, r.grad_norm, r.step) for r in u.trace.records] == \
            [(r.f, r.grad_norm, r.step) for r in v.trace.records]
        assert np.array_equal(u.x, v.x) and u.status == v.status
