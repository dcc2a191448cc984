"""Far-field linearisation, incremental deltas and the gradient-free atom
wiggle on the device, against the reference (golden).  GPU only."""

import math

import numpy as np
import pytest

from conftest import golden_system

pytestmark = pytest.mark.gpu


def test_farfield_linearisation_matches_reference(golden):
    from paper_1810_03358_b200.energy import delta_energy_atom_move, linearize_farfield_coulomb

    s = golden_system(golden, "ff40")
    for atom in (0, 7, 23, 39):
        lin = linearize_farfield_coulomb(s, atom, 7.0)
        ref = golden[f"ff40/lin{atom}"]
        assert lin.e_far0 == pytest.approx(ref[0], rel=1e-12, abs=1e-12)
        np.testing.assert_allclose(lin.coef, ref[1:], rtol=1e-11, atol=1e-12)
        assert np.array_equal(lin.near_idx, golden[f"ff40/near{atom}"])
    for atom, dx, dy, dz, want in golden["ff40/deltas"]:
        lin = linearize_farfield_coulomb(s, int(atom), 7.0)
        got = delta_energy_atom_move(s, lin, [dx, dy, dz])
        assert got == pytest.approx(want, rel=1e-10, abs=1e-10)


def test_incremental_delta_rejects_cutoff_systems(golden):
    from paper_1810_03358_b200.energy import delta_energy_atom_move, linearize_farfield_coulomb

    s = golden_system(golden, "chain12cut")
    lin = linearize_farfield_coulomb(s, 3, 7.0)
    with pytest.raises(ValueError, match="cutoff"):
        delta_energy_atom_move(s, lin, [0.1, 0.0, 0.0])


@pytest.mark.parametrize("name", ["wig40", "wigchain"])
def test_wiggle_tracks_reference(golden, name):
    from paper_1810_03358_b200.optimizers import StopCriteria
    from paper_1810_03358_b200.optimizers.wiggle import WiggleConfig, atom_wiggle

    s = golden_system(golden, name)
    h, seed, epoch, inc, cutoff, iters = golden[f"{name}/cfg"]
    cfg = WiggleConfig(h=h, seed=int(seed), epoch_iterations=int(epoch),
                       use_incremental_coulomb=bool(inc), cutoff=cutoff)
    res = atom_wiggle(s, cfg, StopCriteria(max_iterations=int(iters), gradient_norm_rtol=0.0))
    f = np.array([r.f for r in res.trace.records])
    steps = np.array([r.step for r in res.trace.records])
    ref_f, ref_steps = golden[f"{name}/f"], golden[f"{name}/step"]
    # same random atoms, same accept / reject decisions, same energies
    assert np.array_equal(steps > 0, ref_steps > 0)
    # vertex steps come from parabola fits of probe deltas: roundoff x ~1e3
    np.testing.assert_allclose(steps, ref_steps, rtol=1e-6, atol=1e-12)
    np.testing.assert_allclose(f, ref_f, rtol=1e-9, atol=1e-8)
    calls = np.array([r.value_calls for r in res.trace.records])
    assert np.array_equal(calls, golden[f"{name}/calls"])
    # every accepted move strictly lowered the energy
    assert all(b < a for a, b, st in zip(f, f[1:], steps[1:]) if st > 0)
    assert math.isnan(res.grad_norm)


@pytest.mark.parametrize("inc", [True, False])
def test_graph_wiggle_equals_host_loop(golden, monkeypatch, inc):
    """The graph-resident wiggle (probe batches, parabola vertex, exact check,
    epoch re-evaluation as conditional nodes) makes the host loop's
    decisions with its arithmetic: identical records, coordinates, calls."""
    from paper_1810_03358_b200.optimizers import StopCriteria
    from paper_1810_03358_b200.optimizers.wiggle import WiggleConfig, atom_wiggle
    from paper_1810_03358_b200.synth import make_globule_system

    s = make_globule_system(900, seed=6)
    cfg = WiggleConfig(h=0.05, seed=3, epoch_iterations=25, use_incremental_coulomb=inc,
                       cutoff=7.0)
    out = []
    for host in (True, False):
        if host:
            monkeypatch.setenv("FFMIN_B200_HOST_LOOP", "1")
        else:
            monkeypatch.delenv("FFMIN_B200_HOST_LOOP", raising=False)
        out.append(atom_wiggle(s, cfg, StopCriteria(max_iterations=150, gradient_norm_rtol=0.0)))
    a, b = out
    ra = [(r.iteration, r.f, r.step, r.value_calls, r.best_f) for r in a.trace.records]
    rb = [(r.iteration, r.f, r.step, r.value_calls, r.best_f) for r in b.trace.records]
    assert len(ra) == len(rb) == 151
    assert ra == rb
    assert a.f == b.f and a.status == b.status and np.array_equal(a.x, b.x)
    assert sum(1 for r in a.trace.records if r.step > 0) > 10  # moves were made


def test_exact_deltas_equal_full_recompute_at_scale():
    """The wiggle's exact single-atom probes (O(n) device deltas) against the
    reference's probe_full recipe -- total energy of the moved system minus
    the running total (ffmin/optimizers/wiggle.py:118-127) -- on a 5000-atom
    globule: they agree to the roundoff of the two totals."""
    import oracle as O

    from paper_1810_03358_b200.energy import energy_total, exact_delta_atom_move
    from paper_1810_03358_b200.synth import make_globule_system

    s = make_globule_system(5000, seed=3)
    A = O.Arrays.from_system(s)
    e0 = float(np.sum(O.energy_and_gradient(A, s.coords, False, threads=O.host_threads())[0]))
    assert energy_total(s).total == pytest.approx(e0, rel=1e-11)
    rng = np.random.default_rng(5)
    for atom in rng.integers(0, s.natoms, size=6):
        d = rng.normal(scale=0.2, size=3)
        moved = s.coords.copy()
        moved[atom] += d
        e1 = float(np.sum(O.energy_and_gradient(A, moved, False, threads=O.host_threads())[0]))
        full = e1 - e0  # probe_full
        exact = exact_delta_atom_move(s, int(atom), d)
        assert abs(exact - full) <= 1e-11 * abs(e0) + 1e-9, (atom, exact, full)
        # the device total of the moved system gives the same difference
        dev = energy_total(s.with_coords(moved)).total - energy_total(s).total
        assert abs(dev - full) <= 1e-11 * abs(e0) + 1e-9
