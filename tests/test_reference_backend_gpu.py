"""The boundary proven through the reference's OWN modules: ffmin's energy
layer, oracle and L-BFGS driver, unchanged, with the B200 engine registered
as a third kernel backend exactly as INTEGRATION.md section 2 shows (the
three-line "cuda" branch in ffmin.kernels.get_backend, kernels.py:1006-1024).

The reference package is test data here, not product: it is located through
FFMIN_REF_SRC (a directory holding the ``ffmin`` package) or
/root/reference/pkg/src, and the module is skipped when neither exists (the
GPU box has no /root/reference; profiles/r02_reference_backend.log records
a run with the package staged next to the repository).
"""

import os
import sys
from pathlib import Path

import numpy as np
import pytest

from conftest import golden_arrays

pytestmark = pytest.mark.gpu

CASES = ["chain10", "chain14", "cloud24", "cloud24c7", "explicit8", "chain200", "chain12cut",
         "globule1500"]


def _ref_src():
    for cand in (os.environ.get("FFMIN_REF_SRC"), "/root/reference/pkg/src"):
        if cand and (Path(cand) / "ffmin" / "__init__.py").exists():
            return cand
    return None


@pytest.fixture(scope="module")
def ffmin_cuda():
    """ffmin with get_backend("cuda") -> CUDA_BACKEND."""
    src = _ref_src()
    if src is None:
        pytest.skip("reference package not staged (set FFMIN_REF_SRC)")
    sys.path.insert(0, src)
    import ffmin
    import ffmin.energy
    import ffmin.kernels

    from paper_1810_03358_b200.kernels import CUDA_BACKEND

    orig = ffmin.kernels.get_backend

    def get_backend(name=None):
        if name == "cuda":  # the maintainer's patch
            return CUDA_BACKEND
        return orig(name)

    mods = (ffmin.kernels, ffmin.energy, ffmin)
    for m in mods:
        m.get_backend = get_backend
    yield ffmin
    for m in mods:
        m.get_backend = orig


def _ref_system(ffmin, G, name, coords=None):
    from ffmin.model import AngleTerm, AtomSpec, BondTerm, DihedralTerm
    from ffmin.model import MolecularSystem, NonbondedPolicy

    kw, c = golden_arrays(G, name)
    atoms = tuple(AtomSpec(i, f"A{i}", float(q), float(s), float(e)) for i, (q, s, e) in
                  enumerate(zip(kw["q"], kw["sigma"], kw["epsilon"])))
    return MolecularSystem(
        atoms=atoms, coords=np.array(c if coords is None else coords),
        bonds=tuple(BondTerm(int(i), int(j), float(k), float(r)) for (i, j), k, r in
                    zip(kw["bond_idx"], kw["bond_K"], kw["bond_r0"])),
        angles=tuple(AngleTerm(int(i), int(j), int(k), float(kk), float(a)) for (i, j, k), kk, a
                     in zip(kw["ang_idx"], kw["ang_K"], kw["ang_t0"])),
        dihedrals=tuple(DihedralTerm(int(i), int(j), int(k), int(l), *map(float, v))
                        for (i, j, k, l), v in zip(kw["dih_idx"], kw["dih_V"])),
        nonbonded=NonbondedPolicy(excluded=frozenset(map(tuple, kw["excluded"].tolist())),
                                  scaled14=frozenset(map(tuple, kw["scaled14"].tolist())),
                                  s14=kw["s14"], cutoff=kw["cutoff"]))


@pytest.mark.parametrize("name", CASES)
def test_reference_energy_layer_on_cuda_backend(ffmin_cuda, golden, name):
    """ffmin.energy.energy_and_gradient / energy_total with backend="cuda"
    equal the golden numba results to 1e-10 (FP64)."""
    from ffmin.energy import energy_and_gradient, energy_total

    s = _ref_system(ffmin_cuda, golden, name)
    bd, g = energy_and_gradient(s, np.float64, "cuda")
    got = [bd.stretch, bd.bend, bd.torsion, bd.coulomb, bd.vdw]
    np.testing.assert_allclose(got, golden[f"{name}/egrad_f64"], rtol=1e-10, atol=1e-9)
    ref = golden[f"{name}/grad_f64"]
    assert np.max(np.abs(g - ref)) <= 1e-10 * np.max(np.abs(ref))
    be = energy_total(s, np.float64, "cuda")
    np.testing.assert_allclose([be.stretch, be.bend, be.torsion, be.coulomb, be.vdw],
                               golden[f"{name}/energy_f64"], rtol=1e-10, atol=1e-9)


def test_reference_errors_on_cuda_backend(ffmin_cuda, golden):
    from ffmin.energy import EnergyEvaluationError, energy_and_gradient, energy_total

    s = _ref_system(ffmin_cuda, golden, "collinear")
    msgs = []
    for fn in (energy_total, energy_and_gradient):
        try:
            fn(s, np.float64, "cuda")
            msgs.append("")
        except EnergyEvaluationError as e:
            msgs.append(str(e))
    assert msgs == golden["collinear/messages"].tolist()
    bad = _ref_system(ffmin_cuda, golden, "coincident")
    with pytest.raises(EnergyEvaluationError, match="coincident"):
        energy_and_gradient(bad, np.float64, "cuda")


@pytest.mark.parametrize("name", ["conv60", "conv200"])
def test_reference_lbfgs_on_cuda_backend(ffmin_cuda, golden, name):
    """ffmin.optimizers.lbfgs driving ffmin.oracle.MolecularOracle(backend=
    "cuda") reaches the reference's (numba) minimum to 1e-9."""
    from ffmin.optimizers import StopCriteria, lbfgs, make_linesearch
    from ffmin.oracle import MolecularOracle

    s = _ref_system(ffmin_cuda, golden, name)
    ref_f, _, _, tol = golden[f"{name}/final"]
    res = lbfgs(MolecularOracle(s, backend="cuda"), s.coords.ravel(), m=5,
                linesearch=make_linesearch("par"),
                stop=StopCriteria(max_iterations=20000, gradient_norm_tol=tol,
                                  gradient_norm_rtol=0.0))
    assert res.f == pytest.approx(float(ref_f), rel=1e-9)


def test_reference_lbfgs500_trace_on_cuda_backend(ffmin_cuda, golden):
    """configs[0] through the reference driver on the cuda backend: the
    first 20 records equal the numba trace to 1e-8."""
    from ffmin.optimizers import StopCriteria, lbfgs, make_linesearch
    from ffmin.oracle import MolecularOracle

    s = _ref_system(ffmin_cuda, golden, "lbfgs500")
    res = lbfgs(MolecularOracle(s, backend="cuda"), s.coords.ravel(), m=3,
                linesearch=make_linesearch("par"),
                stop=StopCriteria(max_iterations=20, gradient_norm_tol=1e-3,
                                  gradient_norm_rtol=0.0))
    f = np.array([r.f for r in res.trace.records])
    np.testing.assert_allclose(f, golden["lbfgs500/f_trace"][:len(f)], rtol=1e-8)
