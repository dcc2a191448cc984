"""Potential energy and analytic gradient on the B200 (mirrors ffmin/energy.py).

Same functions, arguments, return types and error behaviour as the
reference energy layer; every evaluation runs in the CUDA engine
(engine.DeviceSystem).  NumPy inputs take the host path (coordinates copied
in, results copied out, one synchronisation: the reference-facing call);
device-resident callers use the oracle in oracle.py or engine.DeviceSystem
directly.

dtype selects the kernel precision exactly as in the reference:
float64 -> FP64 everywhere; float32 -> the O(N^2) pair sweep in FP32 with
FP64 accumulation (bonded terms stay FP64).  As in the reference, the
energy layer reports gradients in the requested dtype and energies as
Python floats.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as N
from .constants import COULOMB_KJ_ANGSTROM
from .engine import engine_for, precision_of
from .model import MolecularSystem


class EnergyEvaluationError(ValueError):
    """Degenerate or invalid geometry in a named interaction term."""


@dataclass(frozen=True)
class EnergyBreakdown:
    stretch: float
    bend: float
    torsion: float
    coulomb: float
    vdw: float

    @property
    def total(self):
        # computed as the sum, never stored separately (ffmin/energy.py:38-41)
        return self.stretch + self.bend + self.torsion + self.coulomb + self.vdw


def _check_backend(backend):
    if backend not in (None, "cuda") and getattr(backend, "name", None) != "cuda":
        raise ValueError(f"unknown kernel backend {backend!r}: this framework runs the "
                         "'cuda' backend only")


def _bond_name(system, row):
    i, j = system.topology.bond_idx[row]
    return f"stretch term {row} (atoms {i}-{j})"


def _angle_name(system, row):
    i, j, k = system.topology.ang_idx[row]
    return f"bend term {row} (atoms {i}-{j}-{k})"


def _dihedral_name(system, row):
    i, j, k, l = system.topology.dih_idx[row]
    return f"torsion term {row} (atoms {i}-{j}-{k}-{l})"


def raise_status(system, st, grad, order=None):
    """Turn engine status words into the reference's typed errors, in the
    order the reference raises them (ffmin/energy.py:133-174)."""
    st = np.asarray(st).reshape(-1)
    nb = int(st[N.ST_NB_BAD_I]), int(st[N.ST_NB_BAD_J])

    def nb_err():
        if nb[0] >= 0:
            raise EnergyEvaluationError(f"nonbonded pair ({nb[0]},{nb[1]}): coincident atoms")

    def bond_err():
        if st[N.ST_BOND] >= 0:
            raise EnergyEvaluationError(
                f"{_bond_name(system, int(st[N.ST_BOND]))}: coincident endpoints")

    def angle_err():
        if st[N.ST_ANGLE] >= 0:
            what = "zero-length arm or collinear geometry" if grad else "zero-length arm"
            raise EnergyEvaluationError(f"{_angle_name(system, int(st[N.ST_ANGLE]))}: {what}")

    def dih_err():
        if st[N.ST_DIHEDRAL] >= 0:
            raise EnergyEvaluationError(
                f"{_dihedral_name(system, int(st[N.ST_DIHEDRAL]))}: degenerate plane")

    if order is None:
        # energy_and_gradient checks bond, angle, dihedral, nonbonded;
        # energy_total evaluates the nonbonded sums first
        order = (bond_err, angle_err, dih_err, nb_err) if grad else (nb_err, angle_err, dih_err)
    for f in order:
        f()


def _eval(system, dtype, backend, grad, flags=None):
    _check_backend(backend)
    eng = engine_for(system.topology)
    return eng.eval_host(system.coords, precision_of(dtype), grad=grad, flags=flags)


def _breakdown(en):
    return EnergyBreakdown(stretch=float(en[0]), bend=float(en[1]), torsion=float(en[2]),
                           coulomb=float(en[3]), vdw=float(en[4]))


def energy_stretch(system: MolecularSystem, dtype=np.float64, backend=None) -> float:
    en, st, _ = _eval(system, dtype, backend, False, N.FFM_ENERGY | N.FFM_NO_NB)
    return float(en[0])  # the reference stretch energy kernel has no check


def energy_bend(system: MolecularSystem, dtype=np.float64, backend=None) -> float:
    en, st, _ = _eval(system, dtype, backend, False, N.FFM_ENERGY | N.FFM_NO_NB)
    if st[N.ST_ANGLE] >= 0:
        raise EnergyEvaluationError(f"{_angle_name(system, int(st[N.ST_ANGLE]))}: zero-length arm")
    return float(en[1])


def energy_torsion(system: MolecularSystem, dtype=np.float64, backend=None) -> float:
    en, st, _ = _eval(system, dtype, backend, False, N.FFM_ENERGY | N.FFM_NO_NB)
    if st[N.ST_DIHEDRAL] >= 0:
        raise EnergyEvaluationError(
            f"{_dihedral_name(system, int(st[N.ST_DIHEDRAL]))}: degenerate plane")
    return float(en[2])


def _nb_energies(system, dtype, backend):
    en, st, _ = _eval(system, dtype, backend, False, N.FFM_ENERGY | N.FFM_NO_TERMS)
    if st[N.ST_NB_BAD_I] >= 0:
        raise EnergyEvaluationError(
            f"nonbonded pair ({int(st[0])},{int(st[1])}): coincident atoms")
    return float(en[3]), float(en[4])


def energy_coulomb(system: MolecularSystem, dtype=np.float64, backend=None) -> float:
    return _nb_energies(system, dtype, backend)[0]


def energy_vdw(system: MolecularSystem, dtype=np.float64, backend=None) -> float:
    return _nb_energies(system, dtype, backend)[1]


def energy_total(system: MolecularSystem, dtype=np.float64, backend=None) -> EnergyBreakdown:
    """All five terms in one device evaluation (ffmin/energy.py:133-141)."""
    en, st, _ = _eval(system, dtype, backend, False)
    raise_status(system, st, grad=False)
    return _breakdown(en)


def energy_and_gradient(system: MolecularSystem, dtype=np.float64, backend=None):
    """One fused sweep: (EnergyBreakdown, flattened analytic gradient)
    (ffmin/energy.py:144-174).  The gradient comes back in `dtype`."""
    en, st, g = _eval(system, dtype, backend, True)
    raise_status(system, st, grad=True)
    return _breakdown(en), g.reshape(-1).astype(np.dtype(dtype), copy=False)


def gradient_total(system: MolecularSystem, dtype=np.float64, backend=None):
    """Analytic gradient of the total energy, flattened to length 3n."""
    return energy_and_gradient(system, dtype, backend)[1]


def finite_difference_gradient(system: MolecularSystem, step=1e-5, dtype=np.float64,
                               backend=None):
    """Central-difference gradient of energy_total (ffmin/energy.py:182-198).
    The 6n displaced geometries are evaluated as device batches."""
    if not step > 0:
        raise ValueError(f"FD step must be > 0, got {step}")
    import torch

    from .engine import require_cuda
    require_cuda()
    _check_backend(backend)
    eng = engine_for(system.topology)
    n = system.natoms
    base = np.array(system.coords, dtype=np.float64).reshape(-1)
    g = np.zeros(base.size)
    chunk = max(1, min(3 * n, 4096 // max(1, n // 256 + 1)))
    for k0 in range(0, 3 * n, chunk):
        ks = np.arange(k0, min(3 * n, k0 + chunk))
        batch = np.repeat(base[None, :], 2 * len(ks), axis=0)
        batch[0::2][np.arange(len(ks)), ks] += step
        batch[1::2][np.arange(len(ks)), ks] -= step
        coords = torch.from_numpy(batch.reshape(-1, n, 3)).cuda(eng.device)
        en, st = eng.eval_batch(coords, precision_of(dtype))
        en = en.cpu().numpy()
        st = st.cpu().numpy()
        for r in range(len(ks)):
            for row in (2 * r, 2 * r + 1):
                raise_status(system, st[row], grad=False)
        tot = en.sum(axis=1)
        g[ks] = (tot[0::2] - tot[1::2]) / (2.0 * step)
    return g


def exact_delta_atom_move(system: MolecularSystem, atom: int, delta, dtype=np.float64,
                          backend=None) -> float:
    """Exact O(n) energy change for moving one atom (ffmin/energy.py:284-313),
    evaluated by the device delta kernel."""
    import torch

    _check_backend(backend)
    delta = np.asarray(delta, dtype=np.float64).reshape(3)
    newpos = system.coords[atom] + delta
    eng = engine_for(system.topology)
    dev = eng.device
    coords = torch.from_numpy(np.ascontiguousarray(system.coords)).to(dev)
    out, st = eng.atom_delta(coords, torch.tensor([atom], dtype=torch.int32, device=dev),
                             torch.from_numpy(newpos.reshape(1, 3)).to(dev))
    out = out.cpu().numpy()[0]
    st = st.cpu().numpy()[0]
    if st[0] >= 0:
        raise EnergyEvaluationError(f"nonbonded pair ({atom},{int(st[0])}): coincident atoms")
    if st[1] >= 0:
        raise EnergyEvaluationError(f"{_angle_name(system, int(st[1]))}: zero-length arm")
    if st[2] >= 0:
        raise EnergyEvaluationError(f"{_dihedral_name(system, int(st[2]))}: degenerate plane")
    # reference summation order: de + dea + ded + dec + dev
    return float(out[2]) + float(out[3]) + float(out[4]) + float(out[0]) + float(out[1])


# re-export the constant under its conventional name (ffmin/energy.py:316-317)
C_COULOMB = COULOMB_KJ_ANGSTROM
