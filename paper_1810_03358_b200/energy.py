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
    eng = engine_for(system.topology, precision=dtype)
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
    _check_backend(backend)
    out, st = atom_deltas(system, [atom], np.asarray(delta, np.float64).reshape(1, 3))
    _raise_delta(system, atom, st[0])
    o = out[0]
    # reference summation order: de + dea + ded + dec + dev
    return float(o[2]) + float(o[3]) + float(o[4]) + float(o[0]) + float(o[1])


@dataclass(frozen=True)
class NeighborList:
    """Symmetric within-cutoff adjacency (ffmin/energy.py:44-49)."""

    cutoff: float
    neighbors: tuple


@dataclass(frozen=True)
class FarFieldLinearization:
    """First-order model of one atom's far-field Coulomb sum
    (ffmin/energy.py:52-68)."""

    atom: int
    cutoff: float
    ref_pos: np.ndarray
    e_far0: float
    coef: np.ndarray
    near_idx: np.ndarray


def _dev_coords(system):
    import torch

    eng = engine_for(system.topology)
    return eng, torch.from_numpy(np.array(system.coords, dtype=np.float64)).to(eng.device)


def build_neighbor_list(system: MolecularSystem, cutoff: float) -> NeighborList:
    """Within-cutoff adjacency by a brute-force pair scan on the device
    (ffmin/energy.py:201-212)."""
    if not cutoff > 0:
        raise ValueError(f"cutoff must be > 0, got {cutoff}")
    import torch

    _, c = _dev_coords(system)
    n = system.natoms
    out = []
    for i0 in range(0, n, 4096):
        d = torch.cdist(c[i0:i0 + 4096], c)
        d[torch.arange(d.shape[0], device=c.device), torch.arange(i0, i0 + d.shape[0],
                                                               device=c.device)] = float("inf")
        rows = (d <= cutoff).cpu().numpy()
        out.extend(np.nonzero(r)[0].astype(np.int64) for r in rows)
    return NeighborList(cutoff=float(cutoff), neighbors=tuple(out))


def linearize_farfield_coulomb(system: MolecularSystem, atom: int,
                               cutoff: float) -> FarFieldLinearization:
    """Split one atom's Coulomb sum at `cutoff` and linearise the far part
    (ffmin/energy.py:215-240), one device kernel."""
    if not 0 <= atom < system.natoms:
        raise ValueError(f"atom index {atom} out of range for {system.natoms} atoms")
    if not cutoff > 0:
        raise ValueError(f"cutoff must be > 0, got {cutoff}")
    eng, c = _dev_coords(system)
    e, m, b = eng.farfield(c, atom, cutoff)
    if int(b.item()) >= 0:
        raise EnergyEvaluationError(f"nonbonded pair ({atom},{int(b.item())}): coincident atoms")
    e = e.cpu().numpy()
    return FarFieldLinearization(atom=int(atom), cutoff=float(cutoff),
                                 ref_pos=system.coords[atom].copy(), e_far0=float(e[0]),
                                 coef=e[1:4].copy(),
                                 near_idx=np.nonzero(m.cpu().numpy())[0].astype(np.int64))


def delta_energy_atom_move(system: MolecularSystem, lin: FarFieldLinearization, delta) -> float:
    """Energy change of moving lin.atom by delta with the far field
    linearised (ffmin/energy.py:243-281); valid while the system still has
    the coordinates lin was built from."""
    if system.topology.cutoff is not None:
        raise ValueError("incremental delta requires a system nonbonded cutoff of none")
    out, st = atom_deltas(system, [lin.atom], np.asarray(delta, np.float64).reshape(1, 3),
                          lin_cutoff=lin.cutoff)
    _raise_delta(system, lin.atom, st[0])
    o = out[0]
    return float(o[2]) + float(o[3]) + float(o[4]) + float(o[0]) + float(o[1]) + float(o[5])


def atom_deltas(system: MolecularSystem, atoms, deltas, lin_cutoff=None, coords_d=None):
    """Batched single-atom move deltas on the device: rows (k, 5) exact or
    (k, 6) linearised, plus status rows (k, 3), as NumPy."""
    import torch

    eng = engine_for(system.topology)
    if coords_d is None:
        coords_d = torch.from_numpy(np.array(system.coords, dtype=np.float64)).to(eng.device)
    atoms = np.asarray(atoms, dtype=np.int64).reshape(-1)
    newpos = system.coords[atoms] + np.asarray(deltas, np.float64).reshape(-1, 3)
    out, st = eng.atom_delta(coords_d, torch.from_numpy(atoms.astype(np.int32)).to(eng.device),
                             torch.from_numpy(newpos).to(eng.device), lin_cutoff=lin_cutoff)
    return out.cpu().numpy(), st.cpu().numpy()


def _raise_delta(system, atom, st):
    if st[0] >= 0:
        raise EnergyEvaluationError(f"nonbonded pair ({atom},{int(st[0])}): coincident atoms")
    if st[1] >= 0:
        raise EnergyEvaluationError(f"{_angle_name(system, int(st[1]))}: zero-length arm")
    if st[2] >= 0:
        raise EnergyEvaluationError(f"{_dihedral_name(system, int(st[2]))}: degenerate plane")


# re-export the constant under its conventional name (ffmin/energy.py:316-317)
C_COULOMB = COULOMB_KJ_ANGSTROM
