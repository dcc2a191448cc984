"""paper_1810_03358_b200: B200-native force-field energy minimisation.

A drop-in for the hot path of the ffmin reference (arXiv 1810.03358): the
O(N^2) Lennard-Jones + Coulomb energy and analytic gradient behind every
minimiser, evaluated by hand-written sm_100a CUDA kernels (csrc/) through a
C ABI (include/ffmin_b200.h), with the reference's model / energy / oracle /
optimiser API on top.  There is no CPU execution path.
"""

__version__ = "0.1.0"

from .constants import COULOMB_KJ_ANGSTROM
from .model import (
    AngleTerm,
    AtomSpec,
    BondTerm,
    DihedralTerm,
    ModelError,
    MolecularSystem,
    NonbondedPolicy,
    Topology,
    build_default_exclusions,
)
from .synth import make_chain_system, make_globule_system, perturbed_copy

_LAZY = {
    # energy layer (imports torch + the native engine on first use)
    "EnergyBreakdown": "energy", "EnergyEvaluationError": "energy",
    "energy_total": "energy", "energy_and_gradient": "energy", "gradient_total": "energy",
    "energy_stretch": "energy", "energy_bend": "energy", "energy_torsion": "energy",
    "energy_coulomb": "energy", "energy_vdw": "energy",
    "finite_difference_gradient": "energy", "exact_delta_atom_move": "energy",
    "C_COULOMB": "energy",
    "DeviceSystem": "engine", "engine_for": "engine",
    "get_backend": "kernels", "KernelBackend": "kernels", "CUDA_BACKEND": "kernels",
    "ObjectiveOracle": "oracle", "FunctionOracle": "oracle", "MolecularOracle": "oracle",
    "DeviceMolecularOracle": "oracle",
}


def __getattr__(name):
    mod = _LAZY.get(name)
    if mod is None:
        raise AttributeError(f"module {__name__!r} has no attribute {name!r}")
    import importlib

    return getattr(importlib.import_module(f".{mod}", __name__), name)
