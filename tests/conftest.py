import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden" / "golden_v1.npz"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden():
    return np.load(GOLDEN, allow_pickle=False)


def golden_arrays(G, name):
    """(kwargs for MolecularSystem.from_arrays, coords) of a golden case."""
    cut = float(G[f"{name}/cutoff"])
    kw = dict(
        q=G[f"{name}/q"], sigma=G[f"{name}/sigma"], epsilon=G[f"{name}/epsilon"],
        bond_idx=G[f"{name}/bond_idx"], bond_K=G[f"{name}/bond_K"],
        bond_r0=G[f"{name}/bond_r0"], ang_idx=G[f"{name}/ang_idx"],
        ang_K=G[f"{name}/ang_K"], ang_t0=G[f"{name}/ang_t0"], dih_idx=G[f"{name}/dih_idx"],
        dih_V=G[f"{name}/dih_V"], excluded=G[f"{name}/excluded"],
        scaled14=G[f"{name}/scaled14"], s14=float(G[f"{name}/s14"]),
        cutoff=None if cut <= 0 else cut)
    return kw, G[f"{name}/coords"]


def golden_system(G, name):
    from paper_1810_03358_b200.model import MolecularSystem

    kw, coords = golden_arrays(G, name)
    return MolecularSystem.from_arrays(coords=coords, **kw)


def oracle_arrays(G, name):
    import oracle as O

    kw, coords = golden_arrays(G, name)
    ex, sc = kw["excluded"], kw["scaled14"]
    si = np.concatenate([ex[:, 0], sc[:, 0]])
    sj = np.concatenate([ex[:, 1], sc[:, 1]])
    ss = np.concatenate([np.zeros(len(ex)), np.full(len(sc), kw["s14"])])
    A = O.Arrays(kw["q"], kw["sigma"], kw["epsilon"], si, sj, ss, kw["cutoff"], kw["bond_idx"],
                 kw["bond_K"], kw["bond_r0"], kw["ang_idx"], kw["ang_K"], kw["ang_t0"],
                 kw["dih_idx"], kw["dih_V"])
    return A, coords


def has_cuda():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False
