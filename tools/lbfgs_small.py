"""Short graph-resident L-BFGS run on a golden system (profiling aid)."""
import sys
import numpy as np
sys.path.insert(0, '.')
from paper_1810_03358_b200.model import MolecularSystem
from paper_1810_03358_b200.oracle import MolecularOracle
from paper_1810_03358_b200.optimizers import StopCriteria, lbfgs, make_linesearch
G = np.load("tests/golden/golden_v1.npz")
name = sys.argv[1] if len(sys.argv) > 1 else "conv200"
it = int(sys.argv[2]) if len(sys.argv) > 2 else 20
cut = float(G[f"{name}/cutoff"])
s = MolecularSystem.from_arrays(
    G[f"{name}/q"], G[f"{name}/sigma"], G[f"{name}/epsilon"], G[f"{name}/coords"],
    G[f"{name}/bond_idx"], G[f"{name}/bond_K"], G[f"{name}/bond_r0"],
    G[f"{name}/ang_idx"], G[f"{name}/ang_K"], G[f"{name}/ang_t0"], G[f"{name}/dih_idx"],
    G[f"{name}/dih_V"], excluded=G[f"{name}/excluded"], scaled14=G[f"{name}/scaled14"],
    s14=float(G[f"{name}/s14"]), cutoff=None if cut <= 0 else cut)
res = lbfgs(MolecularOracle(s), s.coords.ravel(), m=5, linesearch=make_linesearch("par"),
            stop=StopCriteria(max_iterations=it, gradient_norm_rtol=0.0))
print(res.iterations, res.f)
