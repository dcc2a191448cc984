"""Wall time per L-BFGS iteration of a golden system (graph-resident path).
usage: python tools/lbfgs_time.py [conv200] [iters] [--synth N]"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1810_03358_b200.model import MolecularSystem
from paper_1810_03358_b200.oracle import MolecularOracle
from paper_1810_03358_b200.optimizers import StopCriteria, lbfgs, make_linesearch
from paper_1810_03358_b200.synth import make_globule_system

name = sys.argv[1] if len(sys.argv) > 1 else "conv200"
it = int(sys.argv[2]) if len(sys.argv) > 2 else 200
if name.startswith("globule"):
    s = make_globule_system(int(name[7:]), seed=1)
else:
    G = np.load("tests/golden/golden_v1.npz")
    cut = float(G[f"{name}/cutoff"])
    s = MolecularSystem.from_arrays(
        G[f"{name}/q"], G[f"{name}/sigma"], G[f"{name}/epsilon"], G[f"{name}/coords"],
        G[f"{name}/bond_idx"], G[f"{name}/bond_K"], G[f"{name}/bond_r0"],
        G[f"{name}/ang_idx"], G[f"{name}/ang_K"], G[f"{name}/ang_t0"], G[f"{name}/dih_idx"],
        G[f"{name}/dih_V"], excluded=G[f"{name}/excluded"], scaled14=G[f"{name}/scaled14"],
        s14=float(G[f"{name}/s14"]), cutoff=None if cut <= 0 else cut)
for rep in range(2):
    o = MolecularOracle(s)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = lbfgs(o, s.coords.ravel(), m=5, linesearch=make_linesearch("par"),
                stop=StopCriteria(max_iterations=it, gradient_norm_rtol=0.0))
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"{name} n={s.natoms}: {res.iterations} it in {dt*1e3:.1f} ms = "
          f"{dt/res.iterations*1e3:.3f} ms/it; value calls {o.value_calls} "
          f"({o.value_calls/res.iterations:.2f}/it) grad calls {o.grad_calls}; f={res.f:.6f}")
