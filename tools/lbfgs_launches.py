"""A bounded graph-resident L-BFGS run on a globule, for an ncu launch list
(device time per iteration vs wall time; tuning aid).
usage: python tools/lbfgs_launches.py N PREC(0=f64,1=f32) ITERS"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1810_03358_b200.oracle import MolecularOracle
from paper_1810_03358_b200.optimizers import StopCriteria, lbfgs, make_linesearch
from paper_1810_03358_b200.synth import make_globule_system

n, prec, it = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
s = make_globule_system(n, seed=1)
dt = np.float32 if prec else np.float64
o = MolecularOracle(s, dt)
lbfgs(o, s.coords.ravel(), m=5, linesearch=make_linesearch("par"),
      stop=StopCriteria(max_iterations=2, gradient_norm_rtol=1e-6))  # capture the graph
o.value_calls = o.grad_calls = 0
torch.cuda.synchronize()
t0 = time.perf_counter()
res = lbfgs(o, s.coords.ravel(), m=5, linesearch=make_linesearch("par"),
            stop=StopCriteria(max_iterations=it, gradient_norm_rtol=1e-6))
torch.cuda.synchronize()
w = time.perf_counter() - t0
print(f"n={n} {res.iterations} it {w * 1e3 / res.iterations:.3f} ms/it value calls "
      f"{o.value_calls} grad calls {o.grad_calls}")
