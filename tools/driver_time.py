"""Wall time per iteration of the graph-resident drivers on a synthetic
globule (the second run of each reuses the captured graph).
usage: python tools/driver_time.py [natoms] [iters]"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1810_03358_b200.oracle import MolecularOracle
from paper_1810_03358_b200.optimizers import (StopCriteria, cg, fgm, lbfgs, make_linesearch,
                                              steepest_descent)
from paper_1810_03358_b200.synth import make_globule_system

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 100
s = make_globule_system(n, seed=1)
runs = {"sd": lambda o: steepest_descent(o, s.coords.ravel(), make_linesearch("par"), stop),
        "fgm": lambda o: fgm(o, s.coords.ravel(), make_linesearch("par"), stop),
        "cg": lambda o: cg(o, s.coords.ravel(), "prp+", make_linesearch("par"), stop),
        "lbfgs": lambda o: lbfgs(o, s.coords.ravel(), m=5, linesearch=make_linesearch("par"),
                                 stop=stop)}
stop = StopCriteria(max_iterations=iters, gradient_norm_rtol=1e-6)
for name, run in runs.items():
    o = MolecularOracle(s)
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = run(o)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        print(f"{name:6s} rep {rep}: {res.iterations} it {dt*1e3:8.1f} ms = "
              f"{dt/max(1, res.iterations)*1e3:.3f} ms/it  f={res.f:.6f}", flush=True)
