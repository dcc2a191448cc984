"""e2e cost parts of MolecularOracle.value_and_gradient at 100k (FP32).
usage: python tools/e2e_parts.py"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1810_03358_b200 import _native as N
from paper_1810_03358_b200.oracle import MolecularOracle
from paper_1810_03358_b200.synth import make_globule_system

s = make_globule_system(100000, seed=0)
o = MolecularOracle(s, np.float32)
pinned = torch.empty(3 * s.natoms, dtype=torch.float64).pin_memory()
pinned.numpy()[:] = s.coords.ravel()
host = pinned.numpy()
xd = torch.from_numpy(s.coords.ravel().copy()).cuda()
en, st = o.engine.new_outputs()
g = torch.empty((s.natoms, 3), dtype=torch.float64, device="cuda")


def wall(f, reps=20):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        f()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return 1e3 * float(np.median(ts))


print(f"engine.eval + sync          {wall(lambda: o.engine.eval(o._x, N.FFM_F32, grad=g, energies=en, status=st)):.3f} ms")
print(f"oracle v&g, device vector   {wall(lambda: o.value_and_gradient(xd)):.3f} ms")
print(f"oracle v&g, pinned host     {wall(lambda: o.value_and_gradient(host)):.3f} ms")
print(f"oracle v&g, pageable host   {wall(lambda: o.value_and_gradient(s.coords.ravel().copy())):.3f} ms")
