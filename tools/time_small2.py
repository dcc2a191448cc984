"""Breakdown of a small-system evaluation by skipping parts (flags)."""
import sys
import numpy as np, torch
sys.path.insert(0, '.')
from paper_1810_03358_b200 import _native as N
from paper_1810_03358_b200.synth import make_globule_system
from paper_1810_03358_b200.engine import DeviceSystem
n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
s = make_globule_system(n, seed=0)
eng = DeviceSystem(s.topology)
c = torch.from_numpy(s.coords.copy()).cuda()
g = torch.empty_like(c)
en, st = eng.new_outputs()
for prec in (0, 1):
    row = []
    for name, fl, grad in (("E", N.FFM_ENERGY, None), ("E-noNB", N.FFM_ENERGY | N.FFM_NO_NB, None),
                           ("E-noT", N.FFM_ENERGY | N.FFM_NO_TERMS, None),
                           ("E-none", N.FFM_ENERGY | N.FFM_NO_TERMS | N.FFM_NO_NB, None),
                           ("G", N.FFM_ENERGY | N.FFM_GRAD, g), ("G-noNB", N.FFM_ENERGY | N.FFM_GRAD | N.FFM_NO_NB, g),
                           ("G-noT", N.FFM_ENERGY | N.FFM_GRAD | N.FFM_NO_TERMS, g)):
        for _ in range(20):
            eng.eval(c, prec, grad=grad, energies=en, status=st, flags=fl)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(300):
            eng.eval(c, prec, grad=grad, energies=en, status=st, flags=fl)
        e1.record()
        torch.cuda.synchronize()
        row.append(f"{name} {e0.elapsed_time(e1) / 300 * 1e3:5.1f}")
    print(n, "f64" if prec == 0 else "f32", "  ".join(row))
