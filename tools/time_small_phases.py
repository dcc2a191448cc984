"""Phase times of the fused small-system evaluation (globaltimer stamps per
CTA): P0 pack, P1 terms + tiles, sync, P2 gather/reduce, tail.
usage: python tools/time_small_phases.py N PREC GRAD"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1810_03358_b200 import _native as N
from paper_1810_03358_b200.engine import DeviceSystem
from paper_1810_03358_b200.synth import make_globule_system

n, prec, grad = (int(a) for a in sys.argv[1:4])
s = make_globule_system(n, seed=0)
eng = DeviceSystem(s.topology)
c = torch.from_numpy(s.coords.copy()).cuda()
g = torch.empty_like(c)
en, st = eng.new_outputs()
fl = N.FFM_ENERGY | (N.FFM_GRAD if grad else 0) | N.FFM_NO_GRAPH
eng.eval(c, prec, grad=g if grad else None, energies=en, status=st, flags=fl)
torch.cuda.synchronize()
grids = np.zeros(4, np.int32)
clk = torch.zeros((8192, 8), dtype=torch.int64, device="cuda")
N.check(eng.lib.ffm_debug_phase_clock(eng.handle, N.ptr(clk), grids.ctypes.data), "clk")
G = int(grids[2 * prec + grad])
for rep in range(5):
    eng.eval(c, prec, grad=g if grad else None, energies=en, status=st, flags=fl)
torch.cuda.synchronize()
t = clk[:G].cpu().numpy().astype(np.float64)
t -= t[:, 0].min()
t /= 1e3
print(f"n={n} prec={prec} grad={grad} grid={G}")
names = ["start", "after P0 sync", "P1 done", "after P1 sync", "P2 done", "end"]
for k, nm in enumerate(names):
    print(f"  {nm:14s} min {t[:, k].min():7.2f} us  max {t[:, k].max():7.2f} us")
d = t[:, 2] - t[:, 1]
print(f"  P1 work per CTA: max {d.max():.2f} us at CTA {int(d.argmax())}, median {np.median(d):.2f}")
d = t[:, 4] - t[:, 3]
print(f"  P2 work per CTA: max {d.max():.2f} us at CTA {int(d.argmax())}, median {np.median(d):.2f}")
N.check(eng.lib.ffm_debug_phase_clock(eng.handle, None, grids.ctypes.data), "clk")
