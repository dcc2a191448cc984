"""One small-system configuration evaluated repeatedly (ncu target).
usage: python tools/prof_small.py N PREC(0=f64,1=f32) GRAD(0/1) FUSE(0/1) [reps]"""
import sys

import torch

sys.path.insert(0, ".")
from paper_1810_03358_b200 import _native as N
from paper_1810_03358_b200.engine import DeviceSystem
from paper_1810_03358_b200.synth import make_globule_system

n, prec, grad, fuse = (int(a) for a in sys.argv[1:5])
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 20
s = make_globule_system(n, seed=0)
eng = DeviceSystem(s.topology)
c = torch.from_numpy(s.coords.copy()).cuda()
g = torch.empty_like(c)
en, st = eng.new_outputs()
fl = N.FFM_ENERGY | (N.FFM_GRAD if grad else 0) | (0 if fuse else N.FFM_NO_FUSE) | N.FFM_NO_GRAPH
for _ in range(reps):
    eng.eval(c, prec, grad=g if grad else None, energies=en, status=st, flags=fl)
torch.cuda.synchronize()
print("ok", en.cpu().numpy().sum())
