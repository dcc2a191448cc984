"""Median device time of the pair sweep (FFM_TIME_NB) -- tuning aid.
usage: FFMIN_B200_LIB=... python tools/time_nb.py N PREC(0=f64,1=f32) GRAD(0/1)"""
import sys
import numpy as np, torch
sys.path.insert(0, '.')
from paper_1810_03358_b200 import _native as N
from paper_1810_03358_b200.synth import make_globule_system
from paper_1810_03358_b200.engine import DeviceSystem
n, prec, grad = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
s = make_globule_system(n, seed=0)
eng = DeviceSystem(s.topology)
c = torch.from_numpy(s.coords.copy()).cuda()
g = torch.empty_like(c) if grad else None
en, st = eng.new_outputs()
fl = N.FFM_ENERGY | (N.FFM_GRAD if grad else 0) | N.FFM_TIME_NB
ms = []
for k in range(13):
    eng.eval(c, prec, grad=g, energies=en, status=st, flags=fl)
    v = np.zeros(1, np.float32)
    N.check(eng.lib.ffm_system_nb_ms(eng.handle, v.ctypes.data), "nb_ms")
    if k >= 3:
        ms.append(float(v[0]))
e = en.cpu().numpy()
print(f"{np.median(ms):.4f} ms  {n*(n-1)/2/np.median(ms)/1e9:.4f} Tpairs/s  E={e.sum():.6f}")
