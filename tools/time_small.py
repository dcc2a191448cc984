"""Device time per evaluation of small systems: fused one-launch path vs the
kernel chain (FFM_NO_FUSE), graph replay, back to back.
usage: python tools/time_small.py [n1 n2 ...]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1810_03358_b200 import _native as N
from paper_1810_03358_b200.engine import DeviceSystem
from paper_1810_03358_b200.synth import make_globule_system

sizes = [int(a) for a in sys.argv[1:]] or [200, 500, 1000, 2000, 4000]
for n in sizes:
    s = make_globule_system(n, seed=0)
    eng = DeviceSystem(s.topology)
    c = torch.from_numpy(s.coords.copy()).cuda()
    g = torch.empty_like(c)
    en, st = eng.new_outputs()
    row = []
    for prec, tag in ((N.FFM_F64, "f64"), (N.FFM_F32, "f32")):
        for grad in (False, True):
            for extra, name in ((0, "fused"), (N.FFM_NO_FUSE, "chain")):
                fl = N.FFM_ENERGY | (N.FFM_GRAD if grad else 0) | extra
                for _ in range(5):
                    eng.eval(c, prec, grad=g if grad else None, energies=en, status=st, flags=fl)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                reps = 200
                e0.record()
                for _ in range(reps):
                    eng.eval(c, prec, grad=g if grad else None, energies=en, status=st, flags=fl)
                e1.record()
                torch.cuda.synchronize()
                row.append(f"{tag}{'+g' if grad else ''} {name} {e0.elapsed_time(e1) / reps * 1e3:6.1f}us")
    print(f"n={n:5d} ntiles? " + " | ".join(row), flush=True)
    eng.close()
