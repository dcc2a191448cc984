"""Mid-size systems: pair-sweep time (FFM_TIME_NB) and whole evaluation
(graph replay) per N and per plan variant (super-unit edge S, tile mode).
Tuning aid.  usage: python tools/mid_sweep.py [N ...]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1810_03358_b200 import _native as N
from paper_1810_03358_b200.engine import DeviceSystem
from paper_1810_03358_b200.synth import make_globule_system

sizes = [int(a) for a in sys.argv[1:]] or [3000, 5000, 10000, 20000, 30000]
only = os.environ.get("VARIANTS")
PREC = N.FFM_F64 if os.environ.get("PREC") == "f64" else N.FFM_F32
variants = [("auto", {}), ("S128", {"FFM_FORCE_S": "128", "FFM_FORCE_TILES": "0"}), ("S256", {"FFM_FORCE_S": "256", "FFM_FORCE_TILES": "0"}),
            ("tiles256", {"FFM_FORCE_S": "256", "FFM_FORCE_TILES": "1"}),
            ("S512", {"FFM_FORCE_S": "512", "FFM_FORCE_TILES": "0"}),
            ("tiles", {"FFM_FORCE_TILES": "1"})]
for n in sizes:
    s = make_globule_system(n, seed=0)
    c = torch.from_numpy(s.coords.copy()).cuda()
    g = torch.empty_like(c)
    for name, env in variants:
        if only and name not in only.split(","):
            continue
        for k in ("FFM_FORCE_S", "FFM_FORCE_TILES"):
            os.environ.pop(k, None)
        os.environ.update(env)
        eng = DeviceSystem(s.topology)
        en, st = eng.new_outputs()
        fl = N.FFM_ENERGY | (0 if os.environ.get("GRAD") == "0" else N.FFM_GRAD)
        nb = []
        for k in range(8):
            eng.eval(c, PREC, grad=g, energies=en, status=st, flags=fl | N.FFM_TIME_NB)
            v = np.zeros(1, np.float32)
            N.check(eng.lib.ffm_system_nb_ms(eng.handle, v.ctypes.data), "nb_ms")
            if k >= 3:
                nb.append(float(v[0]))
        for _ in range(3):
            eng.eval(c, PREC, grad=g, energies=en, status=st, flags=fl)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 50
        e0.record()
        for _ in range(reps):
            eng.eval(c, PREC, grad=g, energies=en, status=st, flags=fl)
        e1.record()
        torch.cuda.synchronize()
        tot = e0.elapsed_time(e1) / reps
        pairs = n * (n - 1) / 2
        print(f"n={n:6d} {name:6s} S={eng.info['S']:4d} units={eng.info['units']:6d} "
              f"nb={np.median(nb)*1e3:8.1f} us  eval={tot*1e3:8.1f} us  "
              f"{pairs/tot/1e9:7.1f} Gpairs/s  E={float(en.sum()):.6f}", flush=True)
        eng.close()
