"""Batched multi-candidate energy evaluation (configs[3]) per plan variant.
usage: python tools/batch_sweep.py [natoms] [B]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1810_03358_b200 import _native as N
from paper_1810_03358_b200.engine import DeviceSystem
from paper_1810_03358_b200.synth import make_globule_system

n = int(sys.argv[1]) if len(sys.argv) > 1 else 5000
B = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
s = make_globule_system(n, seed=0)
rng = np.random.default_rng(0)
batch = torch.from_numpy(s.coords[None] + rng.normal(scale=0.02, size=(B,) + s.coords.shape)).cuda()
for name, env in (("auto", {}), ("S256", {"FFM_FORCE_S": "256", "FFM_FORCE_TILES": "0"}),
                  ("S512", {"FFM_FORCE_S": "512", "FFM_FORCE_TILES": "0"}),
                  ("S768", {"FFM_FORCE_S": "768", "FFM_FORCE_TILES": "0"}),
                  ("S1024", {"FFM_FORCE_S": "1024", "FFM_FORCE_TILES": "0"}),
                  ("tiles", {"FFM_FORCE_S": "256", "FFM_FORCE_TILES": "1"})):
    for k in ("FFM_FORCE_S", "FFM_FORCE_TILES"):
        os.environ.pop(k, None)
    os.environ.update(env)
    eng = DeviceSystem(s.topology)
    en, st = eng.new_outputs(B)
    for prec, tag in ((N.FFM_F32, "f32"), (N.FFM_F64, "f64")):
        for _ in range(2):
            eng.eval_batch(batch, prec, energies=en, status=st)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            eng.eval_batch(batch, prec, energies=en, status=st)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        print(f"{name:6s} S={eng.info['S']} {tag}: {ms:.3f} ms  {B*n*(n-1)/2/ms/1e9:.3f} Tpairs/s "
              f"E0={float(en[0].sum()):.6f}", flush=True)
    eng.close()
