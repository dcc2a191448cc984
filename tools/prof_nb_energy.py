"""Energy-only evaluations of the 100k globule in FP32 and FP64, for ncu
(development aid): python tools/prof_nb_energy.py [N]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_03358_b200 import _native as N  # noqa: E402
from paper_1810_03358_b200.engine import engine_for  # noqa: E402
from paper_1810_03358_b200.synth import make_globule_system  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
s = make_globule_system(n, seed=0)
eng = engine_for(s.topology)
c = torch.from_numpy(s.coords.copy()).cuda()
for prec in (N.FFM_F32, N.FFM_F64):
    for _ in range(2):
        eng.eval(c, prec)
torch.cuda.synchronize()
print("ok")
