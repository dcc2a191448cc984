"""How much of a small-system evaluation the bonded / scaled-pair term
blocks cost: whole evaluation (graph replay) with the system's terms and
with none (ffm_system_set_terms with zero terms; the 1-4 scaled pairs stay).
usage: python tools/time_terms_share.py [N ...]"""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_03358_b200 import _native as N  # noqa: E402
from paper_1810_03358_b200.engine import DeviceSystem  # noqa: E402
from paper_1810_03358_b200.synth import make_globule_system  # noqa: E402


def eval_us(eng, c, g, prec, reps=50):
    en, st = eng.new_outputs()
    fl = N.FFM_ENERGY | N.FFM_GRAD
    for _ in range(5):
        eng.eval(c, prec, grad=g, energies=en, status=st, flags=fl)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        eng.eval(c, prec, grad=g, energies=en, status=st, flags=fl)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


for n in [int(a) for a in sys.argv[1:]] or [500, 1000, 3000]:
    s = make_globule_system(n, seed=0)
    c = torch.from_numpy(s.coords.copy()).cuda()
    g = torch.empty_like(c)
    for prec, tag in ((N.FFM_F32, "f32"), (N.FFM_F64, "f64")):
        eng = DeviceSystem(s.topology)
        full = eval_us(eng, c, g, prec)
        eng.lib.ffm_system_set_terms.argtypes = [C.c_void_p, C.c_int64] + [C.c_void_p] * 3 + \
            [C.c_int64] + [C.c_void_p] * 3 + [C.c_int64] + [C.c_void_p] * 2
        N.check(eng.lib.ffm_system_set_terms(eng.handle, 0, None, None, None, 0, None, None,
                                             None, 0, None, None), "set_terms")
        bare = eval_us(eng, c, g, prec)
        print(f"n={n:5d} {tag}: with terms {full:6.1f} us, without bonded terms {bare:6.1f} us",
              flush=True)
        eng.close()
