import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_1810_03358_b200 import _native as N
from paper_1810_03358_b200.synth import make_globule_system
from paper_1810_03358_b200.engine import DeviceSystem
for cut in (None, 12.0, 7.0):
    s = make_globule_system(100000, seed=0, cutoff=cut)
    eng = DeviceSystem(s.topology)
    c = torch.from_numpy(s.coords.copy()).cuda(); g = torch.empty_like(c)
    en, st = eng.new_outputs()
    for _ in range(3): eng.eval(c, 1, grad=g, energies=en, status=st)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): eng.eval(c, 1, grad=g, energies=en, status=st)
    e1.record(); torch.cuda.synchronize()
    print(f"cutoff={cut}: {e0.elapsed_time(e1)/10:.3f} ms per energy+grad (100k atoms, f32)  E={en.sum().item():.4f}")
