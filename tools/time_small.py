"""Per-evaluation device time of small systems, graph replays back to back
(launch latency hidden) vs one-at-a-time with a sync (latency exposed)."""
import sys, time
import numpy as np, torch
sys.path.insert(0, '.')
from paper_1810_03358_b200 import _native as N
from paper_1810_03358_b200.synth import make_globule_system
from paper_1810_03358_b200.engine import DeviceSystem
for n in (200, 500, 2000, 10000):
    s = make_globule_system(n, seed=0)
    eng = DeviceSystem(s.topology)
    c = torch.from_numpy(s.coords.copy()).cuda()
    g = torch.empty_like(c)
    en, st = eng.new_outputs()
    out = [str(n), f"S={eng.info['S']}"]
    for prec in (0, 1):
        for grad in (None, g):
            for _ in range(20):
                eng.eval(c, prec, grad=grad, energies=en, status=st)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(200):
                eng.eval(c, prec, grad=grad, energies=en, status=st)
            e1.record()
            torch.cuda.synchronize()
            pipe = e0.elapsed_time(e1) / 200 * 1e3
            t0 = time.perf_counter()
            for _ in range(200):
                eng.eval(c, prec, grad=grad, energies=en, status=st)
                torch.cuda.synchronize()
            lat = (time.perf_counter() - t0) / 200 * 1e6
            out.append(f"{'f64' if prec == 0 else 'f32'}{'G' if grad is not None else 'E'} pipe {pipe:6.1f}us sync {lat:6.1f}us")
    print("  ".join(out))
