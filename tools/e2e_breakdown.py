"""Where the host-API (e2e) time of one 100k-atom FP32 energy+gradient goes.
usage: python tools/e2e_breakdown.py [natoms]"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1810_03358_b200 import _native as N
from paper_1810_03358_b200.energy import energy_and_gradient
from paper_1810_03358_b200.engine import engine_for
from paper_1810_03358_b200.synth import make_globule_system

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
s = make_globule_system(n, seed=0)
eng = engine_for(s.topology)
dev = torch.device("cuda", 0)


def wall(f, reps=10, warm=3):
    for _ in range(warm):
        f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        f()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return 1e3 * float(np.median(ts))


c_dev = torch.from_numpy(s.coords.copy()).to(dev)
g_dev = torch.empty_like(c_dev)
en, st = eng.new_outputs()
print(f"device eval            {wall(lambda: eng.eval(c_dev, N.FFM_F32, grad=g_dev, energies=en, status=st)):.3f} ms")
host = np.ascontiguousarray(s.coords)
pinned = torch.empty((n, 3), dtype=torch.float64).pin_memory()
pinned.numpy()[:] = host
print(f"H2D pageable 2.4MB     {wall(lambda: c_dev.copy_(torch.from_numpy(host))):.3f} ms")
print(f"H2D pinned             {wall(lambda: c_dev.copy_(pinned, non_blocking=True)):.3f} ms")
gh = np.empty((n, 3))
print(f"D2H pageable 2.4MB     {wall(lambda: torch.from_numpy(gh).copy_(g_dev)):.3f} ms")
print(f"D2H pinned             {wall(lambda: pinned.copy_(g_dev, non_blocking=True)):.3f} ms")
g32 = torch.empty((n, 3), dtype=torch.float32, device=dev)
gh32 = np.empty((n, 3), np.float32)
print(f"D2H pageable 1.2MB f32 {wall(lambda: torch.from_numpy(gh32).copy_(g32)):.3f} ms")
print(f"eval_host pageable     {wall(lambda: eng.eval_host(host, N.FFM_F32, grad=True)):.3f} ms")
print(f"eval_host pinned in    {wall(lambda: eng.eval_host(pinned.numpy(), N.FFM_F32, grad=True)):.3f} ms")
print(f"with_coords            {wall(lambda: s.with_coords(host)):.3f} ms")
print(f"energy_and_gradient    {wall(lambda: energy_and_gradient(s.with_coords(pinned.numpy()), np.float32)):.3f} ms")
