"""Per-rank compute time of a row-sharded evaluation, measured one rank at a
time on one GPU (rank 0's share of W; no collective, no waiting between
ranks): the sweep each GPU of a W-GPU job runs.  Tuning aid for the
super-unit re-plan of ffm_system_set_shard.
usage: python tools/shard_time.py [natoms]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1810_03358_b200 import _native as N
from paper_1810_03358_b200.engine import DeviceSystem
from paper_1810_03358_b200.synth import make_globule_system

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
s = make_globule_system(n, seed=0)
c = torch.from_numpy(s.coords.copy()).cuda()
g = torch.empty_like(c)
t1 = None
for W in (1, 2, 4, 8):
    eng = DeviceSystem(s.topology)
    worst = 0.0
    for rank in sorted({0, W - 1}):
        N.check(eng.lib.ffm_system_set_shard(eng.handle, rank, W), "set_shard")
        info = np.zeros(8, np.int64)
        N.check(eng.lib.ffm_system_info(eng.handle, info.ctypes.data), "info")
        en, st = eng.new_outputs()
        for _ in range(3):
            eng.eval(c, N.FFM_F32, grad=g, energies=en, status=st)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            eng.eval(c, N.FFM_F32, grad=g, energies=en, status=st)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        worst = max(worst, ms)
        print(f"W={W} rank {rank}: S={info[2]} units={info[4]} ({info[4] // W}/rank) {ms:.3f} ms",
              flush=True)
    t1 = worst if W == 1 else t1
    print(f"W={W}: slowest rank {worst:.3f} ms -> compute-only efficiency {t1 / (W * worst):.3f}",
          flush=True)
    eng.close()
