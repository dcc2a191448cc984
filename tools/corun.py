"""Co-running experiment: the FP32 and the FP64 energy+gradient sweeps of the
same 100k-atom system on two streams at once (does the idle FP64 pipe add
throughput next to the FP32 sweep?).  Tuning aid.
usage: [FFMIN_B200_LIB=...] python tools/corun.py [N]"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_03358_b200 import _native as N  # noqa: E402
from paper_1810_03358_b200.engine import DeviceSystem  # noqa: E402
from paper_1810_03358_b200.synth import make_globule_system  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
s = make_globule_system(n, seed=0)
e32, e64 = DeviceSystem(s.topology), DeviceSystem(s.topology)
c = torch.from_numpy(s.coords.copy()).cuda()
g32, g64 = torch.empty_like(c), torch.empty_like(c)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
o32, o64 = e32.new_outputs(), e64.new_outputs()


def run(which, reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        if "32" in which:
            e32.eval(c, N.FFM_F32, grad=g32, energies=o32[0], status=o32[1], stream=s1)
        if "64" in which:
            e64.eval(c, N.FFM_F64, grad=g64, energies=o64[0], status=o64[1], stream=s2)
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


for w in ("32", "64", "32+64"):
    run(w, 2)
pairs = n * (n - 1) / 2
for w in ("32", "64", "32+64", "32", "64", "32+64"):
    ms = run(w, 5)
    k = 2 if w == "32+64" else 1
    print(f"{w:6s} {ms:8.3f} ms per round  {k * pairs / ms / 1e9:8.3f} Tpairs/s", flush=True)
