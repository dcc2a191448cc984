"""Per-CTA phase times of the super-unit pair sweep (needs a library built
with -DFFM_UNIT_STAMPS: tools/build_lib_variant.sh stamps -DFFM_UNIT_STAMPS).
Stamps (thread 0): 0 start, 1 j-block staged, 2+ks end of sub-block ks
(ks < 8), 10+q end of warp 0's q-th tile of sub-block 0, 14 end.
usage: FFMIN_B200_LIB=... python tools/unit_phases.py N"""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1810_03358_b200 import _native as N
from paper_1810_03358_b200.engine import DeviceSystem
from paper_1810_03358_b200.synth import make_globule_system

n = int(sys.argv[1])
s = make_globule_system(n, seed=0)
eng = DeviceSystem(s.topology)
c = torch.from_numpy(s.coords.copy()).cuda()
g = torch.empty_like(c)
en, st = eng.new_outputs()
fl = N.FFM_ENERGY | N.FFM_GRAD | N.FFM_NO_GRAPH
for _ in range(3):
    eng.eval(c, N.FFM_F32, grad=g, energies=en, status=st, flags=fl)
units = eng.info["units"]
clk = torch.zeros((units, 16), dtype=torch.int64, device="cuda")
f = eng.lib.ffm_debug_unit_clock
f.argtypes = [C.c_void_p]
assert f(C.c_void_p(clk.data_ptr())) == 0
eng.eval(c, N.FFM_F32, grad=g, energies=en, status=st, flags=fl)
torch.cuda.synchronize()
t = clk.cpu().numpy().astype(np.float64)
assert f(None) == 0
t0 = t[:, 0].min()
T = (t[:, :15] - t0) / 1e3
T[t[:, :15] == 0] = np.nan
S = eng.info["S"]
nsub = min(8, S // 128)
njb = S // 32
print(f"n={n} S={S} units={units} sweep span {np.nanmax(T[:, 14]):.1f} us")
first = T[:, 0] < 0.5
for name, sel in (("first wave", first), ("later", ~first)):
    if not sel.any():
        continue
    X = T[sel]
    row = [np.nanmedian(X[:, 1] - X[:, 0])]
    prev = 1
    for ks in range(nsub):
        row.append(np.nanmedian(X[:, 2 + ks] - X[:, prev]))
        prev = 2 + ks
    row.append(np.nanmedian(X[:, 14] - X[:, prev]))
    tiles = [np.nanmedian(X[:, 10 + q] - (X[:, 9 + q] if q else X[:, 1])) for q in range(min(4, njb // 8))]
    print(f"  {name:10s} ({sel.sum()} CTAs): total {np.nanmedian(X[:, 14] - X[:, 0]):6.2f} us; "
          f"jload {row[0]:.2f}; sub-blocks " + " ".join(f"{v:.2f}" for v in row[1:-1]) +
          f"; tail {row[-1]:.2f}; sub0 tiles(w0) " + " ".join(f"{v:.2f}" for v in tiles))
# slot occupancy: CTA-time over (2 CTA slots per SM x SMs x span), and the
# end-time profile of the last CTAs (the tail)
sms = torch.cuda.get_device_properties(0).multi_processor_count
dur = T[:, 14] - T[:, 0]
span = np.nanmax(T[:, 14])
print(f"  slot occupancy {np.nansum(dur) / (2 * sms * span):.3f} "
      f"(CTA-us {np.nansum(dur):.0f} over {2 * sms} slots x {span:.1f} us)")
ends = np.sort(T[:, 14])
for q in (0.5, 0.75, 0.9, 0.97, 1.0):
    print(f"  {q:.2f} of CTAs done by {ends[min(len(ends) - 1, int(q * len(ends)))]:.1f} us")
starts = np.sort(T[:, 0])
print(f"  last CTA started at {starts[-1]:.1f} us")
