"""Host-side overhead of the device path at small N (development aid)."""
import sys, time
import numpy as np, torch
sys.path.insert(0, '.')
from paper_1810_03358_b200.synth import make_chain_system
from paper_1810_03358_b200.oracle import MolecularOracle
from paper_1810_03358_b200.vecops import DeviceOps
from paper_1810_03358_b200 import _native as N

s = make_chain_system(500, seed=0)
o = MolecularOracle(s)
x = o.initial_point()
ops = DeviceOps()
def t(fn, k=200):
    for _ in range(10): fn()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(k): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / k * 1e6
print(f"oracle.value        {t(lambda: o.value(x)):8.1f} us")
print(f"oracle.val_and_grad {t(lambda: o.value_and_gradient(x)):8.1f} us")
en, st = o.engine.new_outputs()
print(f"engine.eval (async) {t(lambda: o.engine.eval(x.view(-1,3), 0, energies=en, status=st)):8.1f} us")
print(f"engine.eval+sync    {t(lambda: (o.engine.eval(x.view(-1,3), 0, energies=en, status=st), torch.cuda.synchronize())):8.1f} us")
print(f"ops.dot             {t(lambda: ops.dot(x, x)):8.1f} us")
print(f"ops.dots(3)         {t(lambda: ops.dots([(x, x), (x, x), (x, x)])):8.1f} us")
print(f"ops.lincomb         {t(lambda: ops.lincomb(1.0, x, 0.5, x)):8.1f} us")
print(f"torch add           {t(lambda: x + 0.5 * x):8.1f} us")
print(f"empty launch sync   {t(lambda: torch.cuda.synchronize()):8.1f} us")
