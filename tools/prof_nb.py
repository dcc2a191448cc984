"""Launch the pair sweep a few times for ncu (development aid)."""
import sys
import torch
sys.path.insert(0, '.')
from paper_1810_03358_b200.synth import make_globule_system
from paper_1810_03358_b200.engine import engine_for
n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
prec = int(sys.argv[2]) if len(sys.argv) > 2 else 1
s = make_globule_system(n, seed=0)
eng = engine_for(s.topology)
c = torch.from_numpy(s.coords.copy()).cuda()
g = torch.empty_like(c)
for _ in range(3):
    eng.eval(c, prec, grad=g)
torch.cuda.synchronize()
print("ok")
