import os, sys
import numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
os.environ["FFM_FORCE_TILES"] = "1"
from paper_1810_03358_b200 import _native as N
from paper_1810_03358_b200.engine import DeviceSystem
from paper_1810_03358_b200.synth import make_globule_system
dirty = len(sys.argv) > 1 and sys.argv[1] == "dirty"
if dirty:
    from paper_1810_03358_b200.kernels import get_backend
    from conftest import golden_system
    G = np.load("tests/golden/golden_v1.npz")
    kb = get_backend()
    s0 = golden_system(G, "cloud24")
    p = s0.arrays()
    c0 = np.ascontiguousarray(s0.coords)
    print(kb.nb_energy(c0, p["q"], p["sigma"], p["epsilon"], p["scale"], 0.0))
    gout = np.zeros_like(c0)
    print(kb.nb_grad(c0, p["q"], p["sigma"], p["epsilon"], p["scale"], 0.0, gout)[:2])
s = make_globule_system(37, seed=7)
c = torch.from_numpy(s.coords.copy()).cuda()
full = DeviceSystem(s.topology)
gf = torch.empty_like(c)
ef, _ = full.eval(c, N.FFM_F64, grad=gf)
print("full", ef.cpu().numpy())
gs = []
for rank in range(3):
    eng = DeviceSystem(s.topology)
    N.check(eng.lib.ffm_system_set_shard(eng.handle, rank, 3), "set_shard")
    g = torch.empty_like(c)
    e, st = eng.eval(c, N.FFM_F64, grad=g)
    print(rank, e.cpu().numpy(), st.cpu().numpy(), eng.info)
    gs.append(g.cpu().numpy())
    eng.close()
np.save(f"gpurun_out/dbg_tiles_{'dirty' if dirty else 'clean'}.npy", np.array(gs))
print("sum err", np.abs(sum(gs) - gf.cpu().numpy()).max())
