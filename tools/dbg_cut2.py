import sys, numpy as np, torch
sys.path.insert(0, '.')
import oracle as O
from paper_1810_03358_b200 import _native as N
from paper_1810_03358_b200.engine import DeviceSystem
from paper_1810_03358_b200.synth import make_globule_system
for n in (300, 600, 3000):
    for cut in (1000.0, None):
        s = make_globule_system(n, seed=5, cutoff=cut)
        A = O.Arrays.from_system(s)
        ec, ev, _, _, _ = O.nb_eval(A, s.coords, False, threads=8)
        eng = DeviceSystem(s.topology)
        c = torch.from_numpy(s.coords.copy()).cuda()
        out = []
        for fl in (N.FFM_ENERGY, N.FFM_ENERGY | N.FFM_NO_GRAPH, N.FFM_ENERGY | N.FFM_NO_TERMS | N.FFM_NO_GRAPH):
            for prec in (0, 1):
                en, st = eng.eval(c, prec, flags=fl)
                e = en.cpu().numpy()
                out.append(f"{e[3]/ec-1:+.2e},{e[4]/ev-1:+.2e}")
        print(n, cut, eng.info['S'], eng.info['units'], out)
