import sys, numpy as np
sys.path.insert(0, '.')
import oracle as O
from paper_1810_03358_b200.energy import energy_and_gradient
from paper_1810_03358_b200.synth import make_globule_system
for n, cut in ((3000, 7.0), (3000, 1000.0), (30000, 7.0)):
    s = make_globule_system(n, seed=5, cutoff=cut)
    A = O.Arrays.from_system(s)
    e_ref, g_ref, err = O.energy_and_gradient(A, s.coords, True, threads=O.host_threads())
    for dt in (np.float64, np.float32):
        bd, g = energy_and_gradient(s, dt)
        got = np.array([bd.stretch, bd.bend, bd.torsion, bd.coulomb, bd.vdw])
        d = np.abs(g - g_ref).reshape(-1, 3).max(axis=1)
        bad = np.nonzero(d > 1e-6 * np.abs(g_ref).max())[0]
        print(n, cut, np.dtype(dt).name, "E rel", (np.abs(got - e_ref) / np.abs(e_ref)).round(12), "bad atoms", len(bad), bad[:10])
