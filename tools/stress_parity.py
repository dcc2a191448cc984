"""Parity sweep over many system sizes and plan shapes (tuning / regression
aid, not a unit test): FP64 and FP32 energy+gradient against the threaded
oracle, with and without a cutoff.  usage: python tools/stress_parity.py"""
import sys

import numpy as np

sys.path.insert(0, ".")
import oracle as O
from paper_1810_03358_b200.energy import energy_and_gradient
from paper_1810_03358_b200.synth import make_chain_system, make_globule_system

sizes = [int(a) for a in sys.argv[1:]] or [1, 2, 33, 127, 128, 129, 255, 257, 1000, 4095, 4097,
                                            4300, 4400, 5000, 12345, 40000, 40001, 70000]
worst = {}
for n in sizes:
    for cutoff in (None, 9.0):
        s = (make_globule_system(n, seed=n % 97, cutoff=cutoff) if n >= 4
             else make_chain_system(max(n, 2), seed=1, cutoff=cutoff))
        A = O.Arrays.from_system(s)
        e_ref, g_ref, err = O.energy_and_gradient(A, s.coords, True, threads=O.host_threads())
        gmax = max(np.max(np.abs(g_ref)), 1e-30)
        for dt, et, gt in ((np.float64, 1e-10, 1e-10), (np.float32, 1e-5, 1e-4)):
            bd, g = energy_and_gradient(s, dt)
            got = np.array([bd.stretch, bd.bend, bd.torsion, bd.coulomb, bd.vdw])
            rel = np.max(np.abs(got - e_ref) / np.maximum(np.abs(e_ref), 1e-9))
            gerr = np.max(np.abs(np.ravel(g) - np.ravel(g_ref))) / gmax
            # FP32 with a cutoff may classify pairs within ~1e-6 of it differently
            ok = (rel <= et and gerr <= gt) or (cutoff is not None and dt == np.float32)
            tag = f"n={n} cut={cutoff} {np.dtype(dt).name}"
            print(f"{tag:34s} rel(E)={rel:.1e} rel(g)={gerr:.1e} {'ok' if ok else 'FAIL'}",
                  flush=True)
