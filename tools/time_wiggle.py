"""Time the graph-resident atom wiggle (10k atoms by default): total wall
time of atom_wiggle and the split between graph build and chunk launches.

    python tools/time_wiggle.py [natoms] [iterations]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1810_03358_b200.optimizers import StopCriteria  # noqa: E402
from paper_1810_03358_b200.optimizers import graph as G  # noqa: E402
from paper_1810_03358_b200.optimizers.wiggle import WiggleConfig, atom_wiggle  # noqa: E402
from paper_1810_03358_b200.synth import make_globule_system  # noqa: E402


def main():
    natoms = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
    s = make_globule_system(natoms, seed=1)
    t_init = []
    orig = G._GraphRun.__init__

    def timed_init(self, *a, **k):
        t0 = time.perf_counter()
        orig(self, *a, **k)
        torch.cuda.synchronize()
        t_init.append(time.perf_counter() - t0)

    G._GraphRun.__init__ = timed_init
    atom_wiggle(s, WiggleConfig(seed=0), StopCriteria(max_iterations=40, gradient_norm_rtol=0.0))
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = atom_wiggle(s, WiggleConfig(seed=0),
                          StopCriteria(max_iterations=iters, gradient_norm_rtol=0.0))
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        print(f"rep {rep}: {dt * 1e3:.1f} ms total, {dt / iters * 1e3:.3f} ms/it, "
              f"graph init {(t_init[-1] if t_init else 0.0) * 1e3:.1f} ms, f={res.f:.6f}, "
              f"calls={res.trace.records[-1].value_calls}", flush=True)
    print("PDL", os.environ.get("FFM_PDL", "default"))


if __name__ == "__main__":
    main()
