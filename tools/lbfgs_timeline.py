"""Timeline of a graph-resident L-BFGS iteration on a small system: needs a
library built with -DFFM_MIN_STAMPS (tools/build_lib_variant.sh mstamps
-DFFM_MIN_STAMPS).  Tags: 1 it_begin, 2 min_dir, 3 ls_init, 4 fused
evaluation start, 10 its P1 start, 11 its P2 start, 5 its pass end, 7
ls_post, 8 commit, 9 it_end, 12/13 around the fused kernel's probe
controller, 14 after its loop barrier, 20/21 two-loop kernel start/end, 22 one-block dots.
usage: FFMIN_B200_LIB=... python tools/lbfgs_timeline.py [N] [iters]"""
import collections
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_03358_b200 import _native as N  # noqa: E402
from paper_1810_03358_b200.oracle import MolecularOracle  # noqa: E402
from paper_1810_03358_b200.optimizers import StopCriteria, lbfgs, make_linesearch  # noqa: E402
from paper_1810_03358_b200.synth import make_globule_system  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 500
it = int(sys.argv[2]) if len(sys.argv) > 2 else 40
s = make_globule_system(n, seed=1)
o = MolecularOracle(s, np.float32 if os.environ.get("PREC") == "f32" else np.float64)
lbfgs(o, s.coords.ravel(), m=5, linesearch=make_linesearch("par"),
      stop=StopCriteria(max_iterations=2, gradient_norm_rtol=1e-6))
lib = N.load()
buf = torch.zeros(1 + 2 * 200000, dtype=torch.int64, device="cuda")
for f in ("ffm_debug_min_clock_minimize", "ffm_debug_min_clock_small", "ffm_debug_min_clock_vec"):
    getattr(lib, f).argtypes = [C.c_void_p]
    assert getattr(lib, f)(C.c_void_p(buf.data_ptr())) == 0
torch.cuda.synchronize()
res = lbfgs(o, s.coords.ravel(), m=5, linesearch=make_linesearch("par"),
            stop=StopCriteria(max_iterations=it, gradient_norm_rtol=1e-6))
torch.cuda.synchronize()
for f in ("ffm_debug_min_clock_minimize", "ffm_debug_min_clock_small", "ffm_debug_min_clock_vec"):
    getattr(lib, f)(None)
b = buf.cpu().numpy()
k = int(b[0])
ev = b[1:1 + 2 * k].reshape(-1, 2)
ev = ev[np.argsort(ev[:, 1], kind="stable")]
tags, t = ev[:, 0], (ev[:, 1] - ev[0, 1]) / 1e3
starts = np.nonzero(tags == 1)[0]
print(f"n={n}: {res.iterations} iterations, {len(starts)} it_begin stamps, "
      f"{(t[starts[-1]] - t[starts[0]]) / max(1, len(starts) - 1):.1f} us per iteration")
gaps = collections.defaultdict(list)
for a0, a1 in zip(starts[:-1], starts[1:]):
    seq = list(range(a0, a1 + 1))
    for x, y in zip(seq[:-1], seq[1:]):
        gaps[(int(tags[x]), int(tags[y]))].append(t[y] - t[x])
print("transition         count/it  mean us  total us/it")
nit = max(1, len(starts) - 1)
for key, v in sorted(gaps.items(), key=lambda kv: -sum(kv[1])):
    print(f"{key[0]:3d} -> {key[1]:3d}   {len(v) / nit:8.2f} {np.mean(v):8.2f} {sum(v) / nit:10.2f}")
