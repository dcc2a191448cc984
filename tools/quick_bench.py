"""Quick device timing of ffm_eval (energy+grad) -- development aid."""
import sys, time
import numpy as np, torch
sys.path.insert(0, '.')
from paper_1810_03358_b200.synth import make_globule_system
from paper_1810_03358_b200.engine import engine_for

for n in [int(a) for a in (sys.argv[1:] or ["10000", "30000", "100000"])]:
    s = make_globule_system(n, seed=0)
    eng = engine_for(s.topology)
    c = torch.from_numpy(s.coords).cuda()
    g = torch.empty_like(c)
    en, st = eng.new_outputs()
    pairs = n * (n - 1) / 2
    for prec in (1, 0):
        for flags, grad in ((3, g), (1, None)):
            for _ in range(3):
                eng.eval(c, prec, grad=grad, energies=en, status=st, flags=flags)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 10
            e0.record()
            for _ in range(reps):
                eng.eval(c, prec, grad=grad, energies=en, status=st, flags=flags)
            e1.record(); torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            print(f"n={n:7d} {'f32' if prec else 'f64'} {'E+G' if grad is not None else 'E  '} "
                  f"{ms:8.3f} ms  {pairs/ms/1e9:8.2f} Gpairs/s  info={eng.info}  st={st.cpu().tolist()[:5]}", flush=True)
