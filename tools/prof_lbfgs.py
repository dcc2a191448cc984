"""Host-side profile of a small L-BFGS run (golden conv200) -- tuning aid."""
import cProfile, pstats, sys, time
import numpy as np, torch
sys.path.insert(0, '.')
from paper_1810_03358_b200.model import MolecularSystem
from paper_1810_03358_b200.oracle import MolecularOracle
from paper_1810_03358_b200.optimizers import StopCriteria, lbfgs, make_linesearch

G = np.load("tests/golden/golden_v1.npz")
name = sys.argv[1] if len(sys.argv) > 1 else "conv200"
cut = float(G[f"{name}/cutoff"])
s = MolecularSystem.from_arrays(
    G[f"{name}/q"], G[f"{name}/sigma"], G[f"{name}/epsilon"], G[f"{name}/coords"],
    G[f"{name}/bond_idx"], G[f"{name}/bond_K"], G[f"{name}/bond_r0"],
    G[f"{name}/ang_idx"], G[f"{name}/ang_K"], G[f"{name}/ang_t0"], G[f"{name}/dih_idx"],
    G[f"{name}/dih_V"], excluded=G[f"{name}/excluded"], scaled14=G[f"{name}/scaled14"],
    s14=float(G[f"{name}/s14"]), cutoff=None if cut <= 0 else cut)
ref_f, _, ref_it, tol = G[f"{name}/final"]
stop = StopCriteria(max_iterations=50000, gradient_norm_tol=tol, gradient_norm_rtol=0.0)
lbfgs(MolecularOracle(s), s.coords.ravel(), m=5, linesearch=make_linesearch("par"),
      stop=StopCriteria(max_iterations=3, gradient_norm_rtol=0.0))
torch.cuda.synchronize()
o = MolecularOracle(s)
t0 = time.perf_counter()
res = lbfgs(o, s.coords.ravel(), m=5, linesearch=make_linesearch("par"), stop=stop)
dt = time.perf_counter() - t0
print(f"{name}: {res.iterations} it, {dt:.3f} s, {dt/res.iterations*1e3:.3f} ms/it, "
      f"value calls {o.value_calls} grad calls {o.grad_calls}")
o = MolecularOracle(s)
pr = cProfile.Profile()
pr.enable()
res = lbfgs(o, s.coords.ravel(), m=5, linesearch=make_linesearch("par"), stop=stop)
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(25)
