#!/usr/bin/env python
"""Headline benchmark: all-pairs LJ + Coulomb energy + analytic gradient.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A "step" is one energy + gradient evaluation (one oracle value_and_gradient
call) of a 100,000-atom synthetic protein-like system (BASELINE.json metric
"pair-interactions/sec (energy+grad) at N=10k/100k"), FP32 pair arithmetic
with FP64 accumulation; the FP64 mode is measured alongside.  value = pair
interactions (N(N-1)/2 per step) per second, whole job, inputs resident in
HBM; e2e = the same through the public host API (MolecularOracle.
value_and_gradient on a pinned NumPy vector, copies inside the timed region).

N > 1 (torchrun): the pair triangle is row-sharded over the ranks
(paper_1810_03358_b200.parallel), gradients/energies all-reduced over
NVLink with NCCL; strong scaling, timing = max over ranks.

--impl reference times the reference algorithm on the host: the C
restatement in oracle/ (the reference itself is Python + numba and cannot
be installed here), all host threads, a bounded row slice per step.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "pair-interactions/sec (energy+grad)"
NATOMS = 100_000
FLOP_PER_PAIR = 38  # 27 FP32 ops (10 of them FMA -> +10) + 1 rsqrt, DESIGN.md
FMA_SLOTS_PER_PAIR = 24  # FP32 lane-ops on the FMA pipe per pair (SASS: 2 x 12 packed FFMA2/FMUL2/FADD2 per 2 pairs; r^-2 on MUFU)
FP64_OPS_PER_PAIR = 32  # FP64-pipe operations per pair (ncu: fp64 pipe 66.9% at 12.87 ms)
DFMA_PEAK = 18.49e12  # measured DFMA/s (63.6 per clk per SM, profiles/r01_pipes_microbench.txt)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=("ours", "reference"), default="ours")
    p.add_argument("--natoms", type=int, default=NATOMS)
    p.add_argument("--no-extras", action="store_true", help="skip the secondary configs")
    p.add_argument("--shard", action="store_true",
                   help="use the row-sharded NCCL path even with one rank (testing)")
    return p.parse_args()


def nb_traffic(n):
    """DRAM bytes per pair-sweep launch from the committed ncu capture."""
    try:
        d = json.loads((ROOT / "profiles" / "r01_nb_traffic.json").read_text())
        return d["dram_bytes_per_launch"] if d.get("natoms") == n else None
    except Exception:
        return None


def peaks():
    d = {}
    try:
        d = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        pass
    # FP32 FMA peak measured on this pool (profiles/r01_pipes_microbench.txt):
    # 123.2 FMA/clk/SM at 1965 MHz nominal -> 35.83 TFMA/s
    fma = 35.83e12
    return d, fma


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled DURING the timed
    region: an NVML polling thread (2 ms period; the timed region is only
    ~50 ms, too short for nvidia-smi's 100 ms loop).  Falls back to one
    nvidia-smi query when NVML is unavailable."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
               ("hw_power_brake", "nvmlClocksEventReasonHwPowerBrakeSlowdown"))

    def __init__(self, index, period_s=0.002):
        self.index = index
        self.period = period_s
        self.sm, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._nv = None

    def __enter__(self):
        try:
            import pynvml as nv

            nv.nvmlInit()
            self._nv = nv
            self._h = nv.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = float(nv.nvmlDeviceGetMaxClockInfo(self._h, nv.NVML_CLOCK_SM))
            self._t = threading.Thread(target=self._poll, daemon=True)
            self._t.start()
        except Exception:
            self._nv = None
        return self

    def _poll(self):
        nv = self._nv
        masks = [(name, getattr(nv, attr, 0)) for name, attr in self.REASONS]
        while not self._stop.is_set():
            try:
                self.sm.append(float(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                self.reasons.update(name for name, m in masks if m and (r & m))
            except Exception:
                pass
            time.sleep(self.period)

    def __exit__(self, *a):
        self._stop.set()
        if self._nv is not None:
            self._t.join(1.0)

    def summary(self):
        if not self.sm:
            return self._smi_once()
        return {"sm_mhz": float(np.median(self.sm)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.sm), "source": "nvml 2 ms"}

    def _smi_once(self):
        try:
            out = subprocess.run(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm",
                 "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=10)
            sm, mx = (float(x) for x in out.stdout.strip().split(","))
            return {"sm_mhz": sm, "sm_max_mhz": mx, "reasons": ["unsampled"], "samples": 1,
                    "source": "nvidia-smi after the timed region"}
        except Exception:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}


# ------------------------------------------------------------- reference arm

def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle as O
    from paper_1810_03358_b200.synth import make_globule_system

    n = args.natoms
    s = make_globule_system(n, seed=0)
    A = O.Arrays.from_system(s)
    threads = O.host_threads()
    total_pairs = n * (n - 1) // 2
    # rows [i0, i1) hold sum_{i0 <= i < i1} (n - 1 - i) pairs; five slices of
    # equal pair count cover the triangle, one slice per step
    rows = np.arange(n)
    cum = np.concatenate([[0], np.cumsum(n - 1 - rows)])
    edges = [int(np.searchsorted(cum, total_pairs * k / 5)) for k in range(6)]
    edges[-1] = n
    slices = [(edges[k], edges[k + 1]) for k in range(5)]

    def step(k):
        i0, i1 = slices[k % 5]
        t0 = time.perf_counter()
        O.nb_eval(A, s.coords, True, threads=threads, rows=(i0, i1))
        O.bonded(A, s.coords, True)
        return time.perf_counter() - t0, int(cum[i1] - cum[i0])

    for k in range(args.warmup):
        step(k)
    tot_t, tot_p = 0.0, 0
    for k in range(args.steps):
        dt, npairs = step(k)
        tot_t += dt
        tot_p += npairs
    value = tot_p / tot_t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "pairs/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot_t / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"energy+gradient, {n}-atom synthetic protein-like globule",
                   "natoms": n, "sample": "one fifth of the pair triangle (row slice) per step"},
        "cpu_baseline": {"value": value, "unit": "pairs/s", "cores": threads, "kind": "port",
                         "sample": "row slices of the 100k-atom energy+gradient, 1/5 triangle each"},
        "e2e": {"value": value, "unit": "pairs/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- our arm

def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return

    import torch

    from paper_1810_03358_b200 import _native as N
    from paper_1810_03358_b200.energy import energy_and_gradient
    from paper_1810_03358_b200.engine import DeviceSystem
    from paper_1810_03358_b200.parallel import ShardedSystem, init_from_env
    from paper_1810_03358_b200.synth import make_globule_system
    import torch.distributed as dist

    rank, world, local = init_from_env("nccl")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    n = args.natoms
    s = make_globule_system(n, seed=0)
    lib = N.load()
    sharded = world > 1 or args.shard
    if sharded:
        if not dist.is_initialized():
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29533")
            dist.init_process_group("nccl", rank=0, world_size=1,
                                    device_id=torch.device("cuda", local))
        eng = ShardedSystem(s.topology, device=local)
        handle = eng.engine.handle
    else:
        eng = DeviceSystem(s.topology, local)
        handle = eng.handle
    pairs = n * (n - 1) / 2
    rng = np.random.default_rng(1234)
    base = np.ascontiguousarray(s.coords)
    # a fresh geometry per step (small jitter), resident in HBM
    steps_coords = [torch.from_numpy(base + rng.normal(scale=0.01, size=base.shape)).to(dev)
                    for _ in range(4)]
    grad = torch.empty((n, 3), dtype=torch.float64, device=dev)
    en, st = eng.new_outputs()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > 126 MB L2

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def time_device(prec, steps, warmup, clk=None):
        for k in range(warmup):
            eng.eval(steps_coords[k % 4], prec, grad=grad, energies=en, status=st)
        barrier()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(steps)]
        nb_ms = []
        l0 = lib.ffm_launch_count()
        if clk is not None:
            clk.__enter__()  # sample clocks during the timed steps only
        for k in range(steps):
            flush.zero_()  # L2 flush between timed steps (outside the events)
            ev[k][0].record()
            eng.eval(steps_coords[k % 4], prec, grad=grad, energies=en, status=st,
                     flags=N.FFM_ENERGY | N.FFM_GRAD | N.FFM_TIME_NB)
            ev[k][1].record()
            ms = np.zeros(1, np.float32)
            N.check(lib.ffm_system_nb_ms(handle, ms.ctypes.data), "nb_ms")
            nb_ms.append(float(ms[0]))
        barrier()
        if clk is not None:
            clk.__exit__(None, None, None)
        launches = lib.ffm_launch_count() - l0
        step_ms = [a.elapsed_time(b) for a, b in ev]
        tot = float(np.sum(step_ms))
        if world > 1:
            t = torch.tensor([tot, float(np.mean(nb_ms))], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            tot, nbm = t.tolist()
        else:
            nbm = float(np.mean(nb_ms))
        assert int(st[0]) == -1, "coincident atoms in the benchmark system"
        return tot / steps, nbm, launches

    clk = ClockSampler(local)
    ms32, nb32, launches = time_device(N.FFM_F32, args.steps, args.warmup, clk)
    clocks = clk.summary()
    ms64, nb64, _ = time_device(N.FFM_F64, max(3, args.steps // 2), 2)
    value = pairs / (ms32 * 1e-3)

    # ---- e2e through the public API, host buffers (pinned), FP32 mode: the
    # objective oracle every minimiser calls (value_and_gradient on a NumPy
    # vector -> (float, NumPy float64 gradient)), copies inside the timed region
    pinned = torch.empty(3 * n, dtype=torch.float64).pin_memory()
    if sharded:
        from paper_1810_03358_b200.parallel import ShardedMolecularOracle

        orc = ShardedMolecularOracle(s, np.float32, device=local)
    else:
        from paper_1810_03358_b200.oracle import MolecularOracle

        orc = MolecularOracle(s, np.float32, device=local)
    e2e_times = []
    for k in range(args.warmup + args.steps):
        pinned.numpy()[:] = steps_coords[k % 4].cpu().numpy().reshape(-1)
        host = pinned.numpy()
        barrier()
        t0 = time.perf_counter()
        f, g = orc.value_and_gradient(host)
        t1 = time.perf_counter()
        assert isinstance(g, np.ndarray) and g.shape == (3 * n,)
        if k >= args.warmup:
            e2e_times.append(t1 - t0)
    e2e_s = float(np.mean(e2e_times))
    if world > 1:
        t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())

    measured, fma_peak = peaks()
    flop_peak = 2 * fma_peak
    nb_pairs_per_rank = pairs / world
    achieved = nb_pairs_per_rank * FLOP_PER_PAIR / (nb32 * 1e-3)
    # FMA-pipe fraction: FP32 lane-op slots used per second over the pipe's
    # 128 lane-ops / clk / SM (= fma_peak per second)
    fma_frac = nb_pairs_per_rank * FMA_SLOTS_PER_PAIR / (nb32 * 1e-3) / fma_peak

    line = {
        "metric": METRIC, "value": value, "unit": "pairs/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms32,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32 (pair arithmetic; fp64 accumulation)", "data": "synthetic",
        "config": {"workload": f"energy+gradient of a {n}-atom synthetic protein-like globule "
                               "(LJ + Coulomb all pairs, bonded terms, 1-2/1-3 excluded, 1-4 scaled)",
                   "natoms": n, "pairs_per_step": int(pairs), "parallelism": f"row-shard x{world}",
                   "l2": "flushed (256 MB write) between timed steps",
                   "inputs": "fresh jittered geometry per step, resident in HBM"},
        "value_f64": pairs / (ms64 * 1e-3), "ms_per_step_f64": ms64,
        "e2e": {"value": pairs / e2e_s, "unit": "pairs/s", "h2d_bytes_per_step": n * 3 * 8,
                "d2h_bytes_per_step": n * 3 * 8 + 5 * 8 + 8 * 8,
                "api": "oracle.MolecularOracle(system, np.float32).value_and_gradient(x)"
                       if not sharded else "parallel.ShardedMolecularOracle.value_and_gradient(x)"},
        "roofline": {"bound": "fp32-fma-pipe", "kernel": "nb_units_kernel<float,GRAD>",
                     "achieved": achieved / 1e12, "peak": flop_peak / 1e12, "unit": "TFLOP/s",
                     "frac": achieved / flop_peak, "traffic": nb_traffic(n),
                     "flop_per_pair": FLOP_PER_PAIR, "fma_pipe_frac": fma_frac,
                     "nb_ms": nb32, "nb_ms_f64": nb64,
                     "peak_source": "measured FFMA throughput, profiles/r01_pipes_microbench.txt",
                     "bound_note": "not a dense contraction (north star): the pair sweep is bound "
                                   "by the FP32 FMA pipe; DRAM traffic is under 2% of its time "
                                   "and tensor cores do not apply"},
        "roofline_f64": {"bound": "fp64-pipe", "kernel": "nb_units_kernel<double,GRAD>",
                         "achieved": nb_pairs_per_rank * FP64_OPS_PER_PAIR / (nb64 * 1e-3) / 1e12,
                         "peak": DFMA_PEAK / 1e12, "unit": "T fp64-pipe ops/s",
                         "frac": nb_pairs_per_rank * FP64_OPS_PER_PAIR / (nb64 * 1e-3) / DFMA_PEAK,
                         "ops_per_pair": FP64_OPS_PER_PAIR, "nb_ms": nb64},
        "gpu_launches": int(launches),
        "clocks": clocks,
    }

    if rank == 0 and world == 1:
        line["cpu_baseline"] = cpu_baseline(s)
    if not args.no_extras:
        extras = run_extras(rank, world, local)
        if rank == 0:
            line["extras"] = extras
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist.is_initialized():
        dist.barrier()
        dist.destroy_process_group()


def cpu_baseline(s):
    import oracle as O

    A = O.Arrays.from_system(s)
    threads = O.host_threads()
    n = s.natoms
    t0 = time.perf_counter()
    O.nb_eval(A, s.coords, True, threads=threads)
    O.bonded(A, s.coords, True)
    dt = time.perf_counter() - t0
    return {"value": n * (n - 1) / 2 / dt, "unit": "pairs/s", "cores": threads, "kind": "port",
            "sample": f"one full {n}-atom energy+gradient (oracle/ffmin_oracle.c, "
                      f"{threads} threads), {dt:.2f} s"}


def run_extras(rank, world, local):
    """Secondary BASELINE configs, bounded (about a minute)."""
    import torch

    from paper_1810_03358_b200 import _native as N
    from paper_1810_03358_b200.engine import DeviceSystem
    from paper_1810_03358_b200.synth import make_globule_system

    out = {}
    dev = torch.device("cuda", local)
    if world == 1:
        # configs[1]: single evaluation sweep, N = 3k / 10k / 30k, FP64 and FP32
        sweep = {}
        for n in (3000, 10000, 30000):
            s = make_globule_system(n, seed=0)
            eng = DeviceSystem(s.topology, local)
            c = torch.from_numpy(np.array(s.coords, dtype=np.float64)).to(dev)
            g = torch.empty_like(c)
            en, st = eng.new_outputs()
            for prec, tag in ((N.FFM_F32, "f32"), (N.FFM_F64, "f64")):
                for _ in range(3):
                    eng.eval(c, prec, grad=g, energies=en, status=st)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                reps = 20
                e0.record()
                for _ in range(reps):
                    eng.eval(c, prec, grad=g, energies=en, status=st)
                e1.record()
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / reps
                sweep[f"{n}_{tag}"] = {"ms": ms, "pairs_per_s": n * (n - 1) / 2 / (ms * 1e-3)}
            eng.close()
        out["sweep_energy_grad"] = sweep
        # configs[3]: 1024 candidate geometries of a 5k-atom system per step
        s = make_globule_system(5000, seed=0)
        eng = DeviceSystem(s.topology, local)
        B = 1024
        rng = np.random.default_rng(0)
        batch = torch.from_numpy(s.coords[None] + rng.normal(scale=0.02, size=(B,) + s.coords.shape)).to(dev)
        en, st = eng.new_outputs(B)
        for _ in range(2):
            eng.eval_batch(batch, N.FFM_F32, energies=en, status=st)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            eng.eval_batch(batch, N.FFM_F32, energies=en, status=st)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        out["batched_candidates"] = {"candidates": B, "natoms": 5000, "ms_per_step": ms,
                                     "pairs_per_s": B * 5000 * 4999 / 2 / (ms * 1e-3),
                                     "precision": "f32", "what": "energy only"}
        eng.close()
        # configs[0]: L-BFGS time-to-converge against the reference run
        out["lbfgs_converge"] = lbfgs_converge()
        # configs[2]: optimiser comparison on a 10k-atom globule
        out["optimizer_comparison_10k"] = optimizer_comparison(10000, iters=100)
        # configs[4]: L-BFGS iterations on the 100k-atom system (1 GPU)
        out["lbfgs_100k"] = optimizer_comparison(100000, iters=10, methods=("lbfgs",),
                                                 dtype=np.float32)
    return out


def optimizer_comparison(natoms, iters, methods=("sd", "fgm", "cg", "lbfgs", "wiggle"),
                         dtype=np.float64):
    """Every minimiser from the same perturbed start with the same iteration
    budget: final energy, calls and wall time (device-resident iterates)."""
    import torch

    from paper_1810_03358_b200.oracle import MolecularOracle
    from paper_1810_03358_b200.optimizers import StopCriteria, cg, fgm, lbfgs, make_linesearch
    from paper_1810_03358_b200.optimizers import steepest_descent
    from paper_1810_03358_b200.optimizers.wiggle import WiggleConfig, atom_wiggle
    from paper_1810_03358_b200.synth import make_globule_system

    s = make_globule_system(natoms, seed=1)
    out = {"natoms": natoms, "iterations_budget": iters,
           "precision": "f32" if dtype == np.float32 else "f64"}
    for name in methods:
        stop = StopCriteria(max_iterations=iters, gradient_norm_rtol=1e-6)
        o = MolecularOracle(s, dtype=dtype)
        ls = make_linesearch("par")
        run = {"sd": lambda: steepest_descent(o, s.coords.ravel(), ls, stop),
               "fgm": lambda: fgm(o, s.coords.ravel(), ls, stop),
               "cg": lambda: cg(o, s.coords.ravel(), "prp+", ls, stop),
               "lbfgs": lambda: lbfgs(o, s.coords.ravel(), m=5, linesearch=ls, stop=stop)}
        if name != "wiggle":  # warm-up: capture the method's graph outside the timing
            warm = StopCriteria(max_iterations=2, gradient_norm_rtol=1e-6)
            {"sd": lambda: steepest_descent(o, s.coords.ravel(), ls, warm),
             "fgm": lambda: fgm(o, s.coords.ravel(), ls, warm),
             "cg": lambda: cg(o, s.coords.ravel(), "prp+", ls, warm),
             "lbfgs": lambda: lbfgs(o, s.coords.ravel(), m=5, linesearch=ls, stop=warm)}[name]()
            o.value_calls = o.grad_calls = 0
            ls.reset()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if name == "wiggle":
            # gradient-free: one probe batch per atom move; 20 moves per atom
            # budget unit is scaled so the call count is comparable
            res = atom_wiggle(s, WiggleConfig(seed=0),
                              StopCriteria(max_iterations=iters * 20, gradient_norm_rtol=0.0))
            calls = res.trace.records[-1].value_calls
            gcalls = 0
        else:
            res = run[name]()
            calls, gcalls = o.value_calls, o.grad_calls
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        out[name] = {"f": float(res.f), "iterations": int(res.iterations), "status": res.status,
                     "value_calls": int(calls), "grad_calls": int(gcalls), "seconds": dt,
                     "ms_per_iteration": dt / max(1, res.iterations) * 1e3}
    out["f_start"] = float(MolecularOracle(s, dtype=dtype).value(s.coords.ravel()))
    return out


def lbfgs_converge():
    """configs[0]: L-BFGS minimisation from a perturbed start, run to the
    precision limit like the reference (golden conv200: 200-atom chain,
    minimum jittered by 0.05 A), FP64; time-to-converge beside the
    reference's own run recorded in the golden file (numba, 1 core)."""
    import torch

    from paper_1810_03358_b200.model import MolecularSystem
    from paper_1810_03358_b200.oracle import MolecularOracle
    from paper_1810_03358_b200.optimizers import StopCriteria, lbfgs, make_linesearch

    G = np.load(ROOT / "tests" / "golden" / "golden_v1.npz")
    out = {}
    for name in ("lbfgs500", "conv60", "conv200"):
        cut = float(G[f"{name}/cutoff"])
        s = MolecularSystem.from_arrays(
            G[f"{name}/q"], G[f"{name}/sigma"], G[f"{name}/epsilon"], G[f"{name}/coords"],
            G[f"{name}/bond_idx"], G[f"{name}/bond_K"], G[f"{name}/bond_r0"],
            G[f"{name}/ang_idx"], G[f"{name}/ang_K"], G[f"{name}/ang_t0"], G[f"{name}/dih_idx"],
            G[f"{name}/dih_V"], excluded=G[f"{name}/excluded"], scaled14=G[f"{name}/scaled14"],
            s14=float(G[f"{name}/s14"]), cutoff=None if cut <= 0 else cut)
        if name == "lbfgs500":
            # configs[0]: the reference's bounded 500-atom chain run (m = 3,
            # 300 iterations or |g| <= 1e-3), make_golden.py
            ref_f, _, ref_it = G[f"{name}/final"]
            m = 3
            stop = StopCriteria(max_iterations=300, gradient_norm_tol=1e-3,
                                gradient_norm_rtol=0.0)
        else:
            ref_f, _, ref_it, tol = G[f"{name}/final"]
            m = 5
            stop = StopCriteria(max_iterations=50000, gradient_norm_tol=tol,
                                gradient_norm_rtol=0.0)
        lbfgs(MolecularOracle(s), s.coords.ravel(), m=m, linesearch=make_linesearch("par"),
              stop=StopCriteria(max_iterations=3, gradient_norm_rtol=0.0))  # warm-up
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = lbfgs(MolecularOracle(s), s.coords.ravel(), m=m, linesearch=make_linesearch("par"),
                    stop=stop)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        out[name] = {"natoms": s.natoms, "iterations": res.iterations, "status": res.status,
                     "f": res.f, "ref_f": float(ref_f), "ref_iterations": int(ref_it),
                     "rel_diff_f": abs(res.f - ref_f) / abs(ref_f), "seconds": dt,
                     "ref_seconds_numba_1core": float(G[f"{name}/seconds"])}
        if name == "lbfgs500":
            # a long nonconvex run: roundoff differences eventually pick a
            # different basin, so report how long the f trace follows the
            # reference's within 1e-8 relative
            f = np.array([r.f for r in res.trace.records])
            ref = G[f"{name}/f_trace"]
            k = min(len(f), len(ref))
            bad = np.nonzero(np.abs(f[:k] - ref[:k]) > 1e-8 * np.abs(ref[:k]))[0]
            out[name]["trace_matches_reference_iterations"] = int(bad[0]) if len(bad) else k
    return out


if __name__ == "__main__":
    main()
