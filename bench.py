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

N > 1: the pair triangle is row-sharded over the ranks
(paper_1810_03358_b200.parallel), gradients/energies all-reduced over
NVLink with NCCL; strong scaling, timing = max over ranks.  Launched under
torchrun (one rank per GPU) or, with --gpus N and no WORLD_SIZE in the
environment, bench.py re-executes itself under torchrun with N ranks.  A
WORLD_SIZE that disagrees with --gpus is an error; so are fewer visible
GPUs than ranks, unless --allow-shared-gpu (testing only: ranks share
devices round-robin and complete over gloo; the line says so and its
timings are not a scaling measurement).

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
FP64_OPS_PER_PAIR = 29  # FP64-pipe operations per pair (SASS of the unmasked tile: 29 DFMA/DMUL/DADD per pair)
DFMA_PEAK = 18.49e12  # measured DFMA/s (63.6 per clk per SM, profiles/r01_pipes_microbench.txt)
NOMINAL_FP32_FLOPS = 2 * 128 * 148 * 1965e6  # 128 FFMA lanes / clk / SM at the max SM clock
# the tile loop alone (tools/microbench/pairmix.cu: the sweep's warp_tile on a
# restaged shared-memory j-block at the sweep's occupancy, no global memory,
# masks, staging or reductions), ncu pipe activity, profiles/r02_pipes_microbench.txt
MIX_CEILING = {"fp32_fma_pipe_active": 0.788, "fp64_pipe_active": 0.764}
SWEEP_NCU = {"fp32_fma_pipe_active": 0.756, "fp64_pipe_active": 0.737}  # r02 ncu, 100k


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
    p.add_argument("--native-comm", action="store_true",
                   help="complete sharded evaluations with the engine's own ncclAllReduce "
                        "(ffm_system_set_comm) instead of torch.distributed")
    p.add_argument("--allow-shared-gpu", action="store_true",
                   help="testing: more ranks than GPUs (gloo, devices shared round-robin)")
    return p.parse_args()


def free_port():
    import socket

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def launch_ranks(args):
    """--gpus N > 1 without a torchrun environment: re-execute this script
    under torchrun with N ranks (one per GPU) and return its exit code."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(free_port()), str(Path(__file__).resolve()), *sys.argv[1:]]
    env = dict(os.environ)
    env.setdefault("OMP_NUM_THREADS", "4")
    return subprocess.call(cmd, env=env)


def world_from_env(args):
    """(rank, world, local) of this process; refuses a world that
    disagrees with --gpus so a scaling run can never report the wrong N."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    return int(os.environ.get("RANK", "0")), world, int(os.environ.get("LOCAL_RANK", "0"))


def nb_traffic(n):
    """DRAM bytes per pair-sweep launch from the committed ncu capture."""
    try:
        d = json.loads((ROOT / "profiles" / "r02_nb_traffic.json").read_text())
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
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(launch_ranks(args))
    rank, world, local = world_from_env(args)
    if args.impl == "reference":
        run_reference(args)
        return

    import torch
    import torch.distributed as dist

    from paper_1810_03358_b200 import _native as N
    from paper_1810_03358_b200.engine import DeviceSystem
    from paper_1810_03358_b200.parallel import ShardedSystem
    from paper_1810_03358_b200.synth import make_globule_system

    ngpu = torch.cuda.device_count()
    shared = world > ngpu
    if shared and not args.allow_shared_gpu:
        sys.exit(f"bench.py: {world} ranks but {ngpu} visible GPU(s)")
    local = local % ngpu
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    sharded = world > 1 or args.shard
    backend = "gloo" if shared else "nccl"
    if sharded and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", str(free_port()))
        os.environ.setdefault("RANK", "0")
        os.environ.setdefault("WORLD_SIZE", "1")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    n = args.natoms
    s = make_globule_system(n, seed=0)
    lib = N.load()
    native = args.native_comm and backend == "nccl"
    if sharded:
        eng = ShardedSystem(s.topology, device=local, native=native)
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
        if dist.is_initialized():
            dist.barrier()
        torch.cuda.synchronize()

    def allmax(vals):
        if world == 1:
            return vals
        t = torch.tensor(vals, dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.tolist()

    def time_device(prec, steps, warmup, clk=None):
        for k in range(warmup):
            eng.eval(steps_coords[k % 4], prec, grad=grad, energies=en, status=st)
        barrier()
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(steps)]
        nb_ms = []
        l0 = lib.ffm_launch_count()
        if clk is not None:
            clk.__enter__()  # sample clocks during the timed steps only
        for k in range(steps):
            flush.zero_()  # L2 flush between timed steps (outside the events)
            if world > 1:
                dist.barrier()
            ev[k][0].record()
            if sharded and not eng.native:
                # the partial evaluation, then its completion (all-reduce)
                # timed apart: the per-rank compute and the collective
                eng.engine.eval(steps_coords[k % 4], prec, grad=grad, energies=en, status=st,
                                flags=N.FFM_ENERGY | N.FFM_GRAD | N.FFM_TIME_NB)
                ev[k][1].record()
                eng.combiner.combine(grad, en, st)
            else:
                eng.eval(steps_coords[k % 4], prec, grad=grad, energies=en, status=st,
                         flags=N.FFM_ENERGY | N.FFM_GRAD | N.FFM_TIME_NB)
                ev[k][1].record()
            ev[k][2].record()
            ms = np.zeros(1, np.float32)
            N.check(lib.ffm_system_nb_ms(handle, ms.ctypes.data), "nb_ms")
            nb_ms.append(float(ms[0]))
        barrier()
        if clk is not None:
            clk.__exit__(None, None, None)
        launches = lib.ffm_launch_count() - l0
        step_ms = [a.elapsed_time(c) for a, _, c in ev]
        comm_ms = [b.elapsed_time(c) for _, b, c in ev]
        tot, nbm, comm = allmax([float(np.sum(step_ms)), float(np.mean(nb_ms)),
                                 float(np.mean(comm_ms))])
        nb_min = -allmax([-float(np.mean(nb_ms))])[0]
        assert int(st[0]) == -1, "coincident atoms in the benchmark system"
        return tot / steps, nbm, launches, {"sweep_ms_max_rank": nbm, "sweep_ms_min_rank": nb_min,
                                            "allreduce_ms": comm}

    clk = ClockSampler(local)
    ms32, nb32, launches, parts32 = time_device(N.FFM_F32, args.steps, args.warmup, clk)
    clocks = clk.summary()
    ms64, nb64, _, parts64 = time_device(N.FFM_F64, max(3, args.steps // 2), 3)
    value = pairs / (ms32 * 1e-3)

    # ---- e2e through the public API, host buffers (pinned): the objective
    # oracle every minimiser calls (value_and_gradient on a NumPy vector ->
    # (float, NumPy float64 gradient)), copies inside the timed region; FP32
    # mode (the headline) and FP64 (the reference's default dtype)
    pinned = torch.empty(3 * n, dtype=torch.float64).pin_memory()

    def e2e(dtype, steps):
        if sharded:
            from paper_1810_03358_b200.parallel import ShardedMolecularOracle

            orc = ShardedMolecularOracle(s, dtype, device=local, native=native)
        else:
            from paper_1810_03358_b200.oracle import MolecularOracle

            orc = MolecularOracle(s, dtype, device=local)
        times = []
        for k in range(args.warmup + steps):
            pinned.numpy()[:] = steps_coords[k % 4].cpu().numpy().reshape(-1)
            host = pinned.numpy()
            barrier()
            t0 = time.perf_counter()
            f, g = orc.value_and_gradient(host)
            t1 = time.perf_counter()
            assert isinstance(g, np.ndarray) and g.shape == (3 * n,) and np.isfinite(f)
            if k >= args.warmup:
                times.append(t1 - t0)
        return allmax([float(np.mean(times))])[0]

    e2e_s = e2e(np.float32, args.steps)
    e2e64_s = e2e(np.float64, max(3, args.steps // 2))

    measured, fma_peak = peaks()
    flop_peak = 2 * fma_peak
    nb_pairs_per_rank = pairs / world
    achieved = nb_pairs_per_rank * FLOP_PER_PAIR / (nb32 * 1e-3)
    # FMA-pipe fraction: FP32 lane-op slots used per second over the pipe's
    # 128 lane-ops / clk / SM (= fma_peak per second)
    fma_frac = nb_pairs_per_rank * FMA_SLOTS_PER_PAIR / (nb32 * 1e-3) / fma_peak
    api = ("parallel.ShardedMolecularOracle(system, dtype).value_and_gradient(x)" if sharded
           else "oracle.MolecularOracle(system, dtype).value_and_gradient(x)")
    comm = ("none" if not sharded else
            "engine ncclAllReduce (ffm_system_set_comm)" if eng.native else
            f"torch.distributed {backend} all_reduce (parallel.ShardCombiner)")
    line = {
        "metric": METRIC, "value": value, "unit": "pairs/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms32,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32 (pair arithmetic; fp64 accumulation)", "data": "synthetic",
        "config": {"workload": f"energy+gradient of a {n}-atom synthetic protein-like globule "
                               "(LJ + Coulomb all pairs, bonded terms, 1-2/1-3 excluded, 1-4 scaled)",
                   "natoms": n, "pairs_per_step": int(pairs), "parallelism": f"row-shard x{world}",
                   "completion": comm,
                   "l2": "flushed (256 MB write) between timed steps",
                   "inputs": "fresh jittered geometry per step, resident in HBM"},
        "value_f64": pairs / (ms64 * 1e-3), "ms_per_step_f64": ms64,
        "e2e": {"value": pairs / e2e_s, "unit": "pairs/s", "h2d_bytes_per_step": n * 3 * 8,
                "d2h_bytes_per_step": n * 3 * 8 + 5 * 8 + 8 * 8, "api": api.replace("dtype", "np.float32")},
        "e2e_f64": {"value": pairs / e2e64_s, "unit": "pairs/s", "h2d_bytes_per_step": n * 3 * 8,
                    "d2h_bytes_per_step": n * 3 * 8 + 5 * 8 + 8 * 8,
                    "api": api.replace("dtype", "np.float64")},
        "roofline": {"bound": "fp32-fma-pipe", "kernel": "nb_units_kernel<float,GRAD>",
                     "achieved": achieved / 1e12, "peak": flop_peak / 1e12, "unit": "TFLOP/s",
                     "frac": achieved / flop_peak, "traffic": nb_traffic(n),
                     "flop_per_pair": FLOP_PER_PAIR, "fma_pipe_frac": fma_frac,
                     "nb_ms": nb32, "nb_ms_f64": nb64,
                     "frac_of_nominal": achieved / NOMINAL_FP32_FLOPS,
                     "mix_ceiling": {"fma_pipe_active_tile_loop_alone": MIX_CEILING["fp32_fma_pipe_active"],
                                     "fma_pipe_active_sweep": SWEEP_NCU["fp32_fma_pipe_active"],
                                     "source": "ncu, profiles/r02_pipes_microbench.txt: the sweep's "
                                               "tile loop in isolation keeps the FMA pipe 78.8% "
                                               "busy; the 100k sweep 75.6%"},
                     "peak_source": "measured FFMA throughput, profiles/r01_pipes_microbench.txt "
                                    "(MEASURED_PEAKS.json has no FP32 figure); frac_of_nominal: "
                                    "128 FMA/clk/SM x 148 SMs x 1965 MHz = 74.4 TFLOP/s",
                     "bound_note": "not a dense contraction (north star): the pair sweep is bound "
                                   "by the FP32 FMA pipe; DRAM traffic is under 2% of its time "
                                   "and tensor cores do not apply"},
        "roofline_f64": {"bound": "fp64-pipe", "kernel": "nb_units_kernel<double,GRAD>",
                         "achieved": nb_pairs_per_rank * FP64_OPS_PER_PAIR / (nb64 * 1e-3) / 1e12,
                         "peak": DFMA_PEAK / 1e12, "unit": "T fp64-pipe ops/s",
                         "frac": nb_pairs_per_rank * FP64_OPS_PER_PAIR / (nb64 * 1e-3) / DFMA_PEAK,
                         "ops_per_pair": FP64_OPS_PER_PAIR, "nb_ms": nb64,
                         "mix_ceiling": {"fp64_pipe_active_tile_loop_alone": MIX_CEILING["fp64_pipe_active"],
                                         "fp64_pipe_active_sweep": SWEEP_NCU["fp64_pipe_active"],
                                         "source": "ncu, profiles/r02_pipes_microbench.txt"}},
        "gpu_launches": int(launches),
        "clocks": clocks,
    }
    if sharded:
        line["shards"] = {"f32": parts32, "f64": parts64,
                          "note": "per-rank partial evaluation (sweep) and its completion "
                                  "(all-reduce of 24n + 104 bytes) timed apart, max over ranks"}
        if shared:
            line["shards"]["shared_gpu"] = (f"{world} ranks on {ngpu} GPU(s): testing run, "
                                            "not a scaling measurement")
    if rank == 0 and world == 1:
        line["cpu_baseline"] = cpu_baseline(s)
    if not args.no_extras:
        extras = run_extras(rank, world, local, native)
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


def run_extras(rank, world, local, native=False):
    """Secondary BASELINE configs, bounded (about two minutes with the
    same-run CPU minimiser timings)."""
    import torch

    from paper_1810_03358_b200 import _native as N
    from paper_1810_03358_b200.engine import DeviceSystem
    from paper_1810_03358_b200.synth import make_globule_system

    out = {}
    dev = torch.device("cuda", local)
    if world > 1:
        # configs[4]: L-BFGS on the 100k-atom system, row-sharded over the ranks
        out["lbfgs_100k"] = optimizer_comparison(100000, iters=10, methods=("lbfgs",),
                                                 dtype=np.float32, sharded=True, native=native,
                                                 cpu_iters=0)
        return out
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
    bc = {"candidates": B, "natoms": 5000, "what": "energy only"}
    for prec, tag in ((N.FFM_F32, "f32"), (N.FFM_F64, "f64")):
        for _ in range(2):
            eng.eval_batch(batch, prec, energies=en, status=st)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            eng.eval_batch(batch, prec, energies=en, status=st)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        bc[tag] = {"ms_per_step": ms, "pairs_per_s": B * 5000 * 4999 / 2 / (ms * 1e-3)}
    out["batched_candidates"] = bc
    eng.close()
    # configs[0]: L-BFGS time-to-converge beside the CPU port, same run
    out["lbfgs_converge"] = lbfgs_converge()
    # configs[2]: optimiser comparison on a 10k-atom globule
    out["optimizer_comparison_10k"] = optimizer_comparison(10000, iters=100, cpu_iters=3)
    # configs[4]: L-BFGS iterations on the 100k-atom system (1 GPU)
    out["lbfgs_100k"] = optimizer_comparison(100000, iters=10, methods=("lbfgs",),
                                             dtype=np.float32, cpu_iters=1)
    out["shard_compute_100k"] = shard_compute(local)
    return out


def shard_compute(local, n=100_000):
    """configs[4] on one GPU: every rank's partial FP32 evaluation of a W-way
    row-sharded 100k plan (ffm_system_set_shard), timed alone with CUDA
    events -- the compute each GPU of a W-GPU job runs, without the
    all-reduce (24n bytes per evaluation) and without waiting on other
    ranks."""
    import torch

    from paper_1810_03358_b200 import _native as N
    from paper_1810_03358_b200.engine import DeviceSystem
    from paper_1810_03358_b200.synth import make_globule_system

    s = make_globule_system(n, seed=0)
    dev = torch.device("cuda", local)
    c = torch.from_numpy(np.array(s.coords)).to(dev)
    g = torch.empty_like(c)
    eng = DeviceSystem(s.topology, local)
    en, st = eng.new_outputs()
    out = {"natoms": n, "what": "per-rank partial evaluation (FP32 energy+gradient), ms, "
                                "each rank's share timed alone on one GPU; no collective"}
    for W in (1, 2, 4, 8):
        ms = []
        for rank in range(W):
            N.check(eng.lib.ffm_system_set_shard(eng.handle, rank, W), "set_shard")
            for _ in range(2):
                eng.eval(c, N.FFM_F32, grad=g, energies=en, status=st)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                eng.eval(c, N.FFM_F32, grad=g, energies=en, status=st)
            e1.record()
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1) / 5)
        out[f"W{W}"] = {"max_rank_ms": max(ms), "min_rank_ms": min(ms)}
    eng.close()
    return out


def cpu_lbfgs_per_iteration(system, iters):
    """The CPU port of the reference L-BFGS (oracle/optim.py over the C
    restatement of kernels.py, FP64, all host threads) timed on this box in
    the same run: seconds per iteration = (T(iters) - T(start point only)) /
    iters, bounded to a few iterations."""
    import oracle as O
    import oracle.optim as OO

    A = O.Arrays.from_system(system)
    th = O.host_threads()
    x0 = system.coords.ravel()
    t0 = time.perf_counter()
    OO.lbfgs(A, x0, m=5, max_iterations=0, threads=th)
    t1 = time.perf_counter()
    r = OO.lbfgs(A, x0, m=5, max_iterations=iters, threads=th)
    t2 = time.perf_counter()
    per = ((t2 - t1) - (t1 - t0)) / max(1, r["iterations"])
    return {"ms_per_iteration": per * 1e3, "iterations": r["iterations"], "cores": th,
            "kind": "port", "precision": "f64",
            "what": "oracle/optim.py L-BFGS (ffmin/optimizers/lbfgs.py restated) on "
                    "oracle/ffmin_oracle.c, ls_par, m=5"}


def optimizer_comparison(natoms, iters, methods=("sd", "fgm", "cg", "lbfgs", "wiggle"),
                         dtype=np.float64, sharded=False, native=False, cpu_iters=0):
    """Every minimiser from the same perturbed start with the same iteration
    budget: final energy, calls and wall time (device-resident iterates);
    the CPU port's L-BFGS per-iteration time beside it (cpu_iters > 0)."""
    import torch

    from paper_1810_03358_b200.oracle import MolecularOracle
    from paper_1810_03358_b200.optimizers import StopCriteria, cg, fgm, lbfgs, make_linesearch
    from paper_1810_03358_b200.optimizers import steepest_descent
    from paper_1810_03358_b200.optimizers.wiggle import WiggleConfig, atom_wiggle
    from paper_1810_03358_b200.parallel import ShardedMolecularOracle
    from paper_1810_03358_b200.synth import make_globule_system

    s = make_globule_system(natoms, seed=1)
    out = {"natoms": natoms, "iterations_budget": iters,
           "precision": "f32" if dtype == np.float32 else "f64"}

    def oracle():
        if sharded:
            return ShardedMolecularOracle(s, dtype=dtype, native=native)
        return MolecularOracle(s, dtype=dtype)

    def drive(name, o, ls, stop):
        x0 = s.coords.ravel()
        if name == "sd":
            return steepest_descent(o, x0, ls, stop)
        if name == "fgm":
            return fgm(o, x0, ls, stop)
        if name == "cg":
            return cg(o, x0, "prp+", ls, stop)
        return lbfgs(o, x0, m=5, linesearch=ls, stop=stop)

    for name in methods:
        stop = StopCriteria(max_iterations=iters, gradient_norm_rtol=1e-6)
        if name == "wiggle":
            # gradient-free: one probe batch per atom move, 20 moves per
            # budget unit; a short warm-up run captures its graph first
            atom_wiggle(s, WiggleConfig(seed=0),
                        StopCriteria(max_iterations=40, gradient_norm_rtol=0.0))
            # median of three identical runs: single runs of this
            # host-polled loop (one poll per 64 iterations) occasionally
            # take 2-3x longer on a shared host (tools/time_wiggle.py)
            dts = []
            for _ in range(3):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                res = atom_wiggle(s, WiggleConfig(seed=0),
                                  StopCriteria(max_iterations=iters * 20, gradient_norm_rtol=0.0))
                torch.cuda.synchronize()
                dts.append(time.perf_counter() - t0)
            dt = sorted(dts)[1]
            calls, gcalls = res.trace.records[-1].value_calls, 0
        else:
            o = oracle()
            ls = make_linesearch("par")
            # warm-up: capture the method's graph outside the timing
            drive(name, o, ls, StopCriteria(max_iterations=2, gradient_norm_rtol=1e-6))
            o.value_calls = o.grad_calls = 0
            ls.reset()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            res = drive(name, o, ls, stop)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            calls, gcalls = o.value_calls, o.grad_calls
        out[name] = {"f": float(res.f), "iterations": int(res.iterations), "status": res.status,
                     "value_calls": int(calls), "grad_calls": int(gcalls), "seconds": dt,
                     "ms_per_iteration": dt / max(1, res.iterations) * 1e3}
    out["f_start"] = float(oracle().value(s.coords.ravel()))
    if sharded:
        out["completion"] = "device ncclAllReduce" if native else "torch.distributed all_reduce"
    if cpu_iters > 0:
        out["cpu_lbfgs"] = cpu_lbfgs_per_iteration(s, cpu_iters)
    return out


def lbfgs_converge():
    """configs[0]: L-BFGS minimisation from a perturbed start, FP64, on the
    golden cases (tests/golden/make_golden.py): the bounded 500-atom chain run
    (lbfgs500), the converged 500-atom run (conv500) and the converged
    60/200-atom chains, each beside the CPU port of the reference driver
    (oracle/optim.py on the C oracle, one thread: at 500 atoms more threads
    only add synchronisation) timed in the same run."""
    import torch

    import oracle as O
    import oracle.optim as OO
    from paper_1810_03358_b200.model import MolecularSystem
    from paper_1810_03358_b200.oracle import MolecularOracle
    from paper_1810_03358_b200.optimizers import StopCriteria, lbfgs, make_linesearch

    G = np.load(ROOT / "tests" / "golden" / "golden_v1.npz")
    out = {}
    for name in ("lbfgs500", "conv500", "conv60", "conv200"):
        if f"{name}/q" not in G:
            continue
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
            m, max_it, gtol = 3, 300, 1e-3
        else:
            ref_f, _, ref_it, gtol = G[f"{name}/final"]
            m, max_it = 5, 50000
        stop = StopCriteria(max_iterations=max_it, gradient_norm_tol=gtol, gradient_norm_rtol=0.0)
        lbfgs(MolecularOracle(s), s.coords.ravel(), m=m, linesearch=make_linesearch("par"),
              stop=StopCriteria(max_iterations=3, gradient_norm_rtol=0.0))  # warm-up
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = lbfgs(MolecularOracle(s), s.coords.ravel(), m=m, linesearch=make_linesearch("par"),
                    stop=stop)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        A = O.Arrays.from_system(s)
        t1 = time.perf_counter()
        cpu = OO.lbfgs(A, s.coords.ravel(), m=m, max_iterations=max_it, gtol=gtol, threads=1)
        t2 = time.perf_counter()
        out[name] = {"natoms": s.natoms, "iterations": res.iterations, "status": res.status,
                     "f": res.f, "ref_f": float(ref_f), "ref_iterations": int(ref_it),
                     "rel_diff_f": abs(res.f - ref_f) / abs(ref_f), "seconds": dt,
                     "cpu_port": {"seconds": t2 - t1, "iterations": cpu["iterations"],
                                  "f": cpu["f"], "status": cpu["status"], "cores": 1,
                                  "kind": "port"}}
        if name == "lbfgs500":
            # a bounded run on a nonconvex surface: the trace follows the
            # reference's until roundoff picks another basin; the reference
            # itself (numba vs numpy backends, same run) agrees only for
            # G["lbfgs500/self_horizon"] records (make_golden.py)
            f = np.array([r.f for r in res.trace.records])
            ref = G[f"{name}/f_trace"]
            k = min(len(f), len(ref))
            bad = np.nonzero(np.abs(f[:k] - ref[:k]) > 1e-8 * np.abs(ref[:k]))[0]
            out[name]["trace_matches_reference_iterations"] = int(bad[0]) if len(bad) else k
            if f"{name}/self_horizon" in G:
                out[name]["reference_self_horizon"] = int(G[f"{name}/self_horizon"])
            out[name]["note"] = ("unconverged nonconvex run: final f differs by basin, "
                                 "not a parity criterion; conv500 is the converged check")
    return out


if __name__ == "__main__":
    main()
