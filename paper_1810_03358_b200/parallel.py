"""Row-sharded evaluation over the GPUs of one node (one process per GPU).

The pair triangle is cut into S x S super-units (csrc/ffm_capi.cu); rank r
of W evaluates the units u = r, r + W, r + 2W, ... (heaviest first, so every
rank gets the same work to within one unit) and rank 0 also the O(N) bonded
and 1-4 terms.  Each rank therefore produces a *partial* gradient over all
atoms and partial energies; one NCCL all-reduce (SUM) of the packed
[gradient | energies | error words] vector over NVLink completes them on
every rank.  The error words ride in the same sum: a rank that reports an
error contributes (key + 1, 1), the others (0, 0), and every reporting rank
reports the same key -- bonded terms are evaluated by rank 0 alone, and a
coincident pair is located by the finder over the whole triangle (every
rank holds all coordinates), so any rank that flags one finds the same,
globally first pair; key = sum / count - 1 is exact in float64 (keys <
2^53 / W).  Coordinates are
replicated: every rank runs the same optimiser on the same all-reduced
numbers, so no broadcast is needed per step.

Completion, two ways:

* ``ShardCombiner`` (the default): the engine's partial sums, then one
  ``torch.distributed.all_reduce`` of the packed vector on the evaluation's
  stream (NCCL over NVLink, or gloo).  Tested across processes: gloo world 2
  on CPU (tests/test_parallel_cpu.py) and two processes sharing one GPU with
  the real CUDA shards (tests/test_sharded_gpu.py).
* native (opt-in: ``native=True`` or FFMIN_B200_NATIVE_COMM=1, NCCL groups
  only): the group's communicator is attached to the engine
  (ffm_system_set_comm) and every evaluation ends with encode /
  ncclAllReduce / decode kernels on its stream, so the graph-resident
  drivers capture the all-reduce too.  Exercised on one GPU with a one-rank
  group only (a second rank needs a second GPU: NCCL refuses two ranks on
  one device), hence not the default.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch
import torch.distributed as dist

from . import _native as N



def shard_units(nunits: int, rank: int, world: int):
    """The unit indices rank `rank` evaluates (mirrors ffm_system_set_shard)."""
    return list(range(rank, nunits, world))


def unit_order(nb: int):
    """(r, c) of every unit in evaluation order: off-diagonal first, then the
    diagonal (mirrors ffm_system_create)."""
    off = [(r, c) for r in range(nb) for c in range(r + 1, nb)]
    return off + [(r, r) for r in range(nb)]


class ShardCombiner:
    """All-reduce of one rank's partial evaluation (one collective)."""

    SLOTS = (N.ST_NB_BAD_I, N.ST_BOND, N.ST_ANGLE, N.ST_DIHEDRAL)

    def __init__(self, n, device, group=None):
        self.n = n
        self.group = group
        # [gradient (3n) | energies (5) | error (key + 1) x 4 | reporting ranks x 4]
        self.buf = torch.empty(3 * n + N.FFM_NTERMS + 8, dtype=torch.float64, device=device)

    def combine(self, grad, energies, status):
        """grad (3n,) or None, energies (5,), status (8,) int64 -- local
        partials in, global values out (in place on grad/energies/status)."""
        n3, ne = 3 * self.n, N.FFM_NTERMS
        b = self.buf
        if grad is not None:
            b[:n3].copy_(grad.reshape(-1))
        else:
            b[:n3].zero_()
        b[n3:n3 + ne].copy_(energies)
        st = status
        # error keys: the first coincident pair as i * n + j, the first bad
        # bond / angle / dihedral; -1 = clean
        keys = torch.stack([torch.where(st[N.ST_NB_BAD_I] >= 0,
                                        st[N.ST_NB_BAD_I] * self.n + st[N.ST_NB_BAD_J],
                                        st[N.ST_NB_BAD_I]),
                            st[N.ST_BOND], st[N.ST_ANGLE], st[N.ST_DIHEDRAL]])
        rep = keys >= 0
        b[n3 + ne:n3 + ne + 4].copy_(torch.where(rep, keys + 1, 0))
        b[n3 + ne + 4:].copy_(rep)
        dist.all_reduce(b, op=dist.ReduceOp.SUM, group=self.group)
        if grad is not None:
            grad.reshape(-1).copy_(b[:n3])
        energies.copy_(b[n3:n3 + ne])
        cnt = b[n3 + ne + 4:]
        key = torch.where(cnt > 0, torch.round(b[n3 + ne:n3 + ne + 4] / cnt.clamp(min=1.0)) - 1,
                          -1.0).to(torch.int64)
        k0 = key[0]
        st[N.ST_NB_BAD_I].copy_(torch.where(k0 >= 0, k0 // self.n, -1))
        st[N.ST_NB_BAD_J].copy_(torch.where(k0 >= 0, k0 % self.n, -1))
        st[N.ST_BOND:N.ST_DIHEDRAL + 1].copy_(key[1:])
        return grad, energies, status


class ShardedSystem:
    """This rank's engine handle (a private DeviceSystem with a shard) plus
    the completion of its partial evaluations: on the device (the group's
    NCCL communicator attached to the engine, ffm_system_set_comm: one
    all-reduce inside every evaluation, capturable in the graph-resident
    drivers) or, for other backends, by ShardCombiner from Python."""

    def __init__(self, topo, group=None, device=None, native=None):
        import os

        from .engine import DeviceSystem

        if native is None:
            native = os.environ.get("FFMIN_B200_NATIVE_COMM", "") == "1"

        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.engine = DeviceSystem(topo, device)
        N.check(self.engine.lib.ffm_system_set_shard(self.engine.handle, self.rank, self.world),
                "ffm_system_set_shard")
        self.n = topo.natoms
        self.device = self.engine.device
        self.handle = self.engine.handle
        self.lib = self.engine.lib
        self.combiner = ShardCombiner(self.n, self.device, group)
        self.native = native and self._attach_comm(group)

    def _attach_comm(self, group):
        """The group's ncclComm_t, if its backend is NCCL (created eagerly
        by a one-element all-reduce)."""
        try:
            pg = group if group is not None else dist.distributed_c10d._get_default_group()
            probe = torch.zeros(1, device=self.device)
            dist.all_reduce(probe, group=group)
            backend = pg._get_backend(self.device)
            ptr = int(backend._comm_ptr())
        except Exception:
            return False
        if not ptr:
            return False
        return self.engine.lib.ffm_system_set_comm(self.handle, C.c_void_p(ptr)) == 0

    def new_outputs(self):
        return self.engine.new_outputs()

    def eval(self, coords, precision=N.FFM_F64, grad=None, energies=None, status=None,
             flags=None):
        energies, status = self.engine.eval(coords, precision, grad=grad, energies=energies,
                                            status=status, flags=flags)
        if not self.native:
            self.combiner.combine(grad, energies, status)
        return energies, status


class ShardedMolecularOracle:
    """MolecularOracle over row-sharded GPUs: same interface and call
    accounting, every rank sees identical (all-reduced) values."""

    space = "device"

    def __init__(self, system, dtype=np.float64, group=None, device=None, native=None):
        from .engine import precision_of
        from .oracle import MolecularOracle

        self._base = MolecularOracle.__new__(MolecularOracle)
        MolecularOracle.__init__(self._base, system, dtype, device=device)
        self._base.engine = ShardedSystem(system.topology, group, device, native)
        self.system = system
        self.n = 3 * system.natoms
        self.device = self._base.device
        self.precision = precision_of(dtype)
        self.group = group
        self._t = torch.zeros(1, dtype=torch.float64, device=self.device)

    def agreed_elapsed(self, t):
        """MAX of the ranks' elapsed wall times (one all-reduce), so that a
        max_wall_time budget stops every rank at the same iteration: a rank
        that stopped alone would leave the others waiting in the next
        evaluation's collective."""
        self._t.fill_(float(t))
        dist.all_reduce(self._t, op=dist.ReduceOp.MAX, group=self.group)
        return float(self._t.item())

    def __getattr__(self, name):
        return getattr(self._base, name)

    @property
    def value_calls(self):
        return self._base.value_calls

    @value_calls.setter
    def value_calls(self, v):
        self._base.value_calls = v

    @property
    def grad_calls(self):
        return self._base.grad_calls

    @grad_calls.setter
    def grad_calls(self, v):
        self._base.grad_calls = v

    @property
    def native(self):
        """Evaluations complete on the device (graph-resident drivers apply)."""
        return self._base.engine.native

    def value(self, x):
        return self._base.value(x)

    def gradient(self, x):
        return self._base.gradient(x)

    def value_and_gradient(self, x):
        return self._base.value_and_gradient(x)


def init_from_env(backend="nccl"):
    """torchrun-style initialisation (RANK / WORLD_SIZE / LOCAL_RANK /
    MASTER_ADDR); returns (rank, world, local_rank)."""
    import os

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and not dist.is_initialized():
        if backend == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    return rank, world, local
