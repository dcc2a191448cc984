"""Objective oracles: the only interface optimizers see (mirrors ffmin/oracle.py).

Call accounting is identical to the reference: value(), gradient() and
value_and_gradient() each bump their counters, a fused call bumps both.

``MolecularOracle`` evaluates on the device and takes either NumPy arrays
(reference-facing) or cuda tensors (device-resident); the optimisers always
drive it with device vectors.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native as N
from .energy import raise_status
from .engine import engine_for, precision_of


class ObjectiveOracle:
    """Base class; subclasses implement _value/_gradient/_value_and_gradient."""

    #: vectors this oracle consumes: "host" (NumPy) or "device" (torch cuda)
    space = "host"

    def __init__(self, n):
        self.n = int(n)
        self.value_calls = 0
        self.grad_calls = 0

    def reset_counters(self):
        self.value_calls = 0
        self.grad_calls = 0

    def value(self, x) -> float:
        self.value_calls += 1
        return float(self._value(self._coerce(x)))

    def gradient(self, x):
        self.grad_calls += 1
        return self._out(self._gradient(self._coerce(x)))

    def value_and_gradient(self, x):
        self.value_calls += 1
        self.grad_calls += 1
        f, g = self._value_and_gradient(self._coerce(x))
        return float(f), self._out(g)

    def _coerce(self, x):
        return np.asarray(x, dtype=np.float64)

    def _out(self, g):
        return np.asarray(g, dtype=np.float64)

    def _value_and_gradient(self, x):
        return self._value(x), self._gradient(x)

    def _value(self, x):
        raise NotImplementedError

    def _gradient(self, x):
        raise NotImplementedError


class FunctionOracle(ObjectiveOracle):
    """Wrap plain callables f(x) and optionally g(x) (ffmin/oracle.py:53-73)."""

    def __init__(self, n, f, grad=None, value_and_grad=None):
        super().__init__(n)
        self._f = f
        self._g = grad
        self._fg = value_and_grad

    def _value(self, x):
        return self._f(x)

    def _gradient(self, x):
        if self._g is None:
            raise NotImplementedError("no gradient supplied for this oracle")
        return self._g(x)

    def _value_and_gradient(self, x):
        if self._fg is not None:
            return self._fg(x)
        return super()._value_and_gradient(x)


class MolecularOracle(ObjectiveOracle):
    """Total force-field energy as a function of flattened coordinates
    (ffmin/oracle.py:76-103), evaluated on the device.

    Accepts NumPy arrays (reference-facing: gradients come back as float64
    NumPy arrays, f as a Python float) or cuda float64 tensors (device-
    resident: gradients stay in HBM).  ``space == "device"``, so every
    optimiser driven by it keeps x, g and its vector algebra on the GPU;
    only the 5 energy terms and 8 status words (104 bytes) come back per
    evaluation.  dtype selects the kernel precision; values and gradients
    at the oracle boundary are always float64, as in the reference.
    """

    space = "device"

    def __init__(self, system, dtype=np.float64, backend=None, device=None):
        super().__init__(3 * system.natoms)
        from .energy import _check_backend

        _check_backend(backend)
        self.system = system
        self.dtype = np.dtype(dtype)
        self.backend = backend
        self.precision = precision_of(self.dtype)
        self.engine = engine_for(system.topology, device, precision=self.precision)
        self.device = self.engine.device
        n = system.natoms
        # fixed device buffers: every evaluation replays the same captured
        # CUDA graph (engine.ffm_eval); results: 5 energies + 8 status words
        # in one 104-byte block, read back with a single copy
        self._x = torch.empty((n, 3), dtype=torch.float64, device=self.device)
        self._g = torch.empty((n, 3), dtype=torch.float64, device=self.device)
        self._res = torch.empty(N.FFM_NTERMS + N.FFM_STATUS_WORDS, dtype=torch.float64,
                                device=self.device)
        self._en = self._res[:N.FFM_NTERMS]
        self._st = self._res[N.FFM_NTERMS:].view(torch.int64)
        self._host = torch.empty(N.FFM_NTERMS + N.FFM_STATUS_WORDS, dtype=torch.float64,
                                 pin_memory=True)
        self._host_io = False
        self.last_breakdown = None
        self.evaluations = 0

    def system_at(self, x):
        if isinstance(x, torch.Tensor):
            x = x.detach().cpu().numpy()
        return self.system.with_coords(np.asarray(x, dtype=np.float64))

    def initial_point(self):
        """x0 of the wrapped system as a device vector."""
        return torch.from_numpy(np.array(self.system.coords, dtype=np.float64).reshape(-1)).to(
            self.device)

    def _coerce(self, x):
        if isinstance(x, torch.Tensor):
            self._host_io = False
            if x.device != self.device or x.dtype != torch.float64:
                x = x.to(device=self.device, dtype=torch.float64)
            return x.reshape(-1).contiguous()
        self._host_io = True
        x = np.ascontiguousarray(x, dtype=np.float64).reshape(-1)
        if x.shape[0] != self.n:
            raise ValueError(f"x must have {self.n} entries, got {x.shape[0]}")
        return x

    def _out(self, g):
        return g  # _run already produced the caller's kind of vector

    def _run(self, x, grad):
        # host vectors: one H2D copy straight into the evaluation buffer and
        # one D2H copy of the gradient into a fresh page-locked array (from
        # torch's caching host allocator: DMA at full speed, no staging; the
        # NumPy array owns it), the 104-byte result block alongside; one
        # synchronisation for both
        host = isinstance(x, np.ndarray)
        if host and not x.flags.writeable:
            x = x.copy()  # torch.from_numpy warns on read-only arrays
        self._x.view(-1).copy_(torch.from_numpy(x) if host else x)
        self.engine.eval(self._x, self.precision, grad=self._g if grad else None,
                         energies=self._en, status=self._st)
        self._host.copy_(self._res, non_blocking=True)
        g_out = None
        if grad and host:
            gp = torch.empty(self.n, dtype=torch.float64, pin_memory=True)
            gp.copy_(self._g.view(-1), non_blocking=True)
            g_out = gp.numpy()
        torch.cuda.current_stream(self.device).synchronize()
        vals = self._host.numpy()
        en = vals[:N.FFM_NTERMS].copy()
        st = vals[N.FFM_NTERMS:].view(np.int64).copy()
        self.evaluations += 1
        raise_status(self.system, st, grad=grad)
        self.last_breakdown = en
        # EnergyBreakdown.total order (ffmin/energy.py:38-41)
        f = float(en[0]) + float(en[1]) + float(en[2]) + float(en[3]) + float(en[4])
        if grad and not host:
            g_out = self._g.view(-1).clone()
        return f, g_out

    def _value(self, x):
        return self._run(x, False)[0]

    def _gradient(self, x):
        return self._run(x, True)[1]

    def _value_and_gradient(self, x):
        return self._run(x, True)


# the device-resident oracle is the molecular oracle
DeviceMolecularOracle = MolecularOracle
