"""Vector spaces the optimisers run in.

The reference drivers hold x, g, directions and L-BFGS pairs as NumPy arrays
(ffmin/optimizers/*.py).  Here every driver is written once against a small
vector-algebra interface with two implementations:

  * ``DeviceOps`` -- cuda float64 tensors; dot / axpby / the L-BFGS two-loop
    run in the engine's own kernels (csrc/ffm_vec.cu, through the C ABI),
    deterministic fixed-order reductions, nothing leaves HBM except the
    scalars the control flow needs;
  * ``HostOps``   -- NumPy, for objectives defined on the host (the
    synthetic quadratic benchmarks, user callables).  It is not a fallback
    of the device path: a molecular oracle always selects DeviceOps.
"""

from __future__ import annotations

import ctypes as C
import math

import numpy as np


class HostOps:
    space = "host"

    def asvec(self, x):
        return np.array(x, dtype=np.float64).reshape(-1)

    def copy(self, x):
        return np.array(x, dtype=np.float64, copy=True)

    def zeros_like(self, x):
        return np.zeros_like(x)

    def dot(self, a, b) -> float:
        return float(a @ b)

    def dots(self, pairs):
        return [float(a @ b) for a, b in pairs]

    def norm(self, a) -> float:
        return float(np.linalg.norm(a))

    def lincomb(self, a, x, b=0.0, y=None):
        """a x + b y (new vector)."""
        return a * x if y is None else a * x + b * y

    def div(self, x, a):
        """x / a (the reference normalises by division)."""
        return x / a

    def all_finite(self, x) -> bool:
        return bool(np.all(np.isfinite(x)))

    def to_host(self, x):
        return np.array(x, dtype=np.float64, copy=True)

    def two_loop(self, S, Y, rho, g):
        """Algorithm 3 (ffmin/optimizers/lbfgs.py:53-75) on lists of pairs,
        oldest first."""
        q = g.copy()
        alpha = [0.0] * len(S)
        for i in range(len(S) - 1, -1, -1):
            alpha[i] = rho[i] * float(S[i] @ q)
            q -= alpha[i] * Y[i]
        q *= float(S[-1] @ Y[-1]) / float(Y[-1] @ Y[-1])
        for i in range(len(S)):
            b = rho[i] * float(Y[i] @ q)
            q += (alpha[i] - b) * S[i]
        return -q


class DeviceOps:
    """cuda float64 vectors; algebra through the engine's C ABI."""

    space = "device"

    def __init__(self, device=None):
        import torch

        from . import _native as N

        self.torch = torch
        self.N = N
        self.lib = N.load()
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None
                                   else torch.device(device).index or 0)
        nscr = int(self.lib.ffm_vec_scratch_doubles())
        self._scratch = torch.empty(nscr, dtype=torch.float64, device=self.device)
        self._outs = torch.empty(8, dtype=torch.float64, device=self.device)
        self._host_outs = torch.empty(8, dtype=torch.float64, pin_memory=True)

    def _s(self):
        return C.c_void_p(self.torch.cuda.current_stream(self.device).cuda_stream)

    @staticmethod
    def _p(t):
        return C.c_void_p(t.data_ptr())

    def asvec(self, x):
        t = self.torch
        if isinstance(x, t.Tensor):
            return x.to(device=self.device, dtype=t.float64).reshape(-1).clone()
        return t.from_numpy(np.array(x, dtype=np.float64).reshape(-1)).to(self.device)

    def copy(self, x):
        return x.clone()

    def zeros_like(self, x):
        return self.torch.zeros_like(x)

    def dots(self, pairs):
        """Several dot products: one kernel pass, one host readback."""
        out = []
        for k0 in range(0, len(pairs), 8):
            chunk = pairs[k0:k0 + 8]
            k = len(chunk)
            xs = (C.c_void_p * k)(*[a.data_ptr() for a, _ in chunk])
            ys = (C.c_void_p * k)(*[b.data_ptr() for _, b in chunk])
            self.N.check(self.lib.ffm_dots(chunk[0][0].numel(), k, xs, ys, self._p(self._outs),
                                           self._p(self._scratch), self._s()), "ffm_dots")
            self._host_outs.copy_(self._outs)
            out.extend(self._host_outs[:k].tolist())
        return out

    def dot(self, a, b) -> float:
        return self.dots([(a, b)])[0]

    def norm(self, a) -> float:
        return math.sqrt(self.dot(a, a))

    def lincomb(self, a, x, b=0.0, y=None):
        z = self.torch.empty_like(x)
        self.N.check(self.lib.ffm_axpby(x.numel(), None, float(a), 1.0, self._p(x), None,
                                        float(b), None if y is None else self._p(y),
                                        self._p(z), self._s()), "ffm_axpby")
        return z

    def div(self, x, a):
        return self.lincomb(1.0 / a, x)

    def all_finite(self, x) -> bool:
        return bool(self.torch.isfinite(x).all().item())

    def to_host(self, x):
        return x.detach().cpu().numpy().astype(np.float64, copy=True)

    def two_loop(self, S, Y, rho, g):
        """Algorithm 3 in one cooperative kernel; S, Y: lists of device
        vectors, oldest first (views into the ring buffers)."""
        count = len(S)
        if count == 0:
            raise ValueError("two_loop needs at least one pair")
        # the kernel takes ring slots newest first: pass a stacked view
        base_s, base_y, slots = self._ring_view(S, Y)
        order = (C.c_int32 * count)(*slots[::-1])
        rh = (C.c_double * count)(*rho[::-1])
        d = self.torch.empty_like(g)
        self.N.check(self.lib.ffm_lbfgs_two_loop(g.numel(), count, order, rh, self._p(base_s),
                                                 self._p(base_y), self._p(g), self._p(d),
                                                 self._p(self._scratch), self._s()),
                     "ffm_lbfgs_two_loop")
        return d

    @staticmethod
    def _ring_view(S, Y):
        """(S base tensor, Y base tensor, slot index of each pair) when the
        pairs are rows of two [m, n] ring buffers (LbfgsMemory stores them so)."""
        s0, y0 = S[0], Y[0]
        bs = s0._base if s0._base is not None else s0
        by = y0._base if y0._base is not None else y0
        n = s0.numel()
        slots = []
        for s, y in zip(S, Y):
            ks = (s.data_ptr() - bs.data_ptr()) // (8 * n)
            ky = (y.data_ptr() - by.data_ptr()) // (8 * n)
            if ks != ky:
                raise ValueError("s and y pairs must share a ring slot")
            slots.append(int(ks))
        return bs, by, slots


def ops_for(oracle):
    """The vector space an oracle's points live in."""
    if getattr(oracle, "space", "host") == "device":
        dev = getattr(oracle, "device", None)
        return DeviceOps(dev)
    return HostOps()
