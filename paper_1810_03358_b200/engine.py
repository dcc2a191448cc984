"""Device-resident engine: one HBM plan per (topology, device).

``DeviceSystem`` owns an ``ffm_system`` handle (include/ffmin_b200.h) built
from a ``model.Topology``; all geometries of that topology -- every point an
optimiser visits -- are evaluated against it.  Device buffers are PyTorch
tensors (PyTorch is only the allocator / stream provider here); the arithmetic
is the CUDA code in csrc/.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np
import torch

from . import _native as N

PRECISIONS = {np.dtype(np.float64): N.FFM_F64, np.dtype(np.float32): N.FFM_F32}


def precision_of(dtype) -> int:
    if isinstance(dtype, int) and dtype in (N.FFM_F64, N.FFM_F32):
        return dtype
    if isinstance(dtype, torch.dtype):
        dtype = {torch.float64: np.float64, torch.float32: np.float32}.get(dtype, dtype)
    try:
        return PRECISIONS[np.dtype(dtype)]
    except (KeyError, TypeError):
        raise ValueError(f"unsupported kernel dtype {dtype!r} (use float64 or float32)") from None


def require_cuda():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1810_03358_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU execution path")


def _stream_ptr(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _p(a):
    return None if a is None else C.c_void_p(N.ptr(a))


class DeviceSystem:
    """HBM-resident plan of one topology on one CUDA device."""

    def __init__(self, topo, device=None):
        require_cuda()
        self.lib = N.load()
        dev = torch.device("cuda", torch.cuda.current_device() if device is None else
                           (device.index if isinstance(device, torch.device) else int(device)))
        self.device = dev
        self.n = topo.natoms
        h = C.c_void_p()
        si = np.ascontiguousarray(topo.special_i, dtype=np.int64)
        sj = np.ascontiguousarray(topo.special_j, dtype=np.int64)
        ss = np.ascontiguousarray(topo.special_s, dtype=np.float64)
        cutoff = -1.0 if topo.cutoff is None else float(topo.cutoff)
        with torch.cuda.device(dev):
            N.check(self.lib.ffm_system_create(
                C.byref(h), dev.index, self.n, _p(topo.q), _p(topo.sigma), _p(topo.epsilon),
                len(ss), _p(si), _p(sj), _p(ss), cutoff), "ffm_system_create")
            self.handle = h
            N.check(self.lib.ffm_system_set_terms(
                h, len(topo.bond_K), _p(topo.bond_idx), _p(topo.bond_K), _p(topo.bond_r0),
                len(topo.ang_K), _p(topo.ang_idx), _p(topo.ang_K), _p(topo.ang_t0),
                len(topo.dih_V), _p(topo.dih_idx), _p(topo.dih_V)), "ffm_system_set_terms")
        self.refresh_info()
        self._lock = threading.Lock()
        # host-path result buffers
        self._h_en = np.zeros(N.FFM_NTERMS)
        self._h_st = np.zeros(N.FFM_STATUS_WORDS, np.int64)

    def refresh_info(self):
        info = np.zeros(8, np.int64)
        N.check(self.lib.ffm_system_info(self.handle, _p(info)), "ffm_system_info")
        self.info = dict(zip(("n", "np", "S", "blocks", "units", "special_tiles",
                              "scaled_pairs", "device"), info.tolist()))

    def close(self):
        if getattr(self, "handle", None):
            self.lib.ffm_system_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ----------------------------------------------------------- device
    def new_outputs(self, batch=None):
        shape_e = (N.FFM_NTERMS,) if batch is None else (batch, N.FFM_NTERMS)
        shape_s = (N.FFM_STATUS_WORDS,) if batch is None else (batch, N.FFM_STATUS_WORDS)
        return (torch.empty(shape_e, dtype=torch.float64, device=self.device),
                torch.empty(shape_s, dtype=torch.int64, device=self.device))

    def eval(self, coords, precision=N.FFM_F64, grad=None, energies=None, status=None,
             flags=None, stream=None):
        """Evaluate at device coordinates (n, 3) float64.  Writes the fused
        gradient into ``grad`` (device (n, 3) float64) when given.  Returns
        (energies[5], status[8]) device tensors; nothing is synchronised."""
        self._check_coords(coords)
        if energies is None or status is None:
            energies, status = self.new_outputs()
        f = (N.FFM_ENERGY | (N.FFM_GRAD if grad is not None else 0)) if flags is None else flags
        if grad is not None:
            assert grad.is_cuda and grad.dtype == torch.float64 and grad.is_contiguous()
        N.check(self.lib.ffm_eval(self.handle, precision_of(precision), f, _p(coords),
                                  _p(grad), _p(energies), _p(status), _stream_ptr(stream)),
                "ffm_eval")
        return energies, status

    def eval_batch(self, coords, precision=N.FFM_F64, energies=None, status=None, stream=None):
        """Energies of a batch of geometries, coords (B, n, 3) float64 on device."""
        if not (coords.is_cuda and coords.dtype == torch.float64 and coords.is_contiguous()
                and coords.dim() == 3 and coords.shape[1:] == (self.n, 3)):
            raise ValueError(f"batch coords must be a contiguous cuda float64 (B, {self.n}, 3)")
        b = coords.shape[0]
        if energies is None or status is None:
            energies, status = self.new_outputs(b)
        N.check(self.lib.ffm_eval_batch(self.handle, precision_of(precision), b, _p(coords),
                                        _p(energies), _p(status), _stream_ptr(stream)),
                "ffm_eval_batch")
        return energies, status

    def atom_delta(self, coords, atoms, newpos, out=None, status=None, stream=None,
                   lin_cutoff=None):
        """Energy change of single-atom moves; atoms int32 (k,), newpos
        float64 (k, 3), all on device.  Exact: out (k, 5) = (coulomb, vdw,
        stretch, bend, torsion); with lin_cutoff the far-field linearised
        delta, out (k, 6) with the far term last.  status (k, 3)."""
        self._check_coords(coords)
        k = int(atoms.shape[0])
        w = 5 if lin_cutoff is None else 6
        if out is None:
            out = torch.empty((k, w), dtype=torch.float64, device=self.device)
        if status is None:
            status = torch.empty((k, 3), dtype=torch.int64, device=self.device)
        assert atoms.dtype == torch.int32 and newpos.dtype == torch.float64
        N.check(self.lib.ffm_atom_delta_lin(
            self.handle, _p(coords), k, _p(atoms.contiguous()), _p(newpos.contiguous()),
            0.0 if lin_cutoff is None else float(lin_cutoff), _p(out), _p(status),
            _stream_ptr(stream)), "ffm_atom_delta_lin")
        return out, status

    def farfield(self, coords, atom, cutoff, stream=None):
        """(e0_coef[4], near_mask[n] uint8, bad[1]) device tensors."""
        self._check_coords(coords)
        e = torch.empty(4, dtype=torch.float64, device=self.device)
        m = torch.empty(self.n, dtype=torch.uint8, device=self.device)
        b = torch.empty(1, dtype=torch.int64, device=self.device)
        N.check(self.lib.ffm_farfield_build(self.handle, _p(coords), int(atom), float(cutoff),
                                            _p(e), _p(m), _p(b), _stream_ptr(stream)),
                "ffm_farfield_build")
        return e, m, b

    # ------------------------------------------------------------- host
    def eval_host(self, coords, precision=N.FFM_F64, grad=False, flags=None):
        """Reference-facing path: NumPy (n, 3) float64 in, NumPy out, copies
        and synchronisation inside the C ABI (ffm_eval_host)."""
        c = np.ascontiguousarray(coords, dtype=np.float64)
        if c.shape != (self.n, 3):
            raise ValueError(f"coords must have shape ({self.n}, 3), got {c.shape}")
        g = np.empty((self.n, 3), np.float64) if grad else None
        f = (N.FFM_ENERGY | (N.FFM_GRAD if grad else 0)) if flags is None else flags
        en = np.empty(N.FFM_NTERMS)
        st = np.empty(N.FFM_STATUS_WORDS, np.int64)
        with self._lock, torch.cuda.device(self.device):
            N.check(self.lib.ffm_eval_host(self.handle, precision_of(precision), f, _p(c),
                                           _p(g), _p(en), _p(st)), "ffm_eval_host")
        return en, st, g

    def _check_coords(self, coords):
        if not (isinstance(coords, torch.Tensor) and coords.is_cuda
                and coords.dtype == torch.float64 and coords.is_contiguous()
                and tuple(coords.shape[-2:]) == (self.n, 3)):
            raise ValueError(f"coords must be a contiguous cuda float64 tensor ({self.n}, 3)")


def engine_for(topo, device=None, precision=None) -> DeviceSystem:
    """The (cached) engine of a topology on a device.  ``precision`` (FFM_F64
    / FFM_F32 / a NumPy dtype) names the precision the caller evaluates in:
    where the engine's preferred super-unit edge for it differs from the
    creation default (FP64 on mid-size systems, ffm_preferred_edge) the
    caller gets a second cached engine planned with that edge."""
    require_cuda()
    idx = torch.cuda.current_device() if device is None else (
        device.index if isinstance(device, torch.device) else int(device))
    key = idx
    edge = None
    if precision is not None and os.environ.get("FFM_EDGE_PREF", "1") != "0":
        lib = N.load()
        want, dflt = C.c_int(0), C.c_int(0)
        N.check(lib.ffm_preferred_edge(topo.natoms, precision_of(precision), C.byref(want)),
                "ffm_preferred_edge")
        N.check(lib.ffm_preferred_edge(topo.natoms, N.FFM_F32, C.byref(dflt)),
                "ffm_preferred_edge")
        if want.value != dflt.value:
            key, edge = (idx, "edge", want.value), want.value
    eng = topo.engines.get(key)
    if eng is None:
        eng = DeviceSystem(topo, idx)
        if edge is not None:
            with torch.cuda.device(eng.device):
                N.check(eng.lib.ffm_system_set_edge(eng.handle, edge), "ffm_system_set_edge")
            eng.refresh_info()
        topo.engines[key] = eng
    return eng
