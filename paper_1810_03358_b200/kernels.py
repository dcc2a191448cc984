"""The "cuda" kernel backend: drop-in for ffmin/kernels.py's KernelBackend.

Same function names, signatures and return conventions as the reference
loop/numpy backends (ffmin/kernels.py:596-611, 962-977): kernels never raise
on bad geometry, they report the failing term / pair index (-1 when clean);
energies are float64; gradients are ADDED into ``gout`` in its dtype.  The
precision follows the coordinate dtype (float32 coordinates -> FP32 pair
arithmetic with FP64 accumulation).

Every call runs on the GPU through the C ABI (host buffers in, host buffers
out).  Parameter arrays are uploaded once: the HBM plan is cached on the
identity of the arrays passed (the reference's MolecularSystem caches its
arrays the same way, ffmin/model.py:259-319), so repeated calls with the
same system only move coordinates and results.
"""

from __future__ import annotations

import os
import threading
from collections import OrderedDict

import numpy as np

from . import _native as N
from .engine import DeviceSystem, precision_of
from .model import Topology

_CACHE_SIZE = 16
_cache: OrderedDict = OrderedDict()
_cache_lock = threading.Lock()


def _dense_to_special(scale):
    n = scale.shape[0]
    iu, ju = np.nonzero(np.triu(np.asarray(scale, dtype=np.float64) != 1.0, 1))
    return iu.astype(np.int64), ju.astype(np.int64), np.asarray(scale, np.float64)[iu, ju]


def _z(n):
    return np.zeros(n, np.float64)


def _engine(key_arrays, build, n):
    key = tuple(id(a) for a in key_arrays) + (int(n),)
    with _cache_lock:
        hit = _cache.get(key)
        if hit is not None and all(a is b for a, b in zip(hit[0], key_arrays)):
            _cache.move_to_end(key)
            return hit[1]
    eng = DeviceSystem(build())
    with _cache_lock:
        _cache[key] = (tuple(key_arrays), eng)
        while len(_cache) > _CACHE_SIZE:
            _cache.popitem(last=False)
    return eng


def _topology(n, q=None, sigma=None, epsilon=None, scale=None, cutoff=-1.0, bidx=None, K=None,
              r0=None, aidx=None, aK=None, at0=None, didx=None, dV=None):
    si = sj = ss = np.zeros(0)
    if scale is not None:
        si, sj, ss = _dense_to_special(scale)
    f = lambda a, m=0: np.ascontiguousarray(a, np.float64) if a is not None else _z(m)
    i = lambda a, c: (np.ascontiguousarray(a, np.int64).reshape(-1, c) if a is not None
                      else np.zeros((0, c), np.int64))
    return Topology(
        q=f(q, n), sigma=f(sigma) if sigma is not None else np.ones(n), epsilon=f(epsilon, n),
        labels=None, bond_idx=i(bidx, 2), bond_K=f(K), bond_r0=f(r0), ang_idx=i(aidx, 3),
        ang_K=f(aK), ang_t0=f(at0), dih_idx=i(didx, 4),
        dih_V=f(dV).reshape(-1, 4) if dV is not None else np.zeros((0, 4)),
        special_i=np.asarray(si, np.int64), special_j=np.asarray(sj, np.int64),
        special_s=np.asarray(ss, np.float64),
        cutoff=None if cutoff is None or cutoff <= 0 else float(cutoff), s14=0.5)


def _f64coords(c):
    return np.ascontiguousarray(c, dtype=np.float64)


# ------------------------------------------------------------------ pairs

def nb_energy(coords, q, sigma, epsilon, scale, cutoff):
    n = coords.shape[0]
    eng = _engine((q, sigma, epsilon, scale), lambda: _topology(
        n, q, sigma, epsilon, scale, cutoff), n)
    _ensure_cutoff(eng, cutoff)
    en, st, _ = eng.eval_host(_f64coords(coords), precision_of(coords.dtype), False,
                              N.FFM_ENERGY | N.FFM_NO_TERMS)
    if st[0] >= 0:
        return 0.0, 0.0, int(st[0]), int(st[1])
    return float(en[3]), float(en[4]), -1, -1


def nb_grad(coords, q, sigma, epsilon, scale, cutoff, gout):
    n = coords.shape[0]
    eng = _engine((q, sigma, epsilon, scale), lambda: _topology(
        n, q, sigma, epsilon, scale, cutoff), n)
    _ensure_cutoff(eng, cutoff)
    en, st, g = eng.eval_host(_f64coords(coords), precision_of(coords.dtype), True,
                              N.FFM_ENERGY | N.FFM_GRAD | N.FFM_NO_TERMS)
    if st[0] >= 0:
        return 0.0, 0.0, int(st[0]), int(st[1])
    gout += g.astype(gout.dtype, copy=False)
    return float(en[3]), float(en[4]), -1, -1


def _ensure_cutoff(eng, cutoff):
    # the cached plan was built for one cutoff; a different value needs a new plan
    want = None if cutoff is None or cutoff <= 0 else float(cutoff)
    if eng._cutoff_seen is None:
        eng._cutoff_seen = ("set", want)
    elif eng._cutoff_seen[1] != want:
        raise ValueError("cuda backend: the cutoff of a cached parameter set changed; "
                         "pass fresh parameter arrays")


DeviceSystem._cutoff_seen = None


# ----------------------------------------------------------------- bonded

def _bonded(coords, kind, tables, grad, gout=None):
    n = coords.shape[0]
    kw = dict(zip({"bond": ("bidx", "K", "r0"), "angle": ("aidx", "aK", "at0"),
                   "dihedral": ("didx", "dV")}[kind], tables))
    eng = _engine(tuple(tables), lambda: _topology(n, **kw), n)
    en, st, g = eng.eval_host(_f64coords(coords), precision_of(coords.dtype), grad,
                              N.FFM_ENERGY | (N.FFM_GRAD if grad else 0) | N.FFM_NO_NB)
    col = {"bond": (0, N.ST_BOND), "angle": (1, N.ST_ANGLE), "dihedral": (2, N.ST_DIHEDRAL)}
    ei, si = col[kind]
    bad = int(st[si])
    if bad >= 0:
        return float(en[ei]), bad
    if grad:
        gout += g.astype(gout.dtype, copy=False)
    return float(en[ei]), -1


def bond_energy(coords, bidx, K, r0):
    return _bonded(coords, "bond", (bidx, K, r0), False)[0]


def bond_grad(coords, bidx, K, r0, gout):
    return _bonded(coords, "bond", (bidx, K, r0), True, gout)


def angle_energy(coords, aidx, K, t0):
    return _bonded(coords, "angle", (aidx, K, t0), False)


def angle_grad(coords, aidx, K, t0, gout):
    return _bonded(coords, "angle", (aidx, K, t0), True, gout)


def dihedral_energy(coords, didx, V):
    return _bonded(coords, "dihedral", (didx, V), False)


def dihedral_grad(coords, didx, V, gout):
    return _bonded(coords, "dihedral", (didx, V), True, gout)


# ------------------------------------------------------ single-atom moves

def _delta(eng, coords, atom, newpos):
    import torch

    dev = eng.device
    c = torch.from_numpy(_f64coords(coords)).to(dev)
    out, st = eng.atom_delta(c, torch.tensor([int(atom)], dtype=torch.int32, device=dev),
                             torch.from_numpy(np.asarray(newpos, np.float64).reshape(1, 3)).to(dev))
    return out.cpu().numpy()[0], st.cpu().numpy()[0]


def nb_atom_delta(coords, q, sigma, epsilon, scale, cutoff, atom, newpos):
    n = coords.shape[0]
    eng = _engine((q, sigma, epsilon, scale), lambda: _topology(
        n, q, sigma, epsilon, scale, cutoff), n)
    _ensure_cutoff(eng, cutoff)
    out, st = _delta(eng, coords, atom, newpos)
    if st[0] >= 0:
        return 0.0, 0.0, int(st[0])
    return float(out[0]), float(out[1]), -1


def _rows_delta(coords, atom, newpos, kind, tables, rows):
    n = coords.shape[0]
    rows = np.asarray(rows, np.int64)
    if rows.size == 0:
        return 0.0, -1
    sub = [np.asarray(t)[rows] for t in tables]
    key = {"bond": ("bidx", "K", "r0"), "angle": ("aidx", "aK", "at0"),
           "dihedral": ("didx", "dV")}[kind]
    eng = DeviceSystem(_topology(n, **dict(zip(key, sub))))
    out, st = _delta(eng, coords, atom, newpos)
    eng.close()
    if kind == "bond":
        return float(out[2]), -1
    if kind == "angle":
        return (float(out[3]), -1) if st[1] < 0 else (0.0, int(rows[st[1]]))
    return (float(out[4]), -1) if st[2] < 0 else (0.0, int(rows[st[2]]))


def bond_delta(coords, atom, newpos, bidx, K, r0, rows):
    return _rows_delta(coords, atom, newpos, "bond", (bidx, K, r0), rows)[0]


def angle_delta(coords, atom, newpos, aidx, K, t0, rows):
    return _rows_delta(coords, atom, newpos, "angle", (aidx, K, t0), rows)


def dihedral_delta(coords, atom, newpos, didx, V, rows):
    return _rows_delta(coords, atom, newpos, "dihedral", (didx, V), rows)


def farfield_build(coords, q, scale, atom, cutoff):
    """ffmin/kernels.py:359-387: (e0, cx, cy, cz, near_mask uint8, bad)."""
    n = coords.shape[0]
    eng = _engine((q, scale), lambda: _topology(n, q, None, np.zeros(n), scale, -1.0), n)
    import torch

    c = torch.from_numpy(np.array(_f64coords(coords))).to(eng.device)
    e, m, b = eng.farfield(c, int(atom), float(cutoff))
    e = e.cpu().numpy()
    return float(e[0]), float(e[1]), float(e[2]), float(e[3]), m.cpu().numpy(), int(b.item())


def near_nb_delta(coords, q, sigma, epsilon, scale, atom, newpos, near_idx):
    """ffmin/kernels.py:390-416: exact nonbonded change of moving `atom`
    against the partners in near_idx only -- the exact delta kernel on a
    plan whose other atoms carry no charge and no LJ."""
    n = coords.shape[0]
    near = np.zeros(n, bool)
    near[np.asarray(near_idx, np.int64)] = True
    near[int(atom)] = True
    qn = np.where(near, np.asarray(q, np.float64), 0.0)
    en = np.where(near, np.asarray(epsilon, np.float64), 0.0)
    eng = DeviceSystem(_topology(n, qn, sigma, en, scale, -1.0))
    try:
        out, st = _delta(eng, coords, atom, newpos)
    finally:
        eng.close()
    if st[0] >= 0:
        return 0.0, 0.0, int(st[0])
    return float(out[0]), float(out[1]), -1


_CUDA_FNS = {
    "bond_energy": bond_energy, "bond_grad": bond_grad,
    "angle_energy": angle_energy, "angle_grad": angle_grad,
    "dihedral_energy": dihedral_energy, "dihedral_grad": dihedral_grad,
    "nb_energy": nb_energy, "nb_grad": nb_grad,
    "farfield_build": farfield_build, "near_nb_delta": near_nb_delta,
    "nb_atom_delta": nb_atom_delta, "bond_delta": bond_delta,
    "angle_delta": angle_delta, "dihedral_delta": dihedral_delta,
}


class KernelBackend:
    """Named bundle of kernel functions (ffmin/kernels.py:984-988)."""

    def __init__(self, name, fns):
        self.name = name
        for key, fn in fns.items():
            setattr(self, key, fn)


CUDA_BACKEND = KernelBackend("cuda", _CUDA_FNS)


def get_backend(name=None) -> KernelBackend:
    """Resolve the kernel backend (ffmin/kernels.py:1006-1024).  Order:
    explicit name, FFMIN_BACKEND, default "cuda".  There is one backend."""
    if isinstance(name, KernelBackend):
        return name
    if name is None:
        name = os.environ.get("FFMIN_BACKEND", "").strip().lower() or None
    if name is None or name == "cuda":
        return CUDA_BACKEND
    raise ValueError(f"unknown kernel backend {name!r} (this framework provides 'cuda')")
