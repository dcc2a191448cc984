"""CPU oracle for the B200 path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
``--impl reference``) may import this package.  It is the parity checker,
never the thing measured or shipped: the product package
paper_1810_03358_b200 does not import it and has no CPU execution path.

Contents
  * ffmin_oracle.c  -- C restatement of the reference kernels
    (ffmin/kernels.py loop implementations), built by oracle/Makefile into
    oracle/_build/libffmin_oracle.so;
  * this module     -- ctypes wrapper + the energy-layer assembly of
    ffmin/energy.py:133-174 on top of it;
  * optim.py        -- NumPy restatement of the L-BFGS driver and its line
    search (ffmin/optimizers/lbfgs.py, ffmin/linesearch.py).

Pinning: tests/test_oracle_golden.py checks every function here against
golden vectors produced by the reference itself (tests/golden/make_golden.py
imports ffmin from /root/reference and runs its numba backend).
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "_build" / "libffmin_oracle.so"
C_COULOMB = 1389.38757

_lock = threading.Lock()
_lib = None


def build(force=False) -> Path:
    if force or not LIB.exists() or LIB.stat().st_mtime < (HERE / "ffmin_oracle.c").stat().st_mtime:
        subprocess.run(["make", "-C", str(HERE), "-B" if force else "all"], check=True,
                       capture_output=True)
    return LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            if not LIB.exists():
                build()
            L = C.CDLL(str(LIB))
            P = C.c_void_p
            L.ffo_nb_eval.restype = C.c_int
            L.ffo_nb_eval.argtypes = [C.c_int64, P, P, P, P, P, P, P, C.c_double, P, P, P]
            L.ffo_nb_eval_mt.restype = C.c_int
            L.ffo_nb_eval_mt.argtypes = [C.c_int64, P, P, P, P, P, P, P, C.c_double, C.c_int64,
                                         C.c_int64, C.c_int, P, P, P]
            for name, nargs in (("ffo_bond", 7), ("ffo_angle", 7), ("ffo_dihedral", 6)):
                f = getattr(L, name)
                f.restype = C.c_int64
                f.argtypes = [P, C.c_int64] + [P] * (nargs - 2)
            L.ffo_nb_atom_delta.restype = C.c_int64
            L.ffo_nb_atom_delta.argtypes = [C.c_int64, P, P, P, P, C.c_int64, P, P, C.c_double,
                                            C.c_int64, P, P]
            L.ffo_farfield_build.restype = C.c_int64
            L.ffo_farfield_build.argtypes = [C.c_int64, P, P, C.c_int64, P, P, C.c_int64,
                                             C.c_double, P, P]
            L.ffo_host_threads.restype = C.c_int
            _lib = L
        return _lib


def _p(a):
    return None if a is None else C.c_void_p(a.ctypes.data)


def host_threads() -> int:
    return int(lib().ffo_host_threads())


class Arrays:
    """The kernel inputs of one system, from plain arrays."""

    def __init__(self, q, sigma, epsilon, special_i=(), special_j=(), special_s=(),
                 cutoff=None, bond_idx=None, bond_K=None, bond_r0=None, ang_idx=None,
                 ang_K=None, ang_t0=None, dih_idx=None, dih_V=None):
        f = lambda a: np.ascontiguousarray(np.asarray(a, np.float64).reshape(-1))
        self.q, self.sigma, self.eps = f(q), f(sigma), f(epsilon)
        self.n = self.q.size
        si = np.asarray(special_i, np.int64).reshape(-1)
        sj = np.asarray(special_j, np.int64).reshape(-1)
        ss = np.asarray(special_s, np.float64).reshape(-1)
        lo, hi = np.minimum(si, sj), np.maximum(si, sj)
        order = np.lexsort((hi, lo))
        lo, hi, ss = lo[order], hi[order], ss[order]
        self.sp_ptr = np.zeros(self.n + 1, np.int64)
        np.add.at(self.sp_ptr, lo + 1, 1)
        self.sp_ptr = np.cumsum(self.sp_ptr)
        self.sp_j = np.ascontiguousarray(hi, np.int32)
        self.sp_s = np.ascontiguousarray(ss)
        self._pairs = (lo, hi, ss)
        self.cutoff = -1.0 if cutoff is None else float(cutoff)
        i2 = lambda a, c: np.ascontiguousarray(np.asarray(
            np.zeros((0, c)) if a is None else a, np.int64).reshape(-1, c))
        z = lambda a: f(np.zeros(0) if a is None else a)
        self.bond_idx, self.bond_K, self.bond_r0 = i2(bond_idx, 2), z(bond_K), z(bond_r0)
        self.ang_idx, self.ang_K, self.ang_t0 = i2(ang_idx, 3), z(ang_K), z(ang_t0)
        self.dih_idx = i2(dih_idx, 4)
        self.dih_V = np.ascontiguousarray(np.asarray(
            np.zeros((0, 4)) if dih_V is None else dih_V, np.float64).reshape(-1, 4))

    @classmethod
    def from_system(cls, system):
        """Read the arrays of a paper_1810_03358_b200 (or ffmin-shaped) system."""
        t = getattr(system, "topology", None)
        if t is not None:
            return cls(t.q, t.sigma, t.epsilon, t.special_i, t.special_j, t.special_s,
                       t.cutoff, t.bond_idx, t.bond_K, t.bond_r0, t.ang_idx, t.ang_K,
                       t.ang_t0, t.dih_idx, t.dih_V)
        p = system.arrays()
        nb = system.nonbonded
        ex, sc = sorted(nb.excluded), sorted(nb.scaled14)
        si = [a for a, _ in ex] + [a for a, _ in sc]
        sj = [b for _, b in ex] + [b for _, b in sc]
        ss = [0.0] * len(ex) + [nb.s14] * len(sc)
        return cls(p["q"], p["sigma"], p["epsilon"], si, sj, ss, nb.cutoff, p["bond_idx"],
                   p["bond_K"], p["bond_r0"], p["ang_idx"], p["ang_K"], p["ang_t0"],
                   p["dih_idx"], p["dih_V"])

    def row_specials(self, atom):
        """Sorted (partner, scale) of one atom, both directions."""
        lo, hi, ss = self._pairs
        m1, m2 = lo == atom, hi == atom
        j = np.concatenate([hi[m1], lo[m2]])
        s = np.concatenate([ss[m1], ss[m2]])
        o = np.argsort(j)
        return np.ascontiguousarray(j[o], np.int32), np.ascontiguousarray(s[o])


def nb_eval(A: Arrays, coords, grad=True, threads=1, rows=None, gout=None):
    """(coulomb, vdw, bad_i, bad_j, gradient or None) -- ffmin/kernels.py:285-356.
    threads=1 is the reference loop order; rows=(i0, i1) evaluates a row slice.
    gout (n, 3) float64, when given, is accumulated into like the reference's."""
    c = np.ascontiguousarray(np.asarray(coords, np.float64).reshape(A.n, 3))
    g = (gout if gout is not None else np.zeros((A.n, 3))) if grad else None
    en = np.zeros(2)
    bad = np.zeros(2, np.int64)
    L = lib()
    if threads == 1 and rows is None:
        L.ffo_nb_eval(A.n, _p(c), _p(A.q), _p(A.sigma), _p(A.eps), _p(A.sp_ptr), _p(A.sp_j),
                      _p(A.sp_s), A.cutoff, _p(g), _p(en), _p(bad))
    else:
        i0, i1 = rows if rows is not None else (0, A.n)
        L.ffo_nb_eval_mt(A.n, _p(c), _p(A.q), _p(A.sigma), _p(A.eps), _p(A.sp_ptr),
                         _p(A.sp_j), _p(A.sp_s), A.cutoff, int(i0), int(i1), int(threads),
                         _p(g), _p(en), _p(bad))
    return float(en[0]), float(en[1]), int(bad[0]), int(bad[1]), g


def bonded(A: Arrays, coords, grad=True, gout=None):
    """((stretch, bend, torsion), (bond_bad, angle_bad, dih_bad), gradient)."""
    c = np.ascontiguousarray(np.asarray(coords, np.float64).reshape(A.n, 3))
    g = (gout if gout is not None else np.zeros((A.n, 3))) if grad else None
    L = lib()
    e = [C.c_double(0.0) for _ in range(3)]
    b = L.ffo_bond(_p(c), len(A.bond_K), _p(A.bond_idx), _p(A.bond_K), _p(A.bond_r0), _p(g),
                   C.byref(e[0]))
    a = L.ffo_angle(_p(c), len(A.ang_K), _p(A.ang_idx), _p(A.ang_K), _p(A.ang_t0), _p(g),
                    C.byref(e[1]))
    d = L.ffo_dihedral(_p(c), len(A.dih_V), _p(A.dih_idx), _p(A.dih_V), _p(g), C.byref(e[2]))
    return (e[0].value, e[1].value, e[2].value), (int(b), int(a), int(d)), g


def energy_and_gradient(A: Arrays, coords, grad=True, threads=1):
    """Restates ffmin/energy.py:144-174 (grad=True) / 133-141 (grad=False):
    returns (stretch, bend, torsion, coulomb, vdw), gradient (n*3) or None,
    and the error tuple (kind, index...) or None, raised in reference order."""
    # one shared gradient buffer, filled in the reference's order
    # (bond, angle, dihedral, nonbonded: ffmin/energy.py:153-167)
    g0 = np.zeros((A.n, 3)) if grad else None
    (es, eb, et), (bb, ab, db), _ = bonded(A, coords, grad, g0)
    ec, ev, bi, bj, _ = nb_eval(A, coords, grad, threads, gout=g0)
    if grad:
        errs = [("bond", bb), ("angle", ab), ("dihedral", db), ("nb", bi, bj)]
    else:
        errs = [("nb", bi, bj), ("angle", ab), ("dihedral", db)]
    err = next((e for e in errs if e[1] >= 0), None)
    g = g0.reshape(-1) if grad else None
    return (es, eb, et, ec, ev), g, err


def atom_delta(A: Arrays, coords, atom, delta):
    """Exact single-atom move delta, ffmin/energy.py:284-313:
    (coulomb, vdw, stretch, bend, torsion), bad nonbonded partner."""
    c = np.ascontiguousarray(np.asarray(coords, np.float64).reshape(A.n, 3))
    newpos = c[atom] + np.asarray(delta, np.float64).reshape(3)
    moved = c.copy()
    moved[atom] = newpos
    spj, sps = A.row_specials(atom)
    out = np.zeros(2)
    bad = lib().ffo_nb_atom_delta(A.n, _p(c), _p(A.q), _p(A.sigma), _p(A.eps), len(spj),
                                  _p(spj), _p(sps), A.cutoff, int(atom),
                                  _p(np.ascontiguousarray(newpos)), _p(out))
    # bonded deltas = bonded energies of the terms touching the atom, moved - current
    def sub(idx, *arrs):
        m = np.any(idx == atom, axis=1)
        return (idx[m],) + tuple(a[m] for a in arrs)

    L = lib()
    e = []
    for fn, tabs in ((L.ffo_bond, sub(A.bond_idx, A.bond_K, A.bond_r0)),
                     (L.ffo_angle, sub(A.ang_idx, A.ang_K, A.ang_t0)),
                     (L.ffo_dihedral, sub(A.dih_idx, A.dih_V))):
        tabs = [np.ascontiguousarray(t) for t in tabs]
        vals = []
        for cc in (moved, c):
            v = C.c_double(0.0)
            fn(_p(cc), len(tabs[0]), *[_p(t) for t in tabs], None, C.byref(v))
            vals.append(v.value)
        e.append(vals[0] - vals[1])
    return (float(out[0]), float(out[1]), e[0], e[1], e[2]), int(bad)
