"""Molecular system data model (mirrors ffmin/model.py).

Same types, fields and validation rules as the reference (AtomSpec,
BondTerm, AngleTerm, DihedralTerm, NonbondedPolicy, MolecularSystem,
build_default_exclusions), re-laid-out for the device path:

  * parameters and topology are held as contiguous arrays in one shared
    ``Topology`` object; ``with_coords`` makes a new system that shares it,
    so the HBM-resident plan built for one geometry serves every geometry
    an optimiser visits (ffmin/model.py:249-257 shares its caches the same
    way);
  * the nonbonded policy is kept sparse -- the list of pairs whose scale is
    not 1 -- instead of the dense (n, n) matrix of ffmin/model.py:290-295,
    which cannot exist at the 100k-atom sizes this engine targets.  The
    dense matrix is still available (``arrays()["scale"]``) for small
    systems, for code written against the reference kernels.

The tuple views (``atoms``, ``bonds``, ...) are materialised on first use,
so array-built systems (``MolecularSystem.from_arrays``) of 10^5 atoms cost
no Python objects per atom unless asked.
"""

from __future__ import annotations

import math
from collections import deque
from dataclasses import dataclass

import numpy as np


class ModelError(ValueError):
    """Raised when a system or term fails validation."""


@dataclass(frozen=True)
class AtomSpec:
    """Per-atom force-field parameters (ffmin/model.py:25-45)."""

    id: int
    label: str
    q: float
    sigma: float
    epsilon: float

    def __post_init__(self):
        if self.id < 0:
            raise ModelError(f"atom id must be >= 0, got {self.id}")
        if not (self.sigma > 0.0):
            raise ModelError(f"atom {self.id}: sigma must be > 0, got {self.sigma}")
        if self.epsilon < 0.0:
            raise ModelError(f"atom {self.id}: epsilon must be >= 0, got {self.epsilon}")


@dataclass(frozen=True)
class BondTerm:
    """Harmonic stretch K*(r - r0)^2 (ffmin/model.py:48-63)."""

    i: int
    j: int
    K: float
    r0: float

    def __post_init__(self):
        if self.i == self.j:
            raise ModelError(f"bond ({self.i},{self.j}): endpoints must differ")
        if self.K < 0.0:
            raise ModelError(f"bond ({self.i},{self.j}): K must be >= 0")
        if not (self.r0 > 0.0):
            raise ModelError(f"bond ({self.i},{self.j}): r0 must be > 0")


@dataclass(frozen=True)
class AngleTerm:
    """Harmonic bend K*(theta - theta0)^2, apex j (ffmin/model.py:66-88)."""

    i: int
    j: int
    k: int
    K: float
    theta0: float

    def __post_init__(self):
        if len({self.i, self.j, self.k}) != 3:
            raise ModelError(f"angle ({self.i},{self.j},{self.k}): atoms must be distinct")
        if self.K < 0.0:
            raise ModelError(f"angle ({self.i},{self.j},{self.k}): K must be >= 0")
        if not (0.0 < self.theta0 < math.pi):
            raise ModelError(
                f"angle ({self.i},{self.j},{self.k}): theta0 must lie in (0, pi), "
                f"got {self.theta0}")


@dataclass(frozen=True)
class DihedralTerm:
    """OPLS cosine-series torsion over i-j-k-l (ffmin/model.py:91-112)."""

    i: int
    j: int
    k: int
    l: int
    V1: float
    V2: float
    V3: float
    V4: float

    def __post_init__(self):
        if len({self.i, self.j, self.k, self.l}) != 4:
            raise ModelError(
                f"dihedral ({self.i},{self.j},{self.k},{self.l}): atoms must be distinct")


def _canonical_pairs(pairs, natoms, what):
    out = set()
    for i, j in pairs:
        if i == j:
            raise ModelError(f"{what} pair ({i},{j}): indices must differ")
        a, b = (i, j) if i < j else (j, i)
        if a < 0 or b >= natoms:
            raise ModelError(f"{what} pair ({i},{j}): index out of range for {natoms} atoms")
        out.add((a, b))
    return frozenset(out)


@dataclass(frozen=True)
class NonbondedPolicy:
    """Which pairs interact, at what scale, under what cutoff
    (ffmin/model.py:128-162)."""

    excluded: frozenset = frozenset()
    scaled14: frozenset = frozenset()
    s14: float = 0.5
    cutoff: float | None = None

    def __post_init__(self):
        if self.excluded & self.scaled14:
            raise ModelError("nonbonded policy: excluded and scaled14 pair sets overlap")
        if not (0.0 <= self.s14 <= 1.0):
            raise ModelError(f"nonbonded policy: s14 must be in [0, 1], got {self.s14}")
        if self.cutoff is not None and not (self.cutoff > 0.0):
            raise ModelError(f"nonbonded policy: cutoff must be > 0, got {self.cutoff}")

    def pair_scale(self, i, j):
        key = (i, j) if i < j else (j, i)
        if key in self.excluded:
            return 0.0
        if key in self.scaled14:
            return self.s14
        return 1.0

    @staticmethod
    def no_exclusions(cutoff=None):
        return NonbondedPolicy(frozenset(), frozenset(), 0.5, cutoff)


def _graph_separation_pairs(natoms, bond_idx):
    """(1-2/1-3 pairs, 1-4 pairs) as (i<j) int arrays, by BFS to depth 3 in
    the bond graph -- the rule of ffmin/model.py:165-200."""
    adj = [[] for _ in range(natoms)]
    for i, j in bond_idx.tolist():
        adj[i].append(j)
        adj[j].append(i)
    excl, sc = [], []
    for src in range(natoms):
        if not adj[src]:
            continue
        dist = {src: 0}
        frontier = [src]
        for depth in (1, 2, 3):
            nxt = []
            for u in frontier:
                for v in adj[u]:
                    if v not in dist:
                        dist[v] = depth
                        nxt.append(v)
            frontier = nxt
        for v, d in dist.items():
            if v <= src:
                continue
            if d in (1, 2):
                excl.append((src, v))
            elif d == 3:
                sc.append((src, v))
    e = np.array(excl, dtype=np.int64).reshape(-1, 2)
    s = np.array(sc, dtype=np.int64).reshape(-1, 2)
    return e, s


def build_default_exclusions(natoms, bonds, s14=0.5, cutoff=None):
    """1-2 and 1-3 excluded, 1-4 scaled by s14 (ffmin/model.py:165-200)."""
    for b in bonds:
        if b.i >= natoms or b.j >= natoms:
            raise ModelError(f"bond ({b.i},{b.j}): index out of range for {natoms} atoms")
    bidx = np.array([(b.i, b.j) for b in bonds], dtype=np.int64).reshape(-1, 2)
    e, s = _graph_separation_pairs(natoms, bidx)
    return NonbondedPolicy(frozenset(map(tuple, e.tolist())), frozenset(map(tuple, s.tolist())),
                           s14, cutoff)


class Topology:
    """Parameters, term tables and the sparse pair policy of one system.
    Shared (by reference) between all geometries of that system; also owns
    the per-device engine handles (paper_1810_03358_b200.engine)."""

    def __init__(self, q, sigma, epsilon, labels, bond_idx, bond_K, bond_r0, ang_idx, ang_K,
                 ang_t0, dih_idx, dih_V, special_i, special_j, special_s, cutoff, s14,
                 policy=None):
        self.q = q
        self.sigma = sigma
        self.epsilon = epsilon
        self.labels = labels
        self.bond_idx, self.bond_K, self.bond_r0 = bond_idx, bond_K, bond_r0
        self.ang_idx, self.ang_K, self.ang_t0 = ang_idx, ang_K, ang_t0
        self.dih_idx, self.dih_V = dih_idx, dih_V
        self.special_i, self.special_j, self.special_s = special_i, special_j, special_s
        self.cutoff = cutoff
        self.s14 = s14
        self._policy = policy
        self.engines = {}      # device -> engine.DeviceSystem
        self._atom_terms = None
        for a in (q, sigma, epsilon, bond_idx, bond_K, bond_r0, ang_idx, ang_K, ang_t0,
                  dih_idx, dih_V, special_i, special_j, special_s):
            a.setflags(write=False)

    @property
    def natoms(self):
        return int(self.q.shape[0])


def _f64(a, shape=None):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    return a.reshape(shape) if shape is not None else a


def _i64(a, cols):
    return np.ascontiguousarray(np.asarray(a, dtype=np.int64)).reshape(-1, cols)


class MolecularSystem:
    """Immutable system: atoms, coordinates and interaction terms
    (ffmin/model.py:203-347).  Coordinate updates go through with_coords."""

    __slots__ = ("_topo", "coords", "_atoms", "_bonds", "_angles", "_dihedrals", "_cache",
                 "__weakref__")

    def __init__(self, atoms, coords, bonds=(), angles=(), dihedrals=(), nonbonded=None):
        atoms = tuple(atoms)
        bonds = tuple(bonds)
        angles = tuple(angles)
        dihedrals = tuple(dihedrals)
        nonbonded = nonbonded if nonbonded is not None else NonbondedPolicy()
        n = len(atoms)
        for idx, a in enumerate(atoms):
            if a.id != idx:
                raise ModelError(
                    f"atom ids must be 0..n-1 in order; position {idx} has id {a.id}")
        for b in bonds:
            if not (0 <= b.i < n and 0 <= b.j < n):
                raise ModelError(f"bond ({b.i},{b.j}): index out of range")
        for a in angles:
            if not all(0 <= t < n for t in (a.i, a.j, a.k)):
                raise ModelError(f"angle ({a.i},{a.j},{a.k}): index out of range")
        for d in dihedrals:
            if not all(0 <= t < n for t in (d.i, d.j, d.k, d.l)):
                raise ModelError(f"dihedral ({d.i},{d.j},{d.k},{d.l}): index out of range")
        excl = sorted(_canonical_pairs(nonbonded.excluded, n, "excluded"))
        sc = sorted(_canonical_pairs(nonbonded.scaled14, n, "scaled14"))
        si = np.array([p[0] for p in excl] + [p[0] for p in sc], dtype=np.int64)
        sj = np.array([p[1] for p in excl] + [p[1] for p in sc], dtype=np.int64)
        ss = np.array([0.0] * len(excl) + [nonbonded.s14] * len(sc), dtype=np.float64)
        topo = Topology(
            q=_f64([a.q for a in atoms]), sigma=_f64([a.sigma for a in atoms]),
            epsilon=_f64([a.epsilon for a in atoms]), labels=tuple(a.label for a in atoms),
            bond_idx=_i64([(b.i, b.j) for b in bonds], 2), bond_K=_f64([b.K for b in bonds]),
            bond_r0=_f64([b.r0 for b in bonds]),
            ang_idx=_i64([(a.i, a.j, a.k) for a in angles], 3),
            ang_K=_f64([a.K for a in angles]), ang_t0=_f64([a.theta0 for a in angles]),
            dih_idx=_i64([(d.i, d.j, d.k, d.l) for d in dihedrals], 4),
            dih_V=_f64([(d.V1, d.V2, d.V3, d.V4) for d in dihedrals], (-1, 4)),
            special_i=si, special_j=sj, special_s=ss, cutoff=nonbonded.cutoff,
            s14=nonbonded.s14, policy=nonbonded)
        self._init(topo, coords)
        self._atoms, self._bonds, self._angles, self._dihedrals = atoms, bonds, angles, dihedrals

    def _init(self, topo, coords):
        n = topo.natoms
        c = np.array(coords, dtype=np.float64, copy=True)
        if c.shape != (n, 3):
            raise ModelError(f"coords shape {c.shape} does not match {n} atoms")
        if not np.all(np.isfinite(c)):
            raise ModelError("coords must be finite")
        c.setflags(write=False)
        self._topo = topo
        self.coords = c
        self._atoms = self._bonds = self._angles = self._dihedrals = None
        self._cache = {}

    @classmethod
    def from_arrays(cls, q, sigma, epsilon, coords, bond_idx=None, bond_K=None, bond_r0=None,
                    ang_idx=None, ang_K=None, ang_t0=None, dih_idx=None, dih_V=None,
                    excluded=None, scaled14=None, s14=0.5, cutoff=None, labels=None):
        """Array-built system (no per-atom Python objects).  excluded /
        scaled14 are (k, 2) index arrays; validation matches the reference."""
        q, sigma, epsilon = _f64(q), _f64(sigma), _f64(epsilon)
        n = q.shape[0]
        if sigma.shape != (n,) or epsilon.shape != (n,):
            raise ModelError("q, sigma, epsilon must have one entry per atom")
        if not np.all(sigma > 0.0):
            raise ModelError(f"atom {int(np.argmin(sigma > 0.0))}: sigma must be > 0")
        if not np.all(epsilon >= 0.0):
            raise ModelError(f"atom {int(np.argmin(epsilon >= 0.0))}: epsilon must be >= 0")
        none2 = np.zeros((0, 2), np.int64)
        bond_idx = _i64(none2 if bond_idx is None else bond_idx, 2)
        ang_idx = _i64(np.zeros((0, 3)) if ang_idx is None else ang_idx, 3)
        dih_idx = _i64(np.zeros((0, 4)) if dih_idx is None else dih_idx, 4)
        bond_K = _f64([] if bond_K is None else bond_K)
        bond_r0 = _f64([] if bond_r0 is None else bond_r0)
        ang_K = _f64([] if ang_K is None else ang_K)
        ang_t0 = _f64([] if ang_t0 is None else ang_t0)
        dih_V = _f64(np.zeros((0, 4)) if dih_V is None else dih_V, (-1, 4))
        for name, idx in (("bond", bond_idx), ("angle", ang_idx), ("dihedral", dih_idx)):
            if idx.size and (idx.min() < 0 or idx.max() >= n):
                raise ModelError(f"{name} index out of range")
        if bond_idx.size and np.any(bond_idx[:, 0] == bond_idx[:, 1]):
            raise ModelError("bond endpoints must differ")
        if np.any(bond_K < 0) or np.any(~(bond_r0 > 0)):
            raise ModelError("bond K must be >= 0 and r0 > 0")
        if np.any(ang_K < 0) or np.any(~((ang_t0 > 0) & (ang_t0 < math.pi))):
            raise ModelError("angle K must be >= 0 and theta0 in (0, pi)")
        if not (0.0 <= s14 <= 1.0):
            raise ModelError(f"nonbonded policy: s14 must be in [0, 1], got {s14}")
        if cutoff is not None and not (cutoff > 0.0):
            raise ModelError(f"nonbonded policy: cutoff must be > 0, got {cutoff}")
        ex = _i64(none2 if excluded is None else excluded, 2)
        sc = _i64(none2 if scaled14 is None else scaled14, 2)
        ex = np.sort(ex, axis=1)
        sc = np.sort(sc, axis=1)
        for name, arr in (("excluded", ex), ("scaled14", sc)):
            if arr.size and (arr.min() < 0 or arr.max() >= n or np.any(arr[:, 0] == arr[:, 1])):
                raise ModelError(f"{name} pair index out of range or i == j")
        ex = np.unique(ex, axis=0) if ex.size else ex
        sc = np.unique(sc, axis=0) if sc.size else sc
        if ex.size and sc.size:
            both = np.intersect1d(ex[:, 0] * n + ex[:, 1], sc[:, 0] * n + sc[:, 1])
            if both.size:
                raise ModelError("nonbonded policy: excluded and scaled14 pair sets overlap")
        topo = Topology(
            q=q, sigma=sigma, epsilon=epsilon,
            labels=tuple(labels) if labels is not None else None,
            bond_idx=bond_idx, bond_K=bond_K, bond_r0=bond_r0, ang_idx=ang_idx, ang_K=ang_K,
            ang_t0=ang_t0, dih_idx=dih_idx, dih_V=dih_V,
            special_i=np.concatenate([ex[:, 0], sc[:, 0]]),
            special_j=np.concatenate([ex[:, 1], sc[:, 1]]),
            special_s=np.concatenate([np.zeros(len(ex)), np.full(len(sc), float(s14))]),
            cutoff=None if cutoff is None else float(cutoff), s14=float(s14))
        obj = cls.__new__(cls)
        obj._init(topo, coords)
        return obj

    # ------------------------------------------------------------ views
    @property
    def topology(self) -> Topology:
        return self._topo

    @property
    def natoms(self):
        return self._topo.natoms

    @property
    def atoms(self):
        if self._atoms is None:
            t = self._topo
            labels = t.labels or tuple(f"A{i}" for i in range(t.natoms))
            self._atoms = tuple(AtomSpec(i, labels[i], float(t.q[i]), float(t.sigma[i]),
                                         float(t.epsilon[i])) for i in range(t.natoms))
        return self._atoms

    @property
    def bonds(self):
        if self._bonds is None:
            t = self._topo
            self._bonds = tuple(BondTerm(int(i), int(j), float(k), float(r))
                                for (i, j), k, r in zip(t.bond_idx, t.bond_K, t.bond_r0))
        return self._bonds

    @property
    def angles(self):
        if self._angles is None:
            t = self._topo
            self._angles = tuple(AngleTerm(int(i), int(j), int(k), float(kk), float(a))
                                 for (i, j, k), kk, a in zip(t.ang_idx, t.ang_K, t.ang_t0))
        return self._angles

    @property
    def dihedrals(self):
        if self._dihedrals is None:
            t = self._topo
            self._dihedrals = tuple(
                DihedralTerm(int(i), int(j), int(k), int(l), *map(float, v))
                for (i, j, k, l), v in zip(t.dih_idx, t.dih_V))
        return self._dihedrals

    @property
    def nonbonded(self) -> NonbondedPolicy:
        t = self._topo
        if t._policy is None:
            zero = t.special_s == 0.0
            ex = frozenset(zip(t.special_i[zero].tolist(), t.special_j[zero].tolist()))
            sc = frozenset(zip(t.special_i[~zero].tolist(), t.special_j[~zero].tolist()))
            t._policy = NonbondedPolicy(ex, sc, t.s14, t.cutoff)
        return t._policy

    def with_coords(self, coords):
        """New system sharing the topology (and its device plans)."""
        new = MolecularSystem.__new__(MolecularSystem)
        new._init(self._topo, np.asarray(coords, dtype=np.float64).reshape(self.natoms, 3))
        new._atoms, new._bonds = self._atoms, self._bonds
        new._angles, new._dihedrals = self._angles, self._dihedrals
        return new

    def arrays(self, dtype=np.float64):
        """Kernel-ready arrays, names as ffmin/model.py:298-304.  'scale' is
        the dense matrix, built lazily and only for n <= 20000."""
        key = ("params", np.dtype(dtype).name)
        out = self._cache.get(key)
        if out is None:
            t = self._topo
            cast = (lambda a: a) if np.dtype(dtype) == np.float64 else (
                lambda a: a.astype(dtype))
            out = _ArrayDict(self, {
                "q": cast(t.q), "sigma": cast(t.sigma), "epsilon": cast(t.epsilon),
                "bond_idx": t.bond_idx, "bond_K": cast(t.bond_K), "bond_r0": cast(t.bond_r0),
                "ang_idx": t.ang_idx, "ang_K": cast(t.ang_K), "ang_t0": cast(t.ang_t0),
                "dih_idx": t.dih_idx, "dih_V": cast(t.dih_V),
                "special_i": t.special_i, "special_j": t.special_j,
                "special_s": t.special_s,
                "cutoff": -1.0 if t.cutoff is None else float(t.cutoff),
            }, dtype)
            self._cache[key] = out
        return out

    def atom_terms(self, atom):
        """Row indices of the bonded terms involving atom (ffmin/model.py:321-347)."""
        t = self._topo
        if t._atom_terms is None:
            def rows(idx):
                n = t.natoms
                r = np.repeat(np.arange(idx.shape[0]), idx.shape[1])
                a = idx.reshape(-1)
                order = np.lexsort((r, a))
                ptr = np.zeros(n + 1, np.int64)
                np.add.at(ptr, a + 1, 1)
                return np.cumsum(ptr), r[order]
            t._atom_terms = (rows(t.bond_idx), rows(t.ang_idx), rows(t.dih_idx))
        out = []
        for ptr, r in t._atom_terms:
            out.append(np.unique(r[ptr[atom]:ptr[atom + 1]]))
        return tuple(out)

    def __repr__(self):
        t = self._topo
        return (f"MolecularSystem(natoms={t.natoms}, bonds={len(t.bond_K)}, "
                f"angles={len(t.ang_K)}, dihedrals={len(t.dih_V)}, "
                f"special_pairs={len(t.special_s)}, cutoff={t.cutoff})")


class _ArrayDict(dict):
    """dict of kernel arrays with a lazily built dense 'scale' matrix."""

    DENSE_LIMIT = 20000

    def __init__(self, system, items, dtype):
        super().__init__(items)
        self._system = system
        self._dtype = dtype

    def __missing__(self, key):
        if key != "scale":
            raise KeyError(key)
        t = self._system.topology
        n = t.natoms
        if n > self.DENSE_LIMIT:
            raise ModelError(f"dense scale matrix refused for {n} atoms; use the sparse "
                             "special_i/special_j/special_s arrays")
        scale = np.ones((n, n), dtype=np.float64)
        np.fill_diagonal(scale, 0.0)
        scale[t.special_i, t.special_j] = t.special_s
        scale[t.special_j, t.special_i] = t.special_s
        scale = scale.astype(self._dtype)
        scale.setflags(write=False)
        self["scale"] = scale
        return scale
