"""Synthetic molecules for benchmarks, demos and parity tests.

``make_chain_system`` reproduces ffmin/synth.py:23-72 draw for draw (same
generator, same call order), so a seed gives the identical system the
reference builds -- the golden fixtures rely on it.  It is array-built, so
it scales to 10^5 atoms.

``make_globule_system`` is the "random-protein-like" benchmark system of
BASELINE.json: the same chain chemistry, but folded into a compact cube
(serpentine rows of a zig-zag backbone, 4 A between rows) at about
0.05 atoms / A^3, so coordinates stay within +-(N/0.05)^(1/3)/2 A and FP32
positions keep ~1e-6 A resolution even at 100k atoms.
"""

from __future__ import annotations

import math

import numpy as np

from .model import MolecularSystem


def _chain_params(rng, natoms):
    # ffmin/synth.py:26-37: three uniform draws per atom, in q, sigma, eps order
    u = rng.random(3 * natoms).reshape(natoms, 3)
    sign = np.where(np.arange(natoms) % 2 == 0, 0.2, -0.2)
    q = (0.5 + (1.5 - 0.5) * u[:, 0]) * sign
    sigma = 2.8 + (3.6 - 2.8) * u[:, 1]
    eps = 0.3 + (0.8 - 0.3) * u[:, 2]
    # reference: shift = sum(a.q for a in atoms) / natoms (sequential sum)
    shift = sum(q.tolist()) / natoms
    return q - shift, sigma, eps


def _chain_terms(rng, natoms):
    nb, na, nd = max(natoms - 1, 0), max(natoms - 2, 0), max(natoms - 3, 0)
    ub = rng.random(2 * nb).reshape(nb, 2)                 # K, r0 per bond
    ua = rng.random(2 * na).reshape(na, 2)                 # K, theta0 per angle
    ud = rng.random(3 * nd).reshape(nd, 3)                 # V1..V3 per dihedral
    i = np.arange(natoms, dtype=np.int64)
    bond_idx = np.stack([i[:nb], i[:nb] + 1], axis=1)
    bond_K = 250.0 + (350.0 - 250.0) * ub[:, 0]
    bond_r0 = 1.4 + (1.6 - 1.4) * ub[:, 1]
    ang_idx = np.stack([i[:na], i[:na] + 1, i[:na] + 2], axis=1)
    ang_K = 30.0 + (60.0 - 30.0) * ua[:, 0]
    ang_t0 = 1.8 + (2.0 - 1.8) * ua[:, 1]
    dih_idx = np.stack([i[:nd], i[:nd] + 1, i[:nd] + 2, i[:nd] + 3], axis=1)
    dih_V = np.zeros((nd, 4))
    dih_V[:, 0] = 0.5 + (3.0 - 0.5) * ud[:, 0]
    dih_V[:, 1] = 0.0 + (1.5 - 0.0) * ud[:, 1]
    dih_V[:, 2] = 0.0 + (1.0 - 0.0) * ud[:, 2]
    return bond_idx, bond_K, bond_r0, ang_idx, ang_K, ang_t0, dih_idx, dih_V


def chain_policy_pairs(natoms):
    """Exclusions of a linear chain: 1-2 and 1-3 pairs excluded, 1-4 pairs
    scaled -- build_default_exclusions on a path graph, vectorised."""
    i = np.arange(natoms, dtype=np.int64)
    ex = np.concatenate([np.stack([i[:-1], i[:-1] + 1], 1) if natoms > 1 else np.zeros((0, 2), np.int64),
                         np.stack([i[:-2], i[:-2] + 2], 1) if natoms > 2 else np.zeros((0, 2), np.int64)])
    sc = np.stack([i[:-3], i[:-3] + 3], 1) if natoms > 3 else np.zeros((0, 2), np.int64)
    return ex.reshape(-1, 2), sc.reshape(-1, 2)


def make_chain_system(natoms, seed=0, strain=0.3, s14=0.5, cutoff=None) -> MolecularSystem:
    """Alkane-like chain along x with every term type (ffmin/synth.py:23-72)."""
    if natoms < 2:
        raise ValueError("need at least 2 atoms")
    rng = np.random.default_rng(seed)
    q, sigma, eps = _chain_params(rng, natoms)
    terms = _chain_terms(rng, natoms)
    coords = np.zeros((natoms, 3))
    coords[:, 0] = np.arange(natoms) * 1.5
    if strain > 0:
        coords += rng.normal(scale=strain, size=(natoms, 3))
    ex, sc = chain_policy_pairs(natoms)
    return MolecularSystem.from_arrays(
        q, sigma, eps, coords, *terms, excluded=ex, scaled14=sc, s14=s14, cutoff=cutoff,
        labels=[f"C{i}" for i in range(natoms)] if natoms <= 100000 else None)


def globule_coords(natoms, seed=0, noise=0.1, row_spacing=4.0, step=1.25, zig=0.42):
    """Compact serpentine backbone: rows of `step`-spaced zig-zag atoms along
    x, rows on a (y, z) grid `row_spacing` apart, visited boustrophedon so
    consecutive atoms are always bonded neighbours.  Centered at the origin."""
    rng = np.random.default_rng(seed + 7919)
    lx = max(4, int(round((row_spacing / step * math.sqrt(natoms)) ** (2.0 / 3.0))))
    nrows = -(-natoms // lx)
    g = max(1, int(math.ceil(math.sqrt(nrows))))
    k = np.arange(natoms)
    row, t = k // lx, k % lx
    gz = row // g
    gy = np.where(gz % 2 == 0, row % g, g - 1 - row % g)
    xpos = np.where(row % 2 == 0, t, lx - 1 - t) * step
    c = np.stack([xpos,
                  gy * row_spacing + np.where(t % 2 == 0, -zig, zig),
                  gz * row_spacing], axis=1).astype(np.float64)
    c += rng.normal(scale=noise, size=c.shape)
    c -= c.mean(axis=0)
    return c


def make_globule_system(natoms, seed=0, noise=0.1, s14=0.5, cutoff=None) -> MolecularSystem:
    """Random-protein-like compact chain (the benchmark workload)."""
    if natoms < 4:
        raise ValueError("need at least 4 atoms")
    rng = np.random.default_rng(seed)
    q, sigma, eps = _chain_params(rng, natoms)
    terms = _chain_terms(rng, natoms)
    coords = globule_coords(natoms, seed, noise)
    ex, sc = chain_policy_pairs(natoms)
    return MolecularSystem.from_arrays(q, sigma, eps, coords, *terms, excluded=ex,
                                       scaled14=sc, s14=s14, cutoff=cutoff)


def perturbed_copy(system: MolecularSystem, scale, seed) -> MolecularSystem:
    """Same topology, coordinates jittered by N(0, scale) (ffmin/synth.py:75-83)."""
    rng = np.random.default_rng(seed)
    coords = system.coords + rng.normal(scale=scale, size=system.coords.shape)
    return system.with_coords(coords)
