"""Parity of the B200 energy / gradient path with the oracle and the
reference golden vectors.  GPU only (-m gpu).

Tolerances:
  FP64 mode: energies within 1e-10 relative, gradients within 1e-10 of
             max|g| -- the north star asks for 1e-6;
  FP32 mode: energies within 1e-5 relative, gradients within 1e-4 of max|g|
             (pair arithmetic in FP32, accumulation in FP64), compared with
             the FP64 reference.
"""

import numpy as np
import pytest

import oracle as O
from conftest import golden_system, oracle_arrays

pytestmark = pytest.mark.gpu

CASES = ["chain10", "chain14", "cloud24", "cloud24c7", "explicit8", "chain200", "chain12cut",
         "globule1500"]


@pytest.fixture(scope="module")
def E():
    import paper_1810_03358_b200.energy as energy

    return energy


def _rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-12))


@pytest.mark.parametrize("name", CASES)
def test_fp64_matches_reference(golden, E, name):
    s = golden_system(golden, name)
    bd, g = E.energy_and_gradient(s, np.float64)
    ref_e, ref_g = golden[f"{name}/egrad_f64"], golden[f"{name}/grad_f64"]
    got = [bd.stretch, bd.bend, bd.torsion, bd.coulomb, bd.vdw]
    np.testing.assert_allclose(got, ref_e, rtol=1e-10, atol=1e-9)
    assert np.max(np.abs(g - ref_g)) <= 1e-10 * np.max(np.abs(ref_g))
    assert g.dtype == np.float64
    bd2 = E.energy_total(s, np.float64)
    np.testing.assert_allclose([bd2.stretch, bd2.bend, bd2.torsion, bd2.coulomb, bd2.vdw],
                               golden[f"{name}/energy_f64"], rtol=1e-10, atol=1e-9)


@pytest.mark.parametrize("name", CASES)
def test_fp32_mode_tracks_fp64_reference(golden, E, name):
    s = golden_system(golden, name)
    bd, g = E.energy_and_gradient(s, np.float32)
    assert g.dtype == np.float32 and isinstance(bd.total, float)
    ref_e, ref_g = golden[f"{name}/egrad_f64"], golden[f"{name}/grad_f64"]
    got = [bd.stretch, bd.bend, bd.torsion, bd.coulomb, bd.vdw]
    np.testing.assert_allclose(got, ref_e, rtol=1e-5, atol=1e-4)
    assert np.max(np.abs(g - ref_g)) <= 1e-4 * np.max(np.abs(ref_g))


@pytest.mark.parametrize("name", ["chain200", "globule1500"])
def test_repeated_calls_bit_identical(golden, E, name):
    s = golden_system(golden, name)
    for dt in (np.float64, np.float32):
        a, ga = E.energy_and_gradient(s, dt)
        b, gb = E.energy_and_gradient(s, dt)
        assert a == b and np.array_equal(ga, gb)


def test_coincident_pair_error(golden, E):
    s = golden_system(golden, "coincident")
    for dt in (np.float64, np.float32):
        with pytest.raises(E.EnergyEvaluationError, match=r"nonbonded pair \(3,11\)"):
            E.energy_total(s, dt)
        with pytest.raises(E.EnergyEvaluationError, match=r"nonbonded pair \(3,11\)"):
            E.energy_and_gradient(s, dt)


@pytest.mark.parametrize("mode", ["units", "tiles", "units_sharded"])
def test_coincident_pair_found_in_every_sweep_mode(mode, monkeypatch):
    """Two coincident atoms far apart in index in a 3000-atom system: the
    super-unit chain (finder launched only when flagged, its last block
    finalising), the tile-mode fused evaluation and a sharded plan all
    report the reference's first bad pair, then evaluate cleanly again."""
    from paper_1810_03358_b200.energy import EnergyEvaluationError, energy_and_gradient
    from paper_1810_03358_b200.synth import make_globule_system

    monkeypatch.setenv("FFM_FORCE_TILES", "1" if mode == "tiles" else "0")
    s = make_globule_system(3000, seed=4)
    c = s.coords.copy()
    c[2500] = c[117]  # far from each other in the chain: not an excluded pair
    bad = s.with_coords(c)
    A = O.Arrays.from_system(bad)
    _, _, err = O.energy_and_gradient(A, c, True, threads=O.host_threads())
    assert err is not None
    if mode == "units_sharded":
        from paper_1810_03358_b200 import _native as N
        from paper_1810_03358_b200.engine import engine_for

        eng = engine_for(bad.topology)
        N.check(eng.lib.ffm_system_set_shard(eng.handle, 0, 1), "shard")
    for dt in (np.float64, np.float32):
        with pytest.raises(EnergyEvaluationError, match=r"nonbonded pair \(117,2500\)"):
            energy_and_gradient(bad, dt)
        bd, g = energy_and_gradient(s, dt)  # the status words reset
        assert np.isfinite(bd.total) and np.all(np.isfinite(g))


def test_degenerate_terms_raise_reference_messages(golden, E):
    s = golden_system(golden, "collinear")
    msgs = golden["collinear/messages"].tolist()
    with pytest.raises(E.EnergyEvaluationError) as ei:
        E.energy_total(s)
    assert str(ei.value) == msgs[0]
    with pytest.raises(E.EnergyEvaluationError) as ei:
        E.energy_and_gradient(s)
    assert str(ei.value) == msgs[1]


@pytest.mark.parametrize("name", ["chain14", "cloud24", "chain200"])
def test_exact_atom_deltas(golden, E, name):
    s = golden_system(golden, name)
    for a, d, want in zip(golden[f"{name}/delta_atoms"], golden[f"{name}/delta_moves"],
                          golden[f"{name}/delta_values"]):
        got = E.exact_delta_atom_move(s, int(a), d)
        assert got == pytest.approx(float(want), rel=1e-10, abs=1e-10)


def test_landmarks_and_constant(E):
    from paper_1810_03358_b200.model import AtomSpec, MolecularSystem, NonbondedPolicy

    def pair(r, q=0.0, sigma=3.0, eps=0.1):
        return MolecularSystem(atoms=(AtomSpec(0, "a", q, sigma, eps), AtomSpec(1, "b", q, sigma, eps)),
                               coords=np.array([[0.0, 0, 0], [r, 0, 0]]),
                               nonbonded=NonbondedPolicy.no_exclusions())

    assert E.energy_coulomb(pair(1.0, q=1.0, eps=0.0)) == pytest.approx(1389.38757, abs=1e-5)
    sig, eps = 3.4, 0.9
    assert abs(E.energy_vdw(pair(sig, sigma=sig, eps=eps))) <= 1e-10 * eps
    assert E.energy_vdw(pair(2 ** (1 / 6) * sig, sigma=sig, eps=eps)) == pytest.approx(-eps, rel=1e-10)
    assert E.energy_vdw(pair(0.3 * 3.5, sigma=3.5, eps=0.276)) > 1e6


def test_batch_equals_single_evaluations(golden):
    """eval_batch sweeps with the batch plan (the largest super-unit that
    divides np), single evaluations with the system's own plan: FP64 agrees
    to roundoff of the summation order; FP32 tiles are evaluated by
    different warp splits there, so FP32 agrees to FP32 roundoff."""
    import torch

    from paper_1810_03358_b200.engine import engine_for

    s = golden_system(golden, "globule1500")
    eng = engine_for(s.topology)
    rng = np.random.default_rng(3)
    B = 7
    batch = s.coords[None] + rng.normal(scale=0.05, size=(B,) + s.coords.shape)
    for prec in (0, 1):
        en, st = eng.eval_batch(torch.from_numpy(batch).cuda(), prec)
        en = en.cpu().numpy()
        for b in range(B):
            e1, st1, _ = eng.eval_host(batch[b], prec)
            if prec == 0:
                np.testing.assert_allclose(en[b], e1, rtol=1e-12, atol=1e-9)
            else:
                np.testing.assert_allclose(en[b], e1, rtol=1e-6,
                                           atol=1e-6 * float(np.sum(np.abs(e1))))
        assert np.all(st.cpu().numpy()[:, 0] == -1)


def test_kernel_backend_dropin(golden):
    """The 'cuda' KernelBackend answers the reference kernel signatures."""
    from paper_1810_03358_b200.kernels import get_backend

    kb = get_backend()
    assert kb.name == "cuda"
    s = golden_system(golden, "cloud24")
    p = s.arrays()
    c = np.ascontiguousarray(s.coords)
    A, _ = oracle_arrays(golden, "cloud24")
    ec, ev, _, _, gref = O.nb_eval(A, c, True)
    out = kb.nb_energy(c, p["q"], p["sigma"], p["epsilon"], p["scale"], 0.0)
    assert out[2:] == (-1, -1)
    assert out[0] == pytest.approx(ec, rel=1e-11) and out[1] == pytest.approx(ev, rel=1e-11)
    gout = np.zeros_like(c)
    r = kb.nb_grad(c, p["q"], p["sigma"], p["epsilon"], p["scale"], 0.0, gout)
    assert r[2:] == (-1, -1)
    assert np.max(np.abs(gout - gref)) <= 1e-10 * np.max(np.abs(gref))
    # the reference call with a 7 A cutoff (fresh parameter arrays -> fresh plan)
    A7, _ = oracle_arrays(golden, "cloud24c7")
    s7 = golden_system(golden, "cloud24c7")
    p7 = s7.arrays()
    ec7, ev7, _, _, _ = O.nb_eval(A7, c, False)
    out = kb.nb_energy(c, p7["q"], p7["sigma"], p7["epsilon"], p7["scale"], 7.0)
    assert out[0] == pytest.approx(ec7, rel=1e-11) and out[1] == pytest.approx(ev7, rel=1e-11)
    # bonded kernels on the chain
    s = golden_system(golden, "chain14")
    p = s.arrays()
    c = np.ascontiguousarray(s.coords)
    A, _ = oracle_arrays(golden, "chain14")
    (es, eb, et), _, gb = O.bonded(A, c, True)
    g = np.zeros_like(c)
    e, bad = kb.bond_grad(c, p["bond_idx"], p["bond_K"], p["bond_r0"], g)
    e2, bad2 = kb.angle_grad(c, p["ang_idx"], p["ang_K"], p["ang_t0"], g)
    e3, bad3 = kb.dihedral_grad(c, p["dih_idx"], p["dih_V"], g)
    assert (bad, bad2, bad3) == (-1, -1, -1)
    assert (e, e2, e3) == pytest.approx((es, eb, et), rel=1e-12)
    assert np.max(np.abs(g - gb)) <= 1e-11 * np.max(np.abs(gb))
    # coincident pair through the kernel API
    s = golden_system(golden, "coincident")
    p = s.arrays()
    out = kb.nb_energy(np.ascontiguousarray(s.coords), p["q"], p["sigma"], p["epsilon"],
                       p["scale"], 0.0)
    assert out[2:] == (3, 11)


def test_missing_native_library_fails_loudly(tmp_path):
    from paper_1810_03358_b200 import _native

    with pytest.raises(ImportError, match="missing"):
        _native.load(tmp_path / "nope.so")


# ------------------------------------------------------- full-size checks

@pytest.mark.parametrize("n", [10000, 20000, 30000, 100000])
def test_full_size_against_threaded_oracle(n):
    """BASELINE sizes: the whole FP32 / FP64 gradient against the C oracle
    run on all host cores, and the energy-only sweep's energies (the line
    search's probes).  10k: 8-warp FP32 / 4-warp FP64 CTAs on 256-atom
    units, three FP32 energy-only CTAs per SM; 20k: 4-warp FP32 CTAs (many
    256-atom units); 30k: 512-atom units; 100k: 1024-atom units."""
    from paper_1810_03358_b200.energy import energy_and_gradient, energy_total
    from paper_1810_03358_b200.synth import make_globule_system

    s = make_globule_system(n, seed=1)
    A = O.Arrays.from_system(s)
    e_ref, g_ref, err = O.energy_and_gradient(A, s.coords, True, threads=O.host_threads())
    assert err is None
    gmax = np.max(np.abs(g_ref))
    for dt, et, gt in ((np.float64, 1e-10, 1e-10), (np.float32, 1e-5, 1e-4)):
        bd, g = energy_and_gradient(s, dt)
        got = np.array([bd.stretch, bd.bend, bd.torsion, bd.coulomb, bd.vdw])
        assert _rel(got, e_ref) <= et, (dt, got, e_ref)
        assert np.max(np.abs(g - g_ref)) <= gt * gmax
        be = energy_total(s, dt)
        got_e = np.array([be.stretch, be.bend, be.torsion, be.coulomb, be.vdw])
        assert _rel(got_e, e_ref) <= et, (dt, got_e, e_ref)


def test_full_size_properties():
    """Size-independent properties at N = 100k: translation invariance,
    Newton's third law (net gradient ~ 0), FP32 ~ FP64."""
    from paper_1810_03358_b200.energy import energy_and_gradient
    from paper_1810_03358_b200.synth import make_globule_system

    s = make_globule_system(100000, seed=2)
    bd, g = energy_and_gradient(s, np.float64)
    gm = g.reshape(-1, 3)
    assert np.linalg.norm(gm.sum(axis=0)) <= 1e-9 * np.linalg.norm(g)
    bd2, _ = energy_and_gradient(s.with_coords(s.coords + np.array([3.25, -1.5, 0.75])),
                                 np.float64)
    assert bd2.total == pytest.approx(bd.total, rel=1e-9)
    bd3, g3 = energy_and_gradient(s, np.float32)
    assert bd3.total == pytest.approx(bd.total, rel=1e-5)
    assert np.max(np.abs(g3 - g)) <= 1e-4 * np.max(np.abs(g))


@pytest.mark.parametrize("world", [2, 3, 8])
def test_row_shards_sum_to_the_full_evaluation(world, n=20000):
    """ffm_system_set_shard on one GPU: the partial gradients / energies of
    all ranks, summed, equal the unsharded evaluation (what the NCCL
    all-reduce of parallel.ShardCombiner computes on W GPUs)."""
    import torch

    from paper_1810_03358_b200 import _native as N
    from paper_1810_03358_b200.engine import DeviceSystem
    from paper_1810_03358_b200.synth import make_globule_system

    s = make_globule_system(n, seed=4)
    c = torch.from_numpy(s.coords.copy()).cuda()
    full = DeviceSystem(s.topology)
    g_full = torch.empty_like(c)
    e_full, _ = full.eval(c, N.FFM_F64, grad=g_full)
    g_sum = torch.zeros_like(c)
    e_sum = torch.zeros(5, dtype=torch.float64, device=c.device)
    for rank in range(world):
        eng = DeviceSystem(s.topology)
        N.check(eng.lib.ffm_system_set_shard(eng.handle, rank, world), "set_shard")
        g = torch.empty_like(c)
        e, st = eng.eval(c, N.FFM_F64, grad=g)
        assert int(st[0]) == -1
        assert int(st[5]) == 0  # no spurious close-contact flag from other ranks' slots
        if rank != 0:
            assert float(e[0]) == float(e[1]) == float(e[2]) == 0.0  # bonded on rank 0 only
        g_sum += g
        e_sum += e
        eng.close()
    assert torch.allclose(e_sum, e_full, rtol=1e-12)
    assert float((g_sum - g_full).abs().max()) <= 1e-11 * float(g_full.abs().max())


@pytest.mark.parametrize("world", [2, 8])
def test_sharded_plan_replans_super_units(world):
    """60k atoms: the single-GPU plan uses 1024-atom super-units; a sharded
    plan shrinks them (each rank keeps ~6 waves of units) and the rank sums
    still equal the full evaluation; back to one rank restores the edge."""
    from paper_1810_03358_b200 import _native as N
    from paper_1810_03358_b200.engine import DeviceSystem
    from paper_1810_03358_b200.synth import make_globule_system

    s = make_globule_system(60000, seed=2)
    eng = DeviceSystem(s.topology)
    S0 = eng.info["S"]
    assert S0 == 1024
    N.check(eng.lib.ffm_system_set_shard(eng.handle, 0, world), "set_shard")
    info = np.zeros(8, np.int64)
    N.check(eng.lib.ffm_system_info(eng.handle, info.ctypes.data), "info")
    assert info[2] < S0 and info[4] >= 1700 * world
    N.check(eng.lib.ffm_system_set_shard(eng.handle, 0, 1), "set_shard")
    N.check(eng.lib.ffm_system_info(eng.handle, info.ctypes.data), "info")
    assert info[2] == S0
    eng.close()
    test_row_shards_sum_to_the_full_evaluation(world, n=60000)


def test_kernel_backend_farfield_functions(golden):
    from paper_1810_03358_b200.kernels import get_backend

    kb = get_backend("cuda")
    s = golden_system(golden, "ff40")
    p = s.arrays()
    c = np.ascontiguousarray(s.coords)
    for atom in (0, 23):
        e0, cx, cy, cz, near, bad = kb.farfield_build(c, p["q"], p["scale"], atom, 7.0)
        ref = golden[f"ff40/lin{atom}"]
        assert bad == -1
        np.testing.assert_allclose([e0, cx, cy, cz], ref, rtol=1e-11, atol=1e-12)
        assert np.array_equal(np.nonzero(near)[0], golden[f"ff40/near{atom}"])
        newpos = c[atom] + np.array([0.1, -0.2, 0.05])
        dec, dev, bad = kb.near_nb_delta(c, p["q"], p["sigma"], p["epsilon"], p["scale"],
                                         atom, newpos, np.nonzero(near)[0])
        A, _ = oracle_arrays(golden, "ff40")
        # oracle: exact delta restricted to the near set
        import oracle as OO
        mask = np.zeros(A.n, bool)
        mask[np.nonzero(near)[0]] = True
        mask[atom] = True
        A.q = np.where(mask, A.q, 0.0)
        A.eps = np.where(mask, A.eps, 0.0)
        parts, b2 = OO.atom_delta(A, c, atom, newpos - c[atom])
        assert bad == b2 == -1
        assert dec == pytest.approx(parts[0], rel=1e-10, abs=1e-10)
        assert dev == pytest.approx(parts[1], rel=1e-10, abs=1e-10)


@pytest.mark.parametrize("cutoff", [7.0, 12.0])
def test_cutoff_culling_matches_oracle(cutoff):
    """With a cutoff, super-units and tiles whose bounding boxes are farther
    apart than the cutoff are skipped; the result must equal the oracle's
    (which evaluates every pair and drops r > cutoff, kernels.py:303)."""
    from paper_1810_03358_b200.energy import energy_and_gradient
    from paper_1810_03358_b200.synth import make_globule_system

    s = make_globule_system(30000, seed=5, cutoff=cutoff)
    A = O.Arrays.from_system(s)
    e_ref, g_ref, err = O.energy_and_gradient(A, s.coords, True, threads=O.host_threads())
    assert err is None
    gmax = np.max(np.abs(g_ref))
    # FP32 classifies r <= cutoff from an FP32 r^2 (as the reference's float32
    # kernels do), so pairs within ~1e-6 relative of the cutoff may flip;
    # atoms owning such a pair are exempt from the FP32 gradient check
    from scipy.spatial import cKDTree

    tree = cKDTree(s.coords)
    outer = tree.query_pairs(cutoff * (1 + 1e-5), output_type="ndarray")
    d = np.linalg.norm(s.coords[outer[:, 0]] - s.coords[outer[:, 1]], axis=1)
    edge = outer[d > cutoff * (1 - 1e-5)]
    keep = np.ones(s.natoms, bool)
    keep[edge.ravel()] = False
    assert keep.mean() > 0.95
    for dt, et, gt in ((np.float64, 1e-10, 1e-10), (np.float32, 1e-5, 1e-4)):
        bd, g = energy_and_gradient(s, dt)
        got = np.array([bd.stretch, bd.bend, bd.torsion, bd.coulomb, bd.vdw])
        assert _rel(got, e_ref) <= et
        m = keep if dt is np.float32 else np.ones(s.natoms, bool)
        dg = np.abs(np.reshape(g, (-1, 3)) - np.reshape(g_ref, (-1, 3)))
        assert np.max(dg[m]) <= gt * gmax


@pytest.mark.parametrize("S", [128, 256, 512, 768, 1024])
def test_every_super_unit_size(S, monkeypatch):
    """The unit size is picked from {256, 512, 768, 1024} by system size
    (128 for FP64 callers of mid-size systems, ffm_preferred_edge); force
    each one (FFM_FORCE_S, read at plan creation) on one system, with
    special pairs and a ragged last block, and compare with the oracle."""
    from paper_1810_03358_b200.energy import energy_and_gradient
    from paper_1810_03358_b200.engine import DeviceSystem
    from paper_1810_03358_b200.synth import make_globule_system

    monkeypatch.setenv("FFM_FORCE_S", str(S))
    monkeypatch.setenv("FFM_FORCE_TILES", "0")  # super-unit sweep even at this size
    s = make_globule_system(2900, seed=11)
    assert DeviceSystem(s.topology).info["S"] == S
    A = O.Arrays.from_system(s)
    e_ref, g_ref, err = O.energy_and_gradient(A, s.coords, True, threads=O.host_threads())
    assert err is None
    gmax = np.max(np.abs(g_ref))
    for dt, et, gt in ((np.float64, 1e-10, 1e-10), (np.float32, 1e-5, 1e-4)):
        bd, g = energy_and_gradient(s, dt)
        got = np.array([bd.stretch, bd.bend, bd.torsion, bd.coulomb, bd.vdw])
        assert _rel(got, e_ref) <= et
        assert np.max(np.abs(np.ravel(g) - np.ravel(g_ref))) <= gt * gmax


@pytest.mark.parametrize("n,cutoff", [(37, None), (300, None), (1000, 9.0), (4100, None)])
def test_tile_sweep_matches_oracle_and_unit_sweep(n, cutoff, monkeypatch):
    """Small systems sweep one warp per 128 x 32 tile (nb_tiles_kernel):
    same energies / gradients as the oracle and as the super-unit sweep,
    ragged last blocks, cutoff, and row-sharded partial sums."""
    import torch

    from paper_1810_03358_b200 import _native as N
    from paper_1810_03358_b200.engine import DeviceSystem
    from paper_1810_03358_b200.synth import make_globule_system

    s = make_globule_system(n, seed=7, cutoff=cutoff)
    A = O.Arrays.from_system(s)
    e_ref, g_ref, err = O.energy_and_gradient(A, s.coords, True, threads=O.host_threads())
    assert err is None
    gmax = np.max(np.abs(g_ref))
    c = torch.from_numpy(s.coords.copy()).cuda()
    out = {}
    for tiles in ("1", "0"):
        monkeypatch.setenv("FFM_FORCE_TILES", tiles)
        eng = DeviceSystem(s.topology)
        for prec, et, gt in ((N.FFM_F64, 1e-10, 1e-10), (N.FFM_F32, 1e-5, 1e-4)):
            g = torch.empty_like(c)
            e, st = eng.eval(c, prec, grad=g)
            e = e.cpu().numpy()
            assert int(st[0]) == -1
            assert _rel(e, e_ref) <= et
            assert np.max(np.abs(g.cpu().numpy().ravel() - g_ref.ravel())) <= gt * gmax
            out[(tiles, prec)] = (e, g.cpu().numpy())
        eng.close()
    # row shards of the tile sweep sum to the full evaluation
    monkeypatch.setenv("FFM_FORCE_TILES", "1")
    e_sum, g_sum = 0.0, 0.0
    for rank in range(3):
        eng = DeviceSystem(s.topology)
        N.check(eng.lib.ffm_system_set_shard(eng.handle, rank, 3), "set_shard")
        g = torch.empty_like(c)
        e, st = eng.eval(c, N.FFM_F64, grad=g)
        assert int(st[5]) == 0
        e_sum = e_sum + e.cpu().numpy()
        g_sum = g_sum + g.cpu().numpy()
        eng.close()
    np.testing.assert_allclose(e_sum, out[("1", N.FFM_F64)][0], rtol=1e-12, atol=1e-9)
    assert np.max(np.abs(g_sum - out[("1", N.FFM_F64)][1])) <= 1e-11 * gmax


@pytest.mark.parametrize("n", [1, 2, 3, 31, 32, 33, 128, 129])
def test_tiny_and_block_edge_systems(n):
    """Atom counts at and around the 32-atom block and 128-row sub-block
    edges (and a single atom): energies and gradients equal the oracle's."""
    from paper_1810_03358_b200.energy import energy_and_gradient
    from paper_1810_03358_b200.model import MolecularSystem

    rng = np.random.default_rng(n)
    side = int(np.ceil(max(1, n) ** (1 / 3)))
    grid = np.stack(np.meshgrid(*[np.arange(side)] * 3, indexing="ij"), -1).reshape(-1, 3)
    coords = 3.2 * grid[rng.permutation(len(grid))[:n]] + rng.uniform(-0.4, 0.4, size=(n, 3))
    s = MolecularSystem.from_arrays(rng.uniform(-0.5, 0.5, n), rng.uniform(2.5, 3.5, n),
                                    rng.uniform(0.05, 0.2, n), coords)
    A = O.Arrays.from_system(s)
    e_ref, g_ref, err = O.energy_and_gradient(A, s.coords, True, threads=1)
    if err is not None:
        pytest.skip("random cloud has a coincident pair")
    gmax = max(np.max(np.abs(g_ref)), 1e-300)
    for dt, et, gt in ((np.float64, 1e-10, 1e-10), (np.float32, 1e-5, 1e-4)):
        bd, g = energy_and_gradient(s, dt)
        got = np.array([bd.stretch, bd.bend, bd.torsion, bd.coulomb, bd.vdw])
        assert np.max(np.abs(got - e_ref)) <= et * max(1.0, np.max(np.abs(e_ref)))
        assert np.max(np.abs(np.ravel(g) - np.ravel(g_ref))) <= gt * gmax


@pytest.mark.parametrize("fromx", ["default", "forced", "off"])
@pytest.mark.parametrize("name", ["chain10", "cloud24", "cloud24c7", "chain200", "chain12cut",
                                  "globule1500", "coincident", "collinear", "explicit8"])
def test_fused_small_evaluation_equals_kernel_chain(golden, name, fromx, monkeypatch):
    """Small (tile-mode) systems evaluate in one cooperative launch
    (ffm_small.cu) running the same per-item bodies as the kernel chain:
    energies, gradient and status words must be bit-identical, in both
    precisions, with and without the gradient, error cases included -- for
    both kernel variants (fromx: the variant without the packing pass, as
    chosen by size, forced for every size and precision, or never)."""
    import torch

    from paper_1810_03358_b200 import _native as N
    from paper_1810_03358_b200.engine import engine_for

    if fromx == "forced":
        monkeypatch.setenv("FFM_SMALL_FROMX_MAXN", "1000000")
        monkeypatch.setenv("FFM_SMALL_FROMX_F64", "1")
    elif fromx == "off":
        monkeypatch.setenv("FFM_SMALL_FROMX_MAXN", "0")
    s = golden_system(golden, name)
    eng = engine_for(s.topology)
    c = torch.from_numpy(np.ascontiguousarray(s.coords)).cuda()
    lib = N.load()
    for prec in (N.FFM_F64, N.FFM_F32):
        for grad in (False, True):
            base = N.FFM_ENERGY | (N.FFM_GRAD if grad else 0) | N.FFM_NO_GRAPH
            en, st = eng.new_outputs()
            for extra in (0, N.FFM_NO_FUSE):  # first call sizes the workspace
                eng.eval(c, prec, grad=torch.empty_like(c) if grad else None, energies=en,
                         status=st, flags=base | extra)
            out = []
            for extra in (0, N.FFM_NO_FUSE):
                g = torch.full_like(c, np.nan) if grad else None
                en, st = eng.new_outputs()
                torch.cuda.synchronize()
                l0 = lib.ffm_launch_count()
                eng.eval(c, prec, grad=g, energies=en, status=st, flags=base | extra)
                torch.cuda.synchronize()
                out.append((lib.ffm_launch_count() - l0, en.cpu().numpy(), st.cpu().numpy(),
                            None if g is None else g.cpu().numpy()))
            (l_f, e_f, s_f, g_f), (l_c, e_c, s_c, g_c) = out
            assert l_f == 1 and l_c >= 4, (l_f, l_c)
            assert np.array_equal(e_f, e_c, equal_nan=True), (prec, grad, e_f, e_c)
            assert np.array_equal(s_f, s_c), (prec, grad, s_f, s_c)
            if grad:
                assert np.array_equal(g_f, g_c, equal_nan=True)


@pytest.mark.parametrize("S", [256, 512, 1024])
def test_split_last_wave_units(S, monkeypatch):
    """Units of the last wave evaluated in halves (rows [0, nsub/2) and
    [nsub/2, nsub) as separate units with their own partial slots; the
    gather's unit lists take both): forced on small systems of every unit
    edge, against the oracle and summed over row shards."""
    from paper_1810_03358_b200 import _native as N
    from paper_1810_03358_b200.energy import energy_and_gradient
    from paper_1810_03358_b200.engine import DeviceSystem
    from paper_1810_03358_b200.synth import make_globule_system

    import torch

    monkeypatch.setenv("FFM_FORCE_S", str(S))
    monkeypatch.setenv("FFM_FORCE_TILES", "0")
    monkeypatch.setenv("FFM_SPLIT_UNITS", "7")
    s = make_globule_system(4700, seed=12)
    info = DeviceSystem(s.topology).info
    nb = info["np"] // S
    assert info["units"] == nb * (nb + 1) // 2 + 7
    A = O.Arrays.from_system(s)
    e_ref, g_ref, err = O.energy_and_gradient(A, s.coords, True, threads=O.host_threads())
    gmax = np.max(np.abs(g_ref))
    for dt, et, gt in ((np.float64, 1e-10, 1e-10), (np.float32, 1e-5, 1e-4)):
        bd, g = energy_and_gradient(s, dt)
        got = np.array([bd.stretch, bd.bend, bd.torsion, bd.coulomb, bd.vdw])
        assert _rel(got, e_ref) <= et
        assert np.max(np.abs(np.ravel(g) - np.ravel(g_ref))) <= gt * gmax
    c = torch.from_numpy(s.coords.copy()).cuda()
    g_sum = torch.zeros_like(c)
    for rank in range(3):
        eng = DeviceSystem(s.topology)
        N.check(eng.lib.ffm_system_set_shard(eng.handle, rank, 3), "set_shard")
        g = torch.empty_like(c)
        eng.eval(c, N.FFM_F64, grad=g)
        g_sum += g
        eng.close()
    assert float((g_sum.cpu().numpy().ravel() - np.ravel(g_ref)).__abs__().max()) <= 1e-10 * gmax


def test_fp64_preferred_edge_engine():
    """FP64 callers of a mid-size system get an engine planned on 128-atom
    super-units (ffm_preferred_edge / ffm_system_set_edge); FP32 callers and
    other sizes keep the default plan.  Both plans agree with the oracle."""
    import ctypes as C

    from paper_1810_03358_b200 import _native as N
    from paper_1810_03358_b200.energy import energy_and_gradient
    from paper_1810_03358_b200.engine import engine_for
    from paper_1810_03358_b200.oracle import MolecularOracle
    from paper_1810_03358_b200.synth import make_globule_system

    lib = N.load()
    edge = C.c_int(-1)
    for n, e64, e32 in ((500, 0, 0), (5000, 128, 256), (20000, 256, 256), (100000, 1024, 1024)):
        N.check(lib.ffm_preferred_edge(n, N.FFM_F64, C.byref(edge)), "edge")
        assert edge.value == e64, n
        N.check(lib.ffm_preferred_edge(n, N.FFM_F32, C.byref(edge)), "edge")
        assert edge.value == e32, n
    s = make_globule_system(5000, seed=4)
    e_def = engine_for(s.topology)
    e64 = engine_for(s.topology, precision=np.float64)
    assert e_def.info["S"] == 256 and e64.info["S"] == 128 and e64 is not e_def
    assert engine_for(s.topology, precision=np.float32) is e_def
    assert MolecularOracle(s).engine is e64
    assert MolecularOracle(s, np.float32).engine is e_def
    A = O.Arrays.from_system(s)
    e_ref, g_ref, err = O.energy_and_gradient(A, s.coords, True, threads=O.host_threads())
    assert err is None
    bd, g = energy_and_gradient(s, np.float64)
    got = np.array([bd.stretch, bd.bend, bd.torsion, bd.coulomb, bd.vdw])
    assert _rel(got, e_ref) <= 1e-10
    assert np.max(np.abs(np.ravel(g) - np.ravel(g_ref))) <= 1e-10 * np.max(np.abs(g_ref))
    en, st, g_def = e_def.eval_host(s.coords, N.FFM_F64, grad=True)
    assert _rel(en, e_ref) <= 1e-10
    # invalid edges are refused, the plan is unchanged
    assert lib.ffm_system_set_edge(e64.handle, 192) != 0
    assert lib.ffm_system_set_edge(e64.handle, 2048) != 0
    small = engine_for(make_globule_system(600, seed=1).topology)  # tile mode
    assert lib.ffm_system_set_edge(small.handle, 256) != 0
    e64.refresh_info()
    assert e64.info["S"] == 128


def test_edge_128_plan_shards():
    """A 128-edge plan stays 128 when sharded, and its row shards sum to the
    unsharded evaluation (FP64)."""
    import torch

    from paper_1810_03358_b200 import _native as N
    from paper_1810_03358_b200.engine import DeviceSystem
    from paper_1810_03358_b200.synth import make_globule_system

    s = make_globule_system(5000, seed=9)
    c = torch.from_numpy(s.coords.copy()).cuda()
    full = DeviceSystem(s.topology)
    N.check(full.lib.ffm_system_set_edge(full.handle, 128), "set_edge")
    g_full = torch.empty_like(c)
    e_full, _ = full.eval(c, N.FFM_F64, grad=g_full)
    g_sum, e_sum = torch.zeros_like(c), torch.zeros(5, dtype=torch.float64, device="cuda")
    for rank in range(2):
        eng = DeviceSystem(s.topology)
        N.check(eng.lib.ffm_system_set_edge(eng.handle, 128), "set_edge")
        N.check(eng.lib.ffm_system_set_shard(eng.handle, rank, 2), "set_shard")
        eng.refresh_info()
        assert eng.info["S"] == 128
        g = torch.empty_like(c)
        en, _ = eng.eval(c, N.FFM_F64, grad=g)
        g_sum += g
        e_sum += en
        eng.close()
    gmax = float(g_full.abs().max())
    assert float((g_sum - g_full).abs().max()) <= 1e-11 * gmax
    assert float(((e_sum - e_full).abs() / e_full.abs().clamp_min(1e-12)).max()) <= 1e-12
