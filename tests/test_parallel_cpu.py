"""Row-sharding host logic with world_size 2 on CPU (gloo): the unit
partition and the all-reduce that completes the partial gradients /
energies / error words of each rank."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1810_03358_b200.parallel import shard_units, unit_order


def test_units_partition_exactly_and_balanced():
    for nb in (1, 2, 5, 40, 98):
        units = unit_order(nb)
        assert len(units) == nb * (nb + 1) // 2 == len(set(units))
        for world in (1, 2, 3, 4, 8):
            parts = [shard_units(len(units), r, world) for r in range(world)]
            flat = sorted(u for p in parts for u in p)
            assert flat == list(range(len(units)))
            # work of a unit: full square off the diagonal, half on it
            work = [sum(0.5 if units[u][0] == units[u][1] else 1.0 for u in p) for p in parts]
            assert max(work) - min(work) <= 1.0


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, golden_path, q, both=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, os.path.dirname(__file__))
        import oracle as O
        from conftest import oracle_arrays
        from paper_1810_03358_b200 import _native as N
        from paper_1810_03358_b200.parallel import ShardCombiner

        G = np.load(golden_path)
        A, c = oracle_arrays(G, "globule1500")
        n = A.n
        # this rank's share: a row slice of the pair triangle, bonded on rank 0
        edges = np.linspace(0, n, world + 1).astype(int)
        ec, ev, bi, bj, gn = O.nb_eval(A, c, True, threads=2, rows=(edges[rank], edges[rank + 1]))
        (es, eb, et), bad, gb = O.bonded(A, c, True)
        if rank != 0:
            es = eb = et = 0.0
            gb = np.zeros_like(gb)
        grad = torch.from_numpy((gn + gb).reshape(-1).copy())
        energies = torch.tensor([es, eb, et, ec, ev], dtype=torch.float64)
        status = torch.full((N.FFM_STATUS_WORDS,), -1, dtype=torch.int64)
        if rank == 1 or both:  # pretend rank 1 (or every rank) found the first coincident pair
            status[N.ST_NB_BAD_I], status[N.ST_NB_BAD_J] = 7, 9
        if rank == 0:  # and rank 0, which evaluates the bonded terms, a bad angle
            status[N.ST_ANGLE] = 4
        comb = ShardCombiner(n, "cpu")
        comb.combine(grad, energies, status)
        q.put((rank, grad.numpy().copy(), energies.numpy().copy(), status.numpy().copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("both", [False, True])
def test_two_rank_combine_equals_full_evaluation(golden, both):
    """One SUM all-reduce completes gradient, energies and the error words
    (a key reported by one rank or by both)."""
    from conftest import GOLDEN

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, str(GOLDEN), q, both))
             for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    res.sort(key=lambda t: t[0])
    ref_g = golden["globule1500/grad_f64"]
    ref_e = golden["globule1500/egrad_f64"]
    for _, g, e, st in res:
        assert np.max(np.abs(g - ref_g)) <= 1e-12 * np.max(np.abs(ref_g))
        np.testing.assert_allclose(e, ref_e, rtol=1e-12)
        assert st[0] == 7 and st[1] == 9 and st[3] == 4 and st[2] == -1 and st[4] == -1
    # every rank holds bit-identical results (replicated optimiser state)
    assert np.array_equal(res[0][1], res[1][1]) and np.array_equal(res[0][2], res[1][2])
