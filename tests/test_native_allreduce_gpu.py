"""Sharded evaluations completed on the device: the NCCL communicator
attached to the engine (ffm_system_set_comm) all-reduces [gradient |
energies | error words] inside every evaluation, including the ones the
graph-resident drivers capture.  One GPU: a one-rank NCCL group with the
plan sharded as rank 0 of 2, so the all-reduce is the identity on rank 0's
partial sums -- the same numbers parallel.ShardCombiner produces."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.fixture(scope="module")
def nccl1():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield
    dist.destroy_process_group()


def _half(oracle_or_system):
    from paper_1810_03358_b200 import _native as N

    eng = oracle_or_system
    N.check(eng.lib.ffm_system_set_shard(eng.handle, 0, 2), "set_shard")


@pytest.mark.parametrize("n", [3000, 8000])
def test_device_allreduce_equals_python_combiner(nccl1, n):
    from paper_1810_03358_b200 import _native as N
    from paper_1810_03358_b200.parallel import ShardedSystem
    from paper_1810_03358_b200.synth import make_globule_system

    s = make_globule_system(n, seed=8)
    c = s.coords.copy()
    c[n - 10] = c[5]  # a coincident pair: the error words travel too
    outs = []
    for native in (True, False):
        sh = ShardedSystem(s.topology, native=native)
        assert sh.native == native
        _half(sh)
        for coords in (s.coords, c):
            x = torch.from_numpy(np.array(coords)).cuda()
            g = torch.empty_like(x)
            for prec in (N.FFM_F64, N.FFM_F32):
                e, st = sh.eval(x, prec, grad=g)
                outs.append((native, e.cpu().numpy(), st.cpu().numpy(), g.cpu().numpy()))
                e2, st2 = sh.eval(x, prec)
                outs.append((native, e2.cpu().numpy(), st2.cpu().numpy(), None))
        sh.engine.close()
    half = len(outs) // 2
    for a, b in zip(outs[:half], outs[half:]):
        assert np.array_equal(a[1], b[1], equal_nan=True) and np.array_equal(a[2][:5], b[2][:5])
        if a[3] is not None:
            assert np.array_equal(a[3], b[3], equal_nan=True)
    # (whether rank 0's half of the triangle holds the coincident pair depends
    # on the deal; both paths must agree either way -- checked above)


def test_graph_driver_on_sharded_oracle(nccl1, monkeypatch):
    """L-BFGS on a sharded oracle with the device all-reduce: the captured
    iterations (NCCL inside conditional graph bodies) equal the host loop."""
    from paper_1810_03358_b200.optimizers import StopCriteria, lbfgs, make_linesearch
    from paper_1810_03358_b200.parallel import ShardedMolecularOracle
    from paper_1810_03358_b200.synth import make_globule_system

    s = make_globule_system(6000, seed=9)
    res = []
    for host in (True, False):
        if host:
            monkeypatch.setenv("FFMIN_B200_HOST_LOOP", "1")
        else:
            monkeypatch.delenv("FFMIN_B200_HOST_LOOP", raising=False)
        o = ShardedMolecularOracle(s, native=True)
        assert o.native
        _half(o._base.engine)
        r = lbfgs(o, s.coords.ravel(), m=4, linesearch=make_linesearch("par"),
                  stop=StopCriteria(max_iterations=15, gradient_norm_rtol=0.0))
        res.append((r, o))
    (a, oa), (b, ob) = res
    assert "_graph_runs" in ob.__dict__
    ra = [(r.f, r.grad_norm, r.step, r.value_calls, r.grad_calls) for r in a.trace.records]
    rb = [(r.f, r.grad_norm, r.step, r.value_calls, r.grad_calls) for r in b.trace.records]
    assert ra == rb and np.array_equal(a.x, b.x)
