"""Row sharding across processes with the real CUDA shards: two ranks on one
GPU, completed by parallel.ShardCombiner over gloo (CUDA tensors; the
exchange goes through the host, so no kernel of one rank waits on the
other -- NCCL itself refuses two ranks on one device).

Each rank evaluates its share of the super-units (ffm_system_set_shard,
the deal of csrc/ffm_capi.cu) and rank 0 the O(N) terms; one SUM
all-reduce completes them (the reference's contract for this split is a
reduction over the outer index of kernels.py:316-356).
Checked: energies and gradients equal the unsharded evaluation, both ranks
hold bit-identical results, error words survive the reduction, and 15
host-loop L-BFGS iterations on the sharded oracle follow the unsharded run
(a max_wall_time budget stops both ranks at the same iteration)."""

import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

N_ATOMS = 6000


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port),
                      FFMIN_B200_HOST_LOOP="1")
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1810_03358_b200 import _native as N
        from paper_1810_03358_b200.optimizers import StopCriteria, lbfgs, make_linesearch
        from paper_1810_03358_b200.parallel import ShardedMolecularOracle, ShardedSystem
        from paper_1810_03358_b200.synth import make_globule_system

        s = make_globule_system(N_ATOMS, seed=21)
        out = {}
        sh = ShardedSystem(s.topology, device=0)
        assert not sh.native
        x = torch.from_numpy(np.array(s.coords)).cuda()
        bad = x.clone()
        bad[N_ATOMS - 7] = bad[11]  # a coincident pair: the error words travel
        for prec, tag in ((N.FFM_F64, "f64"), (N.FFM_F32, "f32")):
            g = torch.empty_like(x)
            e, st = sh.eval(x, prec, grad=g)
            out[f"e_{tag}"] = e.cpu().numpy()
            out[f"g_{tag}"] = g.cpu().numpy()
            out[f"st_{tag}"] = st.cpu().numpy()
            e, st = sh.eval(bad, prec)
            out[f"bad_{tag}"] = st.cpu().numpy()
        sh.engine.close()
        o = ShardedMolecularOracle(s, device=0)
        r = lbfgs(o, s.coords.ravel(), m=4, linesearch=make_linesearch("par"),
                  stop=StopCriteria(max_iterations=15, gradient_norm_rtol=0.0))
        out["f_trace"] = np.array([t.f for t in r.trace.records])
        out["calls"] = np.array([(t.value_calls, t.grad_calls) for t in r.trace.records])
        out["x"] = np.asarray(r.x)
        # a wall-time budget: the stop decision is the MAX over ranks
        t = lbfgs(o, s.coords.ravel(), m=4, linesearch=make_linesearch("par"),
                  stop=StopCriteria(max_iterations=10_000, max_wall_time=0.3,
                                    gradient_norm_rtol=0.0))
        out["wall_iterations"] = t.iterations
        out["wall_status"] = t.status
        q.put((rank, out))
    except Exception as exc:  # surface the failure in the parent
        q.put((rank, repr(exc)))
        raise
    finally:
        dist.destroy_process_group()


@pytest.fixture(scope="module")
def two_ranks():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(120)
    for r in (0, 1):
        assert not isinstance(res[r], str), res[r]
    assert all(p.exitcode == 0 for p in procs)
    return res


@pytest.fixture(scope="module")
def unsharded():
    from paper_1810_03358_b200 import _native as N
    from paper_1810_03358_b200.engine import DeviceSystem
    from paper_1810_03358_b200.optimizers import StopCriteria, lbfgs, make_linesearch
    from paper_1810_03358_b200.oracle import MolecularOracle
    from paper_1810_03358_b200.synth import make_globule_system

    os.environ["FFMIN_B200_HOST_LOOP"] = "1"
    try:
        s = make_globule_system(N_ATOMS, seed=21)
        eng = DeviceSystem(s.topology, 0)
        x = torch.from_numpy(np.array(s.coords)).cuda()
        out = {}
        for prec, tag in ((N.FFM_F64, "f64"), (N.FFM_F32, "f32")):
            g = torch.empty_like(x)
            e, st = eng.eval(x, prec, grad=g)
            out[f"e_{tag}"] = e.cpu().numpy()
            out[f"g_{tag}"] = g.cpu().numpy()
        eng.close()
        o = MolecularOracle(s, device=0)
        r = lbfgs(o, s.coords.ravel(), m=4, linesearch=make_linesearch("par"),
                  stop=StopCriteria(max_iterations=15, gradient_norm_rtol=0.0))
        out["f_trace"] = np.array([t.f for t in r.trace.records])
        out["calls"] = np.array([(t.value_calls, t.grad_calls) for t in r.trace.records])
        out["x"] = np.asarray(r.x)
        return out
    finally:
        del os.environ["FFMIN_B200_HOST_LOOP"]


def test_ranks_hold_identical_results(two_ranks):
    a, b = two_ranks[0], two_ranks[1]
    for k in a:
        if k.startswith(("st_", "bad_")):  # the five reported words (the rest are rank-local)
            assert np.array_equal(a[k][:5], b[k][:5]), k
        elif isinstance(a[k], np.ndarray):
            assert np.array_equal(a[k], b[k], equal_nan=True), k
        else:
            assert a[k] == b[k], k


@pytest.mark.parametrize("tag,tol", [("f64", 1e-12), ("f32", 1e-6)])
def test_sharded_evaluation_equals_unsharded(two_ranks, unsharded, tag, tol):
    """Partial sums of two ranks all-reduced = the one-rank evaluation
    (summation order differs: tolerance, not bits)."""
    r = two_ranks[0]
    np.testing.assert_allclose(r[f"e_{tag}"], unsharded[f"e_{tag}"], rtol=tol, atol=0)
    g, gu = r[f"g_{tag}"], unsharded[f"g_{tag}"]
    assert np.max(np.abs(g - gu)) <= tol * np.max(np.abs(gu))
    assert (r[f"st_{tag}"][:5] == -1).all()


@pytest.mark.parametrize("tag", ["f64", "f32"])
def test_error_words_survive_the_reduction(two_ranks, tag):
    """The first coincident pair is reported by whichever rank flags it and
    decoded identically on both (key = sum / count - 1)."""
    st = two_ranks[0][f"bad_{tag}"]
    assert (st[0], st[1]) == (11, N_ATOMS - 7)


def test_sharded_lbfgs_follows_unsharded(two_ranks, unsharded):
    r = two_ranks[0]
    assert len(r["f_trace"]) == len(unsharded["f_trace"]) == 16
    # two summation orders of the same FP64 sums: roundoff amplified over
    # 15 steepest-descent-like iterations from a strained start (measured 1e-9)
    np.testing.assert_allclose(r["f_trace"], unsharded["f_trace"], rtol=1e-7, atol=0)
    assert np.array_equal(r["calls"][:, 1], unsharded["calls"][:, 1])
    assert np.max(np.abs(r["calls"][:, 0] - unsharded["calls"][:, 0])) <= 3
    assert np.max(np.abs(r["x"] - unsharded["x"])) <= 1e-5


def test_wall_time_budget_stops_ranks_together(two_ranks):
    assert two_ranks[0]["wall_status"] == "time_budget"
    assert two_ranks[0]["wall_iterations"] == two_ranks[1]["wall_iterations"]
