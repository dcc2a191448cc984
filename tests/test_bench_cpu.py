"""bench.py's rank handling (CPU only): --gpus N without a torchrun
environment re-executes under torch.distributed.run with N ranks on
127.0.0.1; a WORLD_SIZE that disagrees with --gpus is refused, so a scaling
run can never report the wrong N."""

import argparse
import importlib.util
import subprocess
import sys

import pytest

from conftest import ROOT


@pytest.fixture()
def bench(monkeypatch):
    spec = importlib.util.spec_from_file_location("bench_under_test", ROOT / "bench.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_gpus_n_relaunches_under_torchrun(bench, monkeypatch):
    seen = {}

    def fake_call(cmd, env=None):
        seen["cmd"], seen["env"] = cmd, env
        return 0

    monkeypatch.setattr(subprocess, "call", fake_call)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "2"])
    rc = bench.launch_ranks(argparse.Namespace(gpus=4))
    cmd = seen["cmd"]
    assert rc == 0
    assert cmd[:3] == [sys.executable, "-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--nnodes=1" in cmd
    assert cmd[cmd.index("--master-addr") + 1] == "127.0.0.1"
    assert cmd[-4:] == ["--gpus", "4", "--steps", "2"] and cmd[-5].endswith("bench.py")


def test_mismatched_world_is_refused(bench, monkeypatch):
    monkeypatch.setenv("WORLD_SIZE", "2")
    monkeypatch.setenv("RANK", "1")
    monkeypatch.setenv("LOCAL_RANK", "1")
    with pytest.raises(SystemExit, match="--gpus 4 but WORLD_SIZE=2"):
        bench.world_from_env(argparse.Namespace(gpus=4))
    assert bench.world_from_env(argparse.Namespace(gpus=2)) == (1, 2, 1)
