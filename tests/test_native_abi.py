"""The C ABI: the library builds for sm_100a, loads, and exports exactly the
functions include/ffmin_b200.h declares (no GPU needed)."""

import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "ffmin_b200.h"


def declared():
    src = HEADER.read_text()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return set(re.findall(r"\b(ffm_[a-z0-9_]+)\s*\(", src))


@pytest.fixture(scope="module")
def lib_path():
    from paper_1810_03358_b200 import _build

    return _build.build()


def test_header_declares_the_binding_table():
    from paper_1810_03358_b200._native import SIGNATURES

    assert declared() == set(SIGNATURES)


def test_library_exports_every_declared_symbol(lib_path):
    out = subprocess.run(["nm", "-D", "--defined-only", str(lib_path)], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r" T (ffm_[a-z0-9_]+)$", out, flags=re.M))
    assert declared() <= exported
    assert exported == declared(), f"undeclared exports: {exported - declared()}"


def test_library_loads_and_types_every_entry_point(lib_path):
    from paper_1810_03358_b200 import _native

    lib = _native.load()
    assert lib.ffm_version().decode().startswith("ffmin_b200")
    assert lib.ffm_vec_scratch_doubles() >= 5 * 296
    assert lib.ffm_launch_count() >= 0


def test_library_is_sm100a_code(lib_path):
    out = subprocess.run(["cuobjdump", "--list-elf", str(lib_path)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_pair_kernel_uses_packed_fp32(lib_path):
    sass = subprocess.run(["cuobjdump", "-sass", str(lib_path)], capture_output=True,
                          text=True).stdout
    assert "FFMA2" in sass and "FMUL2" in sass and "MUFU.RSQ" in sass


def test_missing_library_fails_loudly(tmp_path):
    from paper_1810_03358_b200 import _native

    with pytest.raises(ImportError, match="missing"):
        _native.load(tmp_path / "libffmin_b200.so")


def test_energy_layer_refuses_cpu(monkeypatch):
    import torch

    from paper_1810_03358_b200 import engine

    monkeypatch.setattr(torch.cuda, "is_available", lambda: False)
    with pytest.raises(RuntimeError, match="no CPU execution path"):
        engine.require_cuda()
