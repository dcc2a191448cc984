"""Build the native engine (csrc/*.cu) into _lib/libffmin_b200.so.

nvcc cross-compiles sm_100a without a GPU, so this runs anywhere the CUDA
toolkit is installed; the resulting .so lives in-tree and travels with the
repository snapshot to the GPU box.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB_DIR = PKG / "_lib"
LIB = LIB_DIR / "libffmin_b200.so"
INCLUDE = PKG.parent / "include"
SOURCES = ("ffm_pairs.cu", "ffm_terms.cu", "ffm_small.cu", "ffm_vec.cu", "ffm_minimize.cu",
           "ffm_capi.cu")
NVCC_FLAGS = (
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC",
)
# per-file extras: the bonded terms are evaluated without FMA contraction so
# that degeneracy thresholds (ffmin/kernels.py:130-140) see the same roundoff
# as the reference's CPU arithmetic
EXTRA = {"ffm_terms.cu": ("-fmad=false",), "ffm_small.cu": ("-fmad=false",),
         "ffm_minimize.cu": ("-fmad=false",)}


def nvcc_path() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: the CUDA toolkit is required to build libffmin_b200.so")


def _stale() -> bool:
    if not LIB.exists():
        return True
    mtime = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES] + list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h"))
    deps += list(INCLUDE.glob("*.h"))
    return any(d.stat().st_mtime > mtime for d in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not _stale():
        return LIB
    LIB_DIR.mkdir(exist_ok=True)
    objs, cmds = [], []
    for src in SOURCES:
        obj = LIB_DIR / (Path(src).stem + ".o")
        cmds.append([nvcc_path(), *NVCC_FLAGS, *EXTRA.get(src, ()), "-c", "-o", str(obj),
                     str(CSRC / src)])
        objs.append(str(obj))
    # the translation units are independent: compile them in parallel
    from concurrent.futures import ThreadPoolExecutor

    with ThreadPoolExecutor(max_workers=min(len(cmds), os.cpu_count() or 1)) as pool:
        for f in [pool.submit(_run, c, verbose) for c in cmds]:
            f.result()
    tmp = LIB.with_suffix(".so.tmp")
    _run([nvcc_path(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", str(tmp),
          *objs, "-ldl"], verbose)
    os.replace(tmp, LIB)
    for o in objs:
        os.remove(o)
    return LIB


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed ({res.returncode}):\n{res.stderr[-4000:]}")


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
