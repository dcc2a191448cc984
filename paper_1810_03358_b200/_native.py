"""ctypes binding of the C ABI in include/ffmin_b200.h.

The shared library is built in-tree (``python -m paper_1810_03358_b200._build``
or ``__graft_entry__.build()``).  There is no fallback: if the library is
missing or cannot be loaded the import of any compute path raises, so a run
can never silently degrade to a CPU implementation.
"""

from __future__ import annotations

import ctypes as C
import threading
from pathlib import Path

import os

LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libffmin_b200.so"
# development aid: FFMIN_B200_LIB points at an alternative build (tuning sweeps)
if os.environ.get("FFMIN_B200_LIB"):
    LIB_PATH = Path(os.environ["FFMIN_B200_LIB"])

FFM_F64 = 0
FFM_F32 = 1
FFM_ENERGY = 1
FFM_GRAD = 2
FFM_NO_NB = 4
FFM_NO_TERMS = 8
FFM_TIME_NB = 16
FFM_NO_GRAPH = 32
FFM_NO_FUSE = 64
FFM_NTERMS = 5
FFM_STATUS_WORDS = 8
ST_NB_BAD_I, ST_NB_BAD_J, ST_BOND, ST_ANGLE, ST_DIHEDRAL = 0, 1, 2, 3, 4

# every exported symbol and its (restype, argtypes); the CPU test suite checks
# that the library exports exactly what include/ffmin_b200.h declares
_P = C.c_void_p
_I64 = C.c_int64
_I = C.c_int
_D = C.c_double
SIGNATURES = {
    "ffm_version": (C.c_char_p, []),
    "ffm_last_error": (C.c_char_p, []),
    "ffm_system_create": (_I, [C.POINTER(_P), _I, _I64, _P, _P, _P, _I64, _P, _P, _P, _D]),
    "ffm_system_set_terms": (_I, [_P, _I64, _P, _P, _P, _I64, _P, _P, _P, _I64, _P, _P]),
    "ffm_system_destroy": (_I, [_P]),
    "ffm_system_set_shard": (_I, [_P, _I, _I]),
    "ffm_system_set_edge": (_I, [_P, _I]),
    "ffm_preferred_edge": (_I, [_I64, _I, _P]),
    "ffm_system_info": (_I, [_P, _P]),
    "ffm_system_nb_ms": (_I, [_P, _P]),
    "ffm_launch_count": (C.c_longlong, []),
    "ffm_debug_phase_clock": (_I, [_P, _P, _P]),
    "ffm_eval": (_I, [_P, _I, _I, _P, _P, _P, _P, _P]),
    "ffm_eval_host": (_I, [_P, _I, _I, _P, _P, _P, _P]),
    "ffm_eval_batch": (_I, [_P, _I, _I64, _P, _P, _P, _P]),
    "ffm_atom_delta": (_I, [_P, _P, _I64, _P, _P, _P, _P, _P]),
    "ffm_atom_delta_lin": (_I, [_P, _P, _I64, _P, _P, _D, _P, _P, _P]),
    "ffm_farfield_build": (_I, [_P, _P, _I64, _D, _P, _P, _P, _P]),
    "ffm_vec_scratch_doubles": (_I64, []),
    "ffm_dot": (_I, [_I64, _P, _P, _P, _P, _P]),
    "ffm_dots": (_I, [_I64, _I, _P, _P, _P, _P, _P]),
    "ffm_axpby": (_I, [_I64, _P, _D, _D, _P, _P, _D, _P, _P, _P]),
    "ffm_lbfgs_two_loop": (_I, [_I64, _I, _P, _P, _P, _P, _P, _P, _P, _P]),
    "ffm_lbfgs_create": (_I, [_P, _I, _P, C.POINTER(_P)]),
    "ffm_lbfgs_configure": (_I, [_P, _P]),
    "ffm_system_set_comm": (_I, [_P, _P]),
    "ffm_lbfgs_start": (_I, [_P, _P, _P, _D, _D, _D, _P]),
    "ffm_lbfgs_run": (_I, [_P, _P]),
    "ffm_lbfgs_poll": (_I, [_P, _P, _P, _P, _I64, _P, _P]),
    "ffm_lbfgs_result": (_I, [_P, _P, _P, _P]),
    "ffm_lbfgs_best": (_I, [_P, _P, _P]),
    "ffm_lbfgs_set_schedule": (_I, [_P, _P, _I64]),
    "ffm_lbfgs_set_atoms": (_I, [_P, _P, _I64]),
    "ffm_lbfgs_destroy": (_I, [_P]),
}


class LbfgsConfig(C.Structure):
    """ffm_lbfgs_config (include/ffmin_b200.h)."""

    _fields_ = [("m", C.c_int32), ("ls_kind", C.c_int32), ("K", C.c_int32),
                ("use_gradient_start", C.c_int32), ("stop_on_linesearch_failure", C.c_int32),
                ("chunk", C.c_int32), ("max_iterations", C.c_int64),
                ("max_oracle_calls", C.c_int64), ("threshold", C.c_double),
                ("h0", C.c_double), ("eps_h", C.c_double), ("k_plus", C.c_double),
                ("k_minus", C.c_double), ("trust", C.c_double), ("method", C.c_int32),
                ("cg_kind", C.c_int32), ("restart_period", C.c_int32), ("reserved", C.c_int32),
                ("fixed_step", C.c_double), ("momentum", C.c_double),
                ("momentum_kind", C.c_int32), ("reserved2", C.c_int32),
                ("wiggle_h", C.c_double), ("wiggle_cutoff", C.c_double),
                ("wiggle_epoch", C.c_int32), ("reserved3", C.c_int32)]


LBFGS_STATUS = {0: None, 1: "converged", 2: "iteration_budget", 3: "linesearch_failure",
                4: "oracle_budget", 5: "horizon_complete"}
LBFGS_REC_WIDTH = 8
# ffm_lbfgs_config.method / cg_kind codes
METHOD_LBFGS, METHOD_CG, METHOD_SD, METHOD_FGM, METHOD_FIXED, METHOD_OFGM, METHOD_WIGGLE = (
    0, 1, 2, 3, 4, 5, 6)
CG_KINDS = ("fr", "prp", "prp+", "hs", "cd", "ls", "dy")

_lock = threading.Lock()
_lib = None


class NativeError(RuntimeError):
    """A C-ABI call failed (bad arguments or a CUDA runtime error)."""


def load(path: Path | str | None = None):
    """Load (once) and return the native library with typed entry points."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        p = Path(path) if path is not None else LIB_PATH
        if not p.exists():
            raise ImportError(
                f"native engine {p} is missing; build it with "
                "`python -m paper_1810_03358_b200._build` (needs nvcc)")
        lib = C.CDLL(str(p))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if path is None:
            _lib = lib
        return lib


def check(rc: int, what: str = "native call"):
    if rc != 0:
        msg = load().ffm_last_error().decode(errors="replace")
        raise NativeError(f"{what} failed ({rc}): {msg}")


def ptr(a) -> int | None:
    """Raw address of a NumPy array or torch tensor (None for None)."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    return a.ctypes.data
