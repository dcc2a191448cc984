"""The minimal ctypes binding INTEGRATION.md gives a maintainer (section 3),
run as written against the built library: it must evaluate a system to the
same numbers as the package's own path."""

import ctypes as C
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

LIB = Path(__file__).resolve().parents[1] / "paper_1810_03358_b200" / "_lib" / "libffmin_b200.so"


def test_integration_ctypes_stub():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_1810_03358_b200.energy import energy_and_gradient
    from paper_1810_03358_b200.synth import make_globule_system

    s = make_globule_system(1200, seed=21)
    t = s.topology
    n = s.natoms
    q, sigma, eps = t.q, t.sigma, t.epsilon
    si, sj, ss = t.special_i, t.special_j, t.special_s
    nb, bidx, bK, br0 = len(t.bond_K), t.bond_idx, t.bond_K, t.bond_r0
    na, aidx, aK, at0 = len(t.ang_K), t.ang_idx, t.ang_K, t.ang_t0
    nd, didx, dV = len(t.dih_V), t.dih_idx, t.dih_V
    coords = np.ascontiguousarray(s.coords)

    # ---- the stub, as in INTEGRATION.md ----
    lib = C.CDLL(str(LIB))
    P, I64, I, D = C.c_void_p, C.c_int64, C.c_int, C.c_double
    lib.ffm_system_create.argtypes = [C.POINTER(P), I, I64, P, P, P, I64, P, P, P, D]
    lib.ffm_system_set_terms.argtypes = [P, I64, P, P, P, I64, P, P, P, I64, P, P]
    lib.ffm_eval_host.argtypes = [P, I, I, P, P, P, P]
    lib.ffm_last_error.restype = C.c_char_p

    def ptr(a):
        return C.c_void_p(a.ctypes.data) if a is not None else None

    h = P()
    assert lib.ffm_system_create(C.byref(h), 0, n, ptr(q), ptr(sigma), ptr(eps),
                                 len(ss), ptr(si), ptr(sj), ptr(ss), -1.0) == 0
    assert lib.ffm_system_set_terms(h, nb, ptr(bidx), ptr(bK), ptr(br0), na, ptr(aidx),
                                    ptr(aK), ptr(at0), nd, ptr(didx), ptr(dV)) == 0
    energies, status = np.empty(5), np.empty(8, np.int64)
    grad = np.empty((n, 3))
    rc = lib.ffm_eval_host(h, 0, 1 | 2, ptr(coords), ptr(grad), ptr(energies), ptr(status))
    if rc:
        raise RuntimeError(lib.ffm_last_error())
    # ---- end of the stub ----
    lib.ffm_system_destroy.argtypes = [P]
    lib.ffm_system_destroy(h)

    bd, g = energy_and_gradient(s)
    want = np.array([bd.stretch, bd.bend, bd.torsion, bd.coulomb, bd.vdw])
    np.testing.assert_allclose(energies, want, rtol=1e-12)
    g = np.asarray(g).reshape(n, 3)
    np.testing.assert_allclose(grad, g, rtol=0, atol=1e-12 * np.max(np.abs(g)))
    assert status[0] == -1 and status[2] == -1
