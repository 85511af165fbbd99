"""CPU-only checks of the drop-in boundary (include/krylov_b200.h):
the library loads without a GPU, exports every declared symbol, refuses to
compute without a device (no CPU fallback), and its host-side small-matrix
routines reproduce the reference's arithmetic bit for bit."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "krylov_b200.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(kry_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for must in ["kry_sstep_gmres", "kry_standard_gmres", "kry_bcgs_pip", "kry_bcgs_pip2", "kry_bcgs_pip_partial",
                 "kry_cholqr", "kry_store_create", "kry_store_append_block", "kry_store_preprocess_block",
                 "kry_store_finalize_big_panel", "kry_spmv", "kry_mpk", "kry_operator_create_csr",
                 "kry_operator_create_laplace2d", "kry_operator_create_laplace3d"]:
        assert must in syms


def test_library_exports_every_declared_symbol():
    from paper_2402_15033_b200 import _capi
    lib = C.CDLL(_capi.LIB_PATH)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    # and the ctypes table covers the header exactly
    assert sorted(_capi.SIGNATURES) == declared_symbols()


def test_abi_version_and_config_defaults(kb):
    assert kb.lib().kry_abi_version() == 2
    c = kb._capi.kry_solver_config()
    kb.lib().kry_solver_config_default(C.byref(c))
    # krylov::SolverConfig defaults (gmres.hpp:18-24)
    assert (c.restart_len, c.step, c.big_step, c.scheme_kind, c.rel_tol, c.max_iters) == (60, 5, 0, 2, 1e-6, 500000)


def test_no_cpu_fallback(kb):
    if kb.device_count() > 0:
        pytest.skip("a GPU is visible")
    h = C.c_void_p()
    rc = kb.lib().kry_ctx_create(0, 1, 0, None, C.byref(h))
    assert rc == kb._capi.KRY_NO_DEVICE
    assert b"no CPU fallback" in kb.lib().kry_last_error()
    with pytest.raises(kb.DeviceError):
        kb.Context(0)


def test_status_names(kb):
    assert kb.lib().kry_status_name(2) == b"not_positive_definite"
    assert kb.lib().kry_status_name(9) == b"no_device"


GOLD = np.load(os.path.join(ROOT, "tests", "golden", "kernels_golden.npz"))


def test_host_cholesky_matches_reference_bitwise(kb):
    r, piv = kb.try_cholesky(GOLD["chol_s"])
    assert piv == int(GOLD["chol_pivot"][0]) == 0
    np.testing.assert_array_equal(np.triu(r), np.triu(GOLD["chol_r"]))
    r, piv = kb.try_cholesky(GOLD["chol_bad_s"])
    assert piv == int(GOLD["chol_bad_pivot"][0]) == 4
    np.testing.assert_array_equal(np.triu(r), np.triu(GOLD["chol_bad_r"]))


def test_host_lsq_matches_reference_bitwise(kb):
    y, imp, valid = kb.solve_hessenberg_lsq(GOLD["store_H"], 2.5)
    np.testing.assert_array_equal(y, GOLD["lsq_y"])
    assert imp == GOLD["lsq_implicit"][0] and valid == int(GOLD["lsq_implicit"][1])


def test_try_cholesky_against_live_reference(kb, ref, rng):
    for k in (1, 6, 21, 61):
        a = rng.standard_normal((3 * k, k))
        s = a.T @ a
        r1, p1 = kb.try_cholesky(s)
        r2, p2 = ref.try_cholesky(s)
        assert p1 == p2
        np.testing.assert_array_equal(np.triu(r1), np.triu(r2))
