"""Runs the C++ drop-in check (tests/cpp/dropin_test.cpp: the reference's
test scenarios written against include/krylov_b200/krylov.hpp) on the GPU."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_dropin_scenarios():
    exe = os.path.join(ROOT, "tests", "cpp", "dropin_test")
    if not os.path.exists(exe):
        subprocess.run(["make", "-C", os.path.join(ROOT, "tests", "cpp")], check=True)
    p = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stdout + p.stderr
    assert "0 failed" in p.stdout


def test_cpp_dropin_compiles_against_header():
    # the header-only C++ layer compiles standalone (also checked on the CPU build host)
    src = os.path.join(ROOT, "tests", "cpp", "dropin_test.cpp")
    p = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-I", os.path.join(ROOT, "include"), src],
                       capture_output=True, text=True)
    assert p.returncode == 0, p.stderr


def test_reference_sparse_core_tests_pass_against_the_dropin():
    """The reference's own tests/test_sparse_core.cpp (Spmv, MatrixMarket,
    Equilibrate), compiled unchanged against include/krylov_b200 through
    tests/cpp/refcompat (krylov/*.hpp → the drop-in API) and a GoogleTest
    shim; its spmv calls run on the GPU.  Built by __graft_entry__.build()
    where /root/reference exists; the binary travels with the tree."""
    exe = os.path.join(ROOT, "tests", "cpp", "ref_sparse_core")
    if not os.path.exists(exe):
        pytest.skip("ref_sparse_core not built (needs /root/reference at build time)")
    p = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stdout + p.stderr
    assert "13 tests, 13 passed, 0 failed" in p.stdout, p.stdout


# The reference's own failures (the first-pass error
# window of CholQr2.FirstPassErrorTracksKappaSquared fails in the reference
# itself) and the one scheme the device path does not carry (BCGS2 with a
# Householder intra step: HHQR out of scope).  The reference's four
# SEGV tests (two-stage store, Appendix A.1) must pass here.
BLOCK_ORTHO_ALLOWED_FAILURES = {"CholQr2.FirstPassErrorTracksKappaSquared", "Bcgs2.HhqrIntraSyncAccounting"}


def test_reference_block_ortho_tests_compiled_unchanged():
    """The reference's own tests/test_block_ortho.cpp (CholQR / CholQR2, BCGS
    project, BCGS2, BCGS-PIP / PIP2, the BasisStore incl. two-stage), compiled
    unchanged against include/krylov_b200 through tests/cpp/refcompat; every
    orthogonalization and store call runs on the GPU, the test matrices come
    from the reference's own generators (oracle/_ref)."""
    exe = os.path.join(ROOT, "tests", "cpp", "ref_block_ortho")
    if not os.path.exists(exe):
        pytest.skip("ref_block_ortho not built (needs /root/reference at build time)")
    p = subprocess.run([exe], capture_output=True, text=True, timeout=1200)
    failed = {ln.split("]", 1)[1].strip() for ln in p.stdout.splitlines() if ln.startswith("[ FAIL ]")}
    passed = {ln.split("]", 1)[1].strip() for ln in p.stdout.splitlines() if ln.startswith("[  OK  ]")}
    assert "20 tests," in p.stdout, p.stdout + p.stderr
    assert failed <= BLOCK_ORTHO_ALLOWED_FAILURES, p.stdout
    for must in ["BasisStore.TwoStageEqualsPip2WhenBigPanelIsPanel", "BasisStore.TwoStageSyncCounts",
                 "BasisStore.PartialBigPanelFinalizedAtActualWidth", "BasisStore.StatesTrackTwoStageLifecycle",
                 "BasisStore.RawSequenceReconstruction", "Bcgs2.GluedAccumulationStaysOrthogonal",
                 "BcgsPip2.MonotoneFailure"]:
        assert must in passed, p.stdout
