"""Out-of-bounds check of every kernel that touches the basis store
(compute-sanitizer is closed on this GPU pool).  With KRY_GUARD=1 the store
is allocated with a guard column on each side, and the guard columns and
the padding rows [n, ld) of every column hold an all-ones NaN pattern: a
kernel writing outside the basis trips Store::check_guards() at the end of
the solve (a loud KRY_INTERNAL), and a kernel reading the padding would
poison its result (so the golden comparisons catch out-of-bounds reads).
Shapes are chosen so n is not a multiple of 32 (padding rows exist)."""
import numpy as np
import pytest

from test_gpu_solver import GOLDEN, assert_parity, run_golden

pytestmark = pytest.mark.gpu


@pytest.fixture
def guard(monkeypatch):
    monkeypatch.setenv("KRY_GUARD", "1")


@pytest.mark.parametrize("key", ["two_2d100_s60", "two_2d100_s20", "pip2_2d100", "two_3d16_s60", "two_2d48_csr",
                                 "standard_2d32", "pip2_2d64_warm", "two_3d64_s60", "rand20k_two_s60_jac"])
@pytest.mark.parametrize("fused", ["0", "1", "2"])
def test_solves_stay_inside_the_basis(kb, ctx, ref, guard, monkeypatch, key, fused):
    if key not in GOLDEN:
        pytest.skip(f"{key} golden not generated")
    monkeypatch.setenv("KRY_FUSED_MPK", fused)  # per-SpMV, heuristic, forced one-pass MPK
    rep, g = run_golden(kb, ref, key)
    assert_parity(rep, g)


@pytest.mark.parametrize("env", [{"KRY_FUSED_PASS": "1"}, {"KRY_SPECULATE": "0"}, {"KRY_GRAPHS": "1"},
                                 {"KRY_UPDATE_TMA": "0"}, {"KRY_FUSED_PANEL_GRAM": "0"}])
def test_solver_variants_stay_inside_the_basis(kb, ctx, ref, guard, monkeypatch, env):
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    rep, g = run_golden(kb, ref, "two_2d100_s60")
    assert_parity(rep, g)


def test_breakdown_paths_stay_inside_the_basis(kb, ctx, guard):
    # rank collapse inside the first panel: speculative rollback, truncation, seam
    n = 237
    rp = np.arange(n + 1, dtype=np.int64)
    ci = np.arange(n, dtype=np.int64)
    vv = np.array([float(1 + i % 11) for i in range(n)])
    op = kb.CsrOperator(rp, ci, vv)
    for kind, shat in [(3, 60), (2, 0), (1, 0)]:
        rep = kb.sstep_gmres(op, np.ones(n), None, kb.SolverConfig(scheme=kb.OrthoScheme(kb.OrthoKind(kind), shat),
                                                                    big_step=shat))
        assert rep.breakdown


def test_guard_detects_a_write_outside_the_basis(kb, ctx, guard):
    """The check itself: corrupt a padding row through the device pointer of a
    guarded C-ABI store and run a solve with the same workspace shape."""
    import ctypes as C
    st = kb.BasisStore(1000, 60, 5, 60)
    q, ld = C.c_void_p(), C.c_int64()
    kb._check(kb.lib().kry_store_device_ptr(st._h, C.byref(q), C.byref(ld)))
    assert ld.value > 1000  # padding rows exist
    from cuda.bindings import runtime as rt
    zero = np.zeros(1)
    err, = rt.cudaMemcpy(q.value + 1000 * 8, zero.ctypes.data, 8, rt.cudaMemcpyKind.cudaMemcpyHostToDevice)
    assert err == rt.cudaError_t.cudaSuccess  # row n (padding) of column 0 := +0.0
    with pytest.raises(kb.KrylovError, match="guard"):
        kb._check(kb.lib().kry_store_check_guards(st._h))
