"""The committed golden fixtures are what the reference computes: re-run the
reference (oracle/_ref, built from /root/reference by oracle/Makefile) and
require exact equality.  CPU only; skipped where the reference cannot be
rebuilt (the GPU box has no /root/reference, but carries the prebuilt .so)."""
import json
import os

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = json.load(open(os.path.join(ROOT, "tests", "golden", "solver_golden.json")))
KG = np.load(os.path.join(ROOT, "tests", "golden", "kernels_golden.npz"))


@pytest.mark.parametrize("key", ["pip2_2d16", "pip2_2d64", "two_2d64_s60", "two_2d100_s20", "standard_2d32",
                                 "two_3d16_s60", "pip2_2d64_warm", "rand20k_two_s60_jac", "rand20k_pip2_jac"])
def test_reference_reproduces_solver_golden(ref, key):
    g = GOLDEN[key]
    if g["operator"] == "random":
        import os
        import sys
        sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
        from make_golden import random_jacobi_system
        a, b = random_jacobi_system(g["grid"])
    else:
        a = ref.laplace2d(g["grid"], g["grid"]) if g["dims"] == 2 else ref.laplace3d(g["grid"], g["grid"], g["grid"])
        b = ref.spmv(a, np.ones(a.n))
    x0 = None if g["x0"] is None else np.full(a.n, g["x0"])
    rep = ref.solve(a, b, x0, ref.make_config(kind=g["kind"], big_step=g["shat"], shat=g["shat"],
                                              max_iters=g["max_iters"]), standard=g["standard"])
    assert (rep.status, rep.iterations, rep.restarts, rep.reduces) == (g["status"], g["iterations"], g["restarts"],
                                                                       g["reduces"])
    assert rep.cycle_residuals == g["cycle_residuals"]
    assert [int(v) for v in rep.per_block] == g["per_block"]


def test_reference_reproduces_kernel_golden(ref):
    a2 = ref.laplace2d(9, 7)
    np.testing.assert_array_equal(ref.spmv(a2, KG["lap2d_9x7_x"]), KG["lap2d_9x7_y"])
    np.testing.assert_array_equal(ref.mpk(a2, KG["mpk_start"], 5), KG["mpk_V"])
    q, rc, rj, red = ref.bcgs_pip(KG["pip_q"], KG["pip_v"])
    np.testing.assert_array_equal(q, KG["pip_out_q"])
    np.testing.assert_array_equal(rc, KG["pip_out_rcol"])
    assert red == 1


def test_golden_counts_follow_the_sync_model():
    # one-stage PIP2: 2 reduces per block (24 per cycle); two-stage ŝ=m: 13 per cycle
    g = GOLDEN["pip2_2d100"]
    assert set(g["per_block"]) == {2}
    g = GOLDEN["two_2d100_s60"]
    assert set(g["per_block"]) == {1} and set(g["per_big_panel"]) == {1}
    assert g["reduces"] == 13 * (g["restarts"] + 1)
