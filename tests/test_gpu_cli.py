"""The CLI drop-in (tools/krylov_b200 solve) against the reference CLI's
solve path: same JSON report keys (harness.hpp:379-400), same residual CSV
(harness.hpp:402-410), and the reference's golden counts."""
import json
import os
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "tools", "krylov_b200")
GOLDEN = json.load(open(os.path.join(ROOT, "tests", "golden", "solver_golden.json")))
REPORT_KEYS = {"scheme", "n", "m", "s", "shat", "rel_tol", "status", "iterations", "restarts", "initial_residual",
               "final_relative_residual", "breakdown", "breakdown_kappa", "total_reduces", "reduces_per_iteration",
               "wall_seconds", "cycle_residuals"}


@pytest.fixture(scope="module")
def exe():
    if not os.path.exists(EXE):
        subprocess.run(["make", "-C", os.path.join(ROOT, "tools")], check=True)
    return EXE


def run(exe, tmp_path, *args):
    out, hist = tmp_path / "r.json", tmp_path / "h.csv"
    p = subprocess.run([exe, "solve", *args, "--out", str(out), "--history", str(hist)], capture_output=True,
                       text=True, timeout=600)
    assert p.returncode == 0, p.stderr
    return json.load(open(out)), open(hist).read().splitlines(), p.stderr


def check_golden(rep, g):
    assert set(rep) == REPORT_KEYS
    assert (rep["iterations"], rep["restarts"], rep["total_reduces"]) == (g["iterations"], g["restarts"], g["reduces"])
    assert rep["status"] == ["converged", "max_iters", "ortho_breakdown", "stagnation"][g["status"]]
    assert np.allclose(rep["cycle_residuals"], g["cycle_residuals"], rtol=1e-5, atol=1e-13)


def test_cli_grid_two_stage(exe, tmp_path):
    rep, hist, err = run(exe, tmp_path, "--grid", "64", "--scheme", "two-stage", "--shat", "60")
    check_golden(rep, GOLDEN["two_2d64_s60"])
    assert hist[0] == "scheme,m,s,shat,rel_tol,cycle,relative_residual"
    assert len(hist) == 1 + len(rep["cycle_residuals"])
    assert hist[1].startswith("two-stage,60,5,60,9.9999999999999995e-07,1,")  # "%.16e" of 1e-6, as fmt_sci
    assert err.startswith("status=converged iters=180 ")


def test_cli_standard(exe, tmp_path):
    rep, _, _ = run(exe, tmp_path, "--grid", "32", "--scheme", "standard")
    check_golden(rep, GOLDEN["standard_2d32"])


def test_cli_matrix_market_symmetric(exe, tmp_path, ref):
    a = ref.laplace2d(48, 48)
    mtx = tmp_path / "lap48.mtx"
    with open(mtx, "w") as f:  # symmetric storage: lower triangle only
        f.write("%%MatrixMarket matrix coordinate real symmetric\n% 48x48 5-point Laplacian\n")
        ent = [(i, a.col_idx[k], a.vals[k]) for i in range(a.n) for k in range(a.row_ptr[i], a.row_ptr[i + 1])
               if a.col_idx[k] <= i]
        f.write(f"{a.n} {a.n} {len(ent)}\n")
        for i, j, v in ent:
            f.write(f"{int(i) + 1} {int(j) + 1} {float(v)!r}\n")
    rep, _, _ = run(exe, tmp_path, "--matrix", str(mtx), "--scheme", "two-stage")
    check_golden(rep, GOLDEN["two_2d48_csr"])


def test_cli_nine_point_and_scaling_options(exe, tmp_path):
    rep, _, _ = run(exe, tmp_path, "--grid", "40", "--stencil", "9", "--scheme", "bcgs-pip2")
    assert rep["status"] == "converged" and rep["total_reduces"] == 2 * rep["iterations"] // 5
    rep, _, _ = run(exe, tmp_path, "--grid", "40", "--equilibrate", "--scheme", "two-stage")
    assert rep["status"] == "converged"
    rep, _, _ = run(exe, tmp_path, "--grid", "40", "--jacobi", "--scheme", "two-stage")
    assert rep["status"] == "converged"


def test_cli_errors(exe, tmp_path):
    p = subprocess.run([exe, "solve", "--grid", "8"], capture_output=True, text=True)
    assert p.returncode == 1 and p.stderr.startswith("error:")
    p = subprocess.run([exe, "solve", "--grid", "8", "--scheme", "nope", "--out", str(tmp_path / "x")],
                       capture_output=True, text=True)
    assert p.returncode == 1
