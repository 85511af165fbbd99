"""Host-side C++ drop-in utilities (include/krylov_b200/io.hpp) on the CPU:
the Laplacian generators against the reference's (oracle/_ref), bit for bit.
Compiled here with g++; skipped where the reference library is absent."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_laplacian_generators_match_reference(tmp_path, ref):
    if shutil.which("g++") is None:
        pytest.skip("no g++")
    lib = os.path.join(ROOT, "oracle", "_ref")
    exe = str(tmp_path / "gen_check")
    cmd = ["g++", "-std=c++20", "-O1", "-I" + os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "cpp", "host", "gen_check.cpp"), "-L" + lib, "-lkrylov_ref",
           "-L" + os.path.join(ROOT, "paper_2402_15033_b200"), "-lkrylov_b200",
           "-Wl,-rpath," + lib, "-Wl,-rpath," + os.path.join(ROOT, "paper_2402_15033_b200"), "-o", exe]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    p = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert p.returncode == 0, p.stdout + p.stderr
    assert "0 failures" in p.stdout
