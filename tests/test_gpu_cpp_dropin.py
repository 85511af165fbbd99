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
