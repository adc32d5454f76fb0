"""Runs the C++ parity driver (tests/cpp/test_exact_b200.cpp: the reference's
test_attention.cpp cases against include/helixsim/exact_b200.hpp) on the GPU."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_exact_b200_driver():
    subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")])
    out = subprocess.run([os.path.join(ROOT, "tests", "cpp", "test_exact_b200")], capture_output=True, text=True,
                         timeout=300)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "failed: 0" in out.stdout.splitlines()[-1]
