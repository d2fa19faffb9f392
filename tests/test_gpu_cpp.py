"""The header-only C++ drop-in shim (include/ds2ctc.hpp) driven from C++,
checked against the oracle (tests/cpp/shim_test.cpp)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "build", "tests", "shim_test")


def test_cpp_shim_builds():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")], check=True)
    assert os.path.exists(EXE)


@pytest.mark.gpu
def test_cpp_shim_parity():
    if not os.path.exists(EXE):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")], check=True)
    res = subprocess.run([EXE], capture_output=True, text=True, timeout=300)
    print(res.stdout)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "PASS" in res.stdout
