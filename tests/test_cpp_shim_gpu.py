"""GPU: the C++ drop-in (include/tilefabric_b200/tilefabric.hpp) runs the
reference's own test bodies (tests/cpp/shim_parity.cpp) through the C ABI."""
import os
import subprocess

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


@pytest.mark.gpu
def test_cpp_shim_parity():
    exe = os.path.join(ROOT, "tests", "cpp", "shim_parity")
    if not os.path.exists(exe):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout[-4000:])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "[FAIL]" not in r.stdout


def test_cpp_shim_builds():
    # CPU: the drop-in header compiles against the C ABI and links the library.
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")], check=True)
    assert os.path.exists(os.path.join(ROOT, "tests", "cpp", "shim_parity"))
