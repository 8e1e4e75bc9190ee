"""The C++ drop-in headers (include/ttlab/*.hpp) running the reference's own
hot-path test cases on the B200 (tests/cpp/test_dropin.cpp)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "test_dropin")


@pytest.mark.gpu
def test_cpp_dropin_headers():
    if not os.path.exists(BIN):
        subprocess.run(["python", "-c", "import __graft_entry__ as g; g.build()"], cwd=ROOT, check=True)
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASSED" in r.stdout


def test_dropin_headers_compile_without_eigen():
    """The headers build with plain g++ (no Eigen) against the C ABI."""
    out = "/tmp/ttlab_dropin_compile_check"
    r = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-Iinclude", "tests/cpp/test_dropin.cpp"], cwd=ROOT,
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
