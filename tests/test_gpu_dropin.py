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


@pytest.mark.gpu
@pytest.mark.parametrize("suite", ["test_core", "test_blas"])
def test_reference_own_tests_through_the_dropin_headers(suite):
    """proj/tests/test_core.cpp / test_blas.cpp of the reference, compiled UNCHANGED against include/ttlab
    (+ the Eigen / Catch2 stand-ins of oracle/) and linked with libttgpu.so: every split, canonicalization,
    simplify, apply, scprod and expectation in them runs on the B200.  Built by __graft_entry__.build() where
    /root/reference exists; the binaries travel with the snapshot."""
    exe = os.path.join(ROOT, "tests", "cpp", "ref_" + suite)
    if not os.path.exists(exe):
        pytest.skip("tests/cpp/ref_%s not built (needs /root/reference at build time)" % suite)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout[-3000:])
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert r.stdout.strip().splitlines()[-1].startswith("ok:")
