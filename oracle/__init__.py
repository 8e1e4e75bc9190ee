"""CPU oracle for the ttlab MPO·MPS apply + canonical simplification hot path.

TEST INFRASTRUCTURE ONLY.  This package is a numpy/scipy restatement of the
reference algorithm (`/root/reference/proj/include/ttlab/*.hpp`, cited per
function in `ttlab_oracle.py`).  Only `tests/`, `__graft_entry__.smoke()` and
`bench.py`'s `cpu_baseline` / `--impl reference` legs may import it, and only
as the checker or the timed CPU baseline.  The product path
(`paper_2601_16734_b200`) never imports, calls or links anything under
`oracle/`.

Pinning: the reference cannot be compiled in this image (it hard-requires
Eigen3 and Catch2, neither present; proj/CMakeLists.txt:10, tests/CMakeLists.txt:1-2).
The restatement is pinned against the reference's own known-answer tests for
this path (test_core.cpp:73-155, 200-227, 258-265; test_blas.cpp:40-77,
108-142, 181-202, 289-311), re-expressed in `tests/test_oracle_pins.py`, and
its random inputs reproduce the reference generator (`random_uniform_mps`,
mps.hpp:493-514; std::mt19937_64 + std::uniform_real_distribution) bit for bit
against golden vectors dumped by a g++/libstdc++ program
(`oracle/golden_rng.cpp`, fixtures in `tests/golden/`).
"""
