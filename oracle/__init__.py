"""CPU oracle for the ttlab MPO·MPS apply + canonical simplification hot path.

TEST INFRASTRUCTURE ONLY.  This package is a numpy/scipy restatement of the
reference algorithm (`/root/reference/proj/include/ttlab/*.hpp`, cited per
function in `ttlab_oracle.py`).  Only `tests/`, `__graft_entry__.smoke()` and
`bench.py`'s `cpu_baseline` / `--impl reference` legs may import it, and only
as the checker or the timed CPU baseline.  The product path
(`paper_2601_16734_b200`) never imports, calls or links anything under
`oracle/`.

Pinning: against outputs of the reference's own code run in this container.
The reference cannot be built as shipped (it hard-requires Eigen3 and Catch2,
neither present; proj/CMakeLists.txt:10, tests/CMakeLists.txt:1-2), but it is
header-only and uses a small subset of the Eigen API: with the stand-in of
`oracle/eigen_standin/` on the include path its hot-path headers compile
unchanged, from where they lie, into `oracle/_ref/ttlab_ref` (`oracle/Makefile`,
`oracle/ref_driver.cpp`).  `tests/golden/make_ref_fixtures.py` runs the cases of
`tests/ref_cases.py` through it and commits the outputs
(`tests/golden/ref_outputs.npz`); `tests/test_oracle_vs_ref.py` checks this
restatement against them (and `tests/test_gpu_ref_golden.py` the CUDA path).
The dense factorizations under the reference's code are then the stand-in's,
not Eigen's: the pin covers the reference's control flow, truncation rule,
ledger, environments, projection and stop rules on gauge-invariant results.
Older pins stay: the reference's known-answer tests for this path
(test_core.cpp:73-155, 200-227, 258-265; test_blas.cpp:40-77, 108-142, 181-202,
289-311) re-expressed in `tests/test_oracle_pins.py`, and the reference input
generator (`random_uniform_mps`, mps.hpp:493-514; std::mt19937_64 +
std::uniform_real_distribution) reproduced bit for bit (`oracle/golden_rng.cpp`,
fixtures in `tests/golden/`; also checked against `ttlab_ref random_uniform`).
"""
