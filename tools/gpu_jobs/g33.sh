set -u
TTG_PHASES=1 timeout 600 python tools/big_probe.py 22 1024 768 2>&1 | tail -10
timeout 300 tests/cpp/ref_test_core 2>&1 | tail -15
timeout 300 tests/cpp/ref_test_blas 2>&1 | tail -15
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -5
bash tools/ab_env.sh C4 TTG_SVD_BG_LMAX 2048
