set -u
echo "== global-memory poison"
TTG_POISON=1 timeout 1500 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_dropin.py 2>&1 | tail -4
echo "== shared-memory poison build"
TTG_LIB=$PWD/paper_2601_16734_b200/libttgpu_poison.so TTG_POISON=1 timeout 1500 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_dropin.py 2>&1 | tail -4
