set -u
timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -k "grid_large" 2>&1 | tail -3
TTG_PHASES=1 timeout 900 python tools/big_probe.py 20 512 384 c 2>&1 | tail -10
