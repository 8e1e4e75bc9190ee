set -u
timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -k "svd" 2>&1 | tail -4
for lm in 1024 2048; do echo "LMAX=$lm"; TTG_SVD_BG_LMAX=$lm TTG_PHASES=1 timeout 600 python tools/big_probe.py 22 1024 768 2>&1 | tail -14; done
