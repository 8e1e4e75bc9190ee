set -u
timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -k "qr" 2>&1 | tail -2
for c in C4 C3; do bash tools/ab_env.sh $c TTG_SVD_WP 4; done
