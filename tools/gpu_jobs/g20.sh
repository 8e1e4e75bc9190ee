set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -k "qr" 2>&1 | tail -2
for v in 0 512; do TTG_QR_LOOKAHEAD1=$v bash tools/ab_env.sh C4 TTG_SVD_WP 4; done
for v in 0 512; do TTG_QR_LOOKAHEAD1=$v bash tools/ab_env.sh C3 TTG_SVD_WP 4; done
