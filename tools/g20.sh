set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -k "qr" 2>&1 | tail -2
for v in 0 1; do TTG_QR_LOOKAHEAD=$v bash tools/ab_env.sh C4 TTG_SVD_WP 4; done
for v in 0 1; do echo LA=$v; TTG_QR_LOOKAHEAD=$v TTG_PHASES=1 timeout 300 python tools/run_config.py C4 2>&1 | grep "phase\|isometry" | tail -5 | cut -c1-300; done
for v in 0 1; do TTG_QR_LOOKAHEAD=$v bash tools/ab_env.sh C3 TTG_SVD_WP 4; done
