set -u
mkdir -p gpurun_out
for oe in 1 0; do TTG_SVD_OE=$oe TTG_DEBUG_SVD_GRID=1 timeout 300 python tools/wp_probe.py >> gpurun_out/g8_wp.log 2>&1; done
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_config_parity.py -q -x -k "grid or clustered or negligible or config4 or config3" > gpurun_out/g8_tests.log 2>&1
for oe in 1 0; do TTG_SVD_OE=$oe bash tools/ab_env.sh C4 TTG_SVD_WP 4 >> gpurun_out/g8_ab.log 2>&1; done
