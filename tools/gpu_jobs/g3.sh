set -u
mkdir -p gpurun_out
for wp in 0 4 8; do TTG_SVD_WP=$wp TTG_DEBUG_SVD_GRID=1 timeout 300 python tools/wp_probe.py >> gpurun_out/g3_wp.log 2>&1; done
timeout 1500 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/g3_tests.log 2>&1
for wp in 0 8 4; do TTG_SVD_WP=$wp timeout 300 python tools/run_config.py C4 > gpurun_out/g3_C4_wp$wp.log 2>&1; done
