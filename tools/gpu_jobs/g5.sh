set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_canonical.py -q -k "negligible or clustered or retry or grid_large or jacobi_svd_random or from_device" > gpurun_out/g5_tests.log 2>&1
for wp in 8 4; do TTG_SVD_WP=$wp TTG_DEBUG_SVD_GRID=1 timeout 300 python tools/wp_probe.py >> gpurun_out/g5_wp.log 2>&1; done
TTG_PHASES=1 TTG_PRE=1 timeout 300 python tools/run_config.py C4 > gpurun_out/g5_C4_pre1.log 2>&1
TTG_PHASES=1 timeout 300 python tools/run_config.py C4 > gpurun_out/g5_C4_pre2.log 2>&1
TTG_PHASES=1 TTG_SVD_WP=4 timeout 300 python tools/run_config.py C4 > gpurun_out/g5_C4_wp4.log 2>&1
