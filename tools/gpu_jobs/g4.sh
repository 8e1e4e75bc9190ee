set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -k "negligible or clustered or retry or grid_large or jacobi_svd_random" > gpurun_out/g4_tests.log 2>&1
TTG_SVD_WP=8 TTG_DEBUG_SVD_GRID=1 timeout 300 python tools/wp_probe.py > gpurun_out/g4_wp.log 2>&1
TTG_PRE=1 timeout 300 python tools/run_config.py C4 > gpurun_out/g4_C4_pre1.log 2>&1
timeout 300 python tools/run_config.py C4 > gpurun_out/g4_C4_pre2.log 2>&1
TTG_SVD_WP=8 TTG_DEBUG_SVD_GRID=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:jacobi_wp -c 1 -o gpurun_out/g4_wp python tools/wp_probe.py > gpurun_out/g4_ncu.log 2>&1
