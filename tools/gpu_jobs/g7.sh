set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --durations=12 > gpurun_out/g7_tests.log 2>&1
for q in 1 0; do TTG_QFREE=$q bash tools/ab_env.sh C4 TTG_SVD_WP 4 >> gpurun_out/g7_ab.log 2>&1; done
TTG_PHASES=1 timeout 300 python tools/run_config.py C4 > gpurun_out/g7_C4.log 2>&1
timeout 300 python tools/heff_probe.py > gpurun_out/g7_heff.txt 2>&1
