set -u
mkdir -p gpurun_out
bash tools/ab_env.sh C4 TTG_SVD_WP 4 > gpurun_out/g13_ab.log 2>&1
cat gpurun_out/g13_ab.log
TTG_PHASES=1 timeout 300 python tools/run_config.py C4 2>&1 | grep phase | head -4
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
