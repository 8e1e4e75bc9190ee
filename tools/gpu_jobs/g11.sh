set -u
mkdir -p gpurun_out
for bg in 16; do TTG_SVD_BG=$bg bash tools/ab_env.sh C4 TTG_SVD_WP 4; done > gpurun_out/g11_ab.log 2>&1
cat gpurun_out/g11_ab.log
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
