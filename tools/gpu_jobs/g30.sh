set -u
for v in 0 1; do echo "HOST_DIMS=$v"; TTG_HOST_DIMS=$v bash tools/ab_env.sh C4 TTG_SVD_WP 4; done
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
