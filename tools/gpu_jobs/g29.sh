set -u
for v in 0 1; do echo "TM=$v"; TTG_GEMM_TM=$v bash tools/ab_env.sh C4 TTG_SVD_WP 4; done
