set -u
for v in "256 64" "128 32" "64 32" "128 16"; do set -- $v; echo "min=$1 div=$2"; TTG_GEMM_SPLITK_MIN=$1 TTG_GEMM_SPLITK_DIV=$2 bash tools/ab_env.sh C4 TTG_SVD_WP 4; done
