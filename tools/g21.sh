set -u
for c in C2 C1 C3; do for v in "1024 256" "256 64"; do set -- $v; echo "$c min=$1 div=$2"; TTG_GEMM_SPLITK_MIN=$1 TTG_GEMM_SPLITK_DIV=$2 bash tools/ab_env.sh $c TTG_SVD_WP 4; done; done
