set -u
for c in C2 C1 C5; do for v in 2 1; do echo "$c PRE_SMALL=$v"; TTG_PRE_SMALL=$v bash tools/ab_env.sh $c TTG_SVD_WP 4; done; done
TTG_PRE_SMALL=1 timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
