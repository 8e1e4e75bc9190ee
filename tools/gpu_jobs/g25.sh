set -u
for c in C2 C1 C5 C3; do bash tools/ab_env.sh $c TTG_SVD_WP 4; done
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
