set -u
bash tools/ab_env.sh C4 TTG_SVD_WP 4; timeout 300 python tools/run_config.py C4 2>&1 | tail -1 | cut -c1-330
bash tools/ab_env.sh C3 TTG_SVD_WP 4
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
