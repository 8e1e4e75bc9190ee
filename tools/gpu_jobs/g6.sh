set -u
mkdir -p gpurun_out
for pre in 1 2; do for wp in 0 4 8; do
  TTG_PRE=$pre bash tools/ab_env.sh C4 TTG_SVD_WP $wp >> gpurun_out/g6_ab.log 2>&1
done; done
