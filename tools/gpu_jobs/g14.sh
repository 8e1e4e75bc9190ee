set -u
mkdir -p gpurun_out
for v in 0 2048 100000; do TTG_QR_PRE2L=$v bash tools/ab_env.sh C4 TTG_SVD_WP 4; done > gpurun_out/g14_ab.log 2>&1
cat gpurun_out/g14_ab.log
for v in 0 2048 100000; do TTG_QR_PRE2L=$v bash tools/ab_env.sh C3 TTG_SVD_WP 4; done > gpurun_out/g14_ab3.log 2>&1
cat gpurun_out/g14_ab3.log
