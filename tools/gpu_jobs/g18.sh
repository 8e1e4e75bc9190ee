set -u
mkdir -p gpurun_out
for v in "0 0" "16 0" "16 512" "8 512"; do set -- $v; echo "raster=$1 kmin=$2"; TTG_GEMM_RASTER=$1 TTG_GEMM_RASTER_KMIN=$2 bash tools/ab_env.sh C4 TTG_SVD_WP 4; done
