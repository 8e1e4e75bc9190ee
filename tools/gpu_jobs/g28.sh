set -u
timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -k "gemm" 2>&1 | tail -6
for v in 0 1; do echo "TM=$v"; TTG_GEMM_TM=$v timeout 300 python tools/gemm_probe.py 2>&1 | grep "f64"; done
