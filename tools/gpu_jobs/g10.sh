set -u
mkdir -p gpurun_out
for bg in 16; do TTG_BG_DEBUG=1 TTG_SVD_BG=$bg TTG_DEBUG_SVD_GRID=1 timeout 300 python tools/bg_probe.py; done > gpurun_out/g10_probe.txt 2>&1
grep "BG=" gpurun_out/g10_probe.txt; grep "k=1024" gpurun_out/g10_probe.txt | head -4
timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -k "svd or jacobi or grid" 2>&1 | tail -3
