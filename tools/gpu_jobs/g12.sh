set -u
mkdir -p gpurun_out
for bg in 16; do TTG_SVD_BG=$bg TTG_DEBUG_SVD_GRID=1 timeout 300 python tools/bg_probe.py; done > gpurun_out/g12_probe.txt 2>&1
grep "BG=" gpurun_out/g12_probe.txt
