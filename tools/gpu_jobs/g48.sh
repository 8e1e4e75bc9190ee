set -u
for s in 1 2 3 4; do timeout 700 python tools/fuzz_split.py 2000 $s > gpurun_out/fsp$s.log 2>&1; grep "^FAIL" gpurun_out/fsp$s.log | cut -c1-300 | head -8; tail -1 gpurun_out/fsp$s.log; done
timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x 2>&1 | tail -3
bash tools/ab_env.sh C3 TTG_X 0
