set -u
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "fuzz_regression" 2>&1 | tail -3
for s in 2 3 6 7 8; do timeout 900 python tools/fuzz_parity.py 2000 $s > gpurun_out/fuzz_s$s.log 2>&1; grep -A1 "^FAIL" gpurun_out/fuzz_s$s.log | cut -c1-300 | head -12; tail -1 gpurun_out/fuzz_s$s.log; done
for s in 4 9; do timeout 1200 python tools/fuzz_parity.py 600 $s big > gpurun_out/fuzz_big$s.log 2>&1; grep -A1 "^FAIL" gpurun_out/fuzz_big$s.log | cut -c1-300 | head; tail -1 gpurun_out/fuzz_big$s.log; done
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
bash tools/ab_env.sh C4 TTG_X 0
