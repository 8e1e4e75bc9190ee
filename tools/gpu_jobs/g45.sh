set -u
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -6
for s in 2 4; do timeout 900 python tools/fuzz_parity.py 2000 $s > gpurun_out/fuzz_s$s.log 2>&1; grep -A1 "^FAIL" gpurun_out/fuzz_s$s.log | cut -c1-300 | head -12; tail -1 gpurun_out/fuzz_s$s.log; done
timeout 1200 python tools/fuzz_parity.py 600 4 big > gpurun_out/fuzz_big4.log 2>&1; grep -A1 "^FAIL" gpurun_out/fuzz_big4.log | cut -c1-300 | head; tail -1 gpurun_out/fuzz_big4.log
for c in C1 C2 C5; do bash tools/ab_env.sh $c TTG_X 0; done
