set -u
for s in 2 3; do timeout 900 python tools/fuzz_parity.py 1500 $s > gpurun_out/fuzz_s$s.log 2>&1; grep -A1 "^FAIL" gpurun_out/fuzz_s$s.log | cut -c1-300 | head -12; tail -1 gpurun_out/fuzz_s$s.log; done
timeout 1200 python tools/fuzz_parity.py 400 4 big > gpurun_out/fuzz_big.log 2>&1; grep -A1 "^FAIL" gpurun_out/fuzz_big.log | cut -c1-300 | head; tail -1 gpurun_out/fuzz_big.log
timeout 1200 python tools/fuzz_parity.py 3000 6 > gpurun_out/fuzz_s6.log 2>&1; grep -A1 "^FAIL" gpurun_out/fuzz_s6.log | cut -c1-300 | head -20; tail -1 gpurun_out/fuzz_s6.log
