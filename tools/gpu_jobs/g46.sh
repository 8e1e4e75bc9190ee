set -u
for s in 21 22 23 24 25; do timeout 900 python tools/fuzz_parity.py 4000 $s > gpurun_out/fz$s.log 2>&1; grep -A1 "^FAIL" gpurun_out/fz$s.log | cut -c1-400 | head -8; tail -1 gpurun_out/fz$s.log; done
for s in 31 32; do TTG_POISON=1 timeout 900 python tools/fuzz_parity.py 3000 $s > gpurun_out/fzp$s.log 2>&1; grep -A1 "^FAIL" gpurun_out/fzp$s.log | cut -c1-400 | head -8; echo "poison: $(tail -1 gpurun_out/fzp$s.log)"; done
for s in 41 42; do timeout 1500 python tools/fuzz_parity.py 1000 $s big > gpurun_out/fzb$s.log 2>&1; grep -A1 "^FAIL" gpurun_out/fzb$s.log | cut -c1-400 | head -8; echo "big: $(tail -1 gpurun_out/fzb$s.log)"; done
TTG_POISON=1 timeout 1500 python tools/fuzz_parity.py 100 43 huge > gpurun_out/fzh43.log 2>&1; grep -A1 "^FAIL" gpurun_out/fzh43.log | cut -c1-400 | head -8; echo "huge poison: $(tail -1 gpurun_out/fzh43.log)"
