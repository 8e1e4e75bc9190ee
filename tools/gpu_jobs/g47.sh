set -u
for s in 23 25 32; do timeout 900 python tools/fuzz_parity.py 4000 $s > gpurun_out/fz$s.log 2>&1; grep -A1 "^FAIL" gpurun_out/fz$s.log | cut -c1-300 | head -6; tail -1 gpurun_out/fz$s.log; done
timeout 1500 python tools/fuzz_parity.py 1000 41 big > gpurun_out/fzb41.log 2>&1; grep -A1 "^FAIL" gpurun_out/fzb41.log | cut -c1-300 | head -6; tail -1 gpurun_out/fzb41.log
timeout 900 python tools/batch_probe.py 20 10 96 48 2>&1 | tail -3
timeout 900 python tools/batch_probe.py 40 12 128 80 2>&1 | tail -3
