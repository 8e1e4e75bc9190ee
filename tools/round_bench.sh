#!/bin/bash
# Round-end evidence on one GPU: bench lines for every config, the reference arm, and the
# C2 ncu launch list.  Outputs under gpurun_out/rb_*.
set -u
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/rb_smi.txt 2>&1
timeout 400 python bench.py > gpurun_out/rb_C2.json 2> gpurun_out/rb_C2.err
timeout 300 python bench.py --impl reference > gpurun_out/rb_ref_C2.json 2> gpurun_out/rb_ref_C2.err
for c in C1 C5; do timeout 400 python bench.py --config $c > gpurun_out/rb_$c.json 2> gpurun_out/rb_$c.err; done
for c in C3 C4; do timeout 600 python bench.py --config $c --steps 3 --warmup 3 > gpurun_out/rb_$c.json 2> gpurun_out/rb_$c.err; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/rb_launches_C2.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-profile > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/rb_launches_C2.csv > gpurun_out/rb_launches_C2.txt 2>&1
