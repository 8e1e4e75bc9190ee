#!/bin/bash
# Round-end evidence on one GPU: bench lines for every config and the reference arm.
# Outputs under gpurun_out/rb_* (copied to profiles/rNN_bench_*.json by hand).
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/rb_smi.txt 2>&1
timeout 900 python bench.py > gpurun_out/rb_C4.json 2> gpurun_out/rb_C4.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/rb_ref_C4.json 2> gpurun_out/rb_ref_C4.err
for c in C1 C2 C5; do timeout 600 python bench.py --config $c --no-c5 > gpurun_out/rb_$c.json 2> gpurun_out/rb_$c.err; done
timeout 900 python bench.py --config C3 --steps 3 --warmup 3 --no-c5 > gpurun_out/rb_C3.json 2> gpurun_out/rb_C3.err
