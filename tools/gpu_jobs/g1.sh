set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/g1_smi.txt 2>&1
timeout 300 python tools/run_config.py C4 > gpurun_out/g1_C4.log 2>&1
timeout 300 python tools/run_config.py C3 > gpurun_out/g1_C3.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g1_launches_C4.csv python tools/run_once.py C4 > gpurun_out/g1_ncu.log 2>&1
python tools/launch_summary.py gpurun_out/g1_launches_C4.csv > gpurun_out/g1_launches_C4.txt 2>&1
gzip -f gpurun_out/g1_launches_C4.csv
