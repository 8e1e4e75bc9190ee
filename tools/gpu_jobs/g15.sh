set -u
mkdir -p gpurun_out
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g15_launches_C4.csv python tools/run_once.py C4 > gpurun_out/g15_ncu.log 2>&1
python tools/launch_summary.py gpurun_out/g15_launches_C4.csv > gpurun_out/g15_launches_C4.txt 2>&1
gzip -f gpurun_out/g15_launches_C4.csv
cat gpurun_out/g15_launches_C4.txt
