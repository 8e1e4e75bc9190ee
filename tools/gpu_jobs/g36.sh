set -u
bash tools/round_bench.sh
ls -la gpurun_out/rb_*
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02f_launches_C4.csv python tools/run_once.py C4 > gpurun_out/ncu_c4.log 2>&1
tail -2 gpurun_out/ncu_c4.log
wc -l gpurun_out/r02f_launches_C4.csv
