set -u
bash tools/round_bench.sh
bash tools/g15.sh > /dev/null 2>&1
NCU="ncu --set full --clock-control none --import-source on"
timeout 900 $NCU -k regex:jacobi_bg_kernel --launch-skip 90 -c 2 -f -o gpurun_out/r02_jbg_c4 python tools/run_once.py C4 > gpurun_out/g26_c.log 2>&1
ncu -i gpurun_out/r02_jbg_c4.ncu-rep --page details --csv > gpurun_out/r02_jbg_c4.details.csv 2>/dev/null
ncu -i gpurun_out/r02_jbg_c4.ncu-rep --page raw --csv > gpurun_out/r02_jbg_c4.raw.csv 2>/dev/null
python tools/ncu_hot.py gpurun_out/r02_jbg_c4.ncu-rep 30 > gpurun_out/r02_jbg_c4.hot.txt 2>&1
