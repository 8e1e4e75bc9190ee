set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
NCU="ncu --set full --clock-control none --import-source on"
timeout 900 $NCU -k regex:jacobi_bg_kernel --launch-skip 90 -c 4 -f -o gpurun_out/r02_jbg_c4 python tools/run_once.py C4 > gpurun_out/g19_c.log 2>&1
ncu -i gpurun_out/r02_jbg_c4.ncu-rep --page details --csv > gpurun_out/r02_jbg_c4.details.csv 2>/dev/null
ncu -i gpurun_out/r02_jbg_c4.ncu-rep --page raw --csv > gpurun_out/r02_jbg_c4.raw.csv 2>/dev/null
python tools/ncu_hot.py gpurun_out/r02_jbg_c4.ncu-rep 30 > gpurun_out/r02_jbg_c4.hot.txt 2>&1
timeout 600 $NCU -k regex:gemm_tma_kernel --launch-skip 200 -c 2 -f -o gpurun_out/r02_gemm_tma_c4 python tools/run_once.py C4 > gpurun_out/g19_d.log 2>&1
ncu -i gpurun_out/r02_gemm_tma_c4.ncu-rep --page raw --csv > gpurun_out/r02_gemm_tma_c4.raw.csv 2>/dev/null
ncu -i gpurun_out/r02_gemm_tma_c4.ncu-rep --page details --csv > gpurun_out/r02_gemm_tma_c4.details.csv 2>/dev/null
