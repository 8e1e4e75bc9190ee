set -u
timeout 900 python -m pytest tests/test_gpu_ref_golden.py -m gpu -q -x 2>&1 | tail -5
bash tools/ab_env.sh C4 TTG_GEMM_TM 1 2
timeout 300 python tools/gemm_probe.py "C4 Y" 2>&1 | grep f64
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tm -c 2 -f -o gpurun_out/r02_gemm_tm_c4Y python tools/gemm_probe.py "C4 Y" > gpurun_out/ncu_tm.log 2>&1
tail -2 gpurun_out/ncu_tm.log
