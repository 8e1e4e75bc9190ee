set -u
mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on"
timeout 600 $NCU -k regex:expand_mpo --launch-skip 13 -c 2 -f -o gpurun_out/r02_expand_mpo_c4 python tools/run_once.py C4 > gpurun_out/g17_a.log 2>&1
timeout 600 $NCU -k regex:expand_hadamard --launch-skip 11 -c 2 -f -o gpurun_out/r02_expand_had_c3 python tools/run_once.py C3 > gpurun_out/g17_b.log 2>&1
timeout 900 $NCU -k regex:jacobi_bg --launch-skip 60 -c 1 -f -o gpurun_out/r02_jbg_c4 python tools/run_once.py C4 > gpurun_out/g17_c.log 2>&1
for r in r02_expand_mpo_c4 r02_expand_had_c3 r02_jbg_c4; do
  ncu -i gpurun_out/$r.ncu-rep --page details --csv > gpurun_out/$r.details.csv 2>/dev/null
  ncu -i gpurun_out/$r.ncu-rep --page raw --csv > gpurun_out/$r.raw.csv 2>/dev/null
done
python tools/ncu_hot.py gpurun_out/r02_jbg_c4.ncu-rep 40 > gpurun_out/r02_jbg_c4.hot.txt 2>&1
ls -la gpurun_out/*.ncu-rep
