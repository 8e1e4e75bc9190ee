set -u
run() { FUZZ_FROM=222 FUZZ_TO=223 timeout 300 python tools/fuzz_parity.py 224 2 2>&1 | grep -E "cases agree" ; }
echo "baseline: $(run)"
echo "blocking: $(CUDA_LAUNCH_BLOCKING=1 run)"
echo "no early: $(TTG_SVD_EARLY=0 run)"
echo "no precond: $(TTG_SVD_PRECOND=0 run)"
echo "poison: $(TTG_POISON=1 run)"
echo "no grid: $(TTG_SVD_GRID=0 run)"
