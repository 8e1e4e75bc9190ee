set -u
run() { FUZZ_FROM=222 FUZZ_TO=223 timeout 300 python tools/fuzz_parity.py 224 2 2>&1 | grep -E "cases agree" ; }
echo "baseline: $(run)"
echo "QR_SMALL=0: $(TTG_QR_SMALL=0 run)"
echo "PRE_SMALL=2: $(TTG_PRE_SMALL=2 run)"
echo "PRE_SKIP=300: $(TTG_PRE_SKIP=300 run)"
echo "RING=0: $(TTG_SVD_RING=0 run)"
echo "CLUSTER=0: $(TTG_SVD_CLUSTER=0 run)"
echo "QR_PANEL_ALL=0: $(TTG_QR_PANEL_ALL=0 run)"
