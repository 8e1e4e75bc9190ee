set -u
# bisect which earlier calls case 223 of seed 2 needs in order to fail
for from in 0 200 215 220 222 223; do
  FUZZ_FROM=$from FUZZ_TO=223 timeout 300 python tools/fuzz_parity.py 224 2 2>&1 | grep -E "^FAIL case 223|cases agree" | cut -c1-120 | tr '\n' ' '; echo " <- from $from"
done
