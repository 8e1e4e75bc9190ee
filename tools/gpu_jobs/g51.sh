set -u
for s in 61 62 63 64 65 66; do timeout 900 python tools/fuzz_parity.py 4000 $s 2>&1 | grep -E "^FAIL|agree|Error" | cut -c1-300 | head -6; done
for s in 71 72 73 74; do timeout 900 python tools/fuzz_split.py 3000 $s 2>&1 | grep -E "^FAIL|agree|Error" | cut -c1-300 | head -6; done
for s in 81 82; do timeout 900 python tools/fuzz_scalars.py 2000 $s 2>&1 | grep -E "^FAIL|agree|Error" | cut -c1-300 | head -6; done
for s in 91 92; do timeout 1500 python tools/fuzz_parity.py 1500 $s big 2>&1 | grep -E "^FAIL|agree|Error" | cut -c1-300 | head -6; done
