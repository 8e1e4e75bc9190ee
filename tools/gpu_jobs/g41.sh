set -u
export TTG_LIB=$PWD/paper_2601_16734_b200/libttgpu_poison.so
for f in s2_223 s2_521 s3_519; do python tools/fuzz_run_case.py tools/fuzz_cases/fuzz_fail_$f.pkl 2>/dev/null | tail -3; done
timeout 600 python tools/fuzz_parity.py 600 5 2>&1 | grep -E "^FAIL|agree" | cut -c1-260 | head -40
