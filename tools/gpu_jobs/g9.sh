set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --durations=12 > gpurun_out/g9_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/g9_tests.log
timeout 600 python bench.py > gpurun_out/g9_C4.json 2> gpurun_out/g9_C4.err
TTG_PHASES=1 timeout 300 python tools/run_config.py C4 > gpurun_out/g9_C4_phases.log 2>&1
