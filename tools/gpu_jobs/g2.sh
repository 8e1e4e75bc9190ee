set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/g2_smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -k "not config3" --durations=15 > gpurun_out/g2_tests.log 2>&1
timeout 600 python bench.py > gpurun_out/g2_bench.json 2> gpurun_out/g2_bench.err
timeout 400 python bench.py --impl reference --steps 3 > gpurun_out/g2_ref.json 2> gpurun_out/g2_ref.err
