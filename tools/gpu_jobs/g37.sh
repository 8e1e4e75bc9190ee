set -u
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
/usr/bin/time -v timeout 900 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; grep -E "Elapsed|Maximum resident" gpurun_out/final_bench.err; cut -c1-300 gpurun_out/final_bench.json
