set -u
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
bash tools/round_bench.sh
for c in C4 ref_C4 C1 C2 C3 C5; do python - <<PY
import json
d=json.loads(open("gpurun_out/rb_$c.json").read().strip().splitlines()[-1])
print("$c", round(d.get("ms_per_step",0),1), "value", d["value"], "e2e", d.get("e2e",{}).get("value"))
PY
done
