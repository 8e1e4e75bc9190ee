#!/bin/bash
# run_config summary line: seconds, TF/s, per-class (launches, ms)
python tools/run_config.py $1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config'], round(d['seconds'],3), round(d['fp64_tflops_effective'],2), d['isometry_err'], {k:(v['launches'], round(v['ms'],1)) for k,v in d['profile'].items()})"
