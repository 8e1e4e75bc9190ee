#!/bin/bash
# A/B over an environment variable: ab_env.sh CONFIG VAR value1 value2 ...
# prints bench ms/step, per-class profile and Jacobi sweeps for each value
cfg=$1; var=$2; shift 2
for v in "$@"; do
  env $var=$v python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-c5 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); p=d['profile']
print('$cfg', '$var=$v', round(d['ms_per_step'],1), 'ms |', ' '.join(f\"{k} {v['ms']:.1f}ms/{v['launches']}\" for k,v in p.items()), '| jac sweeps', p['svd'].get('jacobi_sweeps'))"
done
