#!/bin/bash
# A/B: bench ms/step and per-class profile for each library given (path or "cur"), config $1
cfg=$1; shift
for lib in "$@"; do
  if [ "$lib" = cur ]; then unset TTG_LIB; else export TTG_LIB=$lib; fi
  python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); p=d['profile']
print('$cfg', '$lib'[-20:], round(d['ms_per_step'],1), 'ms |', ' '.join(f\"{k} {v['ms']:.1f}ms/{v['launches']}\" for k,v in p.items()), '| jac sweeps', p['svd'].get('jacobi_sweeps'))"
done
