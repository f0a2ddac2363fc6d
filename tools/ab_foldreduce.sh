#!/bin/bash
# A/B of the head fold inside the plan-reduce launch (SMES_FOLD_IN_REDUCE) at c2
for v in 1 0 1 0; do
  SMES_FOLD_IN_REDUCE=$v timeout 300 python bench.py --no-cpu --steps 200 > gpurun_out/ab.json 2>/dev/null
  python -c "
import json
d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); print('fold_in_reduce=$v', round(d['value']), round(d['ms_per_step'],4), d['kernels']['plan_reduce']['ms'], d['parity']['ok'] if d.get('parity') else None)"
done
