#!/bin/bash
# A/B of the in-kernel X gather + packed store of mlp_fwd (SMES_FWD_PACK) at c2
for v in 0 1 0 1; do
  SMES_FWD_PACK=$v timeout 300 python bench.py --no-cpu --steps 200 > gpurun_out/ab.json 2>/dev/null
  python -c "
import json
d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); k=d['kernels']
print('pack=$v', round(d['value']), round(d['ms_per_step'],4), {n: k[n]['ms'] for n in ('plan_scatter','mlp_fwd','fc1_wgrad') if n in k})"
done
