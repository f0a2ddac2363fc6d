#!/bin/bash
# A/B of the router weight-gradient split-K factor (SMES_RW_SPLITS) at c2
for v in 64 16 32 8 64 16; do
  SMES_RW_SPLITS=$v timeout 300 python bench.py --no-cpu --steps 200 > gpurun_out/ab.json 2>/dev/null
  python -c "
import json
d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); k=d['kernels']; print('rw_splits=$v', round(d['value']), round(d['ms_per_step'],4), k['router_wgrad']['ms'])"
done
