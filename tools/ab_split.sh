#!/bin/bash
# A/B of the split-K folded wgrad (SMES_WGRAD_SPLIT) at c2
for v in 1 8 1 8 4 16; do
  SMES_WGRAD_SPLIT=$v timeout 300 python bench.py --no-cpu --steps 200 > gpurun_out/ab.json 2>/dev/null
  python -c "
import json
d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); k=d['kernels']; print('split=$v', round(d['value']), round(d['ms_per_step'],4), k['fc2_wgrad_folded']['ms'])"
done
