#!/bin/bash
# A/B of the warp-per-instance scoring combine (SMES_SCORE_KERNEL) on the c4 sweep
for v in 0 1 0 1; do
  SMES_SCORE_KERNEL=$v timeout 300 python bench.py --config c4 --steps 1000 > gpurun_out/ab4.json 2>/dev/null
  python -c "
import json
d=json.loads(open('gpurun_out/ab4.json').read().strip().splitlines()[-1])
print('score_kernel=$v', {b: round(v['p50_ms'],4) for b, v in d['sweep'].items()})"
done
