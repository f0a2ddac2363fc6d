#!/bin/bash
# A/B of programmatic dependent launch (SMES_PDL) on the c2 bench step and the c4 / c1 latency
for v in 0 1 0 1; do
  SMES_PDL=$v timeout 300 python bench.py --no-cpu --steps 200 > gpurun_out/ab.json 2>/dev/null
  python -c "
import json
d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); print('c2 pdl=$v', round(d['value']), round(d['ms_per_step'],4), round(d['e2e']['ms_per_step'],4))"
done
for v in 0 1; do
  SMES_PDL=$v timeout 300 python bench.py --config c1 --no-cpu --steps 200 > gpurun_out/ab.json 2>/dev/null
  python -c "
import json
d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); print('c1 pdl=$v', round(d['value']), round(d['ms_per_step'],4))"
  SMES_PDL=$v timeout 300 python bench.py --config c4 --no-cpu > gpurun_out/ab.json 2>/dev/null
  python -c "
import json
d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); print('c4 pdl=$v', {k: round(v['p50_ms'],4) for k,v in d['sweep'].items()})"
done
