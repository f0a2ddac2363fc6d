#!/bin/bash
# A/B of the CTA-pair wgrad (SMES_GEMM_PAIR_K) at c3
for v in 1 0 1 0; do
  SMES_GEMM_PAIR_K=$v timeout 500 python bench.py --config c3 --steps 20 --no-cpu > gpurun_out/ab.json 2>/dev/null
  python -c "
import json
d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); k=d['kernels']; print('pairK=$v', round(d['value']), round(d['ms_per_step'],3), {x: k[x]['ms'] for x in ('fc1_fwd','fc1_dgrad','fc1_wgrad')}, d['clocks']['sm_mhz'])"
done
