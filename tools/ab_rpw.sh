#!/bin/bash
# A/B of the plan chunk size (router.cu SMES_RPW_DIV, .so variants from tools/variant_build.sh)
cp paper_2602_09386_b200/_smes.so /tmp/_smes_base.so
for v in base rpw1 rpw2 rpw8 base; do
  if [ $v == base ]; then cp /tmp/_smes_base.so paper_2602_09386_b200/_smes.so; else cp build_var/_smes_$v.so paper_2602_09386_b200/_smes.so; fi
  timeout 300 python bench.py --no-cpu --steps 200 > gpurun_out/ab.json 2>/dev/null
  timeout 300 python bench.py --config c4 --steps 1000 > gpurun_out/ab4.json 2>/dev/null
  python -c "
import json
d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); k=d['kernels']
d4=json.loads(open('gpurun_out/ab4.json').read().strip().splitlines()[-1])
print('$v c2', round(d['ms_per_step'],4), {n: k[n]['ms'] for n in ('route','plan_scatter','plan_reduce','unpermute') if n in k})
print('$v c4', {b: round(v['p50_ms'],4) for b, v in d4['sweep'].items()})"
done
cp /tmp/_smes_base.so paper_2602_09386_b200/_smes.so
