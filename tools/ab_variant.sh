#!/bin/bash
# c2 A/B of the in-tree library against a .so variant (tools/variant_build.sh):
#   tools/ab_variant.sh NAME   (build_var/_smes_NAME.so)
cp paper_2602_09386_b200/_smes.so /tmp/_smes_base.so
for v in base $1 base $1; do
  if [ $v == base ]; then cp /tmp/_smes_base.so paper_2602_09386_b200/_smes.so; else cp build_var/_smes_$v.so paper_2602_09386_b200/_smes.so; fi
  timeout 300 python bench.py --no-cpu --steps 200 > gpurun_out/ab.json 2>/dev/null
  python -c "
import json
d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); k=d['kernels']
print('$v', round(d['value']), round(d['ms_per_step'],4), {n: k[n]['ms'] for n in ('mlp_fwd','mlp_dgrad','fc1_wgrad') if n in k})"
done
cp /tmp/_smes_base.so paper_2602_09386_b200/_smes.so
