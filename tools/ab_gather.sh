#!/bin/bash
# A/B of the gathered layer input (SMES_GATHER_X) at c2, and the gather-issuing lane count (.so variants)
cp paper_2602_09386_b200/_smes.so /tmp/_smes_base.so
run() {
  SMES_GATHER_X=$2 timeout 300 python bench.py --no-cpu --steps 200 > gpurun_out/ab.json 2>/dev/null
  python -c "
import json
d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); k=d['kernels']
print('$1 gather=$2', round(d['value']), round(d['ms_per_step'],4), {n: k[n]['ms'] for n in ('plan_scatter','mlp_fwd','fc1_wgrad') if n in k})"
}
run base 0
run base 1
for v in gl1 gl4 gl16; do
  cp build_var/_smes_$v.so paper_2602_09386_b200/_smes.so
  run $v 1
done
cp /tmp/_smes_base.so paper_2602_09386_b200/_smes.so
run base 0
run base 1
