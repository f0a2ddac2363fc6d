for v in 0 1 0 1 0 1; do SMES_FOLD_SIDE=$v timeout 300 python bench.py --no-cpu --steps 200 > gpurun_out/b2.json 2>/dev/null; python -c "
import json
d=json.loads(open('gpurun_out/b2.json').read().strip().splitlines()[-1]); print('side=$v', d['value'], d['ms_per_step'])
"; done
