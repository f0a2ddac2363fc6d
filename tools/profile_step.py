"""Short eager driver for ncu: builds the bench engine of a configuration (bench._make_params,
bench._host_inputs) and runs a few eager fwd+bwd steps with the backward side stream serialised,
so the launch order under ncu is the Python call order.  The launch-site tag of every kernel of
the last step goes to gpurun_out/step_tags.json (tools/ncu_traffic.py maps ncu rows to tags with
it).  Not a benchmark -- numbers under ncu are never reported.

    python tools/profile_step.py [steps] [--config c2|c3]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

import bench
from paper_2602_09386_b200 import SMESEngine, _lib

args = [a for a in sys.argv[1:] if not a.startswith("--")]
cfg = sys.argv[sys.argv.index("--config") + 1] if "--config" in sys.argv else "c2"
if cfg in args:
    args.remove(cfg)
steps = int(args[0]) if args else 3
c = bench.CONFIGS[cfg]
dev = torch.device("cuda", 0)
B = c["B"]
eng = SMESEngine(bench._make_params(c, dev), B, c["ks"], c["ka"], device=dev)
h, y = bench._host_inputs(c, B, 0)
eng.set_inputs(h.to(dev), y.to(dev))
eng.serial = True
eng.keep_logits = False        # as the bench's training step (no router-logit output)
for i in range(steps):
    if i == steps - 1:
        _lib.trace = []
    eng.step()
torch.cuda.synchronize()
tags = [t for t, k in _lib.trace for _ in range(k)]
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump({"config": cfg, "launches_per_step": len(tags), "tags": tags},
          open(os.path.join(ROOT, "gpurun_out", "step_tags.json"), "w"), indent=1)
print("n_act", eng.n_act(), "launches/step", len(tags))
