"""c4 scoring at one batch size, eager, for an ncu launch list:
    ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/c4_launches.py 256"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2602_09386_b200 import SMESEngine  # noqa: E402

Bb = int(sys.argv[1]) if len(sys.argv) > 1 else 256
dev = torch.device("cuda:0")
c = dict(bench.CONFIGS["c4"], beta=0.0)
params = bench._make_params(c, dev)
eng = SMESEngine(params, Bb, c["ks"], c["ka"], device=dev)
eng.keep_logits = False
h_host, y_host = bench._host_inputs(c, Bb, 0)
eng.set_inputs(h_host.to(dev), y_host.to(dev))
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
for _ in range(4):
    flush.zero_()
    eng.score()
torch.cuda.synchronize()
print("ok", Bb)
