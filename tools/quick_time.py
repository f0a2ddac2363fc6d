"""c2 training step through a CUDA graph (no L2 flush) for quick A/B of engine options:
    python tools/quick_time.py [opt=value ...]     e.g. fuse_wgrad=1 csum_from_gemm=1"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2602_09386_b200 import SMESEngine
from tests.helpers import make_case, to_engine_params

opts = {k: bool(int(v)) for k, v in (a.split("=") for a in sys.argv[1:])}
B = 16384
p, h, y, lam, beta = make_case(0, B, 8, 32, 256, 256, 4, 2, d_ff=512)
eng = SMESEngine(to_engine_params(p, lam, beta), B, 4, 2, **opts)
eng.set_inputs(torch.tensor(h, device="cuda"), torch.tensor(y, device="cuda", dtype=torch.float32))
g = eng.capture_step()
for _ in range(5):
    g.replay()
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(20):
    g.replay()
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / 20
print(f"c2 step {opts} {ms:.3f} ms -> {B / ms * 1e3:.0f} samples/s, n_act={eng.n_act()}")
