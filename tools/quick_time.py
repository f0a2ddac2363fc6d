import time, torch, sys
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
from tests.helpers import make_case, to_engine_params
from paper_2602_09386_b200 import SMESEngine
B=16384
p, h, y, lam, beta = make_case(0, B, 8, 32, 256, 256, 4, 2, d_ff=512)
eng = SMESEngine(to_engine_params(p, lam, beta), B, 4, 2)
eng.set_inputs(torch.tensor(h, device="cuda"), torch.tensor(y, device="cuda", dtype=torch.float32))
g = eng.capture_step()
for _ in range(5): g.replay()
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(20): g.replay()
e.record(); torch.cuda.synchronize()
ms = s.elapsed_time(e)/20
print(f"c2 step {ms:.3f} ms  -> {B/ms*1e3:.0f} samples/s, n_act={eng.n_act()}")
