"""Short eager driver for ncu: builds the c2 engine (bench config) and runs a few
eager fwd+bwd steps.  Not a benchmark -- numbers under ncu are never reported."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2602_09386_b200 import ExpertLayer, SMESEngine, SMESParams

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
c = bench.CFG
dev = torch.device("cuda", 0)
g = torch.Generator().manual_seed(0)
u = lambda shape, s: ((torch.rand(*shape, generator=g, dtype=torch.float64) * 2 - 1) * s).float().to(dev)
T, E, d, dff, do = c["T"], c["E"], c["d"], c["d_ff"], c["d_out"]
params = SMESParams(router_w=u((T, E, d), 1e-3 / d ** 0.5), router_b=torch.zeros(T, E, device=dev),
                    layers=[ExpertLayer(u((E, dff, d), d ** -0.5), torch.zeros(E, dff, device=dev), "relu"),
                            ExpertLayer(u((E, do, dff), dff ** -0.5), torch.zeros(E, do, device=dev), "identity")],
                    head_w=u((T, do), do ** -0.5), head_b=torch.zeros(T, device=dev), lb_strength=c["beta"])
eng = SMESEngine(params, c["B"], c["ks"], c["ka"], device=dev)
eng.set_inputs(torch.randn(c["B"], d, generator=g).to(torch.bfloat16).to(dev),
               (torch.rand(T, c["B"], generator=g) < 0.2).float().to(dev))
for _ in range(steps):
    eng.step()
torch.cuda.synchronize()
print("n_act", eng.n_act())
