import numpy as np, torch, sys
sys.path.insert(0, '/root/repo')
import paper_2602_09386_b200 as smes
from paper_2602_09386_b200.balance import _raw_sums
rng = np.random.default_rng(5)
z32 = rng.normal(size=(3, 200, 16)).astype(np.float32)
r = smes.route_batch(torch.tensor(z32), smes.RoutingBudget(1, 2))
print("C", r.chunk_union.shape, "cu sum", int(r.chunk_union.sum()), "ca sum", int(r.chunk_active.sum()), "cm", float(r.chunk_mass.sum()))
raw = _raw_sums(r)
torch.cuda.synchronize()
print("raw", raw.cpu().numpy()[:16], raw.cpu().numpy()[16:32].sum())
