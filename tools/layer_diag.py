"""Per-parameter gradient errors of SMESLayer vs the float64 restatement over a few seeds (c2 shape)."""
import sys, zlib, torch
sys.path.insert(0, '.')
import paper_2602_09386_b200 as smes
from tests.test_gpu_smes_layer import _gpu_masks, _restate, rel
for seed in range(4):
    B, T, E, d, d_out, d_ff, (ks, ka), act = 2048, 8, 32, 256, 256, 512, (4, 2), "relu"
    gen = torch.Generator().manual_seed(seed)
    layer = smes.SMESLayer(d, d_out, E, T, smes.RoutingBudget(ks, ka), d_ff=d_ff, expert_nonlinearity=act, generator=gen)
    with torch.no_grad():
        for p in layer.parameters():
            p.copy_((p * (1000.0 if p is layer.router_weight else 1.0)).bfloat16().float())
            if p.ndim == 2 and p is not layer.router_bias:
                p.add_((torch.randn(p.shape, generator=gen) * 0.1).bfloat16().float().cuda())
    h = torch.randn(B, d, generator=gen).bfloat16().float().cuda().requires_grad_(True)
    R = torch.randn(T, B, d_out, generator=gen).cuda()
    reps, lb = layer(h)
    ((reps * R).sum() + 0.3 * lb).backward()
    eng = layer.routing(B)
    rr, rlb, P, hd = _restate(layer, h, eng.active.long().cpu(), _gpu_masks(layer, eng))
    ((rr * R.double().cpu()).sum() + 0.3 * rlb).backward()
    print(seed, {n: round(rel(p.grad, P[n].grad), 4) for n, p in layer.named_parameters()}, round(rel(h.grad, hd.grad), 4),
          'reps', round(rel(reps.detach(), rr.detach()), 4))
