"""Expert parallelism (paper_2602_09386_b200/ep.py) with n virtual ranks on one GPU.

Each virtual rank routes its own batch shard and owns E/n experts; the loopback transport
moves the fixed slots.  Parity target: the single-process oracle on the
concatenated batch, global-batch mean objective -- selections index-exact given the GPU's
logits, loss / expert / router / head gradients and d_hidden within the bf16 tolerance.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from oracle import smes_oracle as O
from paper_2602_09386_b200 import ExpertLayer, SMESParams
from paper_2602_09386_b200.ep import EPRank, ExpertParallelStep, LoopbackComm
from tests.helpers import make_case, rel

TOL = 2e-2


def _rank_params(p, lam, beta, r, n, dev="cuda"):
    E = p.router_w.shape[1]
    El = E // n
    t = lambda a, dt=torch.float32: torch.as_tensor(np.asarray(a), dtype=dt, device=dev)
    layers = [ExpertLayer(t(w[r * El:(r + 1) * El]), t(b[r * El:(r + 1) * El]), act) for (w, b, act) in p.layers]
    return SMESParams(router_w=t(p.router_w), router_b=t(p.router_b), layers=layers, head_w=t(p.head_w),
                      head_b=t(p.head_b),
                      task_weights=None if p.task_weights is None else t(p.task_weights, torch.float64),
                      task_loss_weights=t(lam), lb_strength=beta)


CASES = {
    # name: (seed, n, B_local, T, E, d, d_ff, ks, ka, router_scale, fuse, peer_put)
    "n2_mlp_fused": (0, 2, 512, 4, 64, 128, 256, 2, 1, 1.0, True, False),
    "n2_mlp_unfused": (1, 2, 384, 4, 64, 128, 256, 2, 1, 1e-3, False, False),
    "n4_t8": (2, 4, 256, 8, 128, 128, 256, 3, 2, 1.0, True, False),
    "n1": (3, 1, 512, 4, 32, 128, 256, 2, 1, 1.0, True, False),
    "n2_peer_put": (4, 2, 512, 4, 64, 128, 256, 2, 1, 1.0, True, True),
    "n4_peer_put": (6, 4, 256, 8, 128, 128, 256, 3, 2, 1.0, True, True),
    # the reference expert (one relu pool, experts.py:17-73): unfolded shard, O kept, P = O head_w^T
    "n2_single_relu": (7, 2, 512, 4, 64, 128, None, 2, 1, 1.0, True, False),
    "n4_single_relu_put": (8, 4, 256, 8, 128, 128, None, 3, 2, 1.0, True, True),
}


@pytest.mark.parametrize("name", list(CASES))
def test_ep_parity(name):
    seed, n, Bl, T, E, d, dff, ks, ka, rs, fuse, put = CASES[name]
    Bg = n * Bl
    p, h, y, lam, beta = make_case(seed, Bg, T, E, d, d, ks, ka, d_ff=dff, router_scale=rs, rand_lam=True)
    ranks = [EPRank(_rank_params(p, lam, beta, r, n), E, r, n, Bl, ks, ka, fuse_mlp=fuse) for r in range(n)]
    for r, rk in enumerate(ranks):
        rk.set_inputs(torch.tensor(h[r * Bl:(r + 1) * Bl], device="cuda"),
                      torch.tensor(y[:, r * Bl:(r + 1) * Bl], device="cuda", dtype=torch.float32))
    step = ExpertParallelStep(ranks, LoopbackComm(ranks, fused=put))
    step.step()
    step.step()          # a second step: slots are reused (stale data must not leak)
    torch.cuda.synchronize()
    for rk in ranks:
        rk.check()
    # --- oracle on the concatenated batch with the GPU's logits
    z = np.concatenate([rk.z.double().cpu().numpy().reshape(Bl, T, E) for rk in ranks], 0).transpose(1, 0, 2)
    assert rel(z, O.router_logits(h, p)) < 1e-5          # RouterBank.logits (routing.py:101-103)
    route = O.route_batch(z, ks, ka, p.task_weights)
    act = np.concatenate([rk.active.cpu().numpy() for rk in ranks], 1)
    assert np.array_equal(act, route.active)
    plan = O.build_execution_plan(route.unions, E)
    f = O.forward_sparse(h, p, ks, ka, logits=z, frozen=route, frozen_plan=plan)
    bw = O.backward(f, p, y, lam, beta)
    preds = np.concatenate([rk.preds.cpu().numpy() for rk in ranks], 1)
    assert rel(preds, f.predictions) < TOL
    lo = ranks[0].loss_out.cpu().numpy()
    assert abs(lo[0] - bw.task_value) <= TOL * abs(bw.task_value)
    assert abs(lo[1] - bw.stats.value) <= 1e-5 * abs(bw.stats.value)
    assert abs(lo[2] - bw.total) <= TOL * abs(bw.total)
    El = E // n
    for li in range(len(p.layers)):
        gw = np.concatenate([rk.shard.g_layers[li][0].cpu().numpy() for rk in ranks], 0)
        gb = np.concatenate([rk.shard.g_layers[li][1].cpu().numpy() for rk in ranks], 0)
        assert rel(gw, bw.layers[li][0]) < TOL, ("W", li)
        assert rel(gb, bw.layers[li][1]) < TOL, ("b", li)
    for rk in ranks:      # replicated gradients are identical on every rank after the all-reduce
        assert rel(rk.g_router_w.cpu().numpy().reshape(T, E, d), bw.router_w) < TOL
        assert rel(rk.g_router_b.cpu().numpy().reshape(T, E), bw.router_b) < TOL
        assert rel(rk.g_head_w.cpu().numpy(), bw.head_w) < TOL
        assert rel(rk.g_head_b.cpu().numpy(), bw.head_b) < TOL
    dh = np.concatenate([rk.d_hidden.cpu().numpy() for rk in ranks], 0)
    assert rel(dh, bw.d_hidden) < TOL
    # dedup: an instance is sent to an owner iff its union meets the owner's experts
    for r, rk in enumerate(ranks):
        cnt = rk.cnt.cpu().numpy()
        for o in range(n):
            want = sum(1 for b in range(Bl) if np.any((route.unions[r * Bl + b] >= o * El) &
                                                     (route.unions[r * Bl + b] < (o + 1) * El)))
            assert cnt[o] == want


def test_ep_capacity_overflow_raises():
    """A workspace too small for the received rows raises StateError instead of writing past it."""
    seed, n, Bl, T, E, d, dff, ks, ka = 5, 2, 512, 4, 64, 128, 256, 2, 1
    p, h, y, lam, beta = make_case(seed, n * Bl, T, E, d, d, ks, ka, d_ff=dff, router_scale=1.0)
    ranks = [EPRank(_rank_params(p, lam, beta, r, n), E, r, n, Bl, ks, ka, capacity_factor=0.05) for r in range(n)]
    for r, rk in enumerate(ranks):
        rk.set_inputs(torch.tensor(h[r * Bl:(r + 1) * Bl], device="cuda"),
                      torch.tensor(y[:, r * Bl:(r + 1) * Bl], device="cuda", dtype=torch.float32))
    ExpertParallelStep(ranks, LoopbackComm(ranks)).step()
    torch.cuda.synchronize()
    from paper_2602_09386_b200.errors import StateError
    with pytest.raises(StateError):
        for rk in ranks:
            rk.check()
