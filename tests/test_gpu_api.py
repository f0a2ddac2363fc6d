"""The reference-facing API (taskmoe names) on the GPU, pinned by the reference's own
known-answer tests (restated, file:line) and by the oracle on identical inputs."""
import math
import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

import paper_2602_09386_b200 as smes
from oracle import smes_oracle as O
from tests.helpers import make_case, rel

BF16_TOL = 2e-2


def f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


# ---------------------------------------------------------------- routing known answers

def test_hand_traced_two_stage_selection():
    # test_routing.py:147-160
    probs = np.array([[0.4, 0.3, 0.2, 0.1], [0.1, 0.5, 0.3, 0.1]])
    z = np.array([[4.0, 3.0, 2.0, 1.0], [1.0, 5.0, 3.0, 1.0]])
    d = smes.progressive_route(torch.tensor(z), smes.RoutingBudget(1, 1), full_probs=torch.tensor(probs))
    assert d.shared.tolist() == [1]
    assert d.adaptive[0].tolist() == [0] and d.adaptive[1].tolist() == [2]
    assert d.union.tolist() == [0, 1, 2]


def test_two_term_weights():
    # test_routing.py:113-120
    r = smes.naive_route_batch(torch.tensor([[[2.0, 1.0, 0.0, -1.0]]]), 2)
    w = r.weights.cpu().numpy()
    assert abs(w[0, 0, 0] - math.exp(2) / (math.exp(2) + math.exp(1))) < 1e-6
    assert abs(w[0, 0, 1] - 0.268941) < 1e-6
    assert w[0, 0, 2] == 0.0 and w[0, 0, 3] == 0.0


def test_identical_logits_union_and_adversarial_bound():
    # test_routing.py:98-111
    z = torch.tensor(np.tile(np.array([3.0, 1.0, 2.0, 0.0]), (3, 1))[:, None, :])
    assert smes.naive_route_batch(z, 2).unions[0].tolist() == [0, 2]
    z = np.full((3, 8), -5.0)
    for t in range(3):
        z[t, 2 * t], z[t, 2 * t + 1] = 2.0, 1.0
    assert smes.naive_route_batch(torch.tensor(z[:, None, :]), 2).unions[0].numel() == 6


def test_tie_goes_to_lowest_index():
    # linalg.py:86-101 / test_linalg.py:106-107: equal logits -> lowest expert index wins
    z = torch.zeros(2, 3, 8)
    z[:, :, 5] = 1.0
    r = smes.route_batch(z, smes.RoutingBudget(2, 1))
    assert r.shared.cpu().tolist() == [[0, 5]] * 3
    assert r.adaptive.cpu().tolist() == [[[1]] * 3] * 2


def test_fully_private_reduces_to_naive():
    # test_routing.py:136-145 (25 seeds)
    for seed in range(25):
        z = torch.tensor(f32(np.random.default_rng(seed).normal(size=(3, 1, 9))))
        prog = smes.route_batch(z, smes.RoutingBudget(0, 2))
        ref = O.route_batch(z.double().numpy(), 0, 2)
        assert np.array_equal(prog.active.cpu().numpy(), ref.active)
        assert rel(prog.weights.cpu().numpy(), ref.weights) < 1e-6


def test_budget_and_input_errors():
    with pytest.raises(smes.ConfigError, match="candidates"):
        smes.progressive_route(torch.zeros(2, 4), smes.RoutingBudget(3, 2))
    with pytest.raises(smes.ShapeError):
        smes.route_batch(torch.zeros(2, 4), smes.RoutingBudget(1, 1))
    z = torch.zeros(2, 3, 6)
    z[1, 2, 3] = float("nan")
    with pytest.raises(smes.NumericsError):
        smes.route_batch(z, smes.RoutingBudget(1, 1))


def test_routing_golden_fixtures(golden_dir):
    """Every reference routing fixture: GPU == oracle on the same (fp32) logits, and the
    oracle on those logits reproduces the reference's recorded selections."""
    g = np.load(os.path.join(golden_dir, "routing_golden.npz"))
    for i in range(int(g["n"])):
        c = lambda k: g[f"c{i}_{k}"]
        tw = c("task_weights") if f"c{i}_task_weights" in g.files else None
        z32 = f32(c("z"))
        ks, ka = int(c("k_shared")), int(c("k_adaptive"))
        r = smes.route_batch(torch.tensor(z32), smes.RoutingBudget(ks, ka), None if tw is None else torch.tensor(tw))
        ref = O.route_batch(z32, ks, ka, tw)
        assert np.array_equal(r.shared.cpu().numpy(), ref.shared), i
        assert np.array_equal(r.adaptive.cpu().numpy(), ref.adaptive), i
        assert np.array_equal(r.active.cpu().numpy(), ref.active), i
        assert rel(r.weights.cpu().numpy(), ref.weights) < 1e-6
        assert [u.tolist() for u in r.unions] == [u.tolist() for u in ref.unions]
        # fixture (reference on f64 logits) agrees unless fp32 rounding moved a near-tie
        same = np.array_equal(ref.active, c("active"))
        assert same or i == 6, i


def test_stage1_fp64_exact_at_reference_init():
    """c2-shaped logits at reference router init (|z| ~ 5e-4, pooled gaps ~1e-10): index-exact."""
    rng = np.random.default_rng(0)
    T, B, E, d = 8, 4096, 32, 256
    h = rng.normal(size=(B, d))
    w = rng.uniform(-1e-3 / 16, 1e-3 / 16, size=(T, E, d))
    z32 = f32(np.einsum("bd,ted->tbe", h, w))
    r = smes.route_batch(torch.tensor(z32), smes.RoutingBudget(4, 2))
    ref = O.route_batch(z32, 4, 2)
    assert np.array_equal(r.shared.cpu().numpy(), ref.shared)
    assert np.array_equal(r.active.cpu().numpy(), ref.active)
    assert O.stage1_margin(z32, 4) < 1e-8   # the case really is precision-critical


# ---------------------------------------------------------------- plan / GEMM / combine

def test_plan_hand_example():
    # test_execution.py:27-37
    p = smes.build_execution_plan([np.array([0, 2]), np.array([2, 3])], num_experts=4)
    assert p.loads.cpu().tolist() == [1, 0, 2, 1]
    assert p.total_rows == 4
    assert list(zip(p.gather_instances.cpu().tolist(), p.gather_experts.cpu().tolist())) == \
        [(0, 0), (0, 2), (1, 2), (1, 3)]
    assert p.segment_offsets.cpu().tolist() == [0, 1, 1, 3, 4]
    assert p.row_index(1, 2) == 2


def test_plan_errors():
    with pytest.raises(smes.ShapeError):
        smes.build_execution_plan([np.array([0, 4])], num_experts=4)
    with pytest.raises(smes.ShapeError):
        smes.build_execution_plan([np.array([1, 1])], num_experts=4)


def test_plan_segment_integrity_seeded():
    # test_execution.py:58-83: packing == lexsort, back-map bijection
    for seed in range(10):
        rng = np.random.default_rng(seed)
        E, B = int(rng.integers(3, 40)), int(rng.integers(1, 300))
        unions = [np.sort(rng.choice(E, size=int(rng.integers(0, min(E, 6) + 1)), replace=False)) for _ in range(B)]
        p = smes.build_execution_plan(unions, E)
        ref = O.build_execution_plan(unions, E)
        assert np.array_equal(p.gather_instances.cpu().numpy(), ref.gather_instances)
        assert np.array_equal(p.gather_experts.cpu().numpy(), ref.gather_experts)
        assert np.array_equal(p.segment_offsets.cpu().numpy(), ref.segment_offsets)


def test_grouped_gemm_and_reconstruct_vs_oracle():
    # test_execution.py:108-118 (per-row oracle) and :173-180 (full pipeline vs oracle)
    rng = np.random.default_rng(3)
    T, B, E, d = 4, 300, 16, 128
    z32 = f32(rng.normal(size=(T, B, E)))
    r = smes.route_batch(torch.tensor(z32), smes.RoutingBudget(2, 1))
    plan = smes.build_execution_plan(r, E)
    h = f32(torch.tensor(rng.normal(size=(B, d))).bfloat16().double().numpy())
    w = torch.tensor(rng.uniform(-1, 1, size=(E, d, d)) / d ** 0.5).bfloat16().double().numpy()
    b = rng.normal(size=(E, d)) * 0.1
    for act in ("identity", "relu"):
        pool = smes.ExpertPool(torch.tensor(w, dtype=torch.float32).cuda(), torch.tensor(b, dtype=torch.float32).cuda(), act)
        x = torch.tensor(h, dtype=torch.float32).cuda()[plan.gather_instances]
        out, pre = smes.grouped_gemm(x, pool, plan, return_preactivation=True)
        ref_plan = O.build_execution_plan(O.route_batch(z32, 2, 1).unions, E)
        ref_out, ref_pre = O.grouped_gemm(h[ref_plan.gather_instances], w, b, act, ref_plan)
        assert rel(out.cpu().numpy(), ref_out) < BF16_TOL
        assert rel(pre.cpu().numpy(), ref_pre) < BF16_TOL
        reps = smes.reconstruct_task_reps(out, plan, r)
        ref_reps = O.reconstruct_task_reps(ref_out, ref_plan, O.route_batch(z32, 2, 1))
        assert rel(reps.cpu().numpy(), ref_reps) < BF16_TOL


def test_grouped_gemm_shape_errors():
    plan = smes.build_execution_plan([np.array([0, 1])], 2)
    pool = smes.ExpertPool(torch.zeros(2, 32, 32).cuda(), torch.zeros(2, 32).cuda())
    with pytest.raises(smes.ShapeError):
        smes.grouped_gemm(torch.zeros(3, 32).cuda(), pool, plan)


# ---------------------------------------------------------------- regularizer / loss

def test_load_stats_and_lb_gradient_vs_oracle():
    rng = np.random.default_rng(5)
    z32 = f32(rng.normal(size=(3, 200, 16)))
    r = smes.route_batch(torch.tensor(z32), smes.RoutingBudget(1, 2))
    ref = O.route_batch(z32, 1, 2)
    for dense in (False, True):
        st = smes.compute_load_stats(r, dense_probs=dense)
        rs = O.compute_load_stats(ref, dense)
        assert np.array_equal(st.counts.cpu().numpy(), rs.counts)
        assert rel(st.frequency.cpu().numpy(), rs.frequency) < 1e-12
        assert rel(st.mass.cpu().numpy(), rs.mass) < 1e-5
        assert abs(st.value - rs.value) < 1e-5 * rs.value
        g = smes.lb_loss_gradient(st, r).cpu().numpy()
        assert rel(g, O.lb_loss_gradient(rs, ref)) < 1e-5


def test_task_loss_and_errors():
    rng = np.random.default_rng(1)
    p = rng.uniform(size=(3, 100))
    p[0, :3] = [0.0, 1.0, 1e-9]      # clamp edges (training.py:47-57)
    y = (rng.uniform(size=(3, 100)) < 0.4).astype(float)
    w = np.array([1.0, 0.5, 2.0])
    got = smes.task_loss(torch.tensor(p, dtype=torch.float32), torch.tensor(y), torch.tensor(w))
    assert abs(got - O.task_loss(f32(p), y, w)) < 1e-6 * abs(got)
    with pytest.raises(smes.NumericsError):
        smes.task_loss(torch.tensor([[0.5, 1.5]]), torch.tensor([[0.0, 1.0]]))
    with pytest.raises(smes.NumericsError):
        smes.task_loss(torch.tensor([[0.5, 0.5]]), torch.tensor([[0.0, 2.0]]))
    assert smes.total_loss(1.0, 2.0, 0.5) == 2.0
    with pytest.raises(smes.NumericsError):
        smes.total_loss(1.0, 2.0, -0.1)


# ---------------------------------------------------------------- forward_sparse / backward

def _model_from_case(p, lam, beta, ks, ka):
    t = lambda a: torch.tensor(np.asarray(a), dtype=torch.float32).cuda()
    # reference form: lists of Affine maps (experts.py:26-38, routing.py:64-87, model.py:36-49)
    pools = [smes.ExpertPool([smes.Affine(t(w[e]), t(b[e])) for e in range(w.shape[0])], act)
             for (w, b, act) in p.layers]
    routers = smes.RouterBank([smes.Affine(t(p.router_w[k]), t(p.router_b[k])) for k in range(p.router_w.shape[0])],
                              None if p.task_weights is None else torch.tensor(p.task_weights))
    heads = [smes.Affine(t(p.head_w[k:k + 1]), t(p.head_b[k:k + 1])) for k in range(p.head_w.shape[0])]
    return smes.MoeModel(None, None, pools if len(pools) > 1 else pools[0], routers, heads,
                         torch.tensor(lam), beta, smes.RoutingBudget(ks, ka))


@pytest.mark.parametrize("d_ff", [None, 256])
def test_forward_sparse_backward_api(d_ff):
    B, T, E, d, ks, ka = 512, 4, 16, 128, 2, 1
    p, h, y, lam, beta = make_case(21, B, T, E, d, d, ks, ka, d_ff=d_ff, rand_lam=True)
    model = _model_from_case(p, lam, beta, ks, ka)
    res = smes.forward_sparse(torch.tensor(h, dtype=torch.float32).cuda(), model)
    z = res.router_logits.double().cpu().numpy()
    r = O.route_batch(z, ks, ka)
    assert np.array_equal(res.routing.active.cpu().numpy(), r.active)
    f = O.forward_sparse(h, p, ks, ka, logits=z, frozen=r)
    assert rel(res.predictions.cpu().numpy(), f.predictions) < BF16_TOL
    bw = smes.backward(res, model, torch.tensor(y))
    ref = O.backward(f, p, y, lam, beta)
    assert abs(bw.task_value - ref.task_value) < BF16_TOL * ref.task_value
    assert abs(bw.lb_value - ref.lb_value) < 1e-5 * ref.lb_value
    g = bw.gradients
    assert list(g)[:2] == (["expert_0.weight", "expert_0.bias"] if d_ff is None else ["expert0_0.weight", "expert0_0.bias"])
    for li in range(len(p.layers)):
        pre = "expert_" if d_ff is None else f"expert{li}_"
        gw = torch.stack([g[f"{pre}{e}.weight"] for e in range(E)]).cpu().numpy()
        assert rel(gw, ref.layers[li][0]) < BF16_TOL
    rw = torch.stack([g[f"router_{t}.weight"] for t in range(T)]).cpu().numpy()
    assert rel(rw, ref.router_w) < BF16_TOL
    assert rel(bw.d_hidden.cpu().numpy(), ref.d_hidden) < BF16_TOL
    # frozen reuse (model.py:284-300, test_model.py:167-175): same selections, same outputs
    res2 = smes.forward_sparse(torch.tensor(h, dtype=torch.float32).cuda(), model, frozen=res)
    assert torch.equal(res2.routing.active, res.routing.active)
    assert torch.allclose(res2.predictions, res.predictions)
    with pytest.raises(smes.StateError):
        smes.backward(res, model, torch.tensor(y))       # stale: the engine ran another forward


def test_deferred_cache_fields_survive_engine_reuse():
    """packed_in / packed_out / expert_flops are filled on first read (model.py:301-324 fills them
    eagerly); a result still alive when the engine runs the next forward keeps its own values."""
    B, T, E, d, ks, ka = 384, 4, 16, 64, 2, 1
    p, h, y, lam, beta = make_case(23, B, T, E, d, d, ks, ka)
    model = _model_from_case(p, lam, beta, ks, ka)
    x = torch.tensor(h, dtype=torch.float32).cuda()
    res = smes.forward_sparse(x, model)
    n_rows = res.plan.total_rows
    assert res.expert_flops == n_rows * d * d
    gi = res.plan.gather_instances
    f = O.forward_sparse(h, p, ks, ka, logits=res.router_logits.double().cpu().numpy())
    # the second forward (another batch through the same cached engine) rewrites the engine rows
    res2 = smes.forward_sparse(torch.tensor(h[::-1].copy(), dtype=torch.float32).cuda(), model)
    assert torch.equal(res.packed_in, res.hidden[gi])
    assert rel(res.packed_out.cpu().numpy(), f.layer_outs[-1]) < BF16_TOL
    assert res.packed_out.shape == (n_rows, d)
    assert res2.packed_out.shape == (res2.plan.total_rows, d)
    assert torch.equal(res2.packed_in, res2.hidden[res2.plan.gather_instances])
    assert res.expert_flops == n_rows * d * d
    with pytest.raises(smes.NumericsError):
        yb = torch.tensor(y)
        yb[1, 3] = 0.5
        smes.backward(res2, model, yb)
    smes.forward_sparse(x, model, keep_cache=False)


def test_encoder_path_vs_autograd():
    """Full reference model (encoder + SMES layer) vs a float64 torch-autograd restatement
    of the same graph with the GPU's selections frozen."""
    gen = torch.Generator().manual_seed(0)
    T, E, d, F, dh, B = 4, 16, 128, 92, 64, 256
    model = smes.init_model(gen, F, dh, d, d, E, T, smes.RoutingBudget(2, 1), lb_strength=0.05,
                            expert_nonlinearity="relu")
    # bf16-representable parameters so both sides see identical operands
    for a in (model.encoder1, model.encoder2):
        a.weight = a.weight.bfloat16().float()
    model.experts.weight = model.experts.weight.bfloat16().float()
    model.routers.weight = model.routers.weight.bfloat16().float() * 1000
    x = torch.randn(B, F, generator=gen).bfloat16().float().cuda()
    y = (torch.rand(T, B, generator=gen) < 0.3).float()
    res = smes.forward_sparse(x, model)
    bw = smes.backward(res, model, y)
    act = res.routing.active.cpu()

    P = {k: v.detach().double().cpu().clone().requires_grad_(True) for k, v in
         [("e1w", model.encoder1.weight), ("e1b", model.encoder1.bias), ("e2w", model.encoder2.weight),
          ("e2b", model.encoder2.bias), ("xw", model.experts.weight), ("xb", model.experts.bias),
          ("rw", model.routers.weight), ("rb", model.routers.bias), ("hw", model.head_w), ("hb", model.head_b)]}
    xd = x.double().cpu()
    st = lambda v: v + (v.bfloat16().double() - v).detach()   # bf16 storage, straight-through gradient
    mid = st(torch.relu(xd @ P["e1w"].T + P["e1b"]))
    h = st(mid @ P["e2w"].T + P["e2b"])
    z = torch.einsum("bd,ted->tbe", h, P["rw"]) + P["rb"][:, None, :]
    zs = torch.gather(z, 2, act)
    w = torch.softmax(zs, dim=2)
    Y = torch.relu(torch.einsum("bd,ejd->bej", h, P["xw"]) + P["xb"][None])      # every expert, every row
    outs = Y[torch.arange(B)[None, :, None], act]                                   # (T, B, K, d_out)
    reps = (w[..., None] * outs).sum(2)
    logit = (reps * P["hw"][:, None, :]).sum(-1) + P["hb"][:, None]
    pred = torch.sigmoid(logit).clamp(1e-7, 1 - 1e-7)
    task = -(y.double() * torch.log(pred) + (1 - y.double()) * torch.log1p(-pred)).sum() / B
    freq = torch.bincount(act.flatten(), minlength=E).double() / (B * T)
    mass = torch.zeros(E, dtype=torch.float64).scatter_add(0, act.flatten(), w.flatten()) / (B * T)
    lb = (E / 3) * (freq * mass).sum()
    (task + 0.05 * lb).backward()
    g = bw.gradients
    pairs = [("encoder1.weight", P["e1w"]), ("encoder1.bias", P["e1b"]), ("encoder2.weight", P["e2w"]),
             ("encoder2.bias", P["e2b"])]
    for name, ref in pairs:
        assert rel(g[name].cpu().numpy(), ref.grad.numpy()) < 3e-2, name
    gw = torch.stack([g[f"expert_{e}.weight"] for e in range(E)]).cpu().numpy()
    assert rel(gw, P["xw"].grad.numpy()) < 3e-2
    assert abs(bw.task_value - float(task)) < 2e-2 * float(task)
