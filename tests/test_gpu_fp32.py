"""fp32 arithmetic mode (BASELINE c1; north star: fp32 outputs within 1e-5 relative).

The forward runs with fp32 operands and activations; its GEMMs are bf16x3 tensor-core products
(csrc/gemm.cu smes_gemm_ragged_m_x3).  Checked against the float64 oracle on the SAME fp32 inputs
and weights (no bf16 rounding anywhere), and against the reference's own recorded layer goldens
through the drop-in ``forward_sparse(..., precision="fp32")``.  Tolerance: 1e-5 relative per tensor
(max|diff| / max|ref|).  Selections are index-exact given the GPU's logits, and the GPU's logits
match the oracle's within 1e-5.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

import paper_2602_09386_b200 as smes
from oracle import smes_oracle as O
from paper_2602_09386_b200.fp32 import SMESForwardF32, split_planes
from tests.helpers import rel, to_engine_params

FP32_TOL = 1e-5


def _f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def make_case_f32(seed, B, T, E, d, d_out, ks, ka, d_ff=None, router_scale=1e-3, last_act=None):
    """Seeded fp32 parameters and input (fp32-representable, so the oracle sees the GPU's operands)."""
    rng = np.random.default_rng(seed)
    p = O.init_layer_params(rng, d, d_out, E, T, d_ff=d_ff, router_scale=router_scale)
    p.layers = [(_f32(w), _f32(rng.normal(size=b.shape) * 0.1), act) for (w, b, act) in p.layers]
    if last_act is not None:
        w, b, _ = p.layers[-1]
        p.layers[-1] = (w, b, last_act)
    p.router_w = _f32(p.router_w)
    p.router_b = _f32(rng.normal(size=p.router_b.shape) * router_scale)
    p.head_w = _f32(p.head_w)
    p.head_b = _f32(rng.normal(size=T) * 0.1)
    h = _f32(rng.normal(size=(B, d)))
    y = (rng.uniform(size=(T, B)) < 0.3).astype(np.float64)
    lam = _f32(rng.uniform(0.5, 2.0, T))
    return p, h, y, lam, 0.01


CASES = {
    # name: (seed, B, T, E, d, d_out, ks, ka, d_ff, router_scale, last_act)
    "c1": (0, 1024, 4, 16, 128, 128, 2, 1, 256, 1e-3, None),            # BASELINE configs[0]
    "c1_trained_router": (1, 1024, 4, 16, 128, 128, 2, 1, 256, 1.0, None),
    "single_relu_pool": (2, 777, 4, 16, 128, 128, 2, 1, None, 1.0, None),
    "single_identity_pool": (3, 512, 3, 16, 64, 96, 1, 2, None, 1.0, "identity"),
    "c2_shape": (4, 2048, 8, 32, 256, 256, 4, 2, 512, 1e-3, None),
}


@pytest.mark.parametrize("name", list(CASES))
def test_fp32_forward_matches_oracle(name):
    seed, B, T, E, d, d_out, ks, ka, d_ff, rs, last_act = CASES[name]
    p, h, y, lam, beta = make_case_f32(seed, B, T, E, d, d_out, ks, ka, d_ff, rs, last_act)
    eng = SMESForwardF32(to_engine_params(p, lam, beta), B, ks, ka)
    eng.set_inputs(torch.tensor(h, dtype=torch.float32, device="cuda"),
                   torch.tensor(y, dtype=torch.float32, device="cuda"))
    eng.forward(with_loss=True)
    torch.cuda.synchronize()
    eng.check_finite()
    # router logits (routing.py:101-103): fp32 GEMM on the tensor cores vs f64
    z = eng.z.double().cpu().numpy().reshape(B, T, E).transpose(1, 0, 2)
    assert rel(z, O.router_logits(h, p)) < FP32_TOL
    # selections: index-exact given the GPU's logits (routing.py:235-281)
    r = O.route_batch(z, ks, ka, p.task_weights)
    assert np.array_equal(eng.shared.cpu().numpy(), r.shared)
    assert np.array_equal(eng.active.cpu().numpy(), r.active)
    assert rel(eng.wsel.cpu().numpy(), np.take_along_axis(r.weights, r.active, axis=2)) < FP32_TOL
    plan = O.build_execution_plan(r.unions, E)
    f = O.forward_sparse(h, p, ks, ka, logits=z, frozen=r, frozen_plan=plan)
    gi = eng.gather_inst.cpu().numpy()
    seg_pad = eng.seg_pad.cpu().numpy()
    keep = np.zeros(len(gi), bool)
    keep[: seg_pad[-1]] = gi[: seg_pad[-1]] >= 0
    assert np.array_equal(gi[keep], plan.gather_instances)
    rows = np.nonzero(keep)[0]
    for li in range(len(p.layers)):
        assert rel(eng.outs[li].cpu().numpy()[rows], f.layer_outs[li]) < FP32_TOL, li
    assert rel(eng.reps.cpu().numpy(), f.task_reps) < FP32_TOL
    assert rel(eng.logits.cpu().numpy(), f.head_logits) < FP32_TOL
    assert rel(eng.preds.cpu().numpy(), f.predictions) < FP32_TOL
    # regularizer + loss (balance.py:54-80, training.py:54-94)
    bw = O.backward(f, p, y, lam, beta)
    st = eng.stats_out.cpu().numpy()
    assert np.array_equal(st[2 * E:3 * E], bw.stats.counts)
    assert rel(st[E:2 * E], bw.stats.mass) < FP32_TOL
    assert abs(st[3 * E] - bw.stats.value) <= FP32_TOL * abs(bw.stats.value)
    lo = eng.loss_out.cpu().numpy()
    assert abs(lo[0] - bw.task_value) <= FP32_TOL * abs(bw.task_value)
    assert abs(lo[2] - bw.total) <= FP32_TOL * abs(bw.total)


@pytest.mark.parametrize("M,N,K,G", [(1000, 64, 128, 1), (3000, 256, 256, 4), (700, 24, 64, 3), (2048, 512, 192, 2)])
def test_x3_gemm_is_fp32_accurate(M, N, K, G):
    """smes_gemm_ragged_m_x3 against an f64 matmul of the same fp32 operands: within the fp32 1e-5
    contract, and at least 100x closer than the GEMM of the bf16-rounded operands (~4e-3 off)."""
    from paper_2602_09386_b200._lib import call, ptr
    g = torch.Generator().manual_seed(M + N)
    rows = [M // G] * G
    seg = [0]
    for r in rows:
        seg.append(seg[-1] + (r + 127) // 128 * 128)
    R = seg[-1]
    a = torch.zeros(R, K)
    for i in range(G):
        a[seg[i]:seg[i] + rows[i]] = torch.randn(rows[i], K, generator=g)
    w = torch.randn(G, N, K, generator=g) / K ** 0.5
    b = torch.randn(G, N, generator=g)
    ad, wd, bd = a.cuda(), w.cuda(), b.cuda()
    out = torch.zeros(R, N, device="cuda")
    segd = torch.tensor(seg, dtype=torch.int32, device="cuda")
    a3, w3 = split_planes(ad), split_planes(wd.view(G * N, K))     # keep the planes alive until the GEMM ran
    call("smes_gemm_ragged_m_x3", ptr(a3), 3 * K, R, ptr(w3), G, N, K, ptr(segd), ptr(bd), 1, ptr(out), N, R,
         torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    ref = torch.zeros(R, N, dtype=torch.float64)
    for i in range(G):
        ref[seg[i]:seg[i + 1]] = torch.relu(a[seg[i]:seg[i + 1]].double() @ w[i].double().T + b[i].double())
    err = rel(out.cpu().numpy(), ref.numpy())
    # the same GEMM on bf16-rounded operands (what the bf16 path computes)
    bf = torch.zeros(R, N, dtype=torch.float64)
    for i in range(G):
        bf[seg[i]:seg[i + 1]] = torch.relu(a[seg[i]:seg[i + 1]].bfloat16().double() @ w[i].bfloat16().double().T
                                           + b[i].double())
    assert err < 1e-5
    assert err < rel(bf.numpy(), ref.numpy()) / 100


def test_split_planes_reconstruct_fp32_exactly():
    x = torch.randn(513, 96, device="cuda") * torch.logspace(-20, 20, 96, device="cuda")
    p = split_planes(x).float()
    s = p[:, :96] + p[:, 96:192] + p[:, 192:]
    assert torch.equal(s, x)


def _golden_model(g):
    t = lambda a: torch.tensor(np.asarray(a), dtype=torch.float32, device="cuda")
    E, T = g["expert_w"].shape[0], g["router_w"].shape[0]
    pool = smes.ExpertPool([smes.Affine(t(g["expert_w"][e]), t(g["expert_b"][e])) for e in range(E)], str(g["act"]))
    routers = smes.RouterBank([smes.Affine(t(g["router_w"][k]), t(g["router_b"][k])) for k in range(T)],
                              g["task_weights"])
    heads = [smes.Affine(t(g["head_w"][k:k + 1]), t(g["head_b"][k:k + 1])) for k in range(T)]
    return smes.MoeModel(None, None, pool, routers, heads, g["lam"], float(g["beta"]),
                         smes.RoutingBudget(int(g["k_shared"]), int(g["k_adaptive"])))


@pytest.mark.parametrize("i", range(5))
def test_fp32_api_against_reference_goldens(golden_dir, i):
    """The reference's recorded f64 outputs (tests/golden/make_golden.py) through the drop-in
    forward_sparse in fp32 mode: selections exact, every forward output within 1e-5."""
    g = np.load(f"{golden_dir}/layer_golden_{i}.npz")
    model = _golden_model(g)
    h = torch.tensor(g["h"], dtype=torch.float32, device="cuda")
    res = smes.forward_sparse(h, model, dense_probs_in_stats=bool(g["dense"]), precision="fp32")
    assert res.precision == "fp32"
    # fp32 rounding of the golden's f64 inputs bounds the agreement (~6e-8 relative per operand)
    assert rel(res.router_logits.cpu().numpy(), g["router_logits"]) < FP32_TOL
    assert np.array_equal(res.routing.shared.cpu().numpy(), g["shared"])
    assert np.array_equal(res.routing.active.cpu().numpy(), g["active"])
    assert rel(res.routing.weights.cpu().numpy(), g["weights"]) < FP32_TOL
    assert np.array_equal(res.plan.gather_instances.cpu().numpy(), g["gather_instances"])
    assert rel(res.packed_out.cpu().numpy(), g["packed_out"]) < FP32_TOL
    assert rel(res.task_reps.cpu().numpy(), g["task_reps"]) < FP32_TOL
    assert rel(res.head_logits.cpu().numpy(), g["head_logits"]) < FP32_TOL
    assert rel(res.predictions.cpu().numpy(), g["predictions"]) < FP32_TOL
    tv = smes.task_loss(res.predictions, torch.tensor(g["labels"], device="cuda"), g["lam"])
    assert abs(tv - float(g["task_value"])) <= FP32_TOL * abs(float(g["task_value"]))
    st = smes.compute_load_stats(res.routing, dense_probs=bool(g["dense"]))
    assert abs(st.value - float(g["lb_value"])) <= FP32_TOL * abs(float(g["lb_value"]))
    with pytest.raises(smes.StateError):
        smes.backward(res, model, torch.tensor(g["labels"]))


def test_fp32_api_with_encoder():
    """forward_sparse(precision='fp32') through a model with the reference's encoder
    (model.py:188-199): logits and predictions within 1e-5 of an f64 recomputation."""
    gen = torch.Generator().manual_seed(5)
    m = smes.init_model(gen, 40, 72, 128, 128, 16, 4, smes.RoutingBudget(2, 1), d_ff=256, lb_strength=0.01)
    x = torch.randn(300, 40, generator=gen).cuda()
    res = smes.forward_sparse(x, m, precision="fp32")
    xd = x.double()
    e1 = xd @ m.encoder1.weight.double().T + m.encoder1.bias.double()
    hid = torch.relu(e1) @ m.encoder2.weight.double().T + m.encoder2.bias.double()
    assert rel(res.hidden.cpu().numpy(), hid.cpu().numpy()) < FP32_TOL
    z = torch.stack([hid @ mp.weight.double().T + mp.bias.double() for mp in m.routers.maps])
    assert rel(res.router_logits.cpu().numpy(), z.cpu().numpy()) < FP32_TOL
