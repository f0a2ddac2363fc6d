"""End-to-end parity of the CUDA SMES layer (fwd + bwd) against the CPU oracle.

Selections are index-exact given the GPU's logits; floats within the north
star's bf16 tolerance (2e-2 relative, per tensor: max|diff| / max|ref|).
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from oracle import smes_oracle as O
from paper_2602_09386_b200 import SMESEngine
from tests.helpers import make_case, rel, to_engine_params

BF16_TOL = 2e-2
FP32_TOL = 1e-5

CASES = {
    # name: (seed, B, T, E, d, d_out, ks, ka, d_ff, router_scale, dense, extra)
    "c1_mlp": (0, 1024, 4, 16, 128, 128, 2, 1, 256, 1e-3, False, {}),
    "c1_single_relu": (1, 1024, 4, 16, 128, 128, 2, 1, None, 1e-3, False, {}),
    "c2_small_batch": (2, 2048, 8, 32, 256, 256, 4, 2, 512, 1e-3, False, {}),
    "dense_stats_taskw": (3, 700, 4, 16, 128, 128, 1, 2, 256, 1.0, True, dict(rand_task_w=True, rand_lam=True)),
    "no_shared": (4, 512, 4, 16, 128, 128, 0, 3, None, 1.0, False, {}),
    "single_identity": (5, 1024, 4, 16, 128, 128, 2, 1, None, 1e-3, False, dict(last_act="identity")),
    "c2_t5_csum_gemm": (6, 1536, 5, 32, 256, 256, 4, 2, 512, 1e-3, False, dict(rand_lam=True)),
    "c2_unfused_mlp": (2, 2048, 8, 32, 256, 256, 4, 2, 512, 1e-3, False, {}),
    "c1_d64_dff384": (8, 777, 4, 16, 64, 128, 2, 1, 384, 1.0, False, dict(rand_task_w=True)),
    "c2_fused_wgrad": (10, 2048, 8, 32, 256, 256, 4, 2, 512, 1e-3, False, {}),
    "c3_shape_d512": (11, 1024, 16, 64, 512, 512, 4, 2, 1024, 1e-3, False, {}),
}
# engine options per case (csum_from_gemm: per-expert sums of C from the folded wgrad's ones column)
ENGINE_OPTS = {"c2_t5_csum_gemm": dict(csum_from_gemm=True), "c2_unfused_mlp": dict(fuse_mlp=False),
               "c2_fused_wgrad": dict(fuse_wgrad=True)}


def run_case(name, fold=True):
    seed, B, T, E, d, d_out, ks, ka, d_ff, rs, dense, extra = CASES[name]
    p, h, y, lam, beta = make_case(seed, B, T, E, d, d_out, ks, ka, d_ff=d_ff, router_scale=rs, **extra)
    eng = SMESEngine(to_engine_params(p, lam, beta), B, ks, ka, dense_probs_in_stats=dense,
                     **ENGINE_OPTS.get(name, {}))
    eng.set_inputs(torch.tensor(h, device="cuda"), torch.tensor(y, device="cuda", dtype=torch.float32))
    eng.forward(with_loss=True)          # inference-style forward: materialises every pool output + task reps
    torch.cuda.synchronize()
    eng.reps_fwd = eng.reps.clone()
    eng.outs_fwd = [o.clone() for o in eng.outs]
    # training step (fused combine backward when sparse; heads folded into an identity last pool)
    eng.forward_a(fold=fold and eng.can_fold)
    eng.forward_b(with_loss=True, train=True)
    eng.backward()
    torch.cuda.synchronize()
    return p, h, y, lam, beta, dense, eng


PARAMS = [(n, True) for n in CASES] + [(n, False) for n in ("c1_mlp", "c2_small_batch", "single_identity")]


@pytest.mark.parametrize("name,fold", PARAMS)
def test_layer_parity(name, fold):
    p, h, y, lam, beta, dense, eng = run_case(name, fold)
    if fold and eng.can_fold:
        assert eng._folded, "identity last pool + sparse stats must take the folded training path"
    T, E, B, ks, ka = eng.T, eng.E, eng.B, eng.ks, eng.ka
    z = eng.z.double().cpu().numpy().reshape(B, T, E).transpose(1, 0, 2)
    # router logits against RouterBank.logits (routing.py:101-103) on the identical bf16 operands
    assert rel(z, O.router_logits(h, p)) < FP32_TOL

    # --- routing: index-exact on the GPU's logits (routing.py:235-281)
    r = O.route_batch(z, ks, ka, p.task_weights)
    assert np.array_equal(eng.shared.cpu().numpy(), r.shared)
    assert np.array_equal(eng.adaptive.cpu().numpy(), r.adaptive)
    assert np.array_equal(eng.active.cpu().numpy(), r.active)
    w_ref = np.take_along_axis(r.weights, r.active, axis=2)
    assert rel(eng.wsel.cpu().numpy(), w_ref) < FP32_TOL
    assert np.array_equal(eng.usize.cpu().numpy(), [u.size for u in r.unions])

    # --- plan: identical packing order once pad rows are dropped (execution.py:85-123)
    plan = O.build_execution_plan(r.unions, E)
    gi = eng.gather_inst.cpu().numpy()
    ge = eng.gather_exp.cpu().numpy()
    seg_pad = eng.seg_pad.cpu().numpy()
    keep = np.zeros(len(gi), bool)
    keep[: seg_pad[-1]] = gi[: seg_pad[-1]] >= 0
    assert np.array_equal(gi[keep], plan.gather_instances)
    assert np.array_equal(ge[keep], plan.gather_experts)
    assert np.array_equal(eng.loads.cpu().numpy(), plan.loads)
    assert np.array_equal(eng.seg_log.cpu().numpy(), plan.segment_offsets)
    assert eng.n_act() == plan.total_rows

    # --- forward values (frozen = the GPU's selections, model.py:284-300)
    f = O.forward_sparse(h, p, ks, ka, logits=z, frozen=r, frozen_plan=plan)
    rows = np.nonzero(keep)[0]
    for li in range(len(p.layers)):
        got = eng.outs_fwd[li][:, :eng.dims[li + 1]].float().cpu().numpy()[rows]
        assert rel(got, f.layer_outs[li]) < BF16_TOL, li
    assert rel(eng.reps_fwd.float().cpu().numpy(), f.task_reps) < BF16_TOL
    assert rel(eng.logits.cpu().numpy(), f.head_logits) < BF16_TOL
    assert rel(eng.preds.cpu().numpy(), f.predictions) < BF16_TOL

    # --- regularizer + loss (balance.py:54-80, training.py:54-94)
    bw = O.backward(f, p, y, lam, beta, dense)
    st = eng.stats_out.cpu().numpy()
    assert np.array_equal(st[2 * E:3 * E], bw.stats.counts)
    assert rel(st[:E], bw.stats.frequency) < 1e-12
    assert rel(st[E:2 * E], bw.stats.mass) < FP32_TOL
    assert abs(st[3 * E] - bw.stats.value) <= FP32_TOL * abs(bw.stats.value)
    lo = eng.loss_out.cpu().numpy()
    assert abs(lo[0] - bw.task_value) <= BF16_TOL * abs(bw.task_value)
    assert abs(lo[2] - bw.total) <= BF16_TOL * abs(bw.total)

    # --- gradients (training.py:119-226)
    for li, (gw, gb) in enumerate(eng.g_layers):
        assert rel(gw.cpu().numpy(), bw.layers[li][0]) < BF16_TOL, ("W", li)
        assert rel(gb.cpu().numpy(), bw.layers[li][1]) < BF16_TOL, ("b", li)
    assert rel(eng.g_router_w.cpu().numpy().reshape(T, E, -1), bw.router_w) < BF16_TOL
    assert rel(eng.g_router_b.cpu().numpy().reshape(T, E), bw.router_b) < BF16_TOL
    assert rel(eng.g_head_w.cpu().numpy(), bw.head_w) < BF16_TOL
    assert rel(eng.g_head_b.cpu().numpy(), bw.head_b) < BF16_TOL
    assert rel(eng.d_hidden.cpu().numpy(), bw.d_hidden) < BF16_TOL


def test_unselected_expert_grads_exactly_zero():
    """test_training.py:107-119: an expert in no packed row gets an exactly-zero block."""
    p, h, y, lam, beta = make_case(7, 256, 2, 16, 128, 128, 1, 1, router_scale=1.0)
    p.router_b[:, 5] = -1e4   # expert 5 never selected
    eng = SMESEngine(to_engine_params(p, lam, beta), 256, 1, 1)
    eng.set_inputs(torch.tensor(h, device="cuda"), torch.tensor(y, device="cuda", dtype=torch.float32))
    eng.step()
    torch.cuda.synchronize()
    assert eng.loads[5].item() == 0
    gw, gb = eng.g_layers[0]
    assert torch.all(gw[5] == 0) and torch.all(gb[5] == 0)


def test_graph_replay_is_deterministic():
    """Bitwise-identical results across CUDA-graph replays (SPEC determinism, test_training.py:168-180)."""
    p, h, y, lam, beta = make_case(9, 2048, 8, 32, 256, 256, 4, 2, d_ff=512)
    eng = SMESEngine(to_engine_params(p, lam, beta), 2048, 4, 2)
    eng.set_inputs(torch.tensor(h, device="cuda"), torch.tensor(y, device="cuda", dtype=torch.float32))
    g = eng.capture_step()
    g.replay()
    torch.cuda.synchronize()
    snap = [t.clone() for t in (eng.g_layers[0][0], eng.g_router_w, eng.d_hidden, eng.loss_out)]
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    for a, b in zip(snap, (eng.g_layers[0][0], eng.g_router_w, eng.d_hidden, eng.loss_out)):
        assert torch.equal(a, b)


def test_gathered_layer_input_is_bit_identical():
    """SMES_GATHER_X mode (mlp_fwd and the fc1 weight gradient read the layer input rows from h by
    TMA gather4, no packed X) and SMES_FWD_PACK mode (mlp_fwd's gather warp copies the rows and
    writes the packed X): the training step's loss, gradients and d_hidden equal the packed-X step
    bit for bit."""
    p, h, y, lam, beta = make_case(11, 2048, 8, 32, 256, 256, 4, 2, d_ff=512)
    outs = []
    for gather, pack in ((False, False), (True, False), (False, True)):
        eng = SMESEngine(to_engine_params(p, lam, beta), 2048, 4, 2)
        eng.gather_x, eng.fwd_pack = gather, pack
        eng.set_inputs(torch.tensor(h, device="cuda"), torch.tensor(y, device="cuda", dtype=torch.float32))
        eng.step()
        torch.cuda.synchronize()
        assert eng._x_gathered == gather and eng._x_packed_by_fwd == pack
        outs.append([t.clone() for t in (eng.loss_out, eng.grad_flat, eng.d_hidden, eng.P)])
    for other in outs[1:]:
        for a, b in zip(outs[0], other):
            assert torch.equal(a, b)


@pytest.mark.parametrize("name", ["c1_mlp", "c2_small_batch", "c3_shape_d512", "c1_single_relu"])
def test_score_matches_oracle(name):
    """Inference scoring (SMESEngine.score, BASELINE c4): predictions and logits from the folded
    heads (no hidden / O / reps writes) against the oracle forward on the GPU's selections."""
    seed, B, T, E, d, d_out, ks, ka, d_ff, rs, dense, extra = CASES[name]
    p, h, y, lam, beta = make_case(seed, B, T, E, d, d_out, ks, ka, d_ff=d_ff, router_scale=rs, **extra)
    eng = SMESEngine(to_engine_params(p, lam, beta), B, ks, ka)
    eng.set_inputs(torch.tensor(h, device="cuda"))
    eng.score()
    torch.cuda.synchronize()
    z = eng.z.double().cpu().numpy().reshape(B, T, E).transpose(1, 0, 2)
    assert rel(z, O.router_logits(h, p)) < FP32_TOL
    r = O.route_batch(z, ks, ka, p.task_weights)
    assert np.array_equal(eng.active.cpu().numpy(), r.active)
    plan = O.build_execution_plan(r.unions, E)
    f = O.forward_sparse(h, p, ks, ka, logits=z, frozen=r, frozen_plan=plan)
    assert rel(eng.logits.cpu().numpy(), f.head_logits) < BF16_TOL
    assert rel(eng.preds.cpu().numpy(), f.predictions) < BF16_TOL
