"""SMESLayer (nn.Module + autograd.Function over the B200 kernels) against a float64 torch-autograd
restatement of the same layer with the GPU's selections frozen (the reference's backward is also
selection-fixed, training.py:119-226): task reps and L_lb forward, then every parameter gradient
and d_hidden for an arbitrary upstream gradient of the reps plus beta * L_lb.  bf16-representable
parameters and inputs, bf16 storage of the hidden activations / outputs / reps modelled with a
straight-through rounding, and the GPU's relu masks on the routed (instance, expert) pairs;
tolerance bf16 2e-2 (per tensor, max|diff| / max|ref|)."""
import zlib

import pytest
import torch

pytestmark = pytest.mark.gpu

import paper_2602_09386_b200 as smes

TOL = 2e-2


def rel(a, b):
    a, b = a.double().cpu(), b.double().cpu()
    return float((a - b).abs().max() / b.abs().max())


def _gpu_masks(layer, eng):
    """The GPU's relu masks of every relu pool, per (instance, expert): a pre-activation within the
    fp32 accumulation error of zero can take either sign, so the restatement applies the GPU's
    decisions (feed the oracle the GPU's masks) for the routed (instance, expert) pairs."""
    B, E = eng.B, layer.num_experts
    um = eng.umask.cpu().long() & 0xFFFFFFFF                              # (B, EW)
    e_idx = torch.arange(E)
    member = ((um[:, e_idx // 32] >> (e_idx % 32)) & 1).bool()            # (B, E)
    rank = member.long().cumsum(1) - 1
    rows = torch.gather(eng.row_of.cpu().long(), 1, rank.clamp(min=0))    # (B, E) packed row if member
    masks = []
    L = len(layer.acts)
    for i, a in enumerate(layer.acts):
        if a != "relu":
            masks.append(None)
            continue
        w = layer.widths[i + 1]
        if i < L - 1:
            words = eng.bits[i].cpu().long() & 0xFFFFFFFF                 # (w_pad / 32, R)
            bit = (words[:, :, None] >> torch.arange(32)) & 1             # (w_pad/32, R, 32)
            per_row = bit.permute(1, 0, 2).reshape(words.shape[1], -1)[:, :w].bool()
        else:
            per_row = eng.outs[-1].cpu()[:, :w].float() > 0
        masks.append((member, per_row[rows]))                              # (B, E, w) for members
    return masks


def _restate(layer, h, act_idx, masks=None):
    """float64 autograd restatement; act_idx (T, B, K) = the GPU's active sets."""
    st = lambda v: v + (v.bfloat16().double() - v).detach()      # bf16 storage, straight-through gradient
    P = {n: p.detach().double().cpu().clone().requires_grad_(True) for n, p in layer.named_parameters()}
    hd = h.detach().double().cpu().clone().requires_grad_(True)
    T, E, K = layer.num_tasks, layer.num_experts, act_idx.shape[2]
    B = hd.shape[0]
    z = torch.einsum("bd,ted->tbe", hd, P["router_weight"]) + P["router_bias"][:, None, :]
    w = torch.softmax(torch.gather(z, 2, act_idx), dim=2)                  # (T, B, K)
    x = hd[:, None, :].expand(B, E, hd.shape[1])
    for i, a in enumerate(layer.acts):
        y = torch.einsum("bei,eoi->beo", x, P[f"weight_{i}"]) + P[f"bias_{i}"][None]
        if a == "relu":
            m = (y > 0).detach()
            if masks is not None and masks[i] is not None:
                member, gm = masks[i]
                m = torch.where(member[:, :, None], gm, m)
            y = y * m
        x = st(y)                                                           # every expert, every row
    outs = x[torch.arange(B)[None, :, None], act_idx]                      # (T, B, K, d_out)
    reps = (w[..., None] * outs).sum(2)
    freq = torch.bincount(act_idx.flatten(), minlength=E).double() / (B * T)
    mass = torch.zeros(E, dtype=torch.float64).scatter_add(0, act_idx.flatten(), w.flatten()) / (B * T)
    lb = (E / K) * (freq * mass).sum()
    return reps, lb, P, hd


CASES = {
    # name: (B, T, E, d_in, d_out, d_ff, budget, act)
    "c2_shape_mlp": (2048, 8, 32, 256, 256, 512, (4, 2), "relu"),
    "c1_shape_relu": (1024, 4, 16, 128, 128, None, (2, 1), "relu"),
    "odd_widths_padded": (300, 3, 10, 20, 12, None, (2, 1), "identity"),
    "odd_mlp_padded": (257, 5, 12, 40, 24, 72, (1, 2), "relu"),
}


@pytest.mark.parametrize("name", list(CASES))
def test_smes_layer_autograd(name):
    B, T, E, d, d_out, d_ff, (ks, ka), act = CASES[name]
    gen = torch.Generator().manual_seed(zlib.crc32(name.encode()))
    layer = smes.SMESLayer(d, d_out, E, T, smes.RoutingBudget(ks, ka), d_ff=d_ff, expert_nonlinearity=act,
                           generator=gen)
    with torch.no_grad():
        for p in layer.parameters():
            p.copy_((p * (1000.0 if p is layer.router_weight else 1.0)).bfloat16().float())
            if p.ndim == 2 and p is not layer.router_bias:
                p.add_((torch.randn(p.shape, generator=gen) * 0.1).bfloat16().float().cuda())
    h = torch.randn(B, d, generator=gen).bfloat16().float().cuda().requires_grad_(True)
    R = torch.randn(T, B, d_out, generator=gen).cuda()
    beta = 0.3
    reps, lb = layer(h)
    assert reps.shape == (T, B, d_out) and lb.ndim == 0
    loss = (reps * R).sum() + beta * lb
    loss.backward()
    eng = layer.routing(B)
    act_idx = eng.active.long().cpu()
    rr, rlb, P, hd = _restate(layer, h, act_idx, _gpu_masks(layer, eng))
    assert rel(reps.detach(), rr.detach()) < TOL
    assert abs(float(lb) - float(rlb)) < 1e-4 * float(rlb)
    ((rr * R.double().cpu()).sum() + beta * rlb).backward()
    for n, p in layer.named_parameters():
        assert p.grad is not None, n
        assert p.grad.shape == p.shape, n
        assert rel(p.grad, P[n].grad) < TOL, n
    assert rel(h.grad, hd.grad) < TOL
    # a second forward of the same batch size reuses the engine; a stale backward is refused
    reps2, lb2 = layer(h)
    assert torch.allclose(reps2, reps)
    reps3, _ = layer(h)
    with pytest.raises(smes.StateError):
        reps2.sum().backward()
