"""Losses and the hand-derived backward -- drop-in for taskmoe/training.py (task_loss,
total_loss, backward, BackwardResult).

``backward`` runs the fused combine/heads/LB backward, the expert dgrad/wgrad
tcgen05 GEMMs, the router GEMMs and the un-permute kernel of the engine that
produced the forward result, then (if the model has an encoder) the encoder's
backward on the same GEMM kernel (training.py:214-222).
"""
from __future__ import annotations

from dataclasses import dataclass

import torch

from ._lib import call, ptr
from .balance import LoadStats, finalize_stats, load_stats
from .errors import NumericsError, ShapeError, StateError
from .model import ForwardResult, MoeModel, _gemm, _round, api_replay
from .routing import _stream

__all__ = ["CLAMP_LO", "CLAMP_HI", "task_loss", "total_loss", "backward", "BackwardResult"]

CLAMP_LO = 1e-7          # training.py:50
CLAMP_HI = 1.0 - 1e-7    # training.py:51


def task_loss(predictions, labels, weights=None) -> float:
    """Weighted clamped BCE averaged over instances (training.py:60-87)."""
    p = torch.as_tensor(predictions, dtype=torch.float32)
    y = torch.as_tensor(labels, dtype=torch.float32)
    if p.ndim == 1:
        p, y = p[None, :], y[None, :]
    if p.shape != y.shape or p.ndim != 2:
        raise ShapeError(f"predictions {tuple(p.shape)} and labels {tuple(y.shape)} must both be (T, B)")
    if p.shape[1] == 0:
        raise ShapeError("task loss of an empty batch")
    T, B = p.shape
    dev = p.device if p.is_cuda else torch.device("cuda")
    p, y = p.to(dev).contiguous(), y.to(dev).contiguous()
    w = torch.ones(T, device=dev) if weights is None else torch.as_tensor(weights, dtype=torch.float32).to(dev)
    if w.shape != (T,):
        raise ShapeError(f"expected {T} task weights, got shape {tuple(w.shape)}")
    if bool((w < 0).any()):
        raise NumericsError("task loss weights must be non-negative")
    nparts = 64
    part = torch.zeros(nparts, dtype=torch.float64, device=dev)
    bad = torch.zeros(1, dtype=torch.int32, device=dev)
    call("smes_bce_loss", T, B, ptr(p), ptr(y), ptr(w.contiguous()), ptr(part), nparts, ptr(bad), _stream())
    flags = int(bad.item())
    if flags & 1:
        raise NumericsError("predictions must lie in [0, 1]")
    if flags & 2:
        raise NumericsError("labels must be 0 or 1")
    return float(part.sum().item()) / B


def total_loss(task_value: float, lb_value: float, lb_strength: float) -> float:
    """training.py:90-94."""
    if lb_strength < 0:
        raise NumericsError(f"regularizer strength must be non-negative, got {lb_strength}")
    return float(task_value) + float(lb_strength) * float(lb_value)


@dataclass
class BackwardResult:
    """training.py:97-103: gradients keyed like MoeModel.parameter_blocks()."""
    gradients: dict
    task_value: float
    lb_value: float
    total: float
    stats: LoadStats
    d_hidden: torch.Tensor | None = None


def backward(result: ForwardResult, model: MoeModel, labels, dense_probs_in_stats: bool = False) -> BackwardResult:
    """Exact gradients of the total loss (training.py:119-226); selections fixed."""
    eng = result._engine
    if getattr(result, "precision", "bf16") == "fp32":
        raise StateError("backward of an fp32-precision forward is not provided (the fp32 mode is forward + "
                         "loss, BASELINE c1); run forward_sparse with precision='bf16' for training")
    if eng is None or result.mode != "sparse":
        raise StateError("backward needs a sparse forward result produced by this package")
    if getattr(eng, "step_id", None) != result._step:
        raise StateError("forward result is stale: its engine has run another forward since")
    y = torch.as_tensor(labels, dtype=torch.float32)
    T, B = result.predictions.shape
    if y.shape != (T, B):
        raise ShapeError(f"labels shape {tuple(y.shape)} does not match predictions ({T}, {B})")
    # pageable labels copy without waiting for the queued forward; pinned ones are copied before
    # returning control (the caller may reuse the buffer)
    y = y.to(eng.dev, non_blocking=not y.is_pinned())
    # the label check runs on the device and is read back with the losses: one host sync per call
    bad = ((y != 0) & (y != 1)).any()
    eng.labels.copy_(y)
    eng.dense = bool(dense_probs_in_stats)
    # loss + LoadStats (training.py:140-142) + fused combine bwd, then the expert / router backward
    api_replay(eng, ("bwd", eng.dense), lambda: (eng.forward_b(with_loss=True, train=True), eng.backward()))
    K = eng.K
    E, Ep = model.num_experts, eng.E
    raw = eng.stats_raw.view(3, Ep)[:, :E].reshape(-1).contiguous()
    out, f32 = finalize_stats(raw, E, K, B, T, eng.dense)
    grads = _logical_gradients(eng, model)
    d_hidden = eng.d_hidden[:, :model.d_in].clone()
    if result._enc is not None:
        grads.update(_encoder_backward(result._enc, model, eng))
    host = torch.cat([eng.loss_out, out[3 * E:], bad.double().view(1)]).cpu()
    if host[4] != 0:
        raise NumericsError("labels must be 0 or 1")
    stats = load_stats(out, f32, float(host[3]), E, K, B, T, eng.dense)
    ordered = {k: grads[k] for k in model.parameter_blocks() if k in grads}
    return BackwardResult(ordered, float(host[0]), float(host[1]), float(host[2]), stats, d_hidden)


def _logical_gradients(eng, model) -> dict:
    """Gradient blocks with the reference's names and shapes (model.py:94-111), sliced out of the
    engine's (possibly shim-padded) stacked gradients.  One copy of the engine's flat gradient
    buffer backs every block, so the result owns its memory (a later step cannot rewrite it) for a
    single device copy instead of one per block."""
    T, E, Ep = model.num_tasks, model.num_experts, eng.E
    pools = model.pools
    dims = [model.d_in] + [p.d_out for p in pools]
    flat = eng.grad_flat.clone()
    own = lambda v: flat[v.data_ptr() // 4 - eng.grad_flat.data_ptr() // 4:][:v.numel()].view(v.shape)
    g = {}
    for li, (gw, gb) in enumerate(eng.g_layers):
        di, do = dims[li], dims[li + 1]
        pre = "expert_" if len(pools) == 1 else f"expert{li}_"
        # one unbind per stack (the views in one call, not 2E indexing ops)
        for e, (w, b) in enumerate(zip(own(gw)[:E, :do, :di].unbind(0), own(gb)[:E, :do].unbind(0))):
            g[f"{pre}{e}.weight"] = w
            g[f"{pre}{e}.bias"] = b
    rw = own(eng.g_router_w).view(T, Ep, eng.d)[:, :E, :dims[0]].unbind(0)
    rb = own(eng.g_router_b).view(T, Ep)[:, :E].unbind(0)
    hw = own(eng.g_head_w)[:, :dims[-1]].split(1)
    hb = own(eng.g_head_b).split(1)
    for t in range(T):
        g[f"router_{t}.weight"] = rw[t]
        g[f"router_{t}.bias"] = rb[t]
        g[f"head_{t}.weight"] = hw[t]
        g[f"head_{t}.bias"] = hb[t]
    return g


def _encoder_backward(enc: dict, model: MoeModel, eng) -> dict:
    """encoder2/encoder1 grads from d_hidden (training.py:214-222) on the tcgen05 GEMM."""
    B, dev = eng.B, eng.dev
    Bp = _round(B, 128)
    d, Fp, F = _round(model.d_in, 8), enc["Fp"], enc["F"]
    dh, dhr = enc["dhp"], enc["dh"]
    s = _stream()
    seg1 = torch.tensor([0, Bp], dtype=torch.int32, device=dev)
    g = {}
    dhid = torch.zeros(Bp, d, dtype=torch.bfloat16, device=dev)
    dhid[:B, :model.d_in] = eng.d_hidden[:, :model.d_in]
    w2 = torch.zeros(1, d, dh, dtype=torch.bfloat16, device=dev)      # MN-major (K = d_in, N = d_hidden)
    w2[0, :model.d_in, :dhr] = model.encoder2.weight
    # encoder2: dW = d_hidden^T mid, db = sum d_hidden, d_mid = d_hidden W2 (x relu mask)
    dw2 = torch.zeros(1, d, dh, device=dev)
    call("smes_gemm_ragged_k", ptr(dhid), d, ptr(enc["mid"]), dh, B, 1, d, dh, ptr(seg1), ptr(dw2), None, s)
    part = torch.zeros(Bp // 128, max(d, dh), device=dev)
    db2 = torch.zeros(1, d, device=dev)
    call("smes_seg_colsum", ptr(dhid), d, Bp, d, ptr(seg1), 1, ptr(part), ptr(db2), s)
    dmid = torch.zeros(Bp, dh, dtype=torch.bfloat16, device=dev)
    _gemm(dhid, d, Bp, w2, dh, d, None, 0, dmid, dh, 0, B, b_mn=1, bits_in=enc["bits"], bits_ld=Bp)
    # encoder1: dW = d_pre^T x, db = sum d_pre
    dw1 = torch.zeros(1, dh, Fp, device=dev)
    call("smes_gemm_ragged_k", ptr(dmid), dh, ptr(enc["xb"]), Fp, B, 1, dh, Fp, ptr(seg1), ptr(dw1), None, s)
    db1 = torch.zeros(1, dh, device=dev)
    call("smes_seg_colsum", ptr(dmid), dh, Bp, dh, ptr(seg1), 1, ptr(part), ptr(db1), s)
    g["encoder1.weight"] = dw1[0, :dhr, :F].contiguous()
    g["encoder1.bias"] = db1[0, :dhr].contiguous()
    g["encoder2.weight"] = dw2[0, :model.d_in, :dhr].contiguous()
    g["encoder2.bias"] = db2[0, :model.d_in].contiguous()
    return g
