"""The SMES layer as a ``torch.nn.Module`` (SURVEY 8(b) "Layer forward").

``SMESLayer(h)`` returns ``(task_reps (T, B, d_out), lb)``: the per-task mixtures of the
selected experts' outputs (reconstruct_task_reps, execution.py:161-191, after route_batch and
the grouped expert pools) and the load-balancing value L_lb = (E/K) <f, p> (balance.py:54-80).
Both are differentiable through a ``torch.autograd.Function`` whose backward runs the B200
kernels: the combine backward from the upstream d_reps plus the LB term (csrc/layer.cu), the
grouped dgrad / wgrad GEMMs of every pool, the router backward and the un-permute
(training.py:160-212).  Selections are piecewise constant, as in the reference's hand-derived
backward (selections fixed).  The heads and the task loss stay outside the layer, so any torch
head / loss can sit on top of it.

Parameters are ``nn.Parameter`` tensors in the reference layouts: ``router_weight`` (T, E, d_in)
and ``router_bias`` (T, E) (RouterBank.maps stacked, routing.py:64-103), and per pool
``weight_{l}`` (E, d_out, d_in) / ``bias_{l}`` (E, d_out) (ExpertPool.layers stacked,
experts.py:26-60).  Any widths: the shim pads to the kernels' granularity (model.py).
"""
from __future__ import annotations

import torch

from . import engine as _engine
from .errors import ConfigError, ShapeError, StateError
from .model import ROUTER_INIT_SCALE, _Pad, pad_params
from .routing import RoutingBudget

__all__ = ["SMESLayer"]

_ACTS = ("identity", "relu")


class _SMESFunction(torch.autograd.Function):
    @staticmethod
    def forward(ctx, h, layer, rw, rb, *pool_params):
        eng, pad = layer._engine(h.shape[0])
        d, d_out = layer.d_in, layer.d_out
        eng.h[:, :d].copy_(h.detach())
        eng.forward_layer()
        eng.step_id += 1
        ctx.eng, ctx.pad, ctx.step, ctx.layer = eng, pad, eng.step_id, layer
        reps = eng.reps[..., :d_out].float()
        lb = eng.stats_out[3 * eng.E].float().clone()
        return reps, lb

    @staticmethod
    def backward(ctx, d_reps, d_lb):
        eng, pad, layer = ctx.eng, ctx.pad, ctx.layer
        if eng.step_id != ctx.step:
            raise StateError("SMESLayer backward after another forward through the same engine; "
                             "call backward before the next forward of this batch size")
        T, B, E = layer.num_tasks, eng.B, layer.num_experts
        dr = torch.zeros(T, B, eng.d_out, dtype=torch.float32, device=eng.dev)
        if d_reps is not None:
            dr[..., :layer.d_out] = d_reps
        eng.backward_reps(dr, float(d_lb) if d_lb is not None else 0.0)
        Ep = eng.E
        dims = pad.dims
        grads = []
        for i, (gw, gb) in enumerate(eng.g_layers):
            grads += [gw[:E, :dims[i + 1], :dims[i]].clone(), gb[:E, :dims[i + 1]].clone()]
        d_rw = eng.g_router_w.view(T, Ep, eng.d)[:, :E, :dims[0]].clone()
        d_rb = eng.g_router_b.view(T, Ep)[:, :E].clone()
        d_h = eng.d_hidden[:, :dims[0]].clone()
        return (d_h, None, d_rw, d_rb, *grads)


class SMESLayer(torch.nn.Module):
    """forward(h (B, d_in)) -> (task_reps (T, B, d_out), lb_value) on the B200 kernels."""

    def __init__(self, d_in: int, d_out: int, num_experts: int, num_tasks: int, budget: RoutingBudget,
                 d_ff: int | None = None, expert_nonlinearity: str = "relu", task_weights=None,
                 generator: torch.Generator | None = None, device="cuda"):
        super().__init__()
        budget.validate(num_experts)
        if expert_nonlinearity not in _ACTS:
            raise ConfigError(f"unknown nonlinearity '{expert_nonlinearity}', expected one of {_ACTS}")
        self.budget = budget
        self.num_experts, self.num_tasks = num_experts, num_tasks
        self.d_in, self.d_out = d_in, d_out
        if d_ff is None:
            self.acts = [expert_nonlinearity]
            widths = [d_in, d_out]
        else:   # BASELINE expert MLP: relu d_in -> d_ff, identity d_ff -> d_out
            self.acts = ["relu", "identity"]
            widths = [d_in, d_ff, d_out]
        self.widths = widths
        u = lambda *s, scale: ((torch.rand(*s, generator=generator, dtype=torch.float64) * 2 - 1) * scale).float()
        # fan-in uniform experts, near-zero routers (model.py:117-156)
        self.router_weight = torch.nn.Parameter(
            u(num_tasks, num_experts, d_in, scale=ROUTER_INIT_SCALE / d_in ** 0.5).to(device))
        self.router_bias = torch.nn.Parameter(torch.zeros(num_tasks, num_experts, device=device))
        for i in range(len(widths) - 1):
            self.register_parameter(f"weight_{i}", torch.nn.Parameter(
                u(num_experts, widths[i + 1], widths[i], scale=1.0 / widths[i] ** 0.5).to(device)))
            self.register_parameter(f"bias_{i}", torch.nn.Parameter(
                torch.zeros(num_experts, widths[i + 1], device=device)))
        tw = torch.ones(num_tasks, dtype=torch.float64) if task_weights is None else \
            torch.as_tensor(task_weights, dtype=torch.float64)
        if tw.shape != (num_tasks,) or bool((tw < 0).any()):
            raise ConfigError("task pooling weights must be non-negative, one per task")
        self.register_buffer("task_weights", tw, persistent=True)
        self._engines = {}

    def pool_params(self) -> list:
        out = []
        for i in range(len(self.widths) - 1):
            out += [getattr(self, f"weight_{i}"), getattr(self, f"bias_{i}")]
        return out

    def _params(self, pad: _Pad) -> _engine.SMESParams:
        T = self.num_tasks
        rw, rb = self.router_weight.detach(), self.router_bias.detach()
        pp = self.pool_params()
        layers = [(pp[2 * i].detach(), pp[2 * i + 1].detach(), a) for i, a in enumerate(self.acts)]
        hw = torch.zeros(T, self.d_out, device=rw.device)      # no heads in the layer form
        if pad.active:
            rw, rb, layers, hw = pad_params(rw, rb, layers, hw, pad)
        return _engine.SMESParams(router_w=rw, router_b=rb,
                                  layers=[_engine.ExpertLayer(w, b, a) for (w, b, a) in layers],
                                  head_w=hw, head_b=torch.zeros(T, device=rw.device), task_weights=self.task_weights,
                                  task_loss_weights=torch.ones(T), lb_strength=0.0)

    def _engine(self, B: int):
        pad = _Pad(None, self.num_tasks, self.num_experts, self.widths)
        eng = self._engines.get(B)
        if eng is None:
            eng = _engine.SMESEngine(self._params(pad), B, self.budget.k_shared, self.budget.k_adaptive,
                                     device=self.router_weight.device, lb_experts=self.num_experts)
            eng.step_id = 0
            self._engines[B] = eng
        else:
            eng.p = self._params(pad)
            eng.refresh_weights()
        return eng, pad

    def forward(self, h: torch.Tensor):
        if h.ndim != 2 or h.shape[1] != self.d_in:
            raise ShapeError(f"hidden has shape {tuple(h.shape)}, layer expects (B, {self.d_in})")
        if h.shape[0] == 0:
            raise ShapeError("forward of an empty batch")
        if not h.is_cuda:
            raise ShapeError("SMESLayer expects a CUDA tensor")
        return _SMESFunction.apply(h, self, self.router_weight, self.router_bias, *self.pool_params())

    def routing(self, B: int):
        """The routing decisions of the last forward of batch size B (device buffers)."""
        eng = self._engines.get(B)
        if eng is None:
            raise StateError(f"no forward of batch size {B} yet")
        return eng
