"""Expert selection -- drop-in for taskmoe/routing.py on CUDA tensors.

``route_batch`` runs the fused sm_100a progressive router (csrc/router.cu):
fp64 Stage I over the pooled dense softmax, exact Stage II on the masked
logits, renormalised weights over each task's active set, the per-instance
union as a bitmask, plus the per-chunk histograms the plan and the
load-balancing statistics consume.  The reference's dense / ragged views
(``weights`` (T,B,E), ``full_probs``, ``unions``) are materialised lazily.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _lib
from ._lib import call, ptr
from .errors import ConfigError, NumericsError, ShapeError

__all__ = ["RoutingBudget", "BatchRouting", "RoutingDecision", "route_batch", "progressive_route",
           "naive_route_batch", "renormalized_weights"]


@dataclass(frozen=True)
class RoutingBudget:
    """Per-task activation budget split into shared and task-adaptive counts (routing.py:36-61)."""

    k_shared: int
    k_adaptive: int

    @property
    def k_total(self) -> int:
        return self.k_shared + self.k_adaptive

    def validate(self, num_experts: int) -> None:
        if self.k_shared < 0 or self.k_adaptive < 0:
            raise ConfigError(f"budget counts must be non-negative, got shared={self.k_shared} "
                              f"adaptive={self.k_adaptive}")
        if self.k_total < 1:
            raise ConfigError("budget must activate at least one expert per task")
        if self.k_total > num_experts:
            raise ConfigError(f"budget k={self.k_total} exceeds expert count {num_experts}: "
                              f"stage-II would have only {num_experts - self.k_shared} candidates "
                              f"for {self.k_adaptive} adaptive picks")


@dataclass(frozen=True)
class RoutingDecision:
    """Expert selection for one instance (routing.py:106-128)."""
    shared: torch.Tensor
    adaptive: tuple
    active: tuple
    union: torch.Tensor
    weights: torch.Tensor
    full_probs: torch.Tensor

    @property
    def num_tasks(self):
        return self.weights.shape[0]

    @property
    def num_experts(self):
        return self.weights.shape[1]


class BatchRouting:
    """Batch routing decisions (routing.py:131-166), device resident.

    Compact internals: ``shared`` (B,K_s), ``adaptive`` (T,B,K_a), ``active``
    (T,B,K) int32, ``wsel`` (T,B,K) fp32 renormalised weights aligned with
    ``active``, ``umask`` (B,ceil(E/32)) union bitmask, ``usize`` (B,).
    """

    def __init__(self, z, T, B, E, budget, task_weights, shared, adaptive, active, wsel, umask, usize,
                 chunk_union, chunk_active, chunk_mass, chunk_dmass, rows_per_warp, probs_in=None,
                 z_strides=None):
        # z: fp32 logits; element (t, b, e) at z_flat[t*st + b*sb + e]
        self.z, self.T, self.B, self.E, self.budget = z, T, B, E, budget
        self.z_st, self.z_sb = z_strides if z_strides is not None else (B * E, E)
        self.task_weights = task_weights
        self.shared_i32, self.adaptive_i32, self.active_i32 = shared, adaptive, active
        self.wsel, self.umask, self.usize = wsel, umask, usize
        self.chunk_union, self.chunk_active, self.chunk_mass, self.chunk_dmass = (chunk_union, chunk_active,
                                                                                  chunk_mass, chunk_dmass)
        self.rows_per_warp = rows_per_warp
        self.probs_in = probs_in
        self._weights = self._probs = self._unions = None

    # -- reference fields
    @property
    def shared(self):
        return self.shared_i32.long()

    @property
    def adaptive(self):
        return self.adaptive_i32.long()

    @property
    def active(self):
        return self.active_i32.long()

    @property
    def weights(self) -> torch.Tensor:
        """(T,B,E) renormalised weights, exactly 0 off each task's active set (routing.py:203-211)."""
        if self._weights is None:
            w = torch.zeros(self.T, self.B, self.E, device=self.wsel.device, dtype=torch.float32)
            w.scatter_(2, self.active, self.wsel)
            self._weights = w
        return self._weights

    @property
    def full_probs(self) -> torch.Tensor:
        """(T,B,E) dense gate softmax (fp64), recomputed by the router kernel on demand."""
        if self._probs is None:
            if self.probs_in is not None:
                self._probs = self.probs_in
            else:
                self._probs = _dense_probs(self)
        return self._probs

    @property
    def unions(self) -> tuple:
        """Per-instance sorted distinct expert indices (routing.py:272).  Host sync."""
        if self._unions is None:
            bits = self.umask.cpu().numpy().view("uint32")
            import numpy as np
            out = []
            for b in range(self.B):
                idx = [j * 32 + i for j, w in enumerate(bits[b]) for i in range(32) if (int(w) >> i) & 1]
                out.append(torch.tensor(idx, dtype=torch.int64))
            self._unions = tuple(out)
        return self._unions

    @property
    def num_tasks(self):
        return self.T

    @property
    def batch_size(self):
        return self.B

    @property
    def num_experts(self):
        return self.E

    @property
    def k_total(self):
        return self.active_i32.shape[2]

    def instance(self, b: int) -> RoutingDecision:
        return RoutingDecision(shared=self.shared[b].clone(),
                               adaptive=tuple(self.adaptive[t, b].clone() for t in range(self.T)),
                               active=tuple(self.active[t, b].clone() for t in range(self.T)),
                               union=self.unions[b].clone(), weights=self.weights[:, b, :].clone(),
                               full_probs=self.full_probs[:, b, :].clone())


def _stream():
    return torch.cuda.current_stream().cuda_stream


def _alloc_routing(T, B, E, ks, ka, dev):
    rpw = call("smes_route_rows_per_warp", B)
    C = call("smes_route_num_chunks", B, rpw)
    i32 = torch.int32
    z = lambda *s, dt=torch.float32: torch.zeros(*s, dtype=dt, device=dev)
    return dict(shared=z(B, ks, dt=i32), adaptive=z(T, B, ka, dt=i32), active=z(T, B, ks + ka, dt=i32),
                wsel=z(T, B, ks + ka), umask=z(B, (E + 31) // 32, dt=i32), usize=z(B, dt=i32),
                chunk_union=z(C, E, dt=i32), chunk_active=z(C, E, dt=i32), chunk_mass=z(C, E, dt=torch.float64),
                chunk_dmass=z(C, E, dt=torch.float64), rows_per_warp=rpw)


def _launch_route(zt, T, B, E, ks, ka, tw, bufs, probs_in=None, probs_out=None, frozen=False, strides=None):
    flag = torch.zeros(1, dtype=torch.int32, device=zt.device)
    st, sb = strides if strides is not None else (B * E, E)
    call("smes_route_batch", ptr(zt), st, sb, ptr(probs_in), ptr(tw), T, B, E, ks, ka, bufs["rows_per_warp"],
         ptr(bufs["shared"]), ptr(bufs["adaptive"]), ptr(bufs["active"]), ptr(bufs["wsel"]), ptr(bufs["umask"]),
         ptr(bufs["usize"]), ptr(bufs["chunk_union"]), ptr(bufs["chunk_active"]), ptr(bufs["chunk_mass"]),
         ptr(bufs["chunk_dmass"]), ptr(probs_out), ptr(flag), int(frozen), _stream())
    return flag


def _as_logits(task_logits) -> torch.Tensor:
    z = torch.as_tensor(task_logits)
    if not z.is_cuda:
        z = z.cuda()
    if z.ndim != 3:
        raise ShapeError(f"expected (T, B, E) logits, got shape {tuple(z.shape)}")
    return z.to(torch.float32).contiguous()


def route_batch(task_logits, budget: RoutingBudget, task_weights=None, full_probs=None) -> BatchRouting:
    """Two-stage routing over a batch of logits (T, B, E) -- routing.py:235-281."""
    z = _as_logits(task_logits)
    T, B, E = z.shape
    budget.validate(E)
    dev = z.device
    tw = torch.ones(T, dtype=torch.float64, device=dev) if task_weights is None else \
        torch.as_tensor(task_weights, dtype=torch.float64).to(dev).contiguous()
    if tw.shape != (T,):
        raise ShapeError(f"expected {T} task weights, got shape {tuple(tw.shape)}")
    probs_in = None
    if full_probs is not None:
        probs_in = torch.as_tensor(full_probs, dtype=torch.float64).to(dev).contiguous()
        if probs_in.shape != z.shape:
            raise ShapeError(f"full_probs shape {tuple(probs_in.shape)} does not match logits {tuple(z.shape)}")
    if B == 0:
        raise ShapeError("route_batch of an empty batch")
    bufs = _alloc_routing(T, B, E, budget.k_shared, budget.k_adaptive, dev)
    flag = _launch_route(z, T, B, E, budget.k_shared, budget.k_adaptive, tw, bufs, probs_in=probs_in)
    if int(flag.item()):
        raise NumericsError("routing logits must be finite")
    rpw = bufs.pop("rows_per_warp")
    return BatchRouting(z, T, B, E, budget, tw, rows_per_warp=rpw, probs_in=probs_in, **bufs)


def frozen_routing(task_logits, frozen: BatchRouting) -> BatchRouting:
    """Selections of ``frozen`` reused, weights / probabilities / statistics recomputed from
    fresh logits (the frozen branch of forward_sparse, model.py:284-300)."""
    z = _as_logits(task_logits)
    T, B, E = z.shape
    ks, ka = frozen.budget.k_shared, frozen.budget.k_adaptive
    bufs = _alloc_routing(T, B, E, ks, ka, z.device)
    bufs["shared"].copy_(frozen.shared_i32)
    bufs["adaptive"].copy_(frozen.adaptive_i32)
    flag = _launch_route(z, T, B, E, ks, ka, frozen.task_weights, bufs, frozen=True)
    # (z here is the caller's fresh (T,B,E) logits, contiguous)
    if int(flag.item()):
        raise NumericsError("routing logits must be finite")
    rpw = bufs.pop("rows_per_warp")
    return BatchRouting(z, T, B, E, frozen.budget, frozen.task_weights, rows_per_warp=rpw, **bufs)


def _dense_probs(r: BatchRouting) -> torch.Tensor:
    probs = torch.empty(r.T, r.B, r.E, dtype=torch.float64, device=r.z.device)
    bufs = _alloc_routing(r.T, r.B, r.E, r.budget.k_shared, r.budget.k_adaptive, r.z.device)
    _launch_route(r.z, r.T, r.B, r.E, r.budget.k_shared, r.budget.k_adaptive, r.task_weights, bufs,
                  probs_out=probs, strides=(r.z_st, r.z_sb))
    return probs


def progressive_route(task_logits, budget: RoutingBudget, task_weights=None, full_probs=None) -> RoutingDecision:
    """Single-instance wrapper, logits (T, E) (routing.py:312-323)."""
    z = _as_logits(torch.as_tensor(task_logits)[:, None, :])
    p = None if full_probs is None else torch.as_tensor(full_probs)[:, None, :]
    return route_batch(z, budget, task_weights, p).instance(0)


def naive_route_batch(task_logits, k: int) -> BatchRouting:
    """Independent per-task top-k (routing.py:284-309) == progressive routing with K_s = 0
    (test_routing.py:136-145)."""
    z = _as_logits(task_logits)
    if not 1 <= k <= z.shape[2]:
        raise ConfigError(f"k={k} out of range for {z.shape[2]} experts")
    return route_batch(z, RoutingBudget(0, k))


def renormalized_weights(logits, active) -> torch.Tensor:
    """Softmax of logits[active] scattered back into a length-E vector (routing.py:190-200)."""
    lg = torch.as_tensor(logits, dtype=torch.float64)
    act = torch.as_tensor(active, dtype=torch.int64)
    sel = lg[act]
    e = torch.exp(sel - sel.max())
    out = torch.zeros_like(lg)
    out[act] = e / e.sum()
    return out
