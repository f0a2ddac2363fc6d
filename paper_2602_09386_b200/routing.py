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

import warnings

from . import _lib
from ._lib import call, ptr
from .errors import ConfigError, NumericsError, ShapeError
from .linalg import Affine, FlopCounter, _dev_tensor
from .stacked import AffineStack

__all__ = ["RoutingBudget", "RouterBank", "BatchRouting", "RoutingDecision", "route_batch", "progressive_route",
           "naive_route_batch", "naive_sparse_route", "renormalized_weights", "compute_global_scores",
           "dense_routing", "stack_decisions"]


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


class RouterBank:
    """One affine router per task (d_in -> E) plus Stage-I pooling weights (routing.py:64-103).

    Reference form ``RouterBank(maps=[Affine, ...], task_weights=None)``; stacked form
    ``RouterBank(weight (T, E, d_in), bias (T, E), task_weights)``.  ``maps[t]`` are views of the
    stacked ``weight`` / ``bias`` the kernels consume."""

    def __init__(self, maps, task_weights=None, *stacked_task_weights):
        if isinstance(maps, torch.Tensor):            # stacked form
            self._stack = AffineStack(weight=maps, bias=task_weights)
            task_weights = stacked_task_weights[0] if stacked_task_weights else None
        else:
            maps = list(maps)
            if not maps:
                raise ConfigError("router bank needs at least one task router")
            e, d = maps[0].d_out, maps[0].d_in
            for i, m in enumerate(maps):
                if m.d_out != e or m.d_in != d:
                    raise ShapeError(f"router {i} has shape ({m.d_out},{m.d_in}), expected ({e},{d})")
            self._stack = AffineStack(items=maps)
        items = self._stack.items
        if not items:
            raise ConfigError("router bank needs at least one task router")
        T = len(items)
        tw = torch.ones(T, dtype=torch.float64) if task_weights is None else \
            torch.as_tensor(task_weights, dtype=torch.float64).detach().cpu()
        if tw.shape != (T,):
            raise ShapeError(f"expected {T} task weights, got shape {tuple(tw.shape)}")
        if bool((tw < 0).any()):
            raise ConfigError("task pooling weights must be non-negative")
        self.task_weights = tw

    @property
    def maps(self) -> list:
        return self._stack.items

    @property
    def weight(self) -> torch.Tensor:
        return self._stack.weight

    @weight.setter
    def weight(self, w):
        self._stack.weight = w

    @property
    def bias(self) -> torch.Tensor:
        return self._stack.bias

    @bias.setter
    def bias(self, b):
        self._stack.bias = b

    @property
    def num_tasks(self) -> int:
        return len(self._stack.items)

    @property
    def num_experts(self) -> int:
        return self._stack.items[0].d_out

    @property
    def d_in(self) -> int:
        return self._stack.items[0].d_in

    def logits(self, hidden, counter: FlopCounter | None = None) -> torch.Tensor:
        """Routing logits of a (B, d_in) batch, (T, B, E) (routing.py:101-103)."""
        h = _dev_tensor(hidden)
        if h.ndim != 2 or h.shape[1] != self.d_in:
            raise ShapeError(f"hidden has shape {tuple(h.shape)}, expected (B, {self.d_in})")
        w = self.weight.to(h.device)
        dt = torch.promote_types(h.dtype, w.dtype)
        z = torch.einsum("bd,ted->tbe", h.to(dt), w.to(dt)) + self.bias.to(h.device, dt)[:, None, :]
        if counter is not None:
            counter.add(self.num_tasks * h.shape[0] * self.d_in * self.num_experts)
        return z

    def __repr__(self) -> str:
        return f"RouterBank(num_tasks={self.num_tasks}, num_experts={self.num_experts}, d_in={self.d_in})"


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
                 z_strides=None, weights=None):
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
        self._weights = weights
        self._probs = self._unions = None

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


_warned_fp64 = False


def _as_logits(task_logits) -> torch.Tensor:
    """fp32 device logits.  The router kernels compare fp32 logits exactly; fp64 logits that are not
    fp32-representable are rounded first (selections are index-exact for the rounded values), which
    is reported once with a warning."""
    global _warned_fp64
    z = torch.as_tensor(task_logits)
    if not z.is_cuda:
        z = z.cuda()
    if z.ndim != 3:
        raise ShapeError(f"expected (T, B, E) logits, got shape {tuple(z.shape)}")
    z32 = z.to(torch.float32).contiguous()
    if z.dtype == torch.float64 and not _warned_fp64 and z.numel() and \
            not bool((z32.double() == z).logical_or(~torch.isfinite(z)).all()):
        _warned_fp64 = True
        warnings.warn("route_batch: float64 logits are rounded to float32 before selection; selections are "
                      "index-exact for the rounded logits", RuntimeWarning, stacklevel=3)
    return z32


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
    if bool((tw < 0).any()):
        raise NumericsError("task weights must be non-negative")
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


def naive_sparse_route(task_logits, k: int) -> RoutingDecision:
    """Independent per-task top-k for one instance, (T, E) logits (routing.py:312-331)."""
    z = torch.as_tensor(task_logits)
    if z.ndim != 2:
        raise ShapeError(f"expected (T, E) logits, got shape {tuple(z.shape)}")
    return naive_route_batch(z[:, None, :], k).instance(0)


def compute_global_scores(full_probs, task_weights=None) -> torch.Tensor:
    """s_e = sum_t w_t p_t[e] for one instance, with simplex validation (routing.py:214-232)."""
    p = _dev_tensor(full_probs, torch.float64)
    if p.ndim != 2:
        raise ShapeError(f"expected (T, E) probabilities, got shape {tuple(p.shape)}")
    w = torch.ones(p.shape[0], dtype=torch.float64, device=p.device) if task_weights is None else \
        _dev_tensor(task_weights, torch.float64)
    if w.shape != (p.shape[0],):
        raise ShapeError(f"expected {p.shape[0]} task weights, got shape {tuple(w.shape)}")
    if bool((w < 0).any()):
        raise NumericsError("task weights must be non-negative")
    if bool((p < 0).any()) or float((p.sum(dim=1) - 1.0).abs().max()) > 1e-6:
        raise NumericsError("each task's probabilities must lie on the simplex")
    return w @ p


def _from_arrays(shared, adaptive, active, unions, weights, full_probs, budget: RoutingBudget) -> BatchRouting:
    """A BatchRouting from reference-shaped arrays (dense_routing / stack_decisions): the compact
    device internals are derived, the statistics partials are whole-batch sums in chunk 0."""
    from .execution import _umask_from_unions
    w = _dev_tensor(weights, torch.float64)
    dev = w.device
    T, B, E = w.shape
    act = _dev_tensor(active, torch.int64)
    sh = _dev_tensor(shared, torch.int64).reshape(B, -1)
    ad = _dev_tensor(adaptive, torch.int64).reshape(T, B, -1)
    probs = _dev_tensor(full_probs, torch.float64)
    umask, _ = _umask_from_unions(unions, E, dev)
    usize = torch.tensor([int(torch.as_tensor(u).numel()) for u in unions], dtype=torch.int32, device=dev)
    rpw = call("smes_route_rows_per_warp", B)
    C = call("smes_route_num_chunks", B, rpw)
    chunk_union = torch.zeros(C, E, dtype=torch.int32, device=dev)
    call("smes_plan_counts", B, E, rpw, ptr(umask), ptr(chunk_union), ptr(torch.zeros(B, dtype=torch.int32, device=dev)),
         _stream())
    chunk_active = torch.zeros(C, E, dtype=torch.int32, device=dev)
    chunk_active[0] = torch.bincount(act.reshape(-1), minlength=E).to(torch.int32)
    chunk_mass = torch.zeros(C, E, dtype=torch.float64, device=dev)
    chunk_mass[0] = w.sum(dim=(0, 1))
    chunk_dmass = torch.zeros(C, E, dtype=torch.float64, device=dev)
    chunk_dmass[0] = probs.sum(dim=(0, 1))
    # logits whose softmax is full_probs (a zero probability becomes a very negative finite logit)
    z = torch.where(probs > 0, torch.log(probs.clamp_min(1e-300)), torch.full_like(probs, -1e30)).float()
    wsel = torch.gather(w, 2, act).float().contiguous()
    return BatchRouting(z.contiguous(), T, B, E, budget, torch.ones(T, dtype=torch.float64, device=dev),
                        sh.to(torch.int32).contiguous(), ad.to(torch.int32).contiguous(),
                        act.to(torch.int32).contiguous(), wsel, umask, usize, chunk_union, chunk_active, chunk_mass,
                        chunk_dmass, rpw, probs_in=probs.contiguous(), weights=w)


def dense_routing(full_probs) -> BatchRouting:
    """Every expert active for every task (routing.py:334-353): the dense baseline's routing view."""
    p = _dev_tensor(full_probs, torch.float64)
    if p.ndim != 3:
        raise ShapeError(f"expected (T, B, E) probabilities, got shape {tuple(p.shape)}")
    T, B, E = p.shape
    idx = torch.arange(E, device=p.device)
    return _from_arrays(idx.expand(B, E), torch.zeros(T, B, 0, dtype=torch.int64, device=p.device),
                        idx.expand(T, B, E), tuple(idx.cpu() for _ in range(B)), p, p, RoutingBudget(E, 0))


def stack_decisions(decisions) -> BatchRouting:
    """Per-instance decisions into batch-major arrays (routing.py:166-181)."""
    if not decisions:
        raise ShapeError("cannot stack an empty decision list")
    t = decisions[0].num_tasks
    d0 = decisions[0]
    budget = RoutingBudget(int(d0.shared.numel()), int(d0.adaptive[0].numel()) if t else 0)
    return _from_arrays(torch.stack([_dev_tensor(d.shared, torch.int64) for d in decisions]),
                        torch.stack([torch.stack([_dev_tensor(d.adaptive[i], torch.int64) for d in decisions])
                                     for i in range(t)]),
                        torch.stack([torch.stack([_dev_tensor(d.active[i], torch.int64) for d in decisions])
                                     for i in range(t)]),
                        tuple(torch.as_tensor(d.union).cpu() for d in decisions),
                        torch.stack([_dev_tensor(d.weights, torch.float64) for d in decisions], dim=1),
                        torch.stack([_dev_tensor(d.full_probs, torch.float64) for d in decisions], dim=1), budget)
