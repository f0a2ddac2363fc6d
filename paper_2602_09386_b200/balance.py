"""Multi-gate load-balancing regularizer -- drop-in for taskmoe/balance.py.

The per-expert sums (selection counts, sparse and dense probability mass)
are produced by the router kernel as per-chunk partials and reduced in a
fixed order (csrc/plan.cu chunk_reduce, csrc/reduce.cu stats_finalize):
deterministic, no float atomics.  Under data parallelism the 3E raw sums are
the one all-reduce of the forward (paper_2602_09386_b200/dp.py).
"""
from __future__ import annotations

from dataclasses import dataclass

import torch

from ._lib import call, ptr
from .errors import StateError
from .routing import BatchRouting, _stream

__all__ = ["LoadStats", "SkewDiagnostics", "compute_load_stats", "lb_loss_gradient", "skew_diagnostics"]


@dataclass(frozen=True)
class LoadStats:
    """LoadStats (balance.py:28-44); arrays are device tensors."""
    frequency: torch.Tensor   # (E,) fp64
    mass: torch.Tensor        # (E,) fp64
    value: float
    counts: torch.Tensor      # (E,) int64
    batch_size: int
    num_tasks: int
    k_budget: int
    from_dense_probs: bool
    freq32: torch.Tensor | None = None


@dataclass(frozen=True)
class SkewDiagnostics:
    cv: float
    max_mean_ratio: float
    dead_fraction: float


def _raw_sums(routing: BatchRouting) -> torch.Tensor:
    E, C = routing.E, routing.chunk_union.shape[0]
    dev = routing.umask.device
    i32 = torch.int32
    raw = torch.zeros(3 * E, dtype=torch.float64, device=dev)
    # every scratch buffer stays referenced until the kernel is queued: a temporary freed inside the
    # argument list could be handed out again by the caching allocator for the next one
    scratch = [torch.zeros(C, E, dtype=i32, device=dev), torch.zeros(E, dtype=i32, device=dev),
               torch.zeros(E + 1, dtype=i32, device=dev), torch.zeros(E + 1, dtype=i32, device=dev),
               torch.zeros(3, dtype=i32, device=dev),
               torch.zeros(call("smes_plan_reduce_work_ints", C, E), dtype=i32, device=dev)]
    base, loads, seg_pad, seg_log, totals, work = scratch
    call("smes_plan_reduce", C, E, ptr(routing.chunk_union), ptr(routing.chunk_active), ptr(routing.chunk_mass),
         ptr(routing.chunk_dmass), ptr(base), ptr(loads), ptr(raw), ptr(seg_pad), ptr(seg_log), ptr(totals), ptr(work),
         None, _stream())
    return raw


def finalize_stats(raw: torch.Tensor, E: int, K: int, B: int, T: int, dense: bool):
    """Device LoadStats arrays from the raw sums: ``out`` = [frequency, mass, counts, value] (fp64)
    and the fp32 frequency the LB gradient kernel reads.  No host sync."""
    out = torch.zeros(3 * E + 1, dtype=torch.float64, device=raw.device)
    f32 = torch.zeros(E, dtype=torch.float32, device=raw.device)
    call("smes_stats_finalize", E, K, 0, float(B * T), int(dense), ptr(raw), ptr(out), ptr(f32), _stream())
    return out, f32


def load_stats(out: torch.Tensor, f32: torch.Tensor, value: float, E: int, K: int, B: int, T: int,
               dense: bool) -> LoadStats:
    return LoadStats(frequency=out[:E], mass=out[E:2 * E], value=value, counts=out[2 * E:3 * E].round().long(),
                     batch_size=B, num_tasks=T, k_budget=K, from_dense_probs=bool(dense), freq32=f32)


def stats_from_raw(raw: torch.Tensor, E: int, K: int, B: int, T: int, dense: bool) -> LoadStats:
    out, f32 = finalize_stats(raw, E, K, B, T, dense)
    return load_stats(out, f32, float(out[3 * E].item()), E, K, B, T, dense)


def compute_load_stats(routing: BatchRouting, dense_probs: bool = False) -> LoadStats:
    """f = counts/(B T), p = mass/(B T), L = (E/K) <f, p> (balance.py:54-80)."""
    B, T, E = routing.batch_size, routing.num_tasks, routing.num_experts
    if B == 0 or T == 0:
        raise StateError("load statistics are undefined for an empty batch")
    return stats_from_raw(_raw_sums(routing), E, routing.k_total, B, T, dense_probs)


def lb_loss_gradient(stats: LoadStats, routing: BatchRouting) -> torch.Tensor:
    """dL/dz = coef P (f - <P, f>), coef = E/(K B T), f detached (balance.py:83-99).  (T, B, E) fp32."""
    B, T, E = routing.batch_size, routing.num_tasks, routing.num_experts
    if (stats.batch_size, stats.num_tasks) != (B, T) or stats.frequency.shape != (E,):
        raise StateError("load stats were computed for a different batch")
    if stats.k_budget != routing.k_total:
        raise StateError("load stats were computed under a different budget")
    coef = E / (stats.k_budget * B * T)
    out = torch.empty(T, B, E, dtype=torch.float32, device=routing.z.device)
    f32 = stats.freq32 if stats.freq32 is not None else stats.frequency.float()
    call("smes_lb_grad", T, B, E, routing.k_total, ptr(routing.active_i32), ptr(routing.wsel), ptr(routing.z),
         routing.z_st, routing.z_sb, ptr(f32), coef, int(stats.from_dense_probs), ptr(out), _stream())
    return out


def skew_diagnostics(stats: LoadStats) -> SkewDiagnostics:
    """balance.py:102-112 (reporting only)."""
    c = stats.counts.double()
    mean = float(c.mean())
    if mean == 0:
        return SkewDiagnostics(0.0, 0.0, 1.0)
    return SkewDiagnostics(float(c.std(unbiased=False) / mean), float(c.max() / mean), float((c == 0).double().mean()))
