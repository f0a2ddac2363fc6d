"""Deduplicated expert execution -- drop-in for taskmoe/execution.py and experts.py.

``build_execution_plan`` runs the device counting sort (csrc/plan.cu):
expert-major, instance-ascending packing identical to the reference's
lexsort, with every expert segment padded to 128 rows in the physical
layout the tcgen05 GEMMs consume.  The reference's logical views
(``segment_offsets``, ``gather_instances``, ``row_keys``...) are derived on
demand.  ``grouped_gemm`` / ``reconstruct_task_reps`` accept and return the
reference's logical (N_act, d) packed layout.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch

from ._lib import call, ptr
from .errors import ConfigError, ShapeError, StateError
from .experts import ExpertPool, init_expert_pool
from .linalg import FlopCounter
from .routing import BatchRouting, _stream

__all__ = ["ExpertPool", "init_expert_pool", "ExecutionPlan", "build_execution_plan", "grouped_gemm",
           "reconstruct_task_reps", "FlopCounter"]

ACT = {"identity": 0, "relu": 1}


def _round(x, m):
    return (x + m - 1) // m * m


class ExecutionPlan:
    """Packing layout for one batch (execution.py:32-82), device resident."""

    def __init__(self, num_experts, batch_size, umax, rows_cap, seg_pad, seg_log, loads, totals, row_of,
                 gather_inst, gather_exp, stats_raw, usize):
        self.num_experts, self.batch_size = num_experts, batch_size
        self.umax, self.rows_cap = umax, rows_cap
        self.seg_pad, self.seg_log, self.loads_i32, self.totals = seg_pad, seg_log, loads, totals
        self.row_of, self.gather_inst, self.gather_exp = row_of, gather_inst, gather_exp
        self.stats_raw, self.usize = stats_raw, usize
        self._phys = None

    # -- reference fields (logical layout)
    @property
    def loads(self):
        return self.loads_i32.long()

    @property
    def total_rows(self) -> int:
        return int(self.totals[2].item())

    @property
    def segment_offsets(self):
        return self.seg_log.long()

    @property
    def physical_rows(self) -> torch.Tensor:
        """Logical packed row -> physical (padded) row."""
        if self._phys is None:
            end = int(self.totals[1].item())
            valid = self.gather_inst[:end] >= 0
            self._phys = torch.nonzero(valid).flatten()
        return self._phys

    @property
    def gather_instances(self):
        return self.gather_inst[self.physical_rows].long()

    @property
    def gather_experts(self):
        return self.gather_exp[self.physical_rows].long()

    @property
    def row_keys(self):
        return self.gather_experts * self.batch_size + self.gather_instances

    def row_lookup(self, instances, experts) -> torch.Tensor:
        """Vectorised back-map (execution.py:67-82); raises StateError on a miss."""
        keys = torch.as_tensor(experts, dtype=torch.int64, device=self.seg_pad.device) * self.batch_size + \
            torch.as_tensor(instances, dtype=torch.int64, device=self.seg_pad.device)
        rk = self.row_keys
        if rk.numel() == 0:
            if keys.numel():
                raise StateError("plan holds no packed rows but lookups were requested")
            return torch.zeros_like(keys)
        pos = torch.searchsorted(rk, keys)
        ok = (pos < rk.numel()) & (rk[pos.clamp(max=rk.numel() - 1)] == keys)
        if not bool(ok.all()):
            raise StateError("plan and routing decision are inconsistent")
        return pos

    def row_index(self, instance: int, expert: int) -> int:
        return int(self.row_lookup(torch.tensor([instance]), torch.tensor([expert]))[0])


def _umask_from_unions(unions, num_experts, dev):
    B = len(unions)
    EW = (num_experts + 31) // 32
    words = torch.zeros(B, EW, dtype=torch.int64)
    umax = 0
    for b, u in enumerate(unions):
        u = torch.as_tensor(u, dtype=torch.int64).flatten().cpu()
        if u.numel() and (int(u.min()) < 0 or int(u.max()) >= num_experts):
            raise ShapeError(f"instance {b} union contains expert index outside [0, {num_experts})")
        if torch.unique(u).numel() != u.numel():
            raise ShapeError(f"instance {b} union contains duplicate expert indices")
        umax = max(umax, u.numel())
        for e in u.tolist():
            words[b, e // 32] |= 1 << (e % 32)
    words = torch.where(words >= 2 ** 31, words - 2 ** 32, words)
    return words.to(torch.int32).to(dev), umax


def build_execution_plan(unions, num_experts: int, device=None) -> ExecutionPlan:
    """Traffic calculation plus gather ordering (execution.py:85-123).  ``unions`` is a
    BatchRouting (device fast path) or a sequence of per-instance index arrays."""
    E = int(num_experts)
    if isinstance(unions, BatchRouting):
        r = unions
        dev = r.umask.device
        B, umask, usize = r.B, r.umask, r.usize
        umax = min(E, r.budget.k_shared + r.T * r.budget.k_adaptive)
        rpw = r.rows_per_warp
        chunk_union, chunk_active, chunk_mass, chunk_dmass = r.chunk_union, r.chunk_active, r.chunk_mass, \
            r.chunk_dmass
    else:
        dev = torch.device(device or "cuda")
        B = len(unions)
        umask, umax = _umask_from_unions(unions, E, dev)
        umax = max(umax, 1)
        rpw = call("smes_route_rows_per_warp", max(B, 1))
        C = call("smes_route_num_chunks", max(B, 1), rpw)
        chunk_union = torch.zeros(C, E, dtype=torch.int32, device=dev)
        usize = torch.zeros(max(B, 1), dtype=torch.int32, device=dev)
        chunk_active = torch.zeros(C, E, dtype=torch.int32, device=dev)
        chunk_mass = torch.zeros(C, E, dtype=torch.float64, device=dev)
        chunk_dmass = torch.zeros_like(chunk_mass)
        if B:
            call("smes_plan_counts", B, E, rpw, ptr(umask), ptr(chunk_union), ptr(usize), _stream())
    C = chunk_union.shape[0]
    i32 = torch.int32
    rows_cap = _round(max(B, 1) * umax + E * 127, 128)
    chunk_base = torch.zeros(C, E, dtype=i32, device=dev)
    loads = torch.zeros(E, dtype=i32, device=dev)
    stats_raw = torch.zeros(3 * E, dtype=torch.float64, device=dev)
    seg_pad = torch.zeros(E + 1, dtype=i32, device=dev)
    seg_log = torch.zeros(E + 1, dtype=i32, device=dev)
    totals = torch.zeros(3, dtype=i32, device=dev)
    ticket = torch.zeros(call("smes_plan_reduce_work_ints", C, E), dtype=i32, device=dev)
    row_of = torch.zeros(max(B, 1), umax, dtype=i32, device=dev)
    gather_inst = torch.full((rows_cap,), -1, dtype=i32, device=dev)
    gather_exp = torch.zeros(rows_cap, dtype=i32, device=dev)
    if B:
        s = _stream()
        call("smes_plan_reduce", C, E, ptr(chunk_union), ptr(chunk_active), ptr(chunk_mass), ptr(chunk_dmass),
             ptr(chunk_base), ptr(loads), ptr(stats_raw), ptr(seg_pad), ptr(seg_log), ptr(totals), ptr(ticket), None, s)
        call("smes_plan_scatter", B, E, 8, rpw, ptr(umask), ptr(chunk_base), ptr(seg_pad), ptr(loads), None, 8,
             None, 8, ptr(row_of), umax, ptr(gather_inst), ptr(gather_exp), None, 8, 8, s)
    return ExecutionPlan(E, B, umax, rows_cap, seg_pad, seg_log, loads, totals, row_of, gather_inst, gather_exp,
                         stats_raw, usize)


def _to_physical(x_logical: torch.Tensor, plan: ExecutionPlan, width: int) -> torch.Tensor:
    xp = torch.zeros(plan.rows_cap, width, dtype=torch.bfloat16, device=plan.seg_pad.device)
    if x_logical.shape[0]:
        xp[plan.physical_rows] = x_logical.to(device=xp.device, dtype=torch.bfloat16)
    return xp


def _gemm_fwd(xp, pool: ExpertPool, plan: ExecutionPlan, act: int) -> torch.Tensor:
    w = pool.weight.to(device=xp.device, dtype=torch.bfloat16).contiguous()
    b = pool.bias.to(device=xp.device, dtype=torch.float32).contiguous()
    out = torch.zeros(plan.rows_cap, pool.d_out, dtype=torch.bfloat16, device=xp.device)
    call("smes_gemm_ragged_m", ptr(xp), pool.d_in, plan.rows_cap, ptr(w), pool.num_experts, pool.d_out, pool.d_in,
         0, ptr(plan.seg_pad), ptr(b), act, None, None, plan.rows_cap, ptr(out), pool.d_out, 0, plan.rows_cap,
         _stream())
    return out


def grouped_gemm(packed_in, pool: ExpertPool, plan: ExecutionPlan, counter: FlopCounter | None = None,
                 return_preactivation: bool = False):
    """act(x[seg_e] W_e^T + b_e) per expert segment (execution.py:126-158), on the tcgen05
    grouped GEMM.  Logical (N_act, d) in and out; bf16 operands, fp32 accumulation."""
    x = torch.as_tensor(packed_in)
    n = plan.total_rows
    if x.ndim != 2 or x.shape[0] != n:
        raise ShapeError(f"packed input has shape {tuple(x.shape)}, plan expects {n} rows")
    if x.shape[0] and x.shape[1] != pool.d_in:
        raise ShapeError(f"packed input width {x.shape[1]} != expert d_in {pool.d_in}")
    if pool.num_experts != plan.num_experts:
        raise ShapeError(f"pool has {pool.num_experts} experts, plan was built for {plan.num_experts}")
    xp = _to_physical(x, plan, pool.d_in)
    rows = plan.physical_rows
    out = _gemm_fwd(xp, pool, plan, ACT[pool.nonlinearity])[rows].float()
    if counter is not None:
        counter.add(n * pool.d_in * pool.d_out)
    if return_preactivation:
        pre = out if pool.nonlinearity == "identity" else _gemm_fwd(xp, pool, plan, 0)[rows].float()
        return out, pre
    return out


def reconstruct_task_reps(packed_out, plan: ExecutionPlan, routing: BatchRouting) -> torch.Tensor:
    """reps[t, b] = sum_k w[t,b,K_t[b,k]] O[pi(b, K_t[b,k])] (execution.py:161-191)."""
    o = torch.as_tensor(packed_out)
    if o.ndim != 2 or o.shape[0] != plan.total_rows:
        raise ShapeError(f"packed output has shape {tuple(o.shape)}, plan expects {plan.total_rows} rows")
    if routing.batch_size != plan.batch_size:
        raise ShapeError(f"routing covers {routing.batch_size} instances, plan {plan.batch_size}")
    T, B, E, K = routing.T, routing.B, routing.E, routing.k_total
    d_out = o.shape[1]
    op = _to_physical(o, plan, d_out)
    reps = torch.zeros(T, B, d_out, dtype=torch.bfloat16, device=op.device)
    grid = call("smes_combine_grid", B, T, d_out)
    call("smes_combine_fwd", T, B, E, K, d_out, plan.umax, ptr(routing.umask), ptr(routing.usize),
         ptr(plan.row_of), ptr(routing.active_i32), ptr(routing.wsel), ptr(op), d_out, None, None, None, 0,
         ptr(reps), None, None, None, None, None, grid, _stream())
    return reps.float()
