"""Expert parallelism (BASELINE config c5): experts sharded E/n per GPU, batch sharded B/n.

The reference has one process holding every expert (model.py:267-324, training.py:119-226).
Here rank r owns experts [r*E_l, (r+1)*E_l) and routes its own B_l instances; routers and task
heads are replicated.  The step is expressed in phases so the same code drives one rank per
process (NCCL or the peer-memory transport) and n virtual ranks on one GPU (tests):

  f1  source: router GEMM -> route -> plan over all E experts (source packing, statistics)
              -> pack h[b] once per owner whose experts U_b meets (+ the owner's mask words)
      [all-reduce LB statistics; all-to-all h / masks / per-expert loads]
  f2  owner : plan over the received instances (local experts) -> expert shard forward
              (folded heads: only P, T floats per row, goes back) -> pack P per source
      [all-to-all P]
  f3  source: place P into its plan order -> LoadStats (global B*T) -> fused training
              combine (loss, dz, row coefficients C) -> pack C per owner
      [all-to-all C]
  b1  owner : place C -> expert shard backward (local expert grads, dW_head share, dX)
              -> un-permute dX to per-instance sums over the local experts
      [all-to-all dh]
  b2  source: router dgrad/wgrad -> d_hidden = dh_router + sum over owners
      [all-reduce of the replicated gradients (routers, heads) and the loss partials]

Semantics: the objective is the global-batch mean (lambda/B_global, LB coefficient with
B_global, statistics over B_global*T), so expert gradients are exact at their owner and the
replicated gradients are sums over ranks; parity is defined against the single-process oracle
on the concatenated batch.  Every buffer is fixed-slot, so no step reads a count on the host.
"""
from __future__ import annotations

import torch

from . import _lib
from ._lib import call, ptr, tcall
from .errors import ConfigError, ShapeError, StateError
from .engine import router_wgrad_splits
from .experts import ExpertShard, refresh_into

U32 = torch.int32   # mask words travel as int32 storage


def _round(x, m):
    return (x + m - 1) // m * m


class EPRank:
    """Buffers and phases of one expert-parallel rank."""

    def __init__(self, params, num_experts: int, rank: int, world: int, batch_size: int, k_shared: int,
                 k_adaptive: int, device=None, capacity_factor: float = 2.0, fuse_mlp: bool = True):
        self.dev = torch.device(device or "cuda")
        p = params
        T, d = p.router_w.shape[0], p.router_w.shape[2]
        E, n, B = int(num_experts), int(world), int(batch_size)
        if p.router_w.shape[1] != E:
            raise ShapeError(f"router bank has {p.router_w.shape[1]} experts, expected {E}")
        if E % n or (E // n) % 32:
            raise ConfigError(f"expert parallelism needs E/n to be a multiple of 32 (E={E}, n={n})")
        El = E // n
        if p.layers[0].weight.shape[0] != El:
            raise ShapeError(f"rank {rank} holds {p.layers[0].weight.shape[0]} experts, expected {El}")
        ks, ka = int(k_shared), int(k_adaptive)
        K = ks + ka
        if K < 1 or K > E:
            raise ConfigError(f"budget k={K} outside [1, {E}]")
        self.p, self.T, self.E, self.El, self.n, self.rank, self.B, self.d = p, T, E, El, n, rank, B, d
        self.ks, self.ka, self.K = ks, ka, K
        self.EW = (E + 31) // 32
        self.wpr = El // 32
        self.umax = min(E, ks + T * ka)
        self.d_out = p.layers[-1].d_out
        self.B_pad = _round(B, 128)
        dev, i32, f32, f64, bf = self.dev, torch.int32, torch.float32, torch.float64, torch.bfloat16
        z = lambda *s, dt=f32: torch.zeros(*s, dtype=dt, device=dev)
        # ---------------- source side (routing over all E experts)
        self.rpw = call("smes_route_rows_per_warp", B)
        self.C = call("smes_route_num_chunks", B, self.rpw)
        self.grid = call("smes_combine_grid", B, T, self.d_out)
        self.rows_src = _round(B * self.umax + E * 127, 128)
        self.ldh = d + 64
        self.h_full = z(B, self.ldh, dt=bf)
        self.h_full[:, d] = 1.0
        self.h = self.h_full[:, :d]
        self.z = z(B, T * E)
        self.shared = z(B, ks, dt=i32)
        self.adaptive = z(T, B, ka, dt=i32)
        self.active = z(T, B, K, dt=i32)
        self.wsel = z(T, B, K)
        self.umask = z(B, self.EW, dt=U32)
        self.usize = z(B, dt=i32)
        self.chunk_union = z(self.C, E, dt=i32)
        self.chunk_active = z(self.C, E, dt=i32)
        self.chunk_mass = z(self.C, E, dt=f64)
        self.chunk_dmass = z(self.C, E, dt=f64)
        self.chunk_base = z(self.C, E, dt=i32)
        self.loads = z(E, dt=i32)
        self.stats_raw = z(3 * E, dt=f64)
        self.seg_pad = z(E + 1, dt=i32)
        self.seg_log = z(E + 1, dt=i32)
        self.totals = z(3, dt=i32)
        self.ticket = z(call("smes_plan_reduce_work_ints", self.C, E), dt=i32)
        self.flag = z(1, dt=i32)            # non-finite logits (route)
        self.cap_flag = z(1, dt=i32)        # owner plan exceeded the shard's row capacity
        self.seg_half = z(2 * E + 1, dt=i32)
        self.row_of = z(B, self.umax, dt=i32)
        self.gather_inst = z(self.rows_src, dt=i32)
        self.gather_exp = z(self.rows_src, dt=i32)
        self.ldp = _round(T, 8)
        self.ldc = _round(T, 16)
        self.P_src = z(self.rows_src, self.ldp)
        self.C_src = z(self.rows_src, self.ldc, dt=bf)
        self.labels = z(T, B)
        self.logits = z(T, B)
        self.preds = z(T, B)
        self.loss_part = z(self.grid, dt=f64)
        self.loss_out = z(3, dt=f64)
        self.stats_out = z(3 * E + 1, dt=f64)
        self.freq32 = z(E)
        self.dz = z(self.B_pad, T * E, dt=bf)
        self.part_db = z(self.grid, T)
        self.seg_router = torch.tensor([0, self.B_pad], dtype=i32, device=dev)
        self.rw_splits = router_wgrad_splits(self.B_pad, T * E, d, dev)
        edges = [min(self.B_pad, (self.B_pad // self.rw_splits) // 128 * 128 * i) for i in range(self.rw_splits)]
        self.seg_router_split = torch.tensor(edges + [self.B_pad], dtype=i32, device=dev)
        self.rw_part = z(self.rw_splits, T * E, d)
        self.rb_part = z(self.rw_splits, T * E)
        self.dh_router = z(B, d)
        self.d_hidden = z(B, d)
        # replicated gradients (routers, heads) in one flat buffer: a single all-reduce
        shapes = [(T * E, d), (T * E,), (T, self.d_out), (T,)]
        sizes = [int(torch.Size(s).numel()) for s in shapes]
        self.rep_grad = z(sum(sizes) + self.grid)        # + the loss partials, reduced together
        views, off = [], 0
        for s_, m in zip(shapes, sizes):
            views.append(self.rep_grad[off:off + m].view(s_))
            off += m
        self.g_router_w, self.g_router_b, self.g_head_w, self.g_head_b = views
        self.loss_part_f32 = self.rep_grad[off:]
        # ---------------- dispatch / return buffers (fixed slots per peer)
        self.idx = z(n, B, dt=i32)
        self.pos = z(n, B, dt=i32)
        self.cnt = z(n, dt=i32)
        self.mask_send = z(n, B, self.wpr, dt=U32)
        self.h_send = z(n, B, d, dt=bf)
        self.slot_rows = B * min(El, self.umax)          # rows one source can own at one owner
        self.P_recv = z(n, self.slot_rows, self.ldp)
        self.C_send = z(n, self.slot_rows, self.ldc, dt=bf)
        self.tab_src = z(n * El, 3, dt=i32)
        self.dh_recv = z(n, B, d)
        # ---------------- owner side (local experts over the n*B received instances)
        Br = n * B
        self.Br = Br
        self.umax_l = min(El, ks + T * ka)
        worst = Br * self.umax_l
        cap = int(capacity_factor * B * self.umax) if capacity_factor else worst
        self.rows_own = _round(min(worst, cap) + El * 127, 128)
        self.h_recv = z(n, B, d, dt=bf)
        self.umask_recv = z(n, B, self.wpr, dt=U32)
        self.cnt_recv = z(n, El, dt=i32)
        self.rpw_o = call("smes_route_rows_per_warp", Br)
        self.C_o = call("smes_route_num_chunks", Br, self.rpw_o)
        self.usize_o = z(Br, dt=i32)
        self.chunk_union_o = z(self.C_o, El, dt=i32)
        self.chunk_zero_i = z(self.C_o, El, dt=i32)
        self.chunk_zero_d = z(self.C_o, El, dt=f64)
        self.chunk_base_o = z(self.C_o, El, dt=i32)
        self.loads_o = z(El, dt=i32)
        self.stats_o = z(3 * El, dt=f64)
        self.seg_pad_o = z(El + 1, dt=i32)
        self.seg_log_o = z(El + 1, dt=i32)
        self.totals_o = z(3, dt=i32)
        self.ticket_o = z(call("smes_plan_reduce_work_ints", self.C_o, El), dt=i32)
        self.seg_half_o = z(2 * El + 1, dt=i32)
        self.row_of_o = z(Br, self.umax_l, dt=i32)
        self.shard = ExpertShard(p.layers, T, self.head_w32(), self.rows_own, dev, fuse_mlp=fuse_mlp)
        self.gather_inst_o = z(self.shard.R, dt=i32)
        self.gather_exp_o = z(self.shard.R, dt=i32)
        self.P_send = z(n, self.slot_rows, self.ldp)
        self.C_recv = z(n, self.slot_rows, self.ldc, dt=bf)
        self.tab_own = z(n * El, 3, dt=i32)
        self.dh_own = z(n, B, d)
        # fused transport: device tables of every rank's receive buffers (set by the transport);
        # the pack / gather kernels then store straight into the peers' slots
        self.peers = None
        self.refresh_weights()

    def head_w32(self):
        if not hasattr(self, "_head_w"):
            self._head_w = self.p.head_w.detach().to(self.dev, torch.float32).contiguous()
        return self._head_w

    def refresh_weights(self):
        """Copy the master parameters into the kernel operands (allocated once, then ``copy_``:
        stable addresses for graph replays)."""
        p, T, E, d = self.p, self.T, self.E, self.d
        tw = p.task_weights if p.task_weights is not None else torch.ones(T)
        lam = p.task_loss_weights if p.task_loss_weights is not None else torch.ones(T)
        refresh_into(self, "wr_bf", p.router_w.detach().reshape(T * E, d), torch.bfloat16)
        refresh_into(self, "br", p.router_b.detach().reshape(T * E), torch.float32)
        self.head_w = self.head_w32()
        self.head_w.copy_(p.head_w.detach())
        refresh_into(self, "head_b", p.head_b.detach(), torch.float32)
        refresh_into(self, "tw", torch.as_tensor(tw).detach(), torch.float64)
        refresh_into(self, "lam", torch.as_tensor(lam).detach(), torch.float32)
        self.beta = float(p.lb_strength)
        self.shard.refresh_weights()

    def set_inputs(self, h: torch.Tensor, labels: torch.Tensor):
        if h.shape != (self.B, self.d) or labels.shape != (self.T, self.B):
            raise ShapeError(f"rank {self.rank}: inputs {tuple(h.shape)} / {tuple(labels.shape)}")
        self.h.copy_(h, non_blocking=True)
        self.labels.copy_(labels, non_blocking=True)

    # ------------------------------------------------------------------ phases
    def _s(self):
        return torch.cuda.current_stream(self.dev).cuda_stream

    def f1(self):
        """Route + source plan + LB statistics + dispatch pack."""
        s, T, E, B, d = self._s(), self.T, self.E, self.B, self.d
        tcall("router_fwd", "smes_gemm_ragged_m", ptr(self.h), self.ldh, B, ptr(self.wr_bf), 1, T * E, d, 0, ptr(self.seg_router),
             ptr(self.br), 0, None, None, 0, ptr(self.z), T * E, 1, B, s)
        tcall("route", "smes_route_batch", ptr(self.z), E, T * E, None, ptr(self.tw), T, B, E, self.ks, self.ka, self.rpw,
             ptr(self.shared), ptr(self.adaptive), ptr(self.active), ptr(self.wsel), ptr(self.umask), ptr(self.usize),
             # no dense-mass statistics (EP trains with the sparse LB reading): the router's fast Stage I
             ptr(self.chunk_union), ptr(self.chunk_active), ptr(self.chunk_mass), None, None,
             ptr(self.flag), 0, s)
        tcall("plan_reduce", "smes_plan_reduce", self.C, E, ptr(self.chunk_union), ptr(self.chunk_active), ptr(self.chunk_mass),
             ptr(self.chunk_dmass), ptr(self.chunk_base), ptr(self.loads), ptr(self.stats_raw), ptr(self.seg_pad),
             ptr(self.seg_log), ptr(self.totals), ptr(self.ticket), ptr(self.seg_half), s)
        # the source plan only places rows (row_of, gather arrays) and zeroes C's pad rows; X is not built
        tcall("plan_scatter", "smes_plan_scatter", B, E, d, self.rpw, ptr(self.umask), ptr(self.chunk_base), ptr(self.seg_pad),
             ptr(self.loads), None, self.ldh, None, d, ptr(self.row_of), self.umax, ptr(self.gather_inst),
             ptr(self.gather_exp), ptr(self.C_src), self.ldc, self.ldc, s)
        if self.peers is not None:
            pr = self.peers
            tcall("ep_pack", "smes_ep_pack_put", B, self.EW, ptr(self.umask), self.n, self.wpr, ptr(self.h), self.ldh, d,
                  self.rank, ptr(self.idx), ptr(self.pos), ptr(self.cnt), ptr(pr["mask"]), ptr(pr["h"]), s)
            tcall("ep_pack", "smes_ep_put_slots", self.n, self.rank, ptr(self.loads), self.El * 4, self.El * 4, None,
                  ptr(pr["cnt"]), s)
            return
        tcall("ep_pack", "smes_ep_pack", B, self.EW, ptr(self.umask), self.n, self.wpr, ptr(self.h), self.ldh, d, ptr(self.idx),
             ptr(self.pos), ptr(self.cnt), ptr(self.mask_send), ptr(self.h_send), s)

    def f2(self):
        """Owner: plan over the received instances -> shard forward -> P per source."""
        s, El, d, Br = self._s(), self.El, self.d, self.Br
        sh = self.shard
        umask = self.umask_recv.view(Br, self.wpr)
        tcall("owner_plan", "smes_plan_counts", Br, El, self.rpw_o, ptr(umask), ptr(self.chunk_union_o), ptr(self.usize_o), s)
        tcall("owner_plan", "smes_plan_reduce", self.C_o, El, ptr(self.chunk_union_o), ptr(self.chunk_zero_i), ptr(self.chunk_zero_d),
             ptr(self.chunk_zero_d), ptr(self.chunk_base_o), ptr(self.loads_o), ptr(self.stats_o), ptr(self.seg_pad_o),
             ptr(self.seg_log_o), ptr(self.totals_o), ptr(self.ticket_o), ptr(self.seg_half_o), s)
        tcall("owner_plan", "smes_ep_capacity_guard", El, sh.R, ptr(self.totals_o), ptr(self.seg_pad_o), ptr(self.loads_o),
             ptr(umask), Br * self.wpr, ptr(self.usize_o), Br, ptr(self.cap_flag), s)
        tcall("owner_scatter", "smes_plan_scatter", Br, El, d, self.rpw_o, ptr(umask), ptr(self.chunk_base_o), ptr(self.seg_pad_o),
             ptr(self.loads_o), ptr(self.h_recv), d, ptr(sh.X), sh.ld_in[0], ptr(self.row_of_o), self.umax_l,
             ptr(self.gather_inst_o), ptr(self.gather_exp_o), ptr(sh.Cm), sh.ldc, sh.ldc, s)
        sh.forward(s, self.seg_pad_o, self.totals_o)
        tcall("ep_segments", "smes_ep_segments", 0, self.n, El, ptr(self.cnt_recv), ptr(self.seg_pad_o), self.slot_rows,
             ptr(self.tab_own), s)
        if self.peers is not None:
            tcall("ep_copy_rows", "smes_ep_copy_rows_put", self.n * El, ptr(self.tab_own), El, self.slot_rows,
                  self.rank, ptr(sh.P), sh.ldp * 4, ptr(self.peers["P"]), self.ldp * 4, self.ldp * 4, s)
            return
        tcall("ep_copy_rows", "smes_ep_copy_rows", self.n * El, ptr(self.tab_own), 0, ptr(sh.P), sh.ldp * 4, ptr(self.P_send),
             self.ldp * 4, self.ldp * 4, s)

    def f3(self):
        """Source: P into plan order -> statistics -> training combine -> C per owner."""
        s, T, E, B, K = self._s(), self.T, self.E, self.B, self.K
        Bg = B * self.n
        tcall("ep_segments", "smes_ep_segments", 1, self.n, self.El, ptr(self.loads), ptr(self.seg_pad), self.slot_rows,
             ptr(self.tab_src), s)
        tcall("ep_copy_rows", "smes_ep_copy_rows", self.n * self.El, ptr(self.tab_src), 1, ptr(self.P_recv), self.ldp * 4,
             ptr(self.P_src), self.ldp * 4, self.ldp * 4, s)
        call("smes_stats_finalize", E, K, 0, float(Bg * T), 0, ptr(self.stats_raw), ptr(self.stats_out), ptr(self.freq32),
             s)
        lb_coef = self.beta * E / (K * Bg * T)
        tcall("combine_train", "smes_combine_train", T, B, E, K, self.umax, ptr(self.umask), ptr(self.usize), ptr(self.row_of),
             ptr(self.active), ptr(self.wsel), ptr(self.head_b), ptr(self.P_src), self.ldp, ptr(self.logits),
             ptr(self.preds), ptr(self.labels), ptr(self.lam), ptr(self.loss_part), 1.0 / Bg, ptr(self.C_src),
             self.ldc, ptr(self.dz), ptr(self.freq32), lb_coef, ptr(self.part_db), None, None, self.grid, s)
        if self.peers is not None:
            tcall("ep_copy_rows", "smes_ep_copy_rows_put", self.n * self.El, ptr(self.tab_src), self.El,
                  self.slot_rows, self.rank, ptr(self.C_src), self.ldc * 2, ptr(self.peers["C"]), self.ldc * 2,
                  self.ldc * 2, s)
            return
        tcall("ep_copy_rows", "smes_ep_copy_rows", self.n * self.El, ptr(self.tab_src), 0, ptr(self.C_src), self.ldc * 2,
             ptr(self.C_send), self.ldc * 2, self.ldc * 2, s)

    def b1(self):
        """Owner: C into its plan order -> shard backward -> per-instance dX sums."""
        s, d, Br = self._s(), self.d, self.Br
        sh = self.shard
        tcall("ep_copy_rows", "smes_ep_copy_rows", self.n * self.El, ptr(self.tab_own), 1, ptr(self.C_recv), self.ldc * 2, ptr(sh.Cm),
             sh.ldc * 2, self.ldc * 2, s)
        sh.backward(s, self.seg_pad_o, self.totals_o)
        tcall("unpermute", "smes_unpermute", Br, d, ptr(self.usize_o), ptr(self.row_of_o), self.umax_l, ptr(sh.dX), d, None,
             ptr(self.dh_own), s)

    def b2(self):
        """Source: router backward and d_hidden; stage the replicated gradients for the all-reduce."""
        s, T, E, B, d = self._s(), self.T, self.E, self.B, self.d
        tcall("router_dgrad", "smes_gemm_ragged_m", ptr(self.dz), T * E, self.B_pad, ptr(self.wr_bf), 1, d, T * E, 1,
             ptr(self.seg_router), None, 0, None, None, 0, ptr(self.dh_router), d, 1, B, s)
        tcall("router_wgrad", "smes_gemm_ragged_k", ptr(self.dz), T * E, ptr(self.h), self.ldh, B, self.rw_splits, T * E, d,
             ptr(self.seg_router_split), ptr(self.rw_part), ptr(self.rb_part), s)
        call("smes_part_reduce", ptr(self.rw_part), self.rw_splits, T * E * d, ptr(self.g_router_w), s)
        call("smes_part_reduce", ptr(self.rb_part), self.rw_splits, T * E, ptr(self.g_router_b), s)
        call("smes_part_reduce", ptr(self.part_db), self.grid, T, ptr(self.g_head_b), s)
        self.g_head_w.copy_(self.shard.g_head_w)
        self.loss_part_f32.copy_(self.loss_part)
        tcall("ep_combine_dh", "smes_ep_combine_dh", B, d, self.n, B, ptr(self.pos), ptr(self.dh_recv), ptr(self.dh_router),
             ptr(self.d_hidden), s)

    def finish(self):
        """After the replicated-gradient all-reduce: the global loss."""
        s = self._s()
        self.loss_part.copy_(self.loss_part_f32)
        call("smes_loss_finalize", self.grid, ptr(self.loss_part), 1.0 / (self.B * self.n), self.beta,
             self.stats_out[3 * self.E:].data_ptr(), ptr(self.loss_out), s)

    def check(self):
        """Raise if the owner plan overflowed its row capacity (reads a device flag: host sync)."""
        if int(self.flag.item()):
            from .errors import NumericsError
            raise NumericsError(f"rank {self.rank}: non-finite router logits")
        if int(self.cap_flag.item()):
            raise StateError(f"rank {self.rank}: expert rows exceeded the shard capacity ({self.shard.R}); "
                             f"raise capacity_factor")

    # slots exchanged by the transports: (send, recv, row_bytes, rows_used)
    def exchanges(self, name):
        if name == "dispatch":
            return [(self.h_send, self.h_recv), (self.mask_send, self.umask_recv), (self.loads.view(self.n, self.El),
                                                                                   self.cnt_recv)]
        if name == "P":
            return [(self.P_send, self.P_recv)]
        if name == "C":
            return [(self.C_send, self.C_recv)]
        if name == "dh":
            return [(self.dh_own, self.dh_recv)]
        raise KeyError(name)


# ---------------------------------------------------------------------- transports
def _recv_tables(ranks_recv, dev):
    """Device pointer tables {name: int64[n]} from per-rank receive tensors."""
    return {k: torch.tensor([t.data_ptr() for t in v], dtype=torch.int64, device=dev) for k, v in ranks_recv.items()}


def _recv_buffers(rank):
    return {"mask": rank.umask_recv, "h": rank.h_recv, "cnt": rank.cnt_recv, "P": rank.P_recv, "C": rank.C_recv,
            "dh": rank.dh_recv}


class LoopbackComm:
    """n virtual ranks in one process (tests, single-GPU runs).  ``fused=False``: slot copies
    between send and receive buffers; ``fused=True``: the ranks' pack / gather kernels store
    straight into each other's receive buffers (the peer-memory code path, on one device)."""

    def __init__(self, ranks, fused: bool = False):
        self.ranks = ranks
        self.fused = fused
        if fused:
            bufs = [_recv_buffers(r) for r in ranks]
            tables = _recv_tables({k: [b[k] for b in bufs] for k in bufs[0]}, ranks[0].dev)
            for r in ranks:
                r.peers = tables

    def all_to_all(self, name):
        n = len(self.ranks)
        if self.fused:
            if name == "dh":
                s = torch.cuda.current_stream(self.ranks[0].dev).cuda_stream
                for r in self.ranks:
                    call("smes_ep_put_slots", n, r.rank, ptr(r.dh_own), r.B * r.d * 4, r.B * r.d * 4, None,
                         ptr(r.peers["dh"]), s)
            return
        pairs = [r.exchanges(name) for r in self.ranks]
        for k in range(len(pairs[0])):
            for dst in range(n):
                recv = pairs[dst][k][1]
                for src in range(n):
                    recv[src].copy_(pairs[src][k][0][dst])

    def all_reduce(self, tensors):
        if len(tensors) == 1:
            return
        acc = tensors[0].clone()
        for t in tensors[1:]:
            acc += t
        for t in tensors:
            t.copy_(acc)


class NcclComm:
    """One rank per process: torch.distributed all_to_all_single over equal fixed slots."""

    def __init__(self, rank, group=None):
        import torch.distributed as dist
        self.dist, self.rank, self.group = dist, rank, group

    def all_to_all(self, name):
        for send, recv in self.rank.exchanges(name):
            self.dist.all_to_all_single(recv.view(-1), send.reshape(-1), group=self.group)

    def all_reduce(self, tensors):
        for t in tensors:
            self.dist.all_reduce(t, group=self.group)


def ipc_peer_pointers(t: torch.Tensor, me: int, n: int, group, mapped: dict) -> torch.Tensor:
    """Map every rank's copy of ``t`` (CUDA IPC; the process group carries the handles) and return
    the n device pointers as an int64 device tensor (entry ``me`` is ``t`` itself).  The IPC handle
    names the cudaMalloc segment holding ``t``, so each rank also publishes the tensor's offset
    inside that segment (caching-allocator tensors rarely sit at a segment base) and the opener
    adds it to the mapped base.  ``mapped`` caches one mapping per (peer, segment)."""
    import ctypes as C
    import torch.distributed as dist
    h = (C.c_uint8 * 64)()
    off = C.c_long(0)
    call("smes_ipc_handle", ptr(t), C.cast(h, C.c_void_p), C.byref(off))
    mine = (bytes(h), int(off.value))
    allh = [None] * n
    dist.all_gather_object(allh, mine, group=group)
    ptrs = []
    for r, (hb, o) in enumerate(allh):
        if r == me:
            ptrs.append(t.data_ptr())
            continue
        base = mapped.get(hb)
        if base is None:        # a segment may hold several buffers
            out = C.c_void_p()
            hh = (C.c_uint8 * 64).from_buffer_copy(hb)
            call("smes_ipc_open", C.cast(hh, C.c_void_p), C.byref(out))
            base = mapped[hb] = out.value
        ptrs.append(base + o)
    return torch.tensor(ptrs, dtype=torch.int64, device=t.device)


class PeerComm:
    """One rank per process, hand-written transport over CUDA-IPC-mapped peer memory
    (NVLink/NVSwitch).  ``fused=True`` (default): the dispatch pack and the P / C segment
    gathers store straight into the peers' receive slots (csrc/ep.cu smes_ep_pack_put,
    smes_ep_copy_rows_put), so an exchange is only the flag handshake (smes_ep_signal_wait);
    ``fused=False``: a put kernel moves the filled send slots (smes_ep_put_slots)."""

    def __init__(self, rank, group=None, fused: bool = True):
        import torch.distributed as dist
        self.dist, self.rank, self.group = dist, rank, group
        self.n, self.me = rank.n, rank.rank
        dev = rank.dev
        self.flags = torch.zeros(self.n, dtype=torch.int32, device=dev)
        self.epoch = 0
        self._bufs = {}
        self._mapped = {}
        self.peer_flags = self._open(self.flags)
        for name in ("dispatch", "P", "C", "dh"):
            for _, recv in rank.exchanges(name):
                self._bufs[recv.data_ptr()] = self._open(recv)
        self.fused = fused
        if fused:
            rank.peers = {k: self._bufs[t.data_ptr()] for k, t in _recv_buffers(rank).items()}
        torch.cuda.synchronize(dev)
        self.dist.barrier(group=self.group)

    def _open(self, t):
        return ipc_peer_pointers(t, self.me, self.n, self.group, self._mapped)

    def close(self):
        """Unmap the peers' segments (after a final synchronize)."""
        torch.cuda.synchronize(self.rank.dev)
        for base in self._mapped.values():
            call("smes_ipc_close", base)
        self._mapped.clear()

    def all_to_all(self, name):
        s = torch.cuda.current_stream(self.rank.dev).cuda_stream
        rk = self.rank
        if self.fused and name != "dh":
            # the data is already in the peers' slots: publish and wait for every peer's
            self.epoch += 1
            call("smes_ep_signal_wait", self.n, self.me, ptr(self.peer_flags), ptr(self.flags), self.epoch, s)
            return
        used = {id(rk.h_send): (rk.cnt, rk.d * 2)}      # mask slots travel whole: empty slots must read zero
        for send, recv in rk.exchanges(name):
            slot_bytes = send[0].numel() * send.element_size()
            rows, row_bytes = used.get(id(send), (None, slot_bytes))
            call("smes_ep_put_slots", self.n, self.me, ptr(send), slot_bytes, row_bytes, ptr(rows),
                 ptr(self._bufs[recv.data_ptr()]), s)
        self.epoch += 1
        call("smes_ep_signal_wait", self.n, self.me, ptr(self.peer_flags), ptr(self.flags), self.epoch, s)

    def all_reduce(self, tensors):
        for t in tensors:
            self.dist.all_reduce(t, group=self.group)


class ExpertParallelStep:
    """Drives the phases of the local rank(s) with a transport between them."""

    def __init__(self, ranks, comm):
        self.ranks = list(ranks)
        self.comm = comm

    def step(self):
        R = self.ranks
        for r in R:
            r.f1()
        self.comm.all_reduce([r.stats_raw for r in R])
        self.comm.all_to_all("dispatch")
        for r in R:
            r.f2()
        self.comm.all_to_all("P")
        for r in R:
            r.f3()
        self.comm.all_to_all("C")
        for r in R:
            r.b1()
        self.comm.all_to_all("dh")
        for r in R:
            r.b2()
        self.comm.all_reduce([r.rep_grad for r in R])
        for r in R:
            r.finish()
