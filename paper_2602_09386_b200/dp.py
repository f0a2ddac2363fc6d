"""Data-parallel SMES step (one process per GPU, torch.distributed over NCCL).

Routing, planning and the expert GEMMs are per instance (taskmoe/routing.py:3-8),
so the batch shards with no data-path exchange.  The SMES path has exactly two
real exchange points:

1. the multi-gate LB statistics are means over the WHOLE mini-batch
   (taskmoe/balance.py:62-70): the per-expert (counts, sparse mass, dense mass)
   sums (3E fp64 values) are all-reduced right after routing, before L_lb and
   before the LB gradient;
2. parameter gradients are averaged (one flat fp32 buffer).

Scaling rule that makes the sharded step equal the single-process step on the
concatenated batch: frequency / mass use the global B*T; the BCE mean
(training.py:148) and the LB coefficient E/(K B T) (balance.py:97) use the
LOCAL batch, because gradients are averaged over ranks.

The orchestration only touches the engine through ``forward_a / forward_b /
backward / stats_raw / grad_flat``, so the CPU tests drive it with an oracle
engine over gloo.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


class DataParallelStep:
    def __init__(self, engine, group=None, use_graphs: bool = True):
        self.eng = engine
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.b_local = engine.B
        self.b_global = engine.B * self.world
        self.use_graphs = use_graphs and torch.cuda.is_available() and engine_is_cuda(engine)
        self._ga = self._gb = None

    # the three segments between the two collectives
    def _part_a(self):
        # one rank: nothing to exchange, the plan reduce also finalizes the LoadStats
        solo = self.world == 1
        if getattr(self.eng, "can_fold", False):
            self.eng.forward_a(fold=True, finalize_stats=solo)     # heads folded into the last pool
        else:
            self.eng.forward_a(finalize_stats=solo)

    def _part_b(self):
        self.eng.forward_b(with_loss=True, batch_times_tasks=float(self.b_global * self.eng.T), train=True,
                           batch_scale=self.b_local, lb_batch=self.b_local, stats_done=self.world == 1,
                           defer_reduce=True)
        self.eng.backward(batch_scale=self.b_local, lb_batch=self.b_local)

    def capture(self, warmup: int = 1):
        """Capture the two compute segments as CUDA graphs (collectives stay eager)."""
        st = torch.cuda.Stream()
        st.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(st):
            for _ in range(warmup):
                self.step_eager()
        torch.cuda.current_stream().wait_stream(st)
        self._ga = torch.cuda.CUDAGraph()
        if self.world == 1:
            # nothing to exchange between the segments: one graph, one launch per step
            self._gb = None
            with torch.cuda.graph(self._ga):
                self._part_a()
                self._part_b()
            return
        self._gb = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self._ga):
            self._part_a()
        with torch.cuda.graph(self._gb):
            self._part_b()

    def _allreduce_stats(self):
        if self.world > 1:
            dist.all_reduce(self.eng.stats_raw, op=dist.ReduceOp.SUM, group=self.group)

    def _allreduce_grads(self):
        if self.world > 1:
            dist.all_reduce(self.eng.grad_flat, op=dist.ReduceOp.SUM, group=self.group)
            self.eng.grad_flat.div_(self.world)
            # the reported objective is the global-batch one: the task term is a per-rank mean over
            # an equal shard (average it), L_lb already uses the all-reduced statistics (identical
            # on every rank), so averaging [task, lb, total] gives the global values
            dist.all_reduce(self.eng.loss_out, op=dist.ReduceOp.SUM, group=self.group)
            self.eng.loss_out.div_(self.world)

    def step_eager(self):
        self._part_a()
        self._allreduce_stats()
        self._part_b()
        self._allreduce_grads()

    def step(self):
        if self._ga is None:
            return self.step_eager()
        self._ga.replay()
        if self._gb is None:
            return
        self._allreduce_stats()
        self._gb.replay()
        self._allreduce_grads()


def engine_is_cuda(engine) -> bool:
    t = getattr(engine, "grad_flat", None)
    return t is not None and t.is_cuda
