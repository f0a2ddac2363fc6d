"""Data-parallel SMES step (one process per GPU, torch.distributed over NCCL).

Routing, planning and the expert GEMMs are per instance (taskmoe/routing.py:3-8),
so the batch shards with no data-path exchange.  The SMES path has exactly two
real exchange points:

1. the multi-gate LB statistics are means over the WHOLE mini-batch
   (taskmoe/balance.py:62-70): the per-expert (counts, sparse mass, dense mass)
   sums (3E fp64 values) are all-reduced right after routing, before L_lb and
   before the LB gradient;
2. parameter gradients are averaged.

Scaling rule that makes the sharded step equal the single-process step on the
concatenated batch: frequency / mass use the global B*T; the BCE mean
(training.py:148) and the LB coefficient E/(K B T) (balance.py:97) use the
LOCAL batch, because gradients are averaged over ranks.

B200 transport:
* ``stats="peer"``: the 3E statistics go through a one-shot all-reduce over CUDA-IPC-mapped
  peer memory (csrc/comm.cu): every rank stores its sums into every peer's slot, raises a flag
  and sums the n slots in rank order -- a few microseconds over NVLink / NVSwitch, graph
  capturable (device-side epoch), so the forward never leaves the CUDA graph.
  ``stats="group"``: a torch.distributed all-reduce (NCCL, or gloo in the CPU tests).
* gradients are reduced in three contiguous buckets of the engine's completion-ordered flat
  buffer ([pools but the last] [last pool + heads] [routers]), each issued on a communication
  stream the moment its producing kernels are enqueued (``engine.on_grads``), so the NCCL
  all-reduces run under the remaining backward kernels instead of after them.
With NCCL and ``stats="peer"`` the whole step, collectives included, is one CUDA graph.

The orchestration only touches the engine through ``forward_a / forward_b /
backward / stats_raw / grad_flat / grad_buckets / on_grads``, so the CPU tests drive it with
an oracle engine over gloo.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from ._lib import call, ptr


class PeerAllReduce:
    """One-shot f64 sum over CUDA-IPC-mapped peer memory (csrc/comm.cu smes_peer_allreduce_f64).
    The process group only carries the IPC handles at construction."""

    def __init__(self, count: int, group=None, device=None):
        from .ep import ipc_peer_pointers
        self.group = group
        self.n = dist.get_world_size(group)
        self.me = dist.get_rank(group)
        self.count = int(count)
        dev = torch.device(device or "cuda")
        self.recv = torch.zeros(2, self.n, self.count, dtype=torch.float64, device=dev)
        self.flags = torch.zeros(self.n, dtype=torch.int32, device=dev)
        self.epoch = torch.zeros(1, dtype=torch.int32, device=dev)
        self._mapped = {}
        self.peer_recv = ipc_peer_pointers(self.recv, self.me, self.n, group, self._mapped)
        self.peer_flags = ipc_peer_pointers(self.flags, self.me, self.n, group, self._mapped)
        torch.cuda.synchronize(dev)
        dist.barrier(group=group)

    def __call__(self, t: torch.Tensor, out: torch.Tensor | None = None):
        """out = sum over ranks of t (in place when out is None), on the current stream."""
        if t.dtype != torch.float64 or t.numel() != self.count:
            raise ValueError(f"peer all-reduce expects {self.count} float64 values")
        s = torch.cuda.current_stream(t.device).cuda_stream
        call("smes_peer_allreduce_f64", self.n, self.me, self.count, ptr(t), ptr(self.peer_recv),
             ptr(self.peer_flags), ptr(self.recv), ptr(self.flags), ptr(self.epoch), ptr(t if out is None else out), s)

    def close(self):
        from ._lib import call as _call
        torch.cuda.synchronize(self.recv.device)
        for base in self._mapped.values():
            _call("smes_ipc_close", base)
        self._mapped.clear()


class DataParallelStep:
    def __init__(self, engine, group=None, use_graphs: bool = True, stats: str = "group", overlap: bool = True):
        self.eng = engine
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.b_local = engine.B
        self.b_global = engine.B * self.world
        self.backend = dist.get_backend(group) if dist.is_initialized() else None
        cuda = torch.cuda.is_available() and engine_is_cuda(engine)
        # collectives inside a captured graph need NCCL; gloo runs eager (CPU tests, one-GPU tests)
        self.use_graphs = use_graphs and cuda and (self.world == 1 or self.backend == "nccl")
        self.stats = stats if self.world > 1 else "none"
        self._peer = PeerAllReduce(3 * engine.E, group, engine.stats_raw.device) if self.stats == "peer" else None
        self.overlap = bool(overlap and self.world > 1 and cuda and hasattr(engine, "grad_buckets"))
        self._comm = torch.cuda.Stream(engine.stats_raw.device) if self.overlap else None
        self._ga = self._gb = None

    # the segments between the collectives
    def _part_a(self):
        # one rank: nothing to exchange, the plan reduce also finalizes the LoadStats
        solo = self.world == 1
        if getattr(self.eng, "can_fold", False):
            self.eng.forward_a(fold=True, finalize_stats=solo)     # heads folded into the last pool
        else:
            self.eng.forward_a(finalize_stats=solo)
        if self._peer is not None:
            self._peer(self.eng.stats_raw)

    def _part_b(self):
        self.eng.forward_b(with_loss=True, batch_times_tasks=float(self.b_global * self.eng.T), train=True,
                           batch_scale=self.b_local, lb_batch=self.b_local, stats_done=self.world == 1,
                           defer_reduce=True)
        if self.overlap:
            self.eng.on_grads = self._grad_bucket
        try:
            self.eng.backward(batch_scale=self.b_local, lb_batch=self.b_local)
        finally:
            self.eng.on_grads = None
        if self.overlap:
            torch.cuda.current_stream(self.eng.stats_raw.device).wait_stream(self._comm)

    def _grad_bucket(self, name, stream):
        """Engine hook: bucket ``name`` of grad_flat is final on ``stream`` -- reduce it on the
        communication stream while the rest of the backward runs."""
        ev = torch.cuda.Event()
        ev.record(stream)
        self._comm.wait_event(ev)
        with torch.cuda.stream(self._comm):
            dist.all_reduce(self.eng.grad_flat[self.eng.grad_buckets[name]], op=dist.ReduceOp.SUM, group=self.group)

    def capture(self, warmup: int = 1):
        """Capture the step as CUDA graphs: one graph when no eager collective sits inside the step
        (one rank, or NCCL with the peer statistics exchange), else two around the statistics."""
        st = torch.cuda.Stream()
        st.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(st):
            for _ in range(warmup):
                self.step_eager()
        torch.cuda.current_stream().wait_stream(st)
        if not self.use_graphs:
            return
        self._ga = torch.cuda.CUDAGraph()
        if self.world == 1 or self.stats == "peer":
            self._gb = None
            with torch.cuda.graph(self._ga):
                self._part_a()
                self._part_b()
                self._finish_grads()
            return
        self._gb = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self._ga):
            self._part_a()
        with torch.cuda.graph(self._gb):
            self._part_b()
            self._finish_grads()

    def _allreduce_stats(self):
        if self.stats == "group":
            dist.all_reduce(self.eng.stats_raw, op=dist.ReduceOp.SUM, group=self.group)

    def _finish_grads(self):
        if self.world > 1:
            if not self.overlap:
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
        self._finish_grads()

    def step(self):
        if self._ga is None:
            return self.step_eager()
        self._ga.replay()
        if self._gb is None:
            return
        self._allreduce_stats()
        self._gb.replay()


def engine_is_cuda(engine) -> bool:
    t = getattr(engine, "grad_flat", None)
    return t is not None and t.is_cuda
