"""Host-fed training loop: each step's inputs come from pinned host memory.

``HostStepPipeline.step(h_host, labels_host)`` is the public per-step call of a training
loop fed from the host.  The H2D copy of step i+1's inputs runs on a copy stream into
a double-buffered device staging area while step i computes.  A step then starts with
a device-to-device move into the engine's input buffers (graph-stable addresses), runs
the fwd+bwd step, and queues a D2H read of its loss into pinned memory.
"""
from __future__ import annotations

import torch


class HostStepPipeline:
    def __init__(self, engine, step_fn=None):
        self.eng = engine
        self.step_fn = step_fn or engine.step
        dev = engine.dev
        self.copy_stream = torch.cuda.Stream(dev)
        self.stage_h = [torch.empty(engine.B, engine.d, dtype=torch.bfloat16, device=dev) for _ in range(2)]
        self.stage_y = [torch.empty(engine.T, engine.B, dtype=torch.float32, device=dev) for _ in range(2)]
        self.ready = [torch.cuda.Event() for _ in range(2)]
        self.free = [torch.cuda.Event() for _ in range(2)]
        self.loss_host = torch.zeros(3, dtype=torch.float64).pin_memory()
        self._fill = 0          # staging slot the next prefetch writes
        self._queue = []        # slots holding inputs not yet consumed (FIFO)

    def prefetch(self, h_host: torch.Tensor, labels_host: torch.Tensor) -> None:
        """Queue the H2D copy of a future step's inputs (pinned host tensors)."""
        if len(self._queue) == 2:
            raise RuntimeError("both staging slots hold unconsumed inputs")
        slot = self._fill
        with torch.cuda.stream(self.copy_stream):
            self.copy_stream.wait_event(self.free[slot])
            self.stage_h[slot].copy_(h_host, non_blocking=True)
            self.stage_y[slot].copy_(labels_host, non_blocking=True)
            self.ready[slot].record(self.copy_stream)
        self._queue.append(slot)
        self._fill = 1 - slot

    def step(self, next_h: torch.Tensor | None = None, next_labels: torch.Tensor | None = None) -> torch.Tensor:
        """Run one step on the oldest prefetched inputs; optionally prefetch the following
        step's inputs so their copy overlaps this step.  Returns the pinned loss tensor
        (valid once the current stream has synchronised)."""
        if not self._queue:
            raise RuntimeError("no inputs prefetched: call prefetch(h_host, labels_host) first")
        cur = torch.cuda.current_stream(self.eng.dev)
        slot = self._queue.pop(0)
        cur.wait_event(self.ready[slot])
        self.eng.h.copy_(self.stage_h[slot])
        self.eng.labels.copy_(self.stage_y[slot])
        self.free[slot].record(cur)
        if next_h is not None:
            self.prefetch(next_h, next_labels)
        self.step_fn()
        self.loss_host.copy_(self.eng.loss_out, non_blocking=True)
        return self.loss_host
