"""Data-parallel orchestration (paper_2602_09386_b200/dp.py) on 2 gloo ranks (CPU).

The DataParallelStep drives an oracle-backed engine with the same interface as
SMESEngine (forward_a / stats_raw / forward_b / backward / grad_flat).  Averaged
gradients and the global L_lb must equal the single-process oracle on the
concatenated batch (SURVEY 8e exactness rule).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import smes_oracle as O

KS, KA, BETA = 1, 2, 0.05


def _case():
    rng = np.random.default_rng(4)
    T, E, d, B = 3, 8, 6, 40
    p = O.init_layer_params(rng, d, d, E, T, d_ff=10, router_scale=1.0)
    h = rng.normal(size=(B, d))
    y = (rng.uniform(size=(T, B)) < 0.4).astype(float)
    lam = rng.uniform(0.5, 1.5, T)
    return p, h, y, lam


class OracleEngine:
    """SMESEngine-shaped wrapper over the CPU oracle (test double for the DP host logic)."""

    def __init__(self, p, h, y, lam):
        self.p, self.h, self.y, self.lam = p, h, y, lam
        self.B, self.T = h.shape[0], y.shape[0]
        self.E = p.router_w.shape[1]
        self.stats_raw = torch.zeros(3 * self.E, dtype=torch.float64)
        self.grad_flat = None

    def forward_a(self, finalize_stats=False):    # the oracle finalizes in forward_b either way
        self.f = O.forward_sparse(self.h, self.p, KS, KA)
        r = self.f.routing
        self.stats_raw[: self.E] = torch.tensor(np.bincount(r.active.ravel(), minlength=self.E), dtype=torch.float64)
        self.stats_raw[self.E: 2 * self.E] = torch.tensor(r.weights.sum(axis=(0, 1)))
        self.stats_raw[2 * self.E:] = torch.tensor(r.full_probs.sum(axis=(0, 1)))

    def forward_b(self, with_loss=True, batch_times_tasks=None, train=False, batch_scale=None, lb_batch=None,
                  stats_done=False, defer_reduce=False):
        raw = self.stats_raw.numpy()
        bt = batch_times_tasks
        freq, mass = raw[: self.E] / bt, raw[self.E: 2 * self.E] / bt
        self.bt = bt
        self.freq, self.mass = freq, mass

    def backward(self, batch_scale=None, lb_batch=None):
        K = KS + KA
        value = float((self.E / K) * np.dot(self.freq, self.mass))
        st = O.LoadStats(self.freq, self.mass, value, None, lb_batch, self.T, K, False)
        bw = O.backward(self.f, self.p, self.y, self.lam, BETA, stats=st, batch_scale=batch_scale)
        parts = [g for pair in bw.layers for g in pair] + [bw.router_w, bw.router_b, bw.head_w, bw.head_b]
        self.grad_flat = torch.tensor(np.concatenate([np.ravel(a) for a in parts]))
        self.lb_value = value
        self.loss_out = torch.tensor([bw.task_value, value, bw.task_value + BETA * value], dtype=torch.float64)


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2602_09386_b200.dp import DataParallelStep
    p, h, y, lam = _case()
    n = h.shape[0] // world
    eng = OracleEngine(p, h[rank * n:(rank + 1) * n], y[:, rank * n:(rank + 1) * n], lam)
    step = DataParallelStep(eng, use_graphs=False)
    step.step()
    if rank == 0:
        out.put((eng.grad_flat.numpy(), eng.lb_value, eng.loss_out.numpy()))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_dp_two_ranks_equals_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    grad, lb, loss = q.get(timeout=120)
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    p, h, y, lam = _case()
    f = O.forward_sparse(h, p, KS, KA)
    bw = O.backward(f, p, y, lam, BETA)
    parts = [g for pair in bw.layers for g in pair] + [bw.router_w, bw.router_b, bw.head_w, bw.head_b]
    ref = np.concatenate([np.ravel(a) for a in parts])
    assert np.abs(grad - ref).max() <= 1e-12 * np.abs(ref).max()
    assert abs(lb - bw.lb_value) < 1e-12
    # the all-reduced objective is the global-batch one (dp.py _allreduce_grads)
    assert np.allclose(loss, [bw.task_value, bw.lb_value, bw.total], rtol=1e-12)
