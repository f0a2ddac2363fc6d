"""Expert-parallel transport semantics on 2 gloo ranks (CPU): the all-to-all of fixed slots
(recv[s] on rank r == send[r] on rank s, for every exchange of a phase) and the all-reduce of
the replicated buffers, through the same NcclComm class the GPU run uses (ep.py)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


class _FakeRank:
    """The exchange surface of EPRank with small CPU slots."""

    def __init__(self, me, n):
        g = torch.Generator().manual_seed(100 + me)
        self.h_send = torch.randn(n, 5, 8, generator=g)
        self.h_recv = torch.zeros(n, 5, 8)
        self.m_send = torch.randint(0, 2 ** 30, (n, 5, 1), generator=g, dtype=torch.int32)
        self.m_recv = torch.zeros(n, 5, 1, dtype=torch.int32)
        self.l_send = torch.arange(n * 4, dtype=torch.int32).view(n, 4) + 1000 * me
        self.l_recv = torch.zeros(n, 4, dtype=torch.int32)
        self.rep = torch.full((7,), float(me + 1))

    def exchanges(self, name):
        assert name == "dispatch"
        return [(self.h_send, self.h_recv), (self.m_send, self.m_recv), (self.l_send, self.l_recv)]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2602_09386_b200.ep import NcclComm
    fr = _FakeRank(rank, world)
    comm = NcclComm(fr)
    comm.all_to_all("dispatch")
    comm.all_reduce([fr.rep])
    out.put((rank, fr.h_recv, fr.m_recv, fr.l_recv, fr.rep))
    dist.barrier()
    dist.destroy_process_group()


def test_slot_all_to_all_and_all_reduce():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, h, m, l, rep = q.get(timeout=120)
        res[r] = (h, m, l, rep)
    for p in procs:
        p.join(timeout=60)
    fakes = [_FakeRank(r, world) for r in range(world)]
    for r in range(world):
        h, m, l, rep = res[r]
        for s in range(world):
            assert torch.equal(h[s], fakes[s].h_send[r])
            assert torch.equal(m[s], fakes[s].m_send[r])
            assert torch.equal(l[s], fakes[s].l_send[r])
        assert torch.all(rep == 3.0)
