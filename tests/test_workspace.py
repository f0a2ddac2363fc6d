"""Workspace page pool (paper_2602_09386_b200/workspace.py): the reference's ledger semantics
(tests/test_workspace.py of taskmoe: first fit, FIFO head-of-line waiting, timeouts, bad
releases, provisioning, virtual-time replay) and, on the GPU, the HBM arena with stream-ordered
release."""
import threading
import time

import numpy as np
import pytest
import torch

from paper_2602_09386_b200 import (ConfigError, DeviceWorkspace, LoadProfile, PoolError, PoolTimeout,
                                   StateError, WorkspacePool, provision, required_pages, simulate_replay)


def test_required_pages_arithmetic():
    assert required_pages(20, 16, 8, elem_bytes=8, page_size=4096) == 1     # 3840 B -> 1 page
    assert required_pages(0, 16, 8) == 0
    assert required_pages(279_000, 256, 256, elem_bytes=2, page_size=1 << 20) == 273   # c2 packed bf16
    for n in (3, 17, 40, 129):
        one, two = required_pages(n, 16, 16, page_size=1024), required_pages(2 * n, 16, 16, page_size=1024)
        assert 2 * one - 1 <= two <= 2 * one
    with pytest.raises(ConfigError):
        required_pages(-1, 4, 4)
    with pytest.raises(ConfigError):
        required_pages(1, 0, 4)


def test_first_fit_lowest_gap_and_holes():
    pool = WorkspacePool(10)
    a = pool.allocate(4)
    b = pool.allocate(3)
    assert (a.start, b.start) == (0, 4)
    pool.release(a)
    assert pool.allocate(2).start == 0
    pool = WorkspacePool(10)
    a, b = pool.allocate(2), pool.allocate(3)
    pool.allocate(5)
    pool.release(a)
    pool.release(b)
    assert pool.allocate(5).start == 0


def test_round_trip_counters_and_peak():
    pool = WorkspacePool(8)
    a, b = pool.allocate(3), pool.allocate(4)
    pool.release(a)
    pool.release(b)
    assert pool.pages_in_use == 0 and pool.held_blocks() == []
    assert pool.allocations == pool.releases == 2
    assert pool.peak_pages_in_use == 7


def test_infeasible_and_bad_release():
    pool = WorkspacePool(4)
    with pytest.raises(PoolError, match="never"):
        pool.allocate(5)
    with pytest.raises(PoolError, match="never"):
        pool.try_allocate(5)
    blk = pool.allocate(2)
    pool.allocate(1)
    pool.release(blk)
    before = pool.held_blocks()
    with pytest.raises(PoolError, match="unknown or already released"):
        pool.release(blk)
    assert pool.held_blocks() == before


def test_timeout_counts_one_wait():
    pool = WorkspacePool(4)
    pool.allocate(4)
    t0 = time.monotonic()
    with pytest.raises(PoolTimeout):
        pool.allocate(1, timeout=0.05)
    assert time.monotonic() - t0 < 2.0
    assert pool.wait_events == 1
    assert pool.try_allocate(0) is not None      # the timed-out waiter left the queue


def test_try_allocate_defers_to_waiters():
    pool = WorkspacePool(4)
    hold = pool.allocate(3)
    th = threading.Thread(target=lambda: pool.release(pool.allocate(2, timeout=5.0)))
    th.start()
    for _ in range(500):
        if pool.wait_events == 1:
            break
        time.sleep(0.002)
    assert pool.try_allocate(1) is None          # one page is free, but a waiter is queued
    pool.release(hold)
    th.join(5.0)
    assert pool.pages_in_use == 0


def test_fifo_head_of_line_order():
    pool = WorkspacePool(4)
    hold = pool.allocate(4)
    order, threads = [], []

    def waiter(tag):
        blk = pool.allocate(2, timeout=5.0)
        order.append(tag)
        time.sleep(0.05)
        pool.release(blk)

    for tag in ("first", "second", "third"):
        th = threading.Thread(target=waiter, args=(tag,))
        th.start()
        threads.append(th)
        for _ in range(500):
            if pool.wait_events >= len(threads):
                break
            time.sleep(0.002)
    pool.release(hold)
    for th in threads:
        th.join(5.0)
    assert order == ["first", "second", "third"]
    assert pool.pages_in_use == 0


@pytest.mark.parametrize("seed", [0, 1])
def test_concurrent_no_overlap(seed):
    pool = WorkspacePool(64)
    owner = [0] * 64
    bad = []

    def worker(wid):
        rng = np.random.default_rng((seed, wid))
        for _ in range(40):
            blk = pool.allocate(int(rng.integers(1, 9)), timeout=10.0)
            for p in range(blk.start, blk.start + blk.num_pages):
                if owner[p]:
                    bad.append(p)
                owner[p] = wid + 1
            for p in range(blk.start, blk.start + blk.num_pages):
                owner[p] = 0
            pool.release(blk)

    ths = [threading.Thread(target=worker, args=(w,)) for w in range(8)]
    for th in ths:
        th.start()
    for th in ths:
        th.join(60.0)
    assert not bad
    assert pool.held_blocks() == [] and pool.allocations == pool.releases == 320


def test_profile_quantiles_and_provisioning(tmp_path):
    prof = LoadProfile(samples=list(range(1, 101)))
    assert [prof.quantile(q) for q in (0.5, 0.99, 1.0, 0.001)] == [50, 99, 100, 1]
    assert LoadProfile(samples=[5, 80, 12, 44]).quantile(1.0) == 80
    assert provision(LoadProfile(samples=[20] * 30), 0.99, 16, 8, concurrency=2) == 2 * required_pages(20, 16, 8)
    with pytest.raises(StateError):
        provision(LoadProfile(), 0.5, 4, 4, concurrency=1)
    with pytest.raises(ConfigError):
        prof.quantile(0.0)
    with pytest.raises(ConfigError):
        prof.quantile(1.5)
    path = str(tmp_path / "s.txt")
    LoadProfile(samples=[4, 99, 0, 17]).save(path)
    assert LoadProfile.load(path).samples == [4, 99, 0, 17]
    open(path, "w").write("12\nhello\n")
    with pytest.raises(ConfigError, match="line 2"):
        LoadProfile.load(path)


def test_replay_policy():
    rng = np.random.default_rng(0)
    samples = rng.integers(10, 200, size=60).tolist()
    cap = provision(LoadProfile(samples=samples), 1.0, 16, 16, concurrency=4)
    res = simulate_replay(cap, [required_pages(n, 16, 16) for n in samples], 4)
    assert res.wait_events == 0 and res.completed == 60
    samples = [100] * 20 + [350] * 8 + [100] * 20
    cap = provision(LoadProfile(samples=samples), 0.5, 16, 16, concurrency=4)
    reqs = [required_pages(n, 16, 16) for n in samples]
    assert max(reqs) <= cap and simulate_replay(cap, reqs, 4).wait_events > 0
    reqs = [required_pages(n, 8, 8) for n in [10, 50, 200, 30, 180, 90] * 5]
    assert simulate_replay(40, reqs, 3) == simulate_replay(40, reqs, 3)
    # hand-checked: pool 4, requests 3,2,2 with 2 workers -> t0 runs 3, 2 waits; t1 runs 2+2
    res = simulate_replay(4, [3, 2, 2], 2)
    assert (res.wait_events, res.peak_pages_in_use, res.completed) == (1, 4, 3)
    # pinned on the reference's simulate_replay (workspace.py:272-319) run in the build container
    r = np.random.default_rng(5).integers(1, 30, size=200).tolist()
    res = simulate_replay(64, r, 5)
    assert (res.wait_events, res.peak_pages_in_use, res.completed) == (45, 64, 200)
    with pytest.raises(PoolError):
        simulate_replay(4, [10], 2)


@pytest.mark.gpu
def test_device_arena_and_stream_ordered_release():
    pool = WorkspacePool(page_count=16, page_size=1 << 16)
    ws = DeviceWorkspace(pool)
    blk = pool.allocate(4)
    x, y = ws.carve(blk, [((1000, 64), torch.bfloat16), ((500,), torch.float32)])
    assert x.is_cuda and x.data_ptr() % 256 == 0 and y.data_ptr() % 256 == 0
    assert x.data_ptr() >= ws.arena.data_ptr() + blk.start * pool.page_size
    with pytest.raises(PoolError, match="cannot hold"):
        ws.carve(blk, [((4 << 16,), torch.float32)])
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        torch.cuda._sleep(50_000_000)               # ~25 ms of queued work on s
        x.fill_(1.0)
    pool.release(blk, stream=s)                     # returns at once; pages held until s drains
    assert pool.held_blocks() == [(0, 4)]
    with pytest.raises(PoolError, match="already released"):
        pool.release(blk, stream=s)
    nxt = pool.allocate(16, timeout=10.0)           # waits for the deferred release, no host sync
    assert nxt.start == 0 and pool.releases == 1
    assert float(x.float().sum()) == 64000.0        # the stream's write landed before the reuse


def test_engine_workspace_bytes_matches_specs():
    """The per-engine block size is the aligned sum of the packed-row buffers (no GPU needed)."""
    from paper_2602_09386_b200.engine import ExpertLayer, SMESParams, row_buffer_specs, workspace_bytes
    T, E, d, dff = 4, 16, 128, 256
    z = lambda *s: torch.zeros(*s)
    p = SMESParams(router_w=z(T, E, d), router_b=z(T, E),
                   layers=[ExpertLayer(z(E, dff, d), z(E, dff), "relu"), ExpertLayer(z(E, d, dff), z(E, d), "identity")],
                   head_w=z(T, d), head_b=z(T))
    specs = row_buffer_specs(T, E, 1000, 2, 1, [d, dff, d], ["relu", "identity"])
    names = [n for n, _, _ in specs]
    assert names[:3] == ["gather_inst", "gather_exp", "X"] and "bits.0" in names and "bits.1" not in names
    R = (1000 * 6 + 16 * 127 + 127) // 128 * 128
    assert dict((n, s) for n, s, _ in specs)["X"] == (R, d + 64)
    nb = workspace_bytes(p, 1000, 2, 1)
    raw = sum(torch.Size(s).numel() * torch.empty((), dtype=dt).element_size() for _, s, dt in specs)
    assert raw <= nb < raw + 256 * len(specs)


@pytest.mark.gpu
def test_engines_share_a_device_workspace_pool():
    """Two scoring engines (BASELINE c4 streams) draw their packed-row buffers from blocks of ONE
    provisioned HBM arena, run concurrently on two CUDA streams, and give identical predictions to
    engines with private buffers (workspace.py:42-262 semantics: one grant per in-flight batch)."""
    from paper_2602_09386_b200 import SMESEngine
    from paper_2602_09386_b200.engine import workspace_bytes
    from tests.helpers import make_case, to_engine_params
    B, T, E, d = 1024, 8, 32, 128
    p, h, y, lam, beta = make_case(21, B, T, E, d, d, 4, 2, d_ff=256)
    params = to_engine_params(p, lam, beta)
    page = 1 << 16
    per = -(-workspace_bytes(params, B, 4, 2) // page)
    pool = WorkspacePool(page_count=2 * per, page_size=page)
    ws = DeviceWorkspace(pool)
    blocks = [pool.allocate(per) for _ in range(2)]
    hs = [torch.tensor(h, device="cuda"), torch.tensor(h[::-1].copy(), device="cuda")]
    shared = [SMESEngine(params, B, 4, 2, workspace=(ws, blk)) for blk in blocks]
    assert shared[0].X.data_ptr() >= ws.arena.data_ptr()
    assert shared[1].X.data_ptr() >= ws.arena.data_ptr() + blocks[1].start * page
    assert shared[0].workspace_nbytes <= per * page
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    torch.cuda.synchronize()
    for eng, x, s in zip(shared, hs, streams):
        with torch.cuda.stream(s):
            eng.set_inputs(x)
            eng.score()
    for blk, s in zip(blocks, streams):
        pool.release(blk, stream=s)          # pages come back once each stream's work is done
    torch.cuda.synchronize()
    for eng, x in zip(shared, hs):
        ref = SMESEngine(params, B, 4, 2)
        ref.set_inputs(x)
        ref.score()
        torch.cuda.synchronize()
        assert torch.equal(eng.preds, ref.preds)
    again = pool.allocate(2 * per, timeout=10.0)
    assert again.start == 0
    with pytest.raises(PoolError, match="cannot hold"):
        SMESEngine(params, B, 4, 2, workspace=(ws, WorkspacePool(1, page).allocate(1)))
