"""The training/scoring router entry (smes_route_batch, not frozen, no dense probabilities in or
out) through both kernels: the expert-per-lane route_kernel and the task-grouped route_tg_kernel
(T, E) in {(8, 32), (4, 32)} with (K_s, K_a) = (4, 2).  Against the oracle on the same fp32
logits: selections and union masks index-exact, weights within fp32 1e-6, and the chunk
histograms summed over chunks equal to the oracle's LoadStats sums (counts exact, sparse mass of
the fp32 weights 1e-6 relative, dense fp64 mass 1e-9)."""
import zlib

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from oracle import smes_oracle as O
from paper_2602_09386_b200 import _lib


def _route(z32, ks, ka, tw, dm=True):
    call, ptr = _lib.call, _lib.ptr
    T, B, E = z32.shape
    K = ks + ka
    dev = "cuda"
    z = torch.tensor(z32, dtype=torch.float32, device=dev).permute(1, 0, 2).contiguous()   # (B, T, E)
    rpw = call("smes_route_rows_per_warp", B)
    C = call("smes_route_num_chunks", B, rpw)
    i32 = lambda *s: torch.zeros(*s, dtype=torch.int32, device=dev)
    f64 = lambda *s: torch.zeros(*s, dtype=torch.float64, device=dev)
    out = dict(shared=i32(B, ks), adaptive=i32(T, B, ka), active=i32(T, B, K),
               wsel=torch.zeros(T, B, K, device=dev), umask=i32(B, (E + 31) // 32), usize=i32(B),
               cu=i32(C, E), ca=i32(C, E), cm=f64(C, E), cd=f64(C, E), flag=i32(1))
    twt = torch.tensor(tw, dtype=torch.float64, device=dev)
    call("smes_route_batch", ptr(z), E, T * E, None, ptr(twt), T, B, E, ks, ka, rpw, ptr(out["shared"]),
         ptr(out["adaptive"]), ptr(out["active"]), ptr(out["wsel"]), ptr(out["umask"]), ptr(out["usize"]),
         ptr(out["cu"]), ptr(out["ca"]), ptr(out["cm"]), ptr(out["cd"]) if dm else None, None, ptr(out["flag"]), 0,
         torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    return {k: v.cpu().numpy() for k, v in out.items()}


CASES = {
    "tg_8x32_random": (8, 32, "random"),
    "tg_8x32_reference_init": (8, 32, "init"),
    "tg_8x32_ties": (8, 32, "ties"),
    "tg_4x32_random": (4, 32, "random"),
    "tg_4x32_ties": (4, 32, "ties"),
    "lane_8x64_random": (8, 64, "random"),     # expert-per-lane kernel for comparison
    # (row, task) kernel (csrc/route_rt.cu): taken when no dense mass is requested
    "rt_16x64_init": (16, 64, "init"),         # c3 / c4 shape, reference-init Stage-I gaps
    "rt_16x64_random": (16, 64, "random"),
    "rt_16x64_ties": (16, 64, "ties"),
    "rt_16x64_tiny": (16, 64, "tiny"),         # gaps ~1e-12: the deviation form still decides them
    "rt_12x64_init": (12, 64, "init"),         # T not a power of two: idle task lanes
    "rt_32x64_random": (32, 64, "random"),
    "rt_8x32_init": (8, 32, "init"),
    "rt_4x16_init": (4, 16, "init"),           # c1 shape
    "rt_3x16_ties": (3, 16, "ties"),
    "rt_5x32_tiny": (5, 32, "tiny"),
    # expert-per-lane kernel without dense statistics: its fp32 deviation-form Stage I (E > 64, c5)
    "lanefast_32x256_init": (32, 256, "init"),
    "lanefast_32x256_ties": (32, 256, "ties"),
    "lanefast_8x128_random": (8, 128, "random"),
    "lanefast_4x96_tiny": (4, 96, "tiny"),
}


@pytest.mark.parametrize("name", list(CASES))
def test_router_kernel_vs_oracle(name):
    T, E, kind = CASES[name]
    ks, ka, B = (2, 1, 3001) if E == 16 else (4, 2, 3000)
    rt = name.startswith("rt_") or name.startswith("lanefast_")
    rng = np.random.default_rng(zlib.crc32(name.encode()))
    if kind == "random":
        z = rng.normal(size=(T, B, E))
    elif kind in ("init", "tiny"):  # reference router init: |z| ~ 5e-4, Stage-I gaps ~1e-10 (tiny: ~1e-8)
        sc = 1e-3 if kind == "init" else 1e-7
        z = np.einsum("bd,ted->tbe", rng.normal(size=(B, 256)), rng.uniform(-sc / 16, sc / 16, size=(T, E, 256)))
    else:                         # heavy ties: 3 distinct values
        z = rng.integers(0, 3, size=(T, B, E)).astype(np.float64)
    z32 = np.asarray(z, dtype=np.float32).astype(np.float64)
    tw = rng.uniform(0.5, 2.0, size=T)
    cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
    _lib.call("smes_route_count_exact", _lib.ptr(cnt))
    try:
        g = _route(z32, ks, ka, tw, dm=not rt)
    finally:
        _lib.call("smes_route_count_exact", None)
    if name.startswith("rt_"):
        assert _lib.call("smes_route_rt_supported", T, E, ks, ka)
    if name.startswith("rt_"):          # (the expert-per-lane kernel does not count its fallback rows)
        n_exact = int(cnt.item())
        if kind == "ties":
            assert n_exact > 0, n_exact           # exact pooled ties go through the fp64 recompute
        if kind == "random":
            assert n_exact < B // 20, n_exact
    ref = O.route_batch(z32, ks, ka, tw)
    assert g["flag"][0] == 0
    assert np.array_equal(g["shared"], ref.shared)
    assert np.array_equal(g["adaptive"], ref.adaptive)
    assert np.array_equal(g["active"], ref.active)
    w_ref = np.take_along_axis(ref.weights, ref.active, axis=2)
    assert np.abs(g["wsel"] - w_ref).max() < 1e-6
    usize = np.array([len(u) for u in ref.unions])
    assert np.array_equal(g["usize"], usize)
    for b in range(0, B, 97):
        bits = np.zeros(E, bool)
        bits[ref.unions[b]] = True
        words = [int(sum(1 << i for i in range(32) if 32 * w + i < E and bits[32 * w + i]))
                 for w in range((E + 31) // 32)]
        assert [int(x) & 0xFFFFFFFF for x in g["umask"][b]] == words
    # chunk histograms -> LoadStats sums
    counts = np.bincount(ref.active.reshape(-1), minlength=E)
    assert np.array_equal(g["ca"].sum(0), counts)
    assert np.array_equal(g["cu"].sum(0), np.bincount(np.concatenate(ref.unions), minlength=E))
    sm = ref.weights.sum(axis=(0, 1))              # sums of fp32 weights: 1e-6 relative
    assert (np.abs(g["cm"].sum(0) - sm) <= 1e-6 * sm + 1e-9).all()
    if not rt:
        assert np.abs(g["cd"].sum(0) - ref.full_probs.sum(axis=(0, 1))).max() < 1e-9 * B * T
