"""The fused router front (csrc/front.cu: router GEMM on tcgen05 -> thread-per-row routing from
TMEM) against the oracle and against the two-kernel path it replaces.

Logits: the front's own z output against RouterBank.logits (routing.py:101-103) in f64 on the same
bf16 operands (fp32 accumulation: 1e-5 relative).  Routing: index-exact against the oracle's
route_batch (routing.py:235-281) on those logits, weights within fp32 1e-6, and bit-identical
selections / union masks / histograms to smes_route_batch (the route kernels) on the same z.
Cases include reference-init logits (Stage-I gaps ~1e-10) and exact ties in both stages."""
import zlib

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from oracle import smes_oracle as O
from paper_2602_09386_b200 import _lib


def _bufs(T, B, E, ks, ka, C, dev="cuda"):
    i32 = lambda *s: torch.zeros(*s, dtype=torch.int32, device=dev)
    f64 = lambda *s: torch.zeros(*s, dtype=torch.float64, device=dev)
    return dict(shared=i32(B, ks), adaptive=i32(T, B, ka), active=i32(T, B, ks + ka),
                wsel=torch.zeros(T, B, ks + ka, device=dev), umask=i32(B, (E + 31) // 32), usize=i32(B),
                cu=i32(C, E), ca=i32(C, E), cm=f64(C, E), cd=f64(C, E), flag=i32(1))


def _front(h, w, b, tw, T, E, ks, ka, dm=True):
    call, ptr = _lib.call, _lib.ptr
    B, d = h.shape
    rpw = call("smes_route_rows_per_warp", B)
    C = call("smes_route_num_chunks", B, rpw)
    out = _bufs(T, B, E, ks, ka, C)
    z = torch.zeros(B, T * E, device="cuda")
    call("smes_route_front", ptr(h), d, ptr(w), ptr(b), ptr(tw), T, B, E, d, ks, ka, 4 * rpw, ptr(out["shared"]),
         ptr(out["adaptive"]), ptr(out["active"]), ptr(out["wsel"]), ptr(out["umask"]), ptr(out["usize"]),
         ptr(out["cu"]), ptr(out["ca"]), ptr(out["cm"]), ptr(out["cd"]) if dm else None, ptr(out["flag"]), ptr(z),
         torch.cuda.current_stream().cuda_stream)
    # the same logits through the two-kernel router
    ref = _bufs(T, B, E, ks, ka, C)
    call("smes_route_batch", ptr(z), E, T * E, None, ptr(tw), T, B, E, ks, ka, rpw, ptr(ref["shared"]),
         ptr(ref["adaptive"]), ptr(ref["active"]), ptr(ref["wsel"]), ptr(ref["umask"]), ptr(ref["usize"]),
         ptr(ref["cu"]), ptr(ref["ca"]), ptr(ref["cm"]), ptr(ref["cd"]), None, ptr(ref["flag"]), 0,
         torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    np_ = lambda d_: {k: v.cpu().numpy() for k, v in d_.items()}
    return np_(out), np_(ref), z.double().cpu().numpy()


CASES = {
    # name: (T, E, d, ks, ka, B, kind)
    "c2_reference_init": (8, 32, 256, 4, 2, 16384, "init"),
    "c2_trained_scale": (8, 32, 256, 4, 2, 5000, "x1000"),
    "c2_ties": (8, 32, 256, 4, 2, 3000, "ties"),
    "c2_d192_ragged_B": (8, 32, 192, 4, 2, 1000, "init"),
    "t2_e16_one_chunk": (2, 16, 64, 2, 1, 300, "x1000"),
    "t5_e32_chunk32": (5, 32, 256, 4, 2, 1536, "init"),
    "t3_e16_chunk16": (3, 16, 128, 2, 1, 640, "x1000"),
    "c1_shape": (4, 16, 128, 2, 1, 1024, "init"),
    "t16_e16": (16, 16, 128, 4, 2, 777, "x1000"),
    "small_B": (8, 32, 256, 4, 2, 5, "x1000"),
    # logits ~1e-7: Stage-I gaps ~1e-12, decided by the deviation form (y = e^x - 1 keeps its
    # relative accuracy); exact ties ("ties") take the fp64 recompute
    "c2_all_rows_exact": (8, 32, 256, 4, 2, 8192, "tiny"),
    "t16_e16_all_rows_exact": (16, 16, 128, 4, 2, 2000, "tiny"),
}
NO_DENSE_MASS = {"c2_reference_init", "c2_all_rows_exact", "t3_e16_chunk16"}


@pytest.mark.parametrize("name", list(CASES))
def test_route_front_vs_oracle_and_route_kernel(name):
    T, E, d, ks, ka, B, kind = CASES[name]
    assert _lib.call("smes_route_front_supported", T, E, d, ks, ka)
    rng = np.random.default_rng(zlib.crc32(name.encode()))
    scale = {"init": 1e-3, "x1000": 1.0, "ties": 0.0, "tiny": 1e-7}[kind] / d ** 0.5
    h = torch.tensor(rng.normal(size=(B, d)), dtype=torch.bfloat16, device="cuda")
    w = torch.tensor(rng.uniform(-scale, scale, size=(T * E, d)), dtype=torch.bfloat16, device="cuda")
    if kind == "ties":      # zero weights, bias in {0, 1, 2} per expert, equal for every task: the pooled
        #                     scores and the logits tie exactly (lowest index wins, routing.py:184-187)
        bias = torch.tensor(np.tile(rng.integers(0, 3, size=E), T), dtype=torch.float32, device="cuda")
    else:
        bias = torch.tensor(rng.normal(size=T * E) * scale, dtype=torch.float32, device="cuda")
    tw_np = rng.uniform(0.5, 2.0, size=T)
    tw = torch.tensor(tw_np, dtype=torch.float64, device="cuda")
    dm = name not in NO_DENSE_MASS          # chunk_dmass NULL: the training steps' variant
    cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
    _lib.call("smes_route_front_count_exact", _lib.ptr(cnt))
    try:
        g, r, z = _front(h, w, bias, tw, T, E, ks, ka, dm)
    finally:
        _lib.call("smes_route_front_count_exact", None)
    n_exact = int(cnt.item())
    if kind == "ties":
        assert n_exact > 0, n_exact               # exact pooled ties go through the fp64 recompute
    if kind == "x1000":
        assert n_exact <= B // 20, n_exact
    assert g["flag"][0] == 0
    # logits against RouterBank.logits on the same bf16 operands
    zr = h.double().cpu().numpy() @ w.double().cpu().numpy().T + bias.double().cpu().numpy()
    assert np.abs(z - zr).max() <= 1e-5 * max(np.abs(zr).max(), 1e-30)
    # bit-identical to the two-kernel router on the same z
    for k in ("shared", "adaptive", "active", "umask", "usize", "cu", "ca"):
        assert np.array_equal(g[k], r[k]), k
    assert np.abs(g["wsel"] - r["wsel"]).max() < 1e-6
    assert np.allclose(g["cm"].sum(0), r["cm"].sum(0), rtol=1e-6, atol=1e-9)
    if dm:      # dense mass from fp32 probabilities: the LoadStats fp32 tolerance
        assert np.allclose(g["cd"].sum(0), r["cd"].sum(0), rtol=1e-5, atol=1e-9)
    # index-exact against the oracle (f64 on the same fp32 logits)
    z3 = z.reshape(B, T, E).transpose(1, 0, 2)
    ref = O.route_batch(z3, ks, ka, tw_np)
    assert np.array_equal(g["shared"], ref.shared)
    assert np.array_equal(g["active"], ref.active)
    w_ref = np.take_along_axis(ref.weights, ref.active, axis=2)
    assert np.abs(g["wsel"] - w_ref).max() < 1e-6
    assert np.array_equal(g["ca"].sum(0), np.bincount(ref.active.reshape(-1), minlength=E))
    if kind == "init" and B >= 16384:
        assert O.stage1_margin(z3, ks) < 1e-8      # gaps far below fp32 resolution were decided exactly


def test_engine_uses_front_and_matches_unfused():
    """The engine's forward with the fused front equals the unfused router GEMM + route kernel."""
    from paper_2602_09386_b200 import SMESEngine
    from tests.helpers import make_case, to_engine_params
    B, T, E, d, ks, ka = 4096, 8, 32, 256, 4, 2
    p, h, y, lam, beta = make_case(3, B, T, E, d, d, ks, ka, d_ff=512)
    outs = []
    for front in (True, False):
        eng = SMESEngine(to_engine_params(p, lam, beta), B, ks, ka)
        assert eng.use_front
        eng.use_front = front
        eng.set_inputs(torch.tensor(h, device="cuda"), torch.tensor(y, device="cuda", dtype=torch.float32))
        eng.step()
        torch.cuda.synchronize()
        outs.append({k: getattr(eng, k).clone() for k in ("z", "active", "wsel", "umask", "stats_raw", "loss_out",
                                                           "grad_flat", "d_hidden")})
    a, b = outs
    assert torch.equal(a["active"], b["active"]) and torch.equal(a["umask"], b["umask"])
    assert (a["z"] - b["z"]).abs().max() <= 1e-5 * b["z"].abs().max()
    assert (a["wsel"] - b["wsel"]).abs().max() < 1e-6
    assert torch.allclose(a["stats_raw"], b["stats_raw"], rtol=1e-6, atol=1e-9)
    assert torch.allclose(a["loss_out"], b["loss_out"], rtol=1e-5)
    assert (a["grad_flat"] - b["grad_flat"]).abs().max() <= 1e-3 * b["grad_flat"].abs().max()
