"""Micro-benchmark of the expert-MLP kernels at the c2 shape (E=32, ~8.7K rows per expert):
fused (csrc/mlp.cu) vs the unfused grouped-GEMM sequence.  CUDA events, L2 flushed.
    python tools/bench_mlp.py [path/to/_smes.so ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2602_09386_b200 import _lib


def run(lib_path):
    _lib._lib = None
    _lib.load(lib_path)
    call, ptr = _lib.call, _lib.ptr
    dev = "cuda"
    g = torch.Generator(device=dev).manual_seed(0)
    E, d, dff, T = 32, 256, 512, 8
    loads = [8700 + (e * 37) % 200 for e in range(E)]
    seg = [0]
    for n in loads:
        seg.append(seg[-1] + (n + 127) // 128 * 128)
    R = seg[-1] + 128
    seg_t = torch.tensor(seg, dtype=torch.int32, device=dev)
    X = (torch.randn(R, d + 64, generator=g, device=dev)).to(torch.bfloat16)
    W1 = (torch.randn(E, dff, d, generator=g, device=dev) / 16).to(torch.bfloat16)
    b1 = torch.randn(E, dff, generator=g, device=dev) * 0.1
    G = (torch.randn(E, 8, dff, generator=g, device=dev) / 20).to(torch.bfloat16)
    c = torch.randn(E, 8, device=dev)
    H = torch.zeros(R, dff + 64, device=dev, dtype=torch.bfloat16)
    bits = torch.zeros(dff // 32, R, dtype=torch.int32, device=dev)
    P = torch.zeros(R, 8, device=dev)
    C = (torch.randn(R, 16, generator=g, device=dev) * 1e-2).to(torch.bfloat16)
    dX = torch.zeros(R, d, device=dev, dtype=torch.bfloat16)
    dH = torch.zeros(R, dff, device=dev, dtype=torch.bfloat16)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream().cuda_stream

    def fwd():
        call("smes_mlp_fwd", ptr(X), d + 64, R, ptr(W1), ptr(b1), ptr(G), ptr(c), 8, E, d, dff, ptr(seg_t), ptr(bits),
             R, ptr(H), dff + 64, ptr(P), 8, st)

    def fwd2():
        call("smes_mlp_fwd2", ptr(X), d + 64, R, ptr(W1), ptr(b1), ptr(G), ptr(c), 8, E, d, dff, ptr(seg_t), ptr(bits),
             R, ptr(H), dff + 64, ptr(P), 8, st)

    def fwd_noh():
        call("smes_mlp_fwd", ptr(X), d + 64, R, ptr(W1), ptr(b1), ptr(G), ptr(c), 8, E, d, dff, ptr(seg_t), ptr(bits),
             R, None, 0, ptr(P), 8, st)

    def fwd_nobits():
        call("smes_mlp_fwd", ptr(X), d + 64, R, ptr(W1), ptr(b1), ptr(G), ptr(c), 8, E, d, dff, ptr(seg_t), None,
             R, None, 0, ptr(P), 8, st)

    def dgrad():
        call("smes_mlp_dgrad", ptr(C), 16, R, ptr(G), 8, ptr(W1), E, d, dff, ptr(seg_t), ptr(bits), R, ptr(dX), d,
             ptr(dH), dff, st)

    def dgrad2():
        call("smes_mlp_dgrad2", ptr(C), 16, R, ptr(G), 8, ptr(W1), E, d, dff, ptr(seg_t), ptr(bits), R, ptr(dX), d,
             ptr(dH), dff, st)

    def dgrad_nodh():
        call("smes_mlp_dgrad", ptr(C), 16, R, ptr(G), 8, ptr(W1), E, d, dff, ptr(seg_t), ptr(bits), R, ptr(dX), d,
             None, 0, st)

    def unfused_fwd():
        call("smes_gemm_ragged_m", ptr(X), d + 64, R, ptr(W1), E, dff, d, 0, ptr(seg_t), ptr(b1), 1, ptr(bits), None, R,
             ptr(H), dff + 64, 0, R, st)
        call("smes_gemm_ragged_m", ptr(H), dff + 64, R, ptr(G), E, 8, dff, 0, ptr(seg_t), ptr(c), 0, None, None, 0,
             ptr(P), 8, 1, R, st)

    out = {}
    only = os.environ.get("ONLY")
    for name, fn in [("mlp_fwd", fwd), ("mlp_fwd2", fwd2), ("mlp_fwd_noH", fwd_noh), ("mlp_fwd_noH_nobits", fwd_nobits), ("mlp_dgrad", dgrad), ("mlp_dgrad2", dgrad2), ("mlp_dgrad_nodH", dgrad_nodh),
                     ("unfused_fwd", unfused_fwd)]:
        if only and not name.startswith(only):
            continue
        for _ in range(3):
            fn()
        ts = []
        for _ in range(20):
            flush.zero_()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            fn()
            e.record()
            torch.cuda.synchronize()
            ts.append(s.elapsed_time(e) * 1000)
        ts.sort()
        out[name] = ts[len(ts) // 2]
    rows = sum(loads)
    print(os.path.basename(lib_path), " ".join(f"{k}={v:.1f}us" for k, v in out.items()), f"rows={rows}")


for p in sys.argv[1:] or [_lib.LIB_PATH]:
    run(p)
