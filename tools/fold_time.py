"""Time smes_fold_heads / smes_unfold_grads at the c2 shape (CUDA events, warm)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2602_09386_b200 import _lib

for path in sys.argv[1:] or [_lib.LIB_PATH]:
    _lib._lib = None
    _lib.load(path)
    call, ptr = _lib.call, _lib.ptr
    E, T, ldg, do, di = 32, 8, 8, 256, 512
    dev = "cuda"
    hw = torch.randn(T, do, device=dev)
    W = torch.randn(E, do, di, device=dev).to(torch.bfloat16)
    b = torch.randn(E, do, device=dev)
    G = torch.zeros(E, ldg, di, device=dev, dtype=torch.bfloat16)
    c = torch.zeros(E, ldg, device=dev)
    work = torch.zeros(call("smes_fold_work_floats", E, T, do, di), device=dev)
    Q = torch.randn(E, ldg, di, device=dev)
    cs = torch.randn(E, T, device=dev)
    dW = torch.zeros(E, do, di, device=dev)
    db = torch.zeros(E, do, device=dev)
    dh = torch.zeros(T, do, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    f = lambda: call("smes_fold_heads", E, T, ldg, do, di, ptr(hw), ptr(W), ptr(b), ptr(G), ptr(c), ptr(work), st)
    u = lambda: call("smes_unfold_grads", E, T, ldg, do, di, ptr(Q), ldg * di, di, 1, ptr(cs), T, ptr(hw), ptr(W),
                     ptr(b), ptr(dW), ptr(db), ptr(work), ptr(dh), st)
    for name, fn in (("fold", f), ("unfold", u)):
        for _ in range(5):
            fn()
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        torch.cuda.synchronize()
        s.record()
        for _ in range(100):
            fn()
        e.record()
        torch.cuda.synchronize()
        print(os.path.basename(path), name, f"{s.elapsed_time(e) / 100 * 1000:.1f} us")
