"""Time the fused router front at c2 (reference-init router weights) for one or more library builds:
    python tools/front_time.py [path/to/_smes_variant.so ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2602_09386_b200 import _lib

paths = sys.argv[1:] or [_lib.LIB_PATH]
for path in paths:
    _lib._lib = None
    _lib.load(path)
    call, ptr = _lib.call, _lib.ptr
    T, B, E, d, ks, ka = 8, 16384, 32, 256, 4, 2
    K = ks + ka
    g = torch.Generator(device="cuda").manual_seed(0)
    h = torch.randn(B, d, device="cuda", generator=g).bfloat16()
    w = ((torch.rand(T * E, d, device="cuda", generator=g) * 2 - 1) * 1e-3 / 16).bfloat16()
    bias = torch.zeros(T * E, device="cuda")
    tw = torch.ones(T, dtype=torch.float64, device="cuda")
    rpw = call("smes_route_rows_per_warp", B)
    C = call("smes_route_num_chunks", B, rpw)
    i32 = lambda *s: torch.zeros(*s, dtype=torch.int32, device="cuda")
    f64 = lambda *s: torch.zeros(*s, dtype=torch.float64, device="cuda")
    sh, ad, ac, ws = i32(B, ks), i32(T, B, ka), i32(T, B, K), torch.zeros(T, B, K, device="cuda")
    um, us, cu, ca, cm, cd, fl = i32(B, 1), i32(B), i32(C, E), i32(C, E), f64(C, E), f64(C, E), i32(1)
    st = torch.cuda.current_stream().cuda_stream
    zo = torch.zeros(B, T * E, device="cuda") if os.environ.get("ZOUT") else None
    f = lambda: call("smes_route_front", ptr(h), d, ptr(w), ptr(bias), ptr(tw), T, B, E, d, ks, ka, 4 * rpw,
                              ptr(sh), ptr(ad), ptr(ac), ptr(ws), ptr(um), ptr(us), ptr(cu), ptr(ca), ptr(cm), ptr(cd) if os.environ.get("DM") else None,
                              ptr(fl), ptr(zo), st)
    cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
    if hasattr(_lib.load(), "smes_route_front_count_exact"):
        call("smes_route_front_count_exact", ptr(cnt))
        f()
        torch.cuda.synchronize()
        print("rows through the fp64 recompute:", int(cnt.item()), "of", B)
        call("smes_route_front_count_exact", None)
    for _ in range(5):
        f()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(50):
        f()
    e.record()
    torch.cuda.synchronize()
    print(os.path.basename(path), f"{s.elapsed_time(e) / 50 * 1000:.1f} us",
          "mean union", float(us.double().mean()))
