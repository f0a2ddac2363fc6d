import sys, os, torch
sys.path.insert(0, os.getcwd())
from paper_2602_09386_b200 import _lib
for path in sys.argv[1:]:
    _lib._lib = None
    lib = _lib.load(path)
    call, ptr = _lib.call, _lib.ptr
    T, B, E = (int(x) for x in os.environ.get("TBE", "8,16384,32").split(","))
    ks, ka = 4, 2
    K = ks + ka
    g = torch.Generator(device="cuda").manual_seed(0)
    z = torch.randn(T, B, E, device="cuda", generator=g) * float(os.environ.get("ZSCALE", "1"))
    # LAYOUT=bte: z stored (B, T, E) as the engines write it (stride_t = E, stride_b = T * E)
    bte = os.environ.get("LAYOUT") == "bte"
    if bte:
        z = z.permute(1, 0, 2).contiguous()
    st_t, st_b = (E, T * E) if bte else (B * E, E)
    tw = torch.ones(T, dtype=torch.float64, device="cuda")
    rpw = call("smes_route_rows_per_warp", B)
    C = call("smes_route_num_chunks", B, rpw)
    i32 = lambda *s: torch.zeros(*s, dtype=torch.int32, device="cuda")
    sh, ad, ac = i32(B, ks), i32(T, B, ka), i32(T, B, K)
    ws = torch.zeros(T, B, K, device="cuda")
    um, us = i32(B, (E + 31) // 32), i32(B)
    cu, ca = i32(C, E), i32(C, E)
    cm, cd = torch.zeros(C, E, dtype=torch.float64, device="cuda"), torch.zeros(C, E, dtype=torch.float64, device="cuda")
    fl = i32(1)
    st = torch.cuda.current_stream().cuda_stream
    f = lambda: call("smes_route_batch", ptr(z), st_t, st_b, None, ptr(tw), T, B, E, ks, ka, rpw, ptr(sh), ptr(ad), ptr(ac), ptr(ws), ptr(um), ptr(us), ptr(cu), ptr(ca), ptr(cm), ptr(cd) if os.environ.get("DM") else None, None, ptr(fl), 0, st)
    for _ in range(5): f()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize(); s.record()
    for _ in range(50): f()
    e.record(); torch.cuda.synchronize()
    print(os.path.basename(path), f"{s.elapsed_time(e)/50*1000:.1f} us", int(us.sum()))
