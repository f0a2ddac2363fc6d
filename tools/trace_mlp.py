"""Wait-cycle attribution of mlp_fwd (experiment build with -DSMES_TRACE, tools/variant_build.sh):
    python tools/trace_mlp.py build_var/_smes_trace.so"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2602_09386_b200 import _lib

NAMES = ["prod:xempty", "prod:wempty", "gprod:gempty", "smma:sempty", "smma:xfull", "smma:wfull",
         "pmma:hfull", "pmma:gfull", "pmma:pempty", "epi:sfull", "epi:hempty", "epi:pfull", "epi:bulk_read",
         "T epi(w4)", "T smma(w1)", "T prod(w0)"]


def main(path):
    _lib._lib = None
    lib = _lib.load(path)
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
    X = torch.randn(R, d + 64, generator=g, device=dev).to(torch.bfloat16)
    W1 = (torch.randn(E, dff, d, generator=g, device=dev) / 16).to(torch.bfloat16)
    b1 = torch.randn(E, dff, generator=g, device=dev) * 0.1
    G = (torch.randn(E, 8, dff, generator=g, device=dev) / 20).to(torch.bfloat16)
    c = torch.randn(E, 8, device=dev)
    H = torch.zeros(R, dff + 64, device=dev, dtype=torch.bfloat16)
    bits = torch.zeros(dff // 32, R, dtype=torch.int32, device=dev)
    P = torch.zeros(R, 8, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    mode = os.environ.get("MODE", "h")

    def fwd():
        call("smes_mlp_fwd2" if os.environ.get("FWD2") else "smes_mlp_fwd", ptr(X), d + 64, R, ptr(W1), ptr(b1), ptr(G), ptr(c), 8, E, d, dff, ptr(seg_t), ptr(bits),
             R, ptr(H) if mode == "h" else None, dff + 64 if mode == "h" else 0, ptr(P), 8, st) if mode != "x" else call("smes_mlp_fwd", ptr(X), d + 64, R, ptr(W1), ptr(b1), ptr(G), ptr(c), 8, E, d, dff, ptr(seg_t), None, R, None, 0, ptr(P), 8, st)

    print("fwd2 pair grid:", lib.smes_debug_trace(None, 3))
    for _ in range(3):
        fwd()
    torch.cuda.synchronize()
    out = np.zeros(148 * 16, dtype=np.uint64)
    lib.smes_debug_trace(None, 1)
    fwd()
    torch.cuda.synchronize()
    lib.smes_debug_trace(out.ctypes.data_as(ctypes.c_void_p), 0)
    t = out.reshape(148, 16).astype(np.float64)
    tot = t[:, 13].mean()
    print("per-CTA epi cycles min/mean/max", t[:, 13].min(), tot, t[:, 13].max(), "units/tiles min/max",
          t[:, 12].min(), t[:, 12].max())
    g0, g1 = out.reshape(148, 16)[:, 10].astype(np.int64), out.reshape(148, 16)[:, 11].astype(np.int64)
    print(f"globaltimer: start spread {(g0.max() - g0.min()) / 1e3:.1f} us, first start -> last end "
          f"{(g1.max() - g0.min()) / 1e3:.1f} us, mean CTA span {(g1 - g0).mean() / 1e3:.1f} us, "
          f"implied SM clock {t[:, 13].mean() / ((g1 - g0).mean()):.3f} GHz")
    print("slowest CTAs", np.argsort(-t[:, 13])[:8], "fastest", np.argsort(t[:, 13])[:8])
    print(f"{os.path.basename(path)} mode={mode} kernel cycles (epi w4) {tot:.0f}")
    for i, n in enumerate(NAMES):
        print(f"  {n:16s} {t[:, i].mean():10.0f}  {t[:, i].mean() / tot * 100:5.1f}%")
    ev = np.zeros(4 * 12 * 64, dtype=np.int64)
    lib.smes_debug_trace(ev.ctypes.data_as(ctypes.c_void_p), 2)
    ev = ev.reshape(4, 12, 64)
    t0 = ev[0, 0, 0]
    print("CTA0 per chunk (cycles from first S start): S_start S_issued epi_gotS epi_ld epi_gotH epi_done P_start P_issued | relu bits sts fence")
    for i in range(24):
        print(f"  {i:2d}", " ".join(f"{int(ev[0, r, i] - t0):8d}" for r in range(12)))


for p in sys.argv[1:]:
    main(p)
