"""Per-chunk timeline of mlp_dgrad on CTA 0 (experiment build with -DSMES_TRACE):
    python tools/trace_dgrad.py build_var/_smes_trace.so"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2602_09386_b200 import _lib

lib = _lib.load(sys.argv[1])
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
W1 = (torch.randn(E, dff, d, generator=g, device=dev) / 16).to(torch.bfloat16)
G = (torch.randn(E, 8, dff, generator=g, device=dev) / 20).to(torch.bfloat16)
bits = torch.randint(0, 2 ** 31, (dff // 32, R), dtype=torch.int32, device=dev, generator=g)
C = (torch.randn(R, 16, generator=g, device=dev) * 1e-2).to(torch.bfloat16)
dX = torch.zeros(R, d, device=dev, dtype=torch.bfloat16)
dH = torch.zeros(R, dff, device=dev, dtype=torch.bfloat16)
st = torch.cuda.current_stream().cuda_stream
f = lambda: call("smes_mlp_dgrad", ptr(C), 16, R, ptr(G), 8, ptr(W1), E, d, dff, ptr(seg_t), ptr(bits), R, ptr(dX),
                 d, ptr(dH), dff, st)
for _ in range(3):
    f()
torch.cuda.synchronize()
f()
torch.cuda.synchronize()
ev = np.zeros(4 * 12 * 64, dtype=np.int64)
lib.smes_debug_trace(ev.ctypes.data_as(ctypes.c_void_p), 2)
ev = ev.reshape(4, 12, 64)
t0 = ev[0, 0, 0]
print("CTA0 per chunk: S_issued | dX: gotH gotD issued | epi: gotS ld gotH done")
for i in range(24):
    print(f"  {i:2d}", " ".join(f"{int(ev[0, r, i] - t0):8d}" for r in range(8)))
