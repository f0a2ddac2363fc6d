import torch
x = torch.empty(143 * 1024 * 1024 // 2, dtype=torch.bfloat16, device="cuda")
y = torch.empty_like(x)
f = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
for name, fn in [("zero_ 143MB", lambda: x.zero_()), ("copy 143MB", lambda: y.copy_(x))]:
    for _ in range(3): fn()
    ts = []
    for _ in range(20):
        f.zero_()
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    t = sorted(ts)[10]
    by = x.numel() * 2 * (1 if "zero" in name else 2)
    print(name, f"{t*1e3:.1f} us", f"{by / t / 1e6:.0f} GB/s")
