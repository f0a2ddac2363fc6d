import sys, torch
sys.path.insert(0, '/root/repo')
from paper_2602_09386_b200._lib import call, ptr
dev = "cuda"
g = torch.Generator(device=dev).manual_seed(1)
I, J = 512, 256
loads = [70000]
seg = [0, 70016]
R = seg[-1]
pb = torch.zeros(R, I, device=dev); pb[:70000] = torch.randn(70000, I, generator=g, device=dev)
qb = torch.zeros(R, J + 64, device=dev); qb[:70000, :J] = torch.randn(70000, J, generator=g, device=dev)
pb, qb = pb.bfloat16(), qb.bfloat16()
seg_t = torch.tensor(seg, dtype=torch.int32, device=dev)
out = torch.full((1, I, J), float("nan"), device=dev)
call("smes_gemm_ragged_k", ptr(pb), I, ptr(qb), J + 64, R, 1, I, J, ptr(seg_t), ptr(out), None, torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
ref = pb.float().T @ qb[:, :J].float()
print("nan", torch.isnan(out).sum().item(), "max err", (out[0] - ref).abs().max().item(), "ref max", ref.abs().max().item())
d = (out[0] - ref).abs()
for i0 in range(0, I, 128):
    for j0 in range(0, J, 64):
        print(i0, j0, round(d[i0:i0+128, j0:j0+64].max().item(), 3), end="; ")
    print()
print("ratio sample", (out[0, :4, :4] / ref[:4, :4]))
