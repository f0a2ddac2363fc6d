"""Two expert-parallel ranks in two PROCESSES sharing one GPU, over the hand-written CUDA-IPC
transport (ep.PeerComm: peer receive buffers mapped with cudaIpcOpenMemHandle, fused pack/put
kernels storing into them, flag-epoch handshakes).  gloo carries the IPC handles and the
replicated-gradient all-reduce.  Every rank checks its share against the single-process oracle
on the concatenated batch (global-batch mean objective).

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/ep2_on_one_gpu.py [--unfused]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import torch.distributed as dist

from oracle import smes_oracle as O
from paper_2602_09386_b200.ep import EPRank, ExpertParallelStep, PeerComm
from tests.helpers import make_case, rel
from tests.test_gpu_ep import _rank_params

dist.init_process_group("gloo")
r, n = dist.get_rank(), dist.get_world_size()
torch.cuda.set_device(0)
fused = "--unfused" not in sys.argv
single = "--single-relu" in sys.argv          # the reference expert: one relu pool
Bl, T, E, d, dff, ks, ka = 512, 4, 64, 128, (None if single else 256), 2, 1
p, h, y, lam, beta = make_case(11, n * Bl, T, E, d, d, ks, ka, d_ff=dff, router_scale=1.0, rand_lam=True)
rk = EPRank(_rank_params(p, lam, beta, r, n), E, r, n, Bl, ks, ka)
rk.set_inputs(torch.tensor(h[r * Bl:(r + 1) * Bl], device="cuda"),
              torch.tensor(y[:, r * Bl:(r + 1) * Bl], device="cuda", dtype=torch.float32))
comm = PeerComm(rk, fused=fused)
step = ExpertParallelStep([rk], comm)
for _ in range(3):           # slots and flag epochs are reused across steps
    step.step()
torch.cuda.synchronize()
rk.check()

z = rk.z.double().cpu().numpy().reshape(Bl, T, E)
allz = [None] * n
dist.all_gather_object(allz, z)
zt = np.concatenate(allz, 0).transpose(1, 0, 2)
route = O.route_batch(zt, ks, ka, p.task_weights)
plan = O.build_execution_plan(route.unions, E)
f = O.forward_sparse(h, p, ks, ka, logits=zt, frozen=route, frozen_plan=plan)
bw = O.backward(f, p, y, lam, beta)
sl = slice(r * Bl, (r + 1) * Bl)
El = E // n
errs = {
    "active": float(not np.array_equal(rk.active.cpu().numpy(), route.active[:, sl])),
    "preds": rel(rk.preds.cpu().numpy(), f.predictions[:, sl]),
    "loss": abs(rk.loss_out[0].item() - bw.task_value) / abs(bw.task_value),
    "lb": abs(rk.loss_out[1].item() - bw.stats.value) / abs(bw.stats.value),
    "router_w": rel(rk.g_router_w.cpu().numpy().reshape(T, E, d), bw.router_w),
    "head_w": rel(rk.g_head_w.cpu().numpy(), bw.head_w),
    "d_hidden": rel(rk.d_hidden.cpu().numpy(), bw.d_hidden[sl]),
}
for li in range(len(p.layers)):
    errs[f"W{li}"] = rel(rk.shard.g_layers[li][0].cpu().numpy(), bw.layers[li][0][r * El:(r + 1) * El])
    errs[f"b{li}"] = rel(rk.shard.g_layers[li][1].cpu().numpy(), bw.layers[li][1][r * El:(r + 1) * El])
bad = {k: v for k, v in errs.items() if not v < (1e-5 if k == "lb" else 2e-2)}
print(f"rank {r} ({'fused put' if fused else 'slot put'}{', single relu pool' if single else ''}): "
      + " ".join(f"{k}={v:.2e}" for k, v in errs.items()), flush=True)
comm.close()
dist.barrier()
dist.destroy_process_group()
if bad:
    raise SystemExit(f"rank {r} mismatches: {bad}")
print(f"EP2 IPC OK rank {r}", flush=True)
