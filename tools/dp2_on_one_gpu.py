"""Two data-parallel ranks of the REAL engine on one GPU (gloo over CUDA tensors): the rank
results must equal one process on the concatenated batch (DP exactness of the step incl. its
backward side stream).  Optional arguments: ``peer`` -- LoadStats through the one-shot CUDA-IPC
peer all-reduce (csrc/comm.cu); ``overlap`` -- gradient buckets reduced on a communication stream
as the backward finishes them.
torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/dp2_on_one_gpu.py [peer] [overlap]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as dist

from paper_2602_09386_b200 import SMESEngine
from paper_2602_09386_b200.dp import DataParallelStep
from tests.helpers import make_case, to_engine_params

dist.init_process_group("gloo")
r, n = dist.get_rank(), dist.get_world_size()
B = 4096
p, h, y, lam, beta = make_case(7, B * n, 8, 32, 256, 256, 4, 2, d_ff=512, router_scale=1.0)
eng = SMESEngine(to_engine_params(p, lam, beta), B, 4, 2)
eng.set_inputs(torch.tensor(h[r * B:(r + 1) * B], device="cuda"),
               torch.tensor(y[:, r * B:(r + 1) * B], device="cuda", dtype=torch.float32))
step = DataParallelStep(eng, stats="peer" if "peer" in sys.argv else "group", overlap="overlap" in sys.argv)
step.capture()
for _ in range(3):
    step.step()
torch.cuda.synchronize()
mine = {k: v.detach().float().cpu().numpy() for k, v in eng.gradients().items()}
loss = eng.loss_out.cpu().numpy().copy()
if r == 0:
    ref = SMESEngine(to_engine_params(p, lam, beta), B * n, 4, 2)
    ref.set_inputs(torch.tensor(h, device="cuda"), torch.tensor(y, device="cuda", dtype=torch.float32))
    ref.step()
    torch.cuda.synchronize()
    refg = {k: v.detach().float().cpu().numpy() for k, v in ref.gradients().items()}
    worst = max(np.abs(mine[k] - refg[k]).max() / max(np.abs(refg[k]).max(), 1e-30) for k in refg)
    lref = ref.loss_out.cpu().numpy()
    print(f"dp2 vs single: max rel grad diff {worst:.3e}; loss {loss} vs {lref}", flush=True)
    # the DP loss is all-reduced (global-batch objective): equal to one process up to fp32 order
    assert worst < 2e-2 and np.allclose(loss, lref, rtol=1e-5)
    print("DP2 OK")
dist.barrier()
dist.destroy_process_group()
