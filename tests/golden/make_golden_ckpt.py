"""Generate the MOECKPT1 golden fixture from the REFERENCE itself (build container only):

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_ckpt.py

Writes ``ckpt_small.bin`` with the reference's ``save_model`` (checkpoint.py:38-66) and
``ckpt_small.npz`` holding every parameter block as the reference's ``load_model`` returns it,
plus a batch and the reference's ``forward_sparse`` predictions (model.py:267) on it.  Kernel-
friendly widths (d multiples of 32, d_out 128); the routers are scaled up from the near-zero
init so routing is decided by clear logit gaps.  The GPU box never reads /root/reference.
"""
import os

import numpy as np

from taskmoe.checkpoint import load_model, save_model
from taskmoe.model import forward_sparse, init_model
from taskmoe.routing import RoutingBudget

OUT = os.path.dirname(os.path.abspath(__file__))

rng = np.random.default_rng(2024)
model = init_model(rng, num_features=16, d_hidden=32, d_in=32, d_out=128, num_experts=8, num_tasks=4,
                   budget=RoutingBudget(2, 1), task_loss_weights=np.array([1.0, 0.5, 2.0, 1.5]),
                   lb_strength=0.02, expert_nonlinearity="relu",
                   router_task_weights=np.array([1.0, 1.0, 3.0, 0.5]))
for m in model.routers.maps:
    m.weight *= 3000.0
path = os.path.join(OUT, "ckpt_small.bin")
save_model(model, seed=77, path=path)
loaded, seed = load_model(path)
x = rng.standard_normal((256, 16))
res = forward_sparse(x, loaded, keep_cache=False)
blocks = {k.replace(".", "__"): v for k, v in loaded.parameter_blocks().items()}
np.savez_compressed(os.path.join(OUT, "ckpt_small.npz"), x=x, predictions=res.predictions, seed=seed,
                    shared=res.routing.shared, active=res.routing.active, **blocks)
print(path, os.path.getsize(path), "bytes")
