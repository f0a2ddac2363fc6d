"""Generate golden fixtures for the SMES hot path from the REFERENCE itself.

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src \
        python tests/golden/make_golden.py

It imports ``taskmoe`` (the reference, read-only) and records, for seeded
small cases, the reference's outputs of ``route_batch`` (routing.py:235),
``build_execution_plan`` (execution.py:85), ``forward_sparse``
(model.py:267), ``compute_load_stats`` (balance.py:54) and ``backward``
(training.py:119).  The fixtures (``*.npz``) are committed; the GPU box never
reads /root/reference.

Layer-input gradient trick: the reference ``backward`` returns parameter
grads only.  To recover d(loss)/d(hidden) exactly from the reference, the
encoder is made the identity on a one-hot batch: x = I_B, encoder1 = I
(relu(I) = I), encoder2.weight = h^T, biases 0, so hidden = h and
grads['encoder2.weight'] = d_hidden^T @ I = d_hidden^T (training.py:214).
"""

from __future__ import annotations

import os
import sys

import numpy as np

import taskmoe as tm
from taskmoe.linalg import Affine
from taskmoe.experts import ExpertPool
from taskmoe.routing import RouterBank, RoutingBudget

OUT = os.path.dirname(os.path.abspath(__file__))


def routing_cases():
    cases = []
    rng = np.random.default_rng(1234)
    specs = [(3, 9, 11, 2, 1), (4, 32, 16, 2, 1), (2, 20, 6, 0, 2), (5, 17, 12, 3, 0),
             (8, 40, 32, 4, 2), (1, 8, 5, 1, 1), (4, 24, 64, 4, 2)]
    for i, (t, b, e, ks, ka) in enumerate(specs):
        z = rng.normal(size=(t, b, e))
        if i == 6:
            z *= 1e-3   # reference-init logit scale: tiny pooled gaps
        w = rng.uniform(0.0, 2.0, size=t) if i % 2 else None
        r = tm.route_batch(z, RoutingBudget(ks, ka), w)
        plan = tm.build_execution_plan(r.unions, e)
        d = dict(z=z, k_shared=ks, k_adaptive=ka, shared=r.shared, adaptive=r.adaptive,
                 active=r.active, weights=r.weights, full_probs=r.full_probs,
                 union_sizes=np.array([u.size for u in r.unions]),
                 union_flat=np.concatenate(r.unions), loads=plan.loads,
                 segment_offsets=plan.segment_offsets, gather_instances=plan.gather_instances,
                 gather_experts=plan.gather_experts, row_keys=plan.row_keys)
        if w is not None:
            d["task_weights"] = w
        cases.append(d)
    # ties: identical logits across experts -> lowest index wins (linalg.py:86-101)
    z = np.zeros((2, 4, 8))
    z[:, :, 3] = 1.0
    r = tm.route_batch(z, RoutingBudget(2, 1))
    cases.append(dict(z=z, k_shared=2, k_adaptive=1, shared=r.shared, adaptive=r.adaptive,
                      active=r.active, weights=r.weights, full_probs=r.full_probs,
                      union_sizes=np.array([u.size for u in r.unions]),
                      union_flat=np.concatenate(r.unions)))
    return cases


def layer_case(seed, b, t, e, d, d_out, ks, ka, act, beta, dense, lam_rand, w_rand, scale):
    rng = np.random.default_rng(seed)
    h = rng.normal(size=(b, d))
    experts = ExpertPool([Affine(rng.uniform(-1, 1, (d_out, d)) / np.sqrt(d),
                                 rng.normal(size=d_out) * 0.1) for _ in range(e)], act)
    tw = rng.uniform(0.2, 1.5, size=t) if w_rand else None
    routers = RouterBank([Affine(rng.uniform(-1, 1, (e, d)) * scale / np.sqrt(d),
                                 rng.normal(size=e) * scale) for _ in range(t)], tw)
    heads = [Affine(rng.uniform(-1, 1, (1, d_out)) / np.sqrt(d_out), rng.normal(size=1) * 0.1)
             for _ in range(t)]
    lam = rng.uniform(0.5, 2.0, size=t) if lam_rand else np.ones(t)
    model = tm.MoeModel(encoder1=Affine(np.eye(b), np.zeros(b)),
                        encoder2=Affine(h.T.copy(), np.zeros(d)),
                        experts=experts, routers=routers, heads=heads,
                        task_loss_weights=lam, lb_strength=beta,
                        budget=RoutingBudget(ks, ka), encoder_nonlinearity="relu")
    x = np.eye(b)
    res = tm.forward_sparse(x, model)
    assert np.abs(res.hidden - h).max() < 1e-12
    labels = (rng.uniform(size=(t, b)) < 0.3).astype(np.float64)
    bw = tm.backward(res, model, labels, dense_probs_in_stats=dense)
    g = bw.gradients
    out = dict(
        h=h, labels=labels, lam=lam, beta=beta, dense=int(dense), k_shared=ks, k_adaptive=ka,
        act=act,
        expert_w=np.stack([l.weight for l in experts.layers]),
        expert_b=np.stack([l.bias for l in experts.layers]),
        router_w=np.stack([m.weight for m in routers.maps]),
        router_b=np.stack([m.bias for m in routers.maps]),
        task_weights=routers.task_weights,
        head_w=np.stack([hd.weight[0] for hd in heads]), head_b=np.array([hd.bias[0] for hd in heads]),
        router_logits=res.router_logits, shared=res.routing.shared, adaptive=res.routing.adaptive,
        active=res.routing.active, weights=res.routing.weights,
        loads=res.plan.loads, segment_offsets=res.plan.segment_offsets,
        gather_instances=res.plan.gather_instances, packed_out=res.packed_out,
        task_reps=res.task_reps, head_logits=res.head_logits, predictions=res.predictions,
        task_value=bw.task_value, lb_value=bw.lb_value, total=bw.total,
        stats_counts=bw.stats.counts, stats_frequency=bw.stats.frequency, stats_mass=bw.stats.mass,
        g_expert_w=np.stack([g[f"expert_{i}.weight"] for i in range(e)]),
        g_expert_b=np.stack([g[f"expert_{i}.bias"] for i in range(e)]),
        g_router_w=np.stack([g[f"router_{i}.weight"] for i in range(t)]),
        g_router_b=np.stack([g[f"router_{i}.bias"] for i in range(t)]),
        g_head_w=np.stack([g[f"head_{i}.weight"][0] for i in range(t)]),
        g_head_b=np.array([g[f"head_{i}.bias"][0] for i in range(t)]),
        d_hidden=g["encoder2.weight"].T.copy(),
    )
    return out


def main():
    rc = routing_cases()
    np.savez_compressed(os.path.join(OUT, "routing_golden.npz"),
                        **{f"c{i}_{k}": v for i, c in enumerate(rc) for k, v in c.items()},
                        n=len(rc))
    specs = [
        # seed, B, T, E, d, d_out, Ks, Ka, act, beta, dense, lam_rand, w_rand, router_scale
        (0, 24, 3, 8, 12, 10, 2, 1, "relu", 0.01, False, False, False, 1.0),
        (1, 32, 4, 16, 16, 16, 2, 1, "relu", 0.05, False, True, True, 1.0),
        (2, 20, 2, 6, 8, 6, 1, 2, "identity", 0.1, True, True, False, 1.0),
        (3, 40, 4, 12, 16, 12, 0, 3, "relu", 0.0, False, False, True, 2.0),
        (4, 16, 3, 10, 8, 8, 3, 1, "relu", 0.02, True, False, False, 1e-3),
    ]
    for i, s in enumerate(specs):
        np.savez_compressed(os.path.join(OUT, f"layer_golden_{i}.npz"), **layer_case(*s))
    print("wrote", len(rc), "routing cases and", len(specs), "layer cases to", OUT)


if __name__ == "__main__":
    sys.exit(main())
