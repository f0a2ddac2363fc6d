"""Shared test helpers: seeded parameters in both the oracle (numpy f64) and the
engine (torch) layouts, bf16-rounded identically so both sides see the same
operands (feed the oracle the identical layer input and weights)."""
from __future__ import annotations

import numpy as np
import torch

from oracle import smes_oracle as O


def bf16_round(a: np.ndarray) -> np.ndarray:
    return torch.from_numpy(np.asarray(a, dtype=np.float32)).to(torch.bfloat16).to(torch.float64).numpy()


def make_case(seed, B, T, E, d, d_out, ks, ka, d_ff=None, router_scale=1e-3, beta=0.01,
              rand_bias=True, rand_task_w=False, rand_lam=False, last_act=None):
    rng = np.random.default_rng(seed)
    p = O.init_layer_params(rng, d, d_out, E, T, d_ff=d_ff, router_scale=router_scale)
    layers = []
    for (w, b, act) in p.layers:
        b = rng.normal(size=b.shape) * 0.1 if rand_bias else b
        layers.append((bf16_round(w), b.astype(np.float32).astype(np.float64), act))
    if last_act is not None:
        w, b, _ = layers[-1]
        layers[-1] = (w, b, last_act)
    p.layers = layers
    p.router_w = bf16_round(p.router_w)
    p.router_b = (rng.normal(size=p.router_b.shape) * router_scale).astype(np.float32).astype(np.float64)
    p.head_w = p.head_w.astype(np.float32).astype(np.float64)
    p.head_b = (rng.normal(size=T) * 0.1).astype(np.float32).astype(np.float64)
    p.task_weights = rng.uniform(0.5, 1.5, T) if rand_task_w else None
    lam = rng.uniform(0.5, 2.0, T).astype(np.float32).astype(np.float64) if rand_lam else np.ones(T)
    h = bf16_round(rng.normal(size=(B, d)))
    y = (rng.uniform(size=(T, B)) < np.resize([0.3, 0.1, 0.05, 0.2], T)[:, None]).astype(np.float64)
    return p, h, y, lam, beta


def to_engine_params(p: O.LayerParams, lam, beta, dev="cuda"):
    from paper_2602_09386_b200 import ExpertLayer, SMESParams
    t = lambda a, dt=torch.float32: torch.as_tensor(np.asarray(a), dtype=dt, device=dev)
    return SMESParams(
        router_w=t(p.router_w), router_b=t(p.router_b),
        layers=[ExpertLayer(t(w), t(b), act) for (w, b, act) in p.layers],
        head_w=t(p.head_w), head_b=t(p.head_b),
        task_weights=None if p.task_weights is None else t(p.task_weights, torch.float64),
        task_loss_weights=t(lam), lb_strength=beta)


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    den = np.abs(b).max()
    return float(np.abs(a - b).max() / den) if den > 0 else float(np.abs(a - b).max())
