"""Model container + sparse forward -- drop-in for taskmoe/model.py (forward_sparse).

``forward_sparse(batch, model, ...)`` keeps the reference signature and
result type.  The encoder (two Affine layers, model.py:188-199) runs on the
same tcgen05 GEMM (one group); the SMES layer runs through a cached
:class:`SMESEngine` (router GEMM -> fused router -> plan -> grouped expert
GEMMs -> head projections -> combine/heads).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import torch

from . import engine as _engine
from ._lib import call, ptr
from .errors import ConfigError, ShapeError, StateError
from .execution import ExecutionPlan, ExpertPool, FlopCounter
from .linalg import Affine, init_affine
from .routing import BatchRouting, RoutingBudget, _stream

__all__ = ["MoeModel", "RouterBank", "ForwardResult", "forward_sparse", "init_model"]

ROUTER_INIT_SCALE = 1e-3   # model.py:32
ENCODER_BIAS_INIT = 0.01   # model.py:33


@dataclass
class RouterBank:
    """T routers d_in -> E, stacked: weight (T, E, d_in), bias (T, E) (routing.py:64-103)."""
    weight: torch.Tensor
    bias: torch.Tensor
    task_weights: torch.Tensor | None = None

    def __post_init__(self):
        if self.weight.ndim != 3 or self.bias.shape != self.weight.shape[:2]:
            raise ShapeError(f"router bank expects weight (T,E,d) and bias (T,E), got {tuple(self.weight.shape)}")
        if self.task_weights is None:
            self.task_weights = torch.ones(self.weight.shape[0], dtype=torch.float64)
        self.task_weights = torch.as_tensor(self.task_weights, dtype=torch.float64)
        if self.task_weights.shape != (self.weight.shape[0],):
            raise ShapeError(f"expected {self.weight.shape[0]} task weights")
        if bool((self.task_weights < 0).any()):
            raise ConfigError("task pooling weights must be non-negative")

    @property
    def num_tasks(self):
        return self.weight.shape[0]

    @property
    def num_experts(self):
        return self.weight.shape[1]

    @property
    def d_in(self):
        return self.weight.shape[2]


@dataclass
class MoeModel:
    """Encoder, expert stack, task routers, task heads (model.py:36-111).  ``experts`` is one
    ExpertPool (the reference expert) or a list of pools chained d -> d_ff -> d_out.
    ``encoder1``/``encoder2`` may be None: the batch is then the encoded hidden (B, d_in)."""
    encoder1: Affine | None
    encoder2: Affine | None
    experts: object
    routers: RouterBank
    head_w: torch.Tensor            # (T, d_out)
    head_b: torch.Tensor            # (T,)
    task_loss_weights: torch.Tensor
    lb_strength: float
    budget: RoutingBudget
    encoder_nonlinearity: str = "relu"
    _engines: dict = field(default_factory=dict, repr=False)

    def __post_init__(self):
        pools = self.pools
        t = self.routers.num_tasks
        if self.head_w.shape != (t, pools[-1].d_out):
            raise ConfigError("heads must map d_out -> 1 for every task")
        self.task_loss_weights = torch.as_tensor(self.task_loss_weights, dtype=torch.float64)
        if self.task_loss_weights.shape != (t,):
            raise ConfigError(f"expected {t} task loss weights")
        if bool((self.task_loss_weights < 0).any()) or self.lb_strength < 0:
            raise ConfigError("loss weights and regularizer strength must be non-negative")
        if self.routers.num_experts != pools[0].num_experts:
            raise ConfigError("router width must equal the expert count")
        self.budget.validate(pools[0].num_experts)

    @property
    def pools(self) -> list:
        return list(self.experts) if isinstance(self.experts, (list, tuple)) else [self.experts]

    @property
    def num_tasks(self):
        return self.routers.num_tasks

    @property
    def num_experts(self):
        return self.routers.num_experts

    @property
    def d_in(self):
        return self.routers.d_in

    @property
    def d_out(self):
        return self.pools[-1].d_out

    def parameter_blocks(self) -> dict:
        """Named parameter views in the reference's order and names (model.py:94-111)."""
        blocks = {}
        if self.encoder1 is not None:
            blocks.update({"encoder1.weight": self.encoder1.weight, "encoder1.bias": self.encoder1.bias,
                           "encoder2.weight": self.encoder2.weight, "encoder2.bias": self.encoder2.bias})
        pools = self.pools
        for li, pool in enumerate(pools):
            for e in range(pool.num_experts):
                pre = f"expert_{e}" if len(pools) == 1 else f"expert{li}_{e}"
                blocks[pre + ".weight"] = pool.weight[e]
                blocks[pre + ".bias"] = pool.bias[e]
        for t in range(self.num_tasks):
            blocks[f"router_{t}.weight"] = self.routers.weight[t]
            blocks[f"router_{t}.bias"] = self.routers.bias[t]
        for t in range(self.num_tasks):
            blocks[f"head_{t}.weight"] = self.head_w[t:t + 1]
            blocks[f"head_{t}.bias"] = self.head_b[t:t + 1]
        return blocks

    def smes_params(self) -> _engine.SMESParams:
        return _engine.SMESParams(
            router_w=self.routers.weight, router_b=self.routers.bias,
            layers=[_engine.ExpertLayer(p.weight, p.bias, p.nonlinearity) for p in self.pools],
            head_w=self.head_w, head_b=self.head_b, task_weights=self.routers.task_weights,
            task_loss_weights=self.task_loss_weights, lb_strength=self.lb_strength)


def init_model(gen: torch.Generator | None, num_features: int, d_hidden: int, d_in: int, d_out: int,
               num_experts: int, num_tasks: int, budget: RoutingBudget, task_loss_weights=None,
               lb_strength: float = 0.0, expert_nonlinearity: str = "identity", encoder_nonlinearity: str = "relu",
               router_task_weights=None, d_ff: int | None = None, device="cuda") -> MoeModel:
    """Fan-in uniform init, near-zero routers (model.py:117-156).  ``d_ff`` adds the
    BASELINE 'expert MLP' (relu d_in -> d_ff, identity d_ff -> d_out)."""
    enc1 = init_affine(gen, d_hidden, num_features, bias_value=ENCODER_BIAS_INIT, device=device)
    enc2 = init_affine(gen, d_in, d_hidden, bias_value=ENCODER_BIAS_INIT, device=device)
    from .execution import init_expert_pool
    if d_ff is None:
        experts = init_expert_pool(gen, num_experts, d_in, d_out, expert_nonlinearity, device)
    else:
        experts = [init_expert_pool(gen, num_experts, d_in, d_ff, "relu", device),
                   init_expert_pool(gen, num_experts, d_ff, d_out, "identity", device)]
    s = ROUTER_INIT_SCALE / d_in ** 0.5
    rw = ((torch.rand(num_tasks, num_experts, d_in, generator=gen, dtype=torch.float64) * 2 - 1) * s).float()
    routers = RouterBank(rw.to(device), torch.zeros(num_tasks, num_experts, device=device), router_task_weights)
    hw = ((torch.rand(num_tasks, d_out, generator=gen, dtype=torch.float64) * 2 - 1) / d_out ** 0.5).float()
    lam = torch.ones(num_tasks) if task_loss_weights is None else torch.as_tensor(task_loss_weights)
    return MoeModel(enc1, enc2, experts, routers, hw.to(device), torch.zeros(num_tasks, device=device), lam,
                    lb_strength, budget, encoder_nonlinearity)


@dataclass
class ForwardResult:
    """Predictions plus what backward needs (model.py:159-185)."""
    mode: str
    predictions: torch.Tensor      # (T, B)
    head_logits: torch.Tensor      # (T, B)
    task_reps: torch.Tensor        # (T, B, d_out)
    routing: BatchRouting
    plan: ExecutionPlan
    expert_flops: int
    hidden: torch.Tensor | None = None
    router_logits: torch.Tensor | None = None
    _engine: object = None
    _step: int = -1
    _enc: dict | None = None

    def mean_union(self) -> float:
        return float(self.routing.usize.double().mean())

    def max_union(self) -> int:
        return int(self.routing.usize.max())


def _round(x, m):
    return (x + m - 1) // m * m


def _gemm(a, lda, rows, w, n, k, bias, act, out, ldc, out_fp32, m_limit, bits_out=None, bits_ld=0, b_mn=0,
          bits_in=None):
    seg = torch.tensor([0, _round(rows, 128)], dtype=torch.int32, device=a.device)
    call("smes_gemm_ragged_m", ptr(a), lda, rows, ptr(w), 1, n, k, b_mn, ptr(seg), ptr(bias), act, ptr(bits_out),
         ptr(bits_in), bits_ld, ptr(out), ldc, out_fp32, m_limit, _stream())


def _encode(x: torch.Tensor, model: MoeModel, eng) -> dict:
    """encoder1 -> act -> encoder2 on the tcgen05 GEMM (model.py:188-199)."""
    B, F = x.shape
    dev = x.device
    Fp = _round(F, 8)
    xb = torch.zeros(B, Fp, dtype=torch.bfloat16, device=dev)
    xb[:, :F] = x
    w1 = torch.zeros(model.encoder1.d_out, Fp, dtype=torch.bfloat16, device=dev)
    w1[:, :F] = model.encoder1.weight
    dh = model.encoder1.d_out
    mid = torch.zeros(_round(B, 128), dh, dtype=torch.bfloat16, device=dev)
    relu = model.encoder_nonlinearity == "relu"
    bits = torch.zeros(dh // 32, _round(B, 128), dtype=torch.int32, device=dev) if relu and dh % 32 == 0 else None
    if relu and bits is None:
        raise ShapeError(f"encoder hidden width {dh} must be a multiple of 32")
    _gemm(xb, Fp, B, w1.reshape(1, dh, Fp).contiguous(), dh, Fp, model.encoder1.bias.float().contiguous(),
          1 if relu else 0, mid, dh, 0, B, bits_out=bits, bits_ld=_round(B, 128))
    w2 = model.encoder2.weight.to(torch.bfloat16).reshape(1, model.d_in, dh).contiguous()
    _gemm(mid, dh, B, w2, model.d_in, dh, model.encoder2.bias.float().contiguous(), 0, eng.h, eng.ldh, 0, B)
    return dict(xb=xb, Fp=Fp, F=F, mid=mid, bits=bits, w1=w1, w2=w2)


def _get_engine(model: MoeModel, B: int, dense: bool = False) -> _engine.SMESEngine:
    key = (B, bool(dense))
    eng = model._engines.get(key)
    if eng is None:
        eng = _engine.SMESEngine(model.smes_params(), B, model.budget.k_shared, model.budget.k_adaptive,
                                 dense_probs_in_stats=dense, device=model.head_w.device)
        eng.step_id = 0
        model._engines[key] = eng
    else:
        eng.p = model.smes_params()
        eng.refresh_weights()
    return eng


def forward_sparse(batch, model: MoeModel, counter: FlopCounter | None = None, frozen: ForwardResult | None = None,
                   keep_cache: bool = True, dense_probs_in_stats: bool = False) -> ForwardResult:
    """Sparse pipeline (model.py:267-324) on the B200 kernels.  With ``frozen`` the previous
    selections are reused and only the mixture weights are recomputed (model.py:284-300)."""
    x = torch.as_tensor(batch)
    if not x.is_cuda:
        x = x.cuda()
    if x.ndim != 2:
        raise ShapeError(f"batch has shape {tuple(x.shape)}, expected 2-D")
    B = x.shape[0]
    if B == 0:
        raise ShapeError("forward of an empty batch")
    eng = _get_engine(model, B, dense_probs_in_stats)
    enc = None
    if model.encoder1 is not None:
        if x.shape[1] != model.encoder1.d_in:
            raise ShapeError(f"batch has shape {tuple(x.shape)}, model expects (B, {model.encoder1.d_in})")
        enc = _encode(x.float(), model, eng)
    else:
        if x.shape[1] != model.d_in:
            raise ShapeError(f"hidden has shape {tuple(x.shape)}, model expects (B, {model.d_in})")
        eng.h.copy_(x)
    if frozen is not None:
        if frozen.mode != "sparse" or frozen.plan is None:
            raise StateError("frozen forward result must come from the sparse pipeline")
        eng.shared.copy_(frozen.routing.shared_i32)
        eng.adaptive.copy_(frozen.routing.adaptive_i32)
    eng.forward_a(frozen=frozen is not None)
    eng.forward_b(with_loss=False)
    eng.step_id += 1
    T, E = eng.T, eng.E
    # the result owns its arrays (the reference returns fresh arrays): clone the engine's buffers so a
    # later forward through the same cached engine cannot rewrite this result's routing or plan
    c = lambda t: t.clone()
    z = c(eng.z)
    routing = BatchRouting(z, T, B, E, model.budget, c(eng.tw), c(eng.shared), c(eng.adaptive), c(eng.active),
                           c(eng.wsel), c(eng.umask), c(eng.usize), c(eng.chunk_union), c(eng.chunk_active),
                           c(eng.chunk_mass), c(eng.chunk_dmass), eng.rpw, z_strides=(E, T * E))
    plan = ExecutionPlan(E, B, eng.umax, eng.rows_cap, c(eng.seg_pad), c(eng.seg_log), c(eng.loads), c(eng.totals),
                         c(eng.row_of), c(eng.gather_inst), c(eng.gather_exp), c(eng.stats_raw), routing.usize)
    n_act = eng.n_act()
    flops = n_act * sum(eng.dims[i] * eng.dims[i + 1] for i in range(len(eng.dims) - 1))
    if counter is not None:
        counter.add(flops)
    return ForwardResult("sparse", eng.preds.clone(), eng.logits.clone(), eng.reps.float(), routing, plan, flops,
                         hidden=eng.h.clone() if keep_cache else None,
                         router_logits=z.view(B, T, E).transpose(0, 1) if keep_cache else None,
                         _engine=eng, _step=eng.step_id, _enc=enc)
