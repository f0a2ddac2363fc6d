"""Model container + sparse forward -- drop-in for taskmoe/model.py.

``MoeModel`` keeps the reference fields (model.py:36-111): ``encoder1``/``encoder2``
(``Affine``), ``experts`` (``ExpertPool``), ``routers`` (``RouterBank``), ``heads``
(a list of T ``Affine`` maps d_out -> 1), ``task_loss_weights``, ``lb_strength``,
``budget``, ``encoder_nonlinearity``.  Two extensions: ``experts`` may be a list of
pools chained d -> d_ff -> d_out (the BASELINE "expert MLP"), and the encoders may be
None (the batch is then the encoded hidden (B, d_in)).

``forward_sparse(batch, model, ...)`` keeps the reference signature and result type.
The encoder runs on the tcgen05 GEMM (one group); the SMES layer runs through a cached
:class:`SMESEngine` (fused router front -> plan -> grouped expert GEMMs -> combine/heads).
Any widths are accepted: the shim zero-pads d, the pool widths and the expert count to the
kernels' granularity (multiples of 32; T*E a multiple of 8).  Padded weight rows/columns are
zero, padded experts carry a -1e30 router bias and are never selected, and every output is
sliced back to the logical shapes, so results equal those of the unpadded layer.
"""
from __future__ import annotations

import os
import weakref
from dataclasses import dataclass, field

import torch

from . import engine as _engine
from ._lib import call, ptr
from .errors import ConfigError, ShapeError, StateError
from .execution import ExecutionPlan
from .experts import ExpertPool, init_expert_pool
from .linalg import Affine, FlopCounter, init_affine
from .routing import BatchRouting, RouterBank, RoutingBudget, _stream
from .stacked import AffineStack

__all__ = ["MoeModel", "RouterBank", "ForwardResult", "forward_sparse", "init_model"]

ROUTER_INIT_SCALE = 1e-3   # model.py:32
ENCODER_BIAS_INIT = 0.01   # model.py:33
DEAD_EXPERT_BIAS = -1e30   # router bias of shim-padded experts: softmax mass exactly 0, never selected


class MoeModel:
    """Encoder, expert pool(s), task routers, task heads (model.py:36-111)."""

    def __init__(self, encoder1: Affine | None, encoder2: Affine | None, experts, routers: RouterBank, heads,
                 task_loss_weights, lb_strength: float, budget: RoutingBudget, encoder_nonlinearity: str = "relu"):
        self.encoder1, self.encoder2 = encoder1, encoder2
        self.experts = experts
        self.routers = routers
        heads = list(heads)
        for i, h in enumerate(heads):
            if h.d_out != 1 or h.d_in != heads[0].d_in:
                raise ConfigError(f"head {i} must map d_out -> 1")
        self._heads = AffineStack(items=heads)
        self.task_loss_weights = torch.as_tensor(task_loss_weights, dtype=torch.float64).detach().cpu()
        self.lb_strength = float(lb_strength)
        self.budget = budget
        self.encoder_nonlinearity = encoder_nonlinearity
        self._engines = {}
        t = self.routers.num_tasks
        pools = self.pools
        if len(self._heads.items) != t:
            raise ConfigError(f"{len(self._heads.items)} heads for {t} routers")
        if self.task_loss_weights.shape != (t,):
            raise ConfigError(f"expected {t} task loss weights")
        if bool((self.task_loss_weights < 0).any()) or self.lb_strength < 0:
            raise ConfigError("loss weights and regularizer strength must be non-negative")
        if (encoder1 is None) != (encoder2 is None):
            raise ConfigError("encoder1 and encoder2 must both be given or both be None")
        if encoder1 is not None:
            if encoder1.d_out != encoder2.d_in:
                raise ConfigError("encoder layer widths do not chain")
            if encoder2.d_out != pools[0].d_in or encoder2.d_out != self.routers.d_in:
                raise ConfigError("encoder output width must match expert and router input")
        elif pools[0].d_in != self.routers.d_in:
            raise ConfigError("expert and router input widths differ")
        for i in range(1, len(pools)):
            if pools[i].d_in != pools[i - 1].d_out or pools[i].num_experts != pools[0].num_experts:
                raise ConfigError(f"expert pool {i} does not chain")
        for i, h in enumerate(self._heads.items):
            if h.d_in != pools[-1].d_out or h.d_out != 1:
                raise ConfigError(f"head {i} must map d_out -> 1")
        if self.routers.num_experts != pools[0].num_experts:
            raise ConfigError("router width must equal the expert count")
        self.budget.validate(pools[0].num_experts)

    # -- reference fields and properties
    @property
    def heads(self) -> list:
        return self._heads.items

    @property
    def head_w(self) -> torch.Tensor:
        """(T, d_out) view of the stacked heads."""
        return self._heads.weight[:, 0, :]

    @property
    def head_b(self) -> torch.Tensor:
        """(T,) view of the stacked head biases."""
        return self._heads.bias[:, 0]

    @property
    def pools(self) -> list:
        return list(self.experts) if isinstance(self.experts, (list, tuple)) else [self.experts]

    @property
    def num_features(self) -> int:
        return self.encoder1.d_in if self.encoder1 is not None else self.d_in

    @property
    def d_hidden(self) -> int:
        return self.encoder1.d_out if self.encoder1 is not None else self.d_in

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
        """Named parameter views in the reference's order and names (model.py:94-111).  A stack of
        pools names its experts ``expert{l}_{e}``."""
        blocks = {}
        if self.encoder1 is not None:
            blocks.update({"encoder1.weight": self.encoder1.weight, "encoder1.bias": self.encoder1.bias,
                           "encoder2.weight": self.encoder2.weight, "encoder2.bias": self.encoder2.bias})
        pools = self.pools
        for li, pool in enumerate(pools):
            for e, layer in enumerate(pool.layers):
                pre = f"expert_{e}" if len(pools) == 1 else f"expert{li}_{e}"
                blocks[pre + ".weight"] = layer.weight
                blocks[pre + ".bias"] = layer.bias
        for t, m in enumerate(self.routers.maps):
            blocks[f"router_{t}.weight"] = m.weight
            blocks[f"router_{t}.bias"] = m.bias
        for t, h in enumerate(self.heads):
            blocks[f"head_{t}.weight"] = h.weight
            blocks[f"head_{t}.bias"] = h.bias
        return blocks

    def num_parameters(self) -> int:
        return sum(v.numel() for v in self.parameter_blocks().values())

    def smes_params(self, pad: "_Pad | None" = None) -> _engine.SMESParams:
        """The layer's parameters in the engine's stacked layouts (zero-padded by ``pad``)."""
        pools = self.pools
        rw, rb = self.routers.weight, self.routers.bias
        layers = [(p.weight, p.bias, p.nonlinearity) for p in pools]
        hw, hb = self.head_w, self.head_b
        if pad is not None and pad.active:
            rw, rb, layers, hw = pad_params(rw, rb, layers, hw, pad)
        return _engine.SMESParams(
            router_w=rw, router_b=rb, layers=[_engine.ExpertLayer(w, b, act) for (w, b, act) in layers],
            head_w=hw, head_b=hb, task_weights=self.routers.task_weights,
            task_loss_weights=self.task_loss_weights, lb_strength=self.lb_strength)

    def __repr__(self) -> str:
        return (f"MoeModel(num_tasks={self.num_tasks}, num_experts={self.num_experts}, d_in={self.d_in}, "
                f"d_out={self.d_out}, pools={len(self.pools)}, budget={self.budget})")


def _round(x, m):
    return (x + m - 1) // m * m


def _pad_out(d_out: int) -> int:
    """The combine kernels tile d_out by 32 lanes x {4, 8} columns x {1, 2, 4, 8} warps."""
    for w in (128, 256, 512, 1024):
        if d_out <= w:
            return w if d_out % 128 or d_out & (d_out - 1) else d_out
    return _round(d_out, 32)


class _Pad:
    """Kernel granularity of the layer: input and hidden widths to multiples of 32, the output width
    to 128 / 256 / 512 / 1024 (combine tiling), T * E to a multiple of 8."""

    def __init__(self, model: "MoeModel | None" = None, T: int = 0, E: int = 0, dims=None, fp32: bool = False):
        if model is not None:
            T, E, dims = model.num_tasks, model.num_experts, [model.d_in] + [p.d_out for p in model.pools]
        self.T, self.E = T, E
        self.dims = list(dims)
        if fp32:   # bf16x3 GEMMs: contraction widths in whole 64-column k-blocks
            self.dims_p = [_round(x, 64) for x in self.dims[:-1]] + [_round(self.dims[-1], 32)]
        else:
            self.dims_p = [_round(x, 32) for x in self.dims[:-1]] + [_pad_out(self.dims[-1])]
        E_p = self.E
        while (self.T * E_p) % 8:
            E_p += 1
        self.E_p = E_p
        self.active = self.dims_p != self.dims or E_p != self.E


def pad_params(rw, rb, layers, hw, pad: _Pad):
    """Zero-padded copies of router / pool / head parameters at the kernels' granularity; the padded
    experts get a -1e30 router bias (never selected, softmax mass exactly 0)."""
    T, E, Ep = pad.T, pad.E, pad.E_p
    dims, dp = pad.dims, pad.dims_p
    dev = rw.device
    z = lambda *s: torch.zeros(*s, dtype=torch.float32, device=dev)
    rw_p = z(T, Ep, dp[0])
    rw_p[:, :E, :dims[0]] = rw
    rb_p = torch.full((T, Ep), DEAD_EXPERT_BIAS, dtype=torch.float32, device=dev)
    rb_p[:, :E] = rb
    lp = []
    for i, (w, b, act) in enumerate(layers):
        w_p = z(Ep, dp[i + 1], dp[i])
        w_p[:E, :dims[i + 1], :dims[i]] = w
        b_p = z(Ep, dp[i + 1])
        b_p[:E, :dims[i + 1]] = b
        lp.append((w_p, b_p, act))
    hw_p = z(T, dp[-1])
    hw_p[:, :dims[-1]] = hw
    return rw_p, rb_p, lp, hw_p


def init_model(gen: torch.Generator | None, num_features: int, d_hidden: int, d_in: int, d_out: int,
               num_experts: int, num_tasks: int, budget: RoutingBudget, task_loss_weights=None,
               lb_strength: float = 0.0, expert_nonlinearity: str = "identity", encoder_nonlinearity: str = "relu",
               router_task_weights=None, d_ff: int | None = None, device="cuda") -> MoeModel:
    """Fan-in uniform init, near-zero routers (model.py:117-156).  ``d_ff`` adds the
    BASELINE 'expert MLP' (relu d_in -> d_ff, identity d_ff -> d_out)."""
    enc1 = init_affine(gen, d_hidden, num_features, bias_value=ENCODER_BIAS_INIT, device=device)
    enc2 = init_affine(gen, d_in, d_hidden, bias_value=ENCODER_BIAS_INIT, device=device)
    if d_ff is None:
        experts = init_expert_pool(gen, num_experts, d_in, d_out, expert_nonlinearity, device)
    else:
        experts = [init_expert_pool(gen, num_experts, d_in, d_ff, "relu", device),
                   init_expert_pool(gen, num_experts, d_ff, d_out, "identity", device)]
    routers = RouterBank([init_affine(gen, num_experts, d_in, scale=ROUTER_INIT_SCALE / d_in ** 0.5, device=device)
                          for _ in range(num_tasks)], router_task_weights)
    heads = [init_affine(gen, 1, d_out, device=device) for _ in range(num_tasks)]
    lam = torch.ones(num_tasks) if task_loss_weights is None else torch.as_tensor(task_loss_weights)
    return MoeModel(enc1, enc2, experts, routers, heads, lam, lb_strength, budget, encoder_nonlinearity)


def heads_from_stacked(head_w: torch.Tensor, head_b: torch.Tensor) -> list:
    """T ``Affine`` heads (1, d_out) from a stacked (T, d_out) weight and (T,) bias."""
    w = torch.as_tensor(head_w)
    b = torch.as_tensor(head_b)
    return [Affine(w[t:t + 1], b[t:t + 1]) for t in range(w.shape[0])]


class _Deferred:
    """A result field computed on first access from data the result already owns."""
    __slots__ = ("fn",)

    def __init__(self, fn):
        self.fn = fn


class _Lazy:
    """Dataclass field descriptor: stores values as given, evaluates a :class:`_Deferred` once on
    first read.  The reference fills these eagerly (model.py:307-324); here the row gathers and
    fp32 widenings nobody reads cost nothing, and reading them later gives the same arrays."""

    def __set_name__(self, owner, name):
        self.key = "_lz_" + name

    def __get__(self, obj, owner=None):
        if obj is None:
            return None                       # the dataclass default
        v = obj.__dict__.get(self.key)
        if isinstance(v, _Deferred):
            v = v.fn()
            obj.__dict__[self.key] = v
        return v

    def __set__(self, obj, value):
        obj.__dict__[self.key] = value


@dataclass
class ForwardResult:
    """Predictions plus what backward needs (model.py:159-185).  Arrays are device tensors."""
    mode: str
    predictions: torch.Tensor      # (T, B)
    head_logits: torch.Tensor      # (T, B)
    task_reps: torch.Tensor        # (T, B, d_out)
    routing: BatchRouting
    plan: ExecutionPlan
    expert_flops: int = _Lazy()    # (the logical row count is a device value: read on first access)
    inputs: torch.Tensor | None = None
    encoder_pre: torch.Tensor | None = None
    encoder_hidden: torch.Tensor | None = None
    hidden: torch.Tensor | None = None
    router_logits: torch.Tensor | None = None
    packed_in: torch.Tensor | None = _Lazy()
    packed_pre: torch.Tensor | None = None
    packed_out: torch.Tensor | None = _Lazy()
    expert_outputs: torch.Tensor | None = None
    _engine: object = None
    _step: int = -1
    _enc: dict | None = None
    _pad: object = None
    precision: str = "bf16"

    def mean_union(self) -> float:
        return float(self.routing.usize.double().mean())

    def max_union(self) -> int:
        return int(self.routing.usize.max())


def _gemm(a, lda, rows, w, n, k, bias, act, out, ldc, out_fp32, m_limit, bits_out=None, bits_ld=0, b_mn=0,
          bits_in=None):
    seg = torch.tensor([0, _round(rows, 128)], dtype=torch.int32, device=a.device)
    call("smes_gemm_ragged_m", ptr(a), lda, rows, ptr(w), 1, n, k, b_mn, ptr(seg), ptr(bias), act, ptr(bits_out),
         ptr(bits_in), bits_ld, ptr(out), ldc, out_fp32, m_limit, _stream())


def _encode(x: torch.Tensor, model: MoeModel, eng) -> dict:
    """encoder1 -> act -> encoder2 on the tcgen05 GEMM (model.py:188-199).  Widths that are not
    multiples of the kernel granularity are zero-padded (the padded columns stay zero)."""
    B, F = x.shape
    dev = x.device
    Fp = _round(F, 8)
    dh = model.encoder1.d_out
    dhp = _round(dh, 32)
    d = model.d_in
    xb = torch.zeros(B, Fp, dtype=torch.bfloat16, device=dev)
    xb[:, :F] = x
    w1 = torch.zeros(dhp, Fp, dtype=torch.bfloat16, device=dev)
    w1[:dh, :F] = model.encoder1.weight
    b1 = torch.zeros(dhp, device=dev)
    b1[:dh] = model.encoder1.bias
    mid = torch.zeros(_round(B, 128), dhp, dtype=torch.bfloat16, device=dev)
    relu = model.encoder_nonlinearity == "relu"
    bits = torch.zeros(dhp // 32, _round(B, 128), dtype=torch.int32, device=dev) if relu else None
    _gemm(xb, Fp, B, w1.reshape(1, dhp, Fp).contiguous(), dhp, Fp, b1, 1 if relu else 0, mid, dhp, 0, B,
          bits_out=bits, bits_ld=_round(B, 128))
    w2 = torch.zeros(1, d, dhp, dtype=torch.bfloat16, device=dev)
    w2[0, :, :dh] = model.encoder2.weight
    _gemm(mid, dhp, B, w2, d, dhp, model.encoder2.bias.float().contiguous(), 0, eng.h, eng.ldh, 0, B)
    return dict(xb=xb, Fp=Fp, F=F, mid=mid, bits=bits, w1=w1, w2=w2, dh=dh, dhp=dhp)


def _encode_f32(x: torch.Tensor, model: MoeModel, eng) -> dict:
    """encoder1 -> act -> encoder2 in fp32 (bf16x3 GEMMs, model.py:188-199)."""
    from .fp32 import split_planes
    B, F = x.shape
    dev = x.device
    Fp = _round(F, 64)
    dh = model.encoder1.d_out
    dhp = _round(dh, 64)
    d = model.d_in
    xf = torch.zeros(B, Fp, device=dev)
    xf[:, :F] = x
    x3 = split_planes(xf)
    w1 = torch.zeros(dhp, Fp, device=dev)
    w1[:dh, :F] = model.encoder1.weight
    b1 = torch.zeros(dhp, device=dev)
    b1[:dh] = model.encoder1.bias
    mid = torch.zeros(B, dhp, device=dev)
    relu = model.encoder_nonlinearity == "relu"
    seg = torch.tensor([0, _round(B, 128)], dtype=torch.int32, device=dev)
    w13 = split_planes(w1)          # operands stay referenced until the GEMMs are queued (stream-ordered reuse)
    call("smes_gemm_ragged_m_x3", ptr(x3), 3 * Fp, B, ptr(w13), 1, dhp, Fp, ptr(seg), ptr(b1),
         1 if relu else 0, ptr(mid), dhp, B, _stream())
    w2 = torch.zeros(d, dhp, device=dev)
    w2[:, :dh] = model.encoder2.weight
    dp = eng.d
    out = torch.zeros(B, dp, device=dev)
    b2 = torch.zeros(dp, device=dev)
    b2[:d] = model.encoder2.bias
    w2p = torch.zeros(dp, dhp, device=dev)
    w2p[:d] = w2
    mid3, w23 = split_planes(mid), split_planes(w2p)
    call("smes_gemm_ragged_m_x3", ptr(mid3), 3 * dhp, B, ptr(w23), 1, dp, dhp, ptr(seg),
         ptr(b2), 0, ptr(out), dp, B, _stream())
    eng.h.copy_(out)
    return dict(mid=mid, dh=dh, dhp=dhp, F=F, Fp=Fp, planes=(x3, w13, mid3, w23))


def _get_engine(model: MoeModel, B: int, dense: bool = False, precision: str = "bf16"):
    if precision not in ("bf16", "fp32"):
        raise ConfigError(f"unknown precision '{precision}', expected 'bf16' or 'fp32'")
    fp32 = precision == "fp32"
    pad = _Pad(model, fp32=fp32)
    key = (B, bool(dense), tuple(pad.dims_p), pad.E_p, tuple(p.nonlinearity for p in model.pools), precision)
    eng = model._engines.get(key)
    if eng is None and fp32:
        from .fp32 import SMESForwardF32
        eng = SMESForwardF32(model.smes_params(pad), B, model.budget.k_shared, model.budget.k_adaptive,
                             device=model.routers.weight.device, lb_experts=model.num_experts,
                             dense_probs_in_stats=dense)
        eng.step_id = 0
        model._engines[key] = eng
    elif eng is None:
        eng = _engine.SMESEngine(model.smes_params(pad), B, model.budget.k_shared, model.budget.k_adaptive,
                                 dense_probs_in_stats=dense, device=model.routers.weight.device,
                                 lb_experts=model.num_experts)
        eng.step_id = 0
        model._engines[key] = eng
    else:
        eng.p = model.smes_params(pad)
        eng.refresh_weights()
    return eng, pad


def forward_sparse(batch, model: MoeModel, counter: FlopCounter | None = None, frozen: ForwardResult | None = None,
                   keep_cache: bool = True, dense_probs_in_stats: bool = False,
                   precision: str = "bf16") -> ForwardResult:
    """Sparse pipeline (model.py:267-324) on the B200 kernels.  With ``frozen`` the previous
    selections are reused and only the mixture weights are recomputed (model.py:284-300).

    ``precision``: "bf16" (default; bf16 operands, fp32 accumulation, the training path) or
    "fp32" (fp32 operands and activations, GEMMs as bf16x3 tensor-core products -- the north
    star's fp32 1e-5 contract; forward only, see fp32.py)."""
    x = torch.as_tensor(batch)
    if not x.is_cuda:
        x = x.cuda()
    if x.ndim != 2:
        raise ShapeError(f"batch has shape {tuple(x.shape)}, expected 2-D")
    B = x.shape[0]
    if B == 0:
        raise ShapeError("forward of an empty batch")
    if model.encoder1 is not None and x.shape[1] != model.encoder1.d_in:
        raise ShapeError(f"batch has shape {tuple(x.shape)}, model expects (B, {model.encoder1.d_in})")
    if model.encoder1 is None and x.shape[1] != model.d_in:
        raise ShapeError(f"hidden has shape {tuple(x.shape)}, model expects (B, {model.d_in})")
    if frozen is not None and (frozen.mode != "sparse" or frozen.plan is None):
        raise StateError("frozen forward result must come from the sparse pipeline")
    eng, pad = _get_engine(model, B, dense_probs_in_stats, precision)
    if precision == "fp32":
        return _forward_sparse_f32(x, model, counter, frozen, keep_cache, eng, pad)
    eng.keep_logits = True
    _settle(eng)
    T, E, Ep = model.num_tasks, model.num_experts, pad.E_p
    d, d_out = model.d_in, model.d_out
    enc = None
    if model.encoder1 is not None:
        enc = _encode(x.float(), model, eng)
    else:
        eng.h[:, :d].copy_(x)
    if frozen is not None:
        eng.shared.copy_(frozen.routing.shared_i32)
        eng.adaptive.copy_(frozen.routing.adaptive_i32)
    fz = frozen is not None
    api_replay(eng, ("fwd", fz, eng.dense), lambda: (eng.forward_a(frozen=fz), eng.forward_b(with_loss=False)))
    eng.step_id += 1
    # the result owns its arrays (the reference returns fresh arrays): clone the engine's buffers so a
    # later forward through the same cached engine cannot rewrite this result's routing or plan
    c = lambda t: t.clone()
    ce = lambda t: t[:, :E].contiguous()           # drop the shim's padded experts
    z = c(eng.z)
    routing = BatchRouting(z, T, B, E, model.budget, c(eng.tw), c(eng.shared), c(eng.adaptive), c(eng.active),
                           c(eng.wsel), c(eng.umask), c(eng.usize), ce(eng.chunk_union), ce(eng.chunk_active),
                           ce(eng.chunk_mass), ce(eng.chunk_dmass), eng.rpw, z_strides=(Ep, T * Ep))
    raw = eng.stats_raw.view(3, Ep)[:, :E].reshape(-1).contiguous()
    plan = ExecutionPlan(E, B, eng.umax, eng.rows_cap, eng.seg_pad[:E + 1].clone(), eng.seg_log[:E + 1].clone(),
                         eng.loads[:E].clone(), c(eng.totals), c(eng.row_of), c(eng.gather_inst),
                         c(eng.gather_exp), raw, routing.usize)
    dims = pad.dims
    per_row = sum(dims[i] * dims[i + 1] for i in range(len(dims) - 1))
    # expert_flops needs the logical row count, a device value: read on first access (a host sync
    # here would stall the caller's next launches behind the whole forward)
    flops = _Deferred(lambda: int(plan.totals[2].item()) * per_row)
    if counter is not None:
        counter.add(flops.fn())
    reps = eng.reps[..., :d_out].float()
    res = ForwardResult("sparse", eng.preds.clone(), eng.logits.clone(), reps, routing, plan, flops,
                        _engine=eng, _step=eng.step_id, _enc=enc, _pad=pad)
    if keep_cache:
        res.inputs = x
        # without encoders the hidden is the batch itself (the kernels read its bf16 copy)
        hidden = x.float() if enc is None else eng.h[:, :d].float()
        res.hidden = hidden
        res.router_logits = z.view(B, T, Ep)[:, :, :E].permute(1, 0, 2)
        if enc is not None:
            res.encoder_hidden = enc["mid"][:B, :enc["dh"]].float()
        # packed_in = hidden[gather_instances] (model.py:301) from arrays the result owns; packed_out
        # reads the engine's expert outputs until the engine's next forward, which first gathers
        # them into a copy this result owns (_settle)
        res.packed_in = _Deferred(lambda: hidden[plan.gather_instances])
        state = {"rows": None}
        res.packed_out = _Deferred(lambda: (state["rows"] if state["rows"] is not None
                                            else eng.outs[-1][plan.physical_rows, :d_out]).float())

        def settle(r):
            if isinstance(r.__dict__.get("_lz_packed_out"), _Deferred):
                state["rows"] = eng.outs[-1][plan.physical_rows, :d_out]
        eng._pending = [(weakref.ref(res), settle)]
    return res


def api_replay(eng, key, launches) -> None:
    """Run ``launches`` -- a fixed launch sequence on the engine's own buffers -- through a CUDA
    graph captured on its second use (the first runs eagerly: it creates the engine's side stream
    and sets kernel attributes).  The API step is host-bound (~50 launches through ctypes); a replay
    is one launch.  SMES_API_GRAPHS=0 keeps every call eager."""
    graphs = eng.__dict__.setdefault("_api_graphs", {})
    g = graphs.get(key)
    if g is None:
        seen = eng.__dict__.setdefault("_api_seen", set())
        if key not in seen or os.environ.get("SMES_API_GRAPHS", "1") == "0":
            seen.add(key)
            launches()
            return
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            launches()
        graphs[key] = g
    g.replay()


def _settle(eng) -> None:
    """Before a forward rewrites the engine's buffers: earlier results still alive take their own
    copy of what their deferred fields read from the engine."""
    for ref, settle in getattr(eng, "_pending", ()):
        r = ref()
        if r is not None:
            settle(r)
    eng._pending = []


def _forward_sparse_f32(x, model: MoeModel, counter, frozen, keep_cache, eng, pad) -> ForwardResult:
    """fp32 forward (fp32.SMESForwardF32): same result type; ``backward`` of it is refused."""
    B = x.shape[0]
    T, E, Ep = model.num_tasks, model.num_experts, pad.E_p
    d, d_out = model.d_in, model.d_out
    enc = None
    if model.encoder1 is not None:
        enc = _encode_f32(x.float(), model, eng)
    else:
        eng.h[:, :d].copy_(x)
    if frozen is not None:
        eng.shared.copy_(frozen.routing.shared_i32)
        eng.adaptive.copy_(frozen.routing.adaptive_i32)
    eng.forward(with_loss=False, frozen=frozen is not None)
    eng.check_finite()
    eng.step_id += 1
    c = lambda t: t.clone()
    ce = lambda t: t[:, :E].contiguous()
    z = c(eng.z)
    routing = BatchRouting(z, T, B, E, model.budget, c(eng.tw), c(eng.shared), c(eng.adaptive), c(eng.active),
                           c(eng.wsel), c(eng.umask), c(eng.usize), ce(eng.chunk_union), ce(eng.chunk_active),
                           ce(eng.chunk_mass), ce(eng.chunk_dmass), eng.rpw, z_strides=(Ep, T * Ep))
    raw = eng.stats_raw.view(3, Ep)[:, :E].reshape(-1).contiguous()
    plan = ExecutionPlan(E, B, eng.umax, eng.rows_cap, eng.seg_pad[:E + 1].clone(), eng.seg_log[:E + 1].clone(),
                         eng.loads[:E].clone(), c(eng.totals), c(eng.row_of), c(eng.gather_inst),
                         c(eng.gather_exp), raw, routing.usize)
    n_act = eng.n_act()
    dims = pad.dims
    flops = n_act * sum(dims[i] * dims[i + 1] for i in range(len(dims) - 1))
    if counter is not None:
        counter.add(flops)
    reps = eng.reps[..., :d_out].clone()
    # mode "sparse" keeps the reference's result contract; _engine is withheld so backward refuses it
    res = ForwardResult("sparse", eng.preds.clone(), eng.logits.clone(), reps, routing, plan, flops,
                        _engine=None, _step=eng.step_id, _enc=enc, _pad=pad)
    res.precision = "fp32"
    if keep_cache:
        res.inputs = x
        res.hidden = eng.h[:, :d].clone()
        res.router_logits = z.view(B, T, Ep)[:, :, :E].permute(1, 0, 2)
        if enc is not None:
            res.encoder_hidden = enc["mid"][:B, :enc["dh"]].clone()
        rows = plan.physical_rows
        res.packed_in = eng.X3[rows, :d].float() + eng.X3[rows, pad.dims_p[0]:pad.dims_p[0] + d].float() + \
            eng.X3[rows, 2 * pad.dims_p[0]:2 * pad.dims_p[0] + d].float()
        res.packed_out = eng.outs[-1][rows, :d_out].clone()
    return res
