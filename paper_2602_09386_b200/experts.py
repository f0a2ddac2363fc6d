"""Expert pools -- drop-in for taskmoe/experts.py -- and the expert shard of the
expert-parallel step.

``ExpertPool`` keeps the reference fields (``layers``: a list of ``Affine`` maps,
``nonlinearity``; experts.py:17-73) over stacked device storage (``weight``
(E, d_out, d_in), ``bias`` (E, d_out)) that the kernels consume.

``ExpertShard`` is used by the expert-parallel step (:mod:`ep`): an owner rank runs its local
experts (reference ``ExpertPool`` / ``grouped_gemm``, experts.py:17-73, execution.py:126-158, and
the expert part of ``backward``, training.py:180-192) on the rows other ranks dispatched to it.
The last (identity) pool is folded into the task heads (csrc/fold.cu), so the shard consumes
the packed layer input X and produces the head projections P of every row; the backward
consumes the row coefficients C (training.py:160-179 after folding) and produces the
parameter gradients of the local experts, the local share of dW_head and the per-row dX.
A single relu pool (the reference expert with ``expert_nonlinearity="relu"``) runs unfolded:
the shard writes the pool outputs O and consumes d_packed.

Buffers are sized by ``rows_cap`` (a multiple of 128); rows follow the plan's padded,
expert-major layout (``seg_pad``), pad rows of X and C are zero.
"""
from __future__ import annotations

import torch

from ._lib import call, ptr, tcall
from .errors import ConfigError, ShapeError
from .linalg import Affine, FlopCounter, _dev_tensor
from .stacked import AffineStack

__all__ = ["ExpertPool", "init_expert_pool", "apply_nonlinearity", "ExpertShard"]

_NONLINEARITIES = ("identity", "relu")


def apply_nonlinearity(name: str, x: torch.Tensor) -> torch.Tensor:
    """experts.py:17-23."""
    if name == "identity":
        return x
    if name == "relu":
        return torch.clamp_min(x, 0.0)
    raise ConfigError(f"unknown nonlinearity '{name}', expected one of {_NONLINEARITIES}")


class ExpertPool:
    """E affine maps d_in -> d_out with one shared nonlinearity (experts.py:26-73).

    Reference form ``ExpertPool(layers=[Affine, ...], nonlinearity="relu")``; stacked form
    ``ExpertPool(weight (E, d_out, d_in), bias (E, d_out), nonlinearity)``.  ``layers[e]`` are views
    of the stacked ``weight`` / ``bias``."""

    def __init__(self, layers, nonlinearity="identity", *stacked_nonlinearity):
        if isinstance(layers, torch.Tensor):          # stacked form
            self._stack = AffineStack(weight=layers, bias=nonlinearity)
            nonlinearity = stacked_nonlinearity[0] if stacked_nonlinearity else "identity"
        else:
            layers = list(layers)
            if not layers:
                raise ConfigError("expert pool needs at least one expert")
        if nonlinearity not in _NONLINEARITIES:
            raise ConfigError(f"unknown nonlinearity '{nonlinearity}', expected one of {_NONLINEARITIES}")
        if not isinstance(layers, torch.Tensor):
            d_in, d_out = layers[0].d_in, layers[0].d_out
            for i, layer in enumerate(layers):
                if layer.d_in != d_in or layer.d_out != d_out:
                    raise ShapeError(f"expert {i} maps {layer.d_in}->{layer.d_out}, expected {d_in}->{d_out}")
            self._stack = AffineStack(items=layers)
        self.nonlinearity = nonlinearity
        if not self._stack.items:
            raise ConfigError("expert pool needs at least one expert")

    @classmethod
    def stacked(cls, weight, bias, nonlinearity="identity") -> "ExpertPool":
        return cls(weight, bias, nonlinearity)

    @property
    def layers(self) -> list:
        return self._stack.items

    @property
    def weight(self) -> torch.Tensor:
        return self._stack.weight

    @weight.setter
    def weight(self, w):
        self._stack.weight = w

    @property
    def bias(self) -> torch.Tensor:
        return self._stack.bias

    @bias.setter
    def bias(self, b):
        self._stack.bias = b

    @property
    def num_experts(self) -> int:
        return len(self._stack.items)

    @property
    def d_in(self) -> int:
        return self._stack.items[0].d_in

    @property
    def d_out(self) -> int:
        return self._stack.items[0].d_out

    def activate(self, pre: torch.Tensor) -> torch.Tensor:
        return apply_nonlinearity(self.nonlinearity, pre)

    def apply_all(self, hidden, counter: FlopCounter | None = None) -> torch.Tensor:
        """Dense path: every expert on every instance, (B, E, d_out) (experts.py:63-73)."""
        h = _dev_tensor(hidden)
        w = self.weight.to(h.device)
        dt = torch.promote_types(h.dtype, w.dtype)
        if h.ndim != 2 or h.shape[1] != self.d_in:
            raise ShapeError(f"hidden has shape {tuple(h.shape)}, expected (B, {self.d_in})")
        out = torch.einsum("bi,eoi->beo", h.to(dt), w.to(dt)) + self.bias.to(h.device, dt)[None]
        if counter is not None:
            counter.add(h.shape[0] * self.d_in * self.d_out * self.num_experts)
        return self.activate(out)

    def __repr__(self) -> str:
        return (f"ExpertPool(num_experts={self.num_experts}, d_in={self.d_in}, d_out={self.d_out}, "
                f"nonlinearity='{self.nonlinearity}')")


def init_expert_pool(gen: torch.Generator | None, num_experts: int, d_in: int, d_out: int,
                     nonlinearity: str = "identity", device="cuda") -> ExpertPool:
    """Fan-in uniform init, zero bias (experts.py:76-84, linalg.py:152-162)."""
    s = 1.0 / d_in ** 0.5
    w = (torch.rand(num_experts, d_out, d_in, generator=gen, dtype=torch.float64) * 2 - 1) * s
    return ExpertPool(w.float().to(device), torch.zeros(num_experts, d_out, device=device), nonlinearity)


def _round(x, m):
    return (x + m - 1) // m * m


def refresh_into(obj, name: str, src: torch.Tensor, dtype) -> torch.Tensor:
    """``obj.name`` <- src (cast to dtype) in place; allocated on first use so device addresses
    captured by a CUDA graph stay valid across weight refreshes."""
    cur = getattr(obj, name, None)
    if cur is None or cur.shape != src.shape or cur.dtype != dtype:
        cur = torch.empty(src.shape, dtype=dtype, device=obj.dev)
        setattr(obj, name, cur)
    cur.copy_(src)
    return cur


class ExpertShard:
    def __init__(self, layers, T: int, head_w: torch.Tensor, rows_cap: int, device, fuse_mlp: bool = True,
                 fuse_wgrad: bool = False):
        # folded heads: [relu ->] identity pools.  Unfolded: one relu pool (the reference expert with
        # expert_nonlinearity="relu"), whose outputs O are kept and projected onto the heads.
        self.folded = layers[-1].act == "identity"
        if len(layers) not in (1, 2) or (len(layers) == 2 and (layers[0].act != "relu" or not self.folded)):
            raise ConfigError("expert shard needs [relu ->] identity expert pools or one relu pool")
        self.dev = torch.device(device)
        self.layers = layers
        self.E = layers[0].weight.shape[0]
        self.T = T
        self.dims = [layers[0].d_in] + [l.d_out for l in layers]
        if any(x % 32 for x in self.dims):
            raise ShapeError(f"expert widths must be multiples of 32, got {self.dims}")
        self.d, self.d_out = self.dims[0], self.dims[-1]
        self.R = _round(rows_cap, 128)
        self.ldg = _round(T, 8)
        self.ldp = self.ldg
        self.ldc = _round(T, 16)
        d, R, E = self.d, self.R, self.E
        L = len(layers)
        self.fuse = bool(fuse_mlp and L == 2 and d % 64 == 0 and d <= 256 and self.dims[1] % 128 == 0
                         and T <= 16)
        self.fuse_wgrad = bool(fuse_wgrad and self.fuse)
        dev, bf, f32 = self.dev, torch.bfloat16, torch.float32
        z = lambda *s, dt=f32: torch.zeros(*s, dtype=dt, device=dev)
        self.ld_in = [w + 64 for w in self.dims[:-1]]
        self.X = z(R, self.ld_in[0], dt=bf)
        self.X[:, d] = 1.0                                 # ones column: bias grads in the wgrad GEMM
        self.H = None
        if L == 2:
            self.H = z(R, self.ld_in[1], dt=bf)
            self.H[:, self.dims[1]] = 1.0
            self.bits = z(self.dims[1] // 32, R, dt=torch.int32)
            self.dH = z(R, self.dims[1], dt=bf)
        self.P = z(R, self.ldp)
        self.Cm = z(R, self.ldc, dt=bf)
        self.dX = z(R, d, dt=bf)
        di = self.dims[-2]
        self.G = z(E, self.ldg, di, dt=bf)
        self.c = z(E, self.ldg)
        self.Qe = z(E, self.ldg, di)                       # per-expert C^T H
        self.csum = z(E, self.ldg)                         # per-expert column sums of C
        self.work = z(call("smes_fold_work_floats", E, T, self.d_out, di))
        shapes = [(E, l.d_out, l.d_in) for l in layers] + [(E, l.d_out) for l in layers]
        sizes = [int(torch.Size(s).numel()) for s in shapes]
        self.grad_flat = z(sum(sizes))
        views, off = [], 0
        for s, n in zip(shapes, sizes):
            views.append(self.grad_flat[off:off + n].view(s))
            off += n
        self.g_layers = [(views[i], views[L + i]) for i in range(L)]
        self.g_head_w = z(T, self.d_out)                   # this shard's share of dW_head
        self.head_w = head_w
        if not self.folded:
            # unfolded single relu pool: O and its relu mask, d_packed = (C head_w) x mask
            self.O = z(R, self.d_out, dt=bf)
            self.bits = z(self.d_out // 32, R, dt=torch.int32)
            self.dO = z(R, self.d_out, dt=bf)
            # one group over every row; callers pass the plan's [0, padded rows] table instead (seg_one)
            self.seg_all = torch.tensor([0, R], dtype=torch.int32, device=dev)
            self.head_w_bf = torch.empty(1, T, self.d_out, dtype=bf, device=dev)
            self.head_wT_bf = torch.zeros(1, self.d_out, self.ldc, dtype=bf, device=dev)
            self.g_head_w3 = self.g_head_w.view(1, T, self.d_out)
        self.refresh_weights()

    def refresh_weights(self):
        """bf16 / fp32 operands, allocated once and refreshed in place (graph-stable addresses)."""
        if not hasattr(self, "w_bf"):
            self.w_bf = [torch.empty(l.weight.shape, dtype=torch.bfloat16, device=self.dev) for l in self.layers]
            self.b32 = [torch.empty(l.bias.shape, dtype=torch.float32, device=self.dev) for l in self.layers]
        for l, w, b in zip(self.layers, self.w_bf, self.b32):
            w.copy_(l.weight.detach())
            b.copy_(l.bias.detach())
        if not self.folded:
            self.head_w_bf[0].copy_(self.head_w)
            self.head_wT_bf[0, :, :self.T].copy_(self.head_w.t())

    # ------------------------------------------------------------------ forward
    def forward(self, s, seg_pad, seg_one=None):
        """P of every packed row (X already scattered; seg_pad = padded expert offsets)."""
        E, R, T = self.E, self.R, self.T
        di = self.dims[-2]
        if not self.folded:
            # O = relu(X W^T + b) (+ mask), then P = O head_w^T over every row (N = T)
            tcall("fc1_fwd", "smes_gemm_ragged_m", ptr(self.X), self.ld_in[0], R, ptr(self.w_bf[0]), E, self.d_out,
                  self.d, 0, ptr(seg_pad), ptr(self.b32[0]), 1, ptr(self.bits), None, R, ptr(self.O), self.d_out, 0,
                  R, s)
            tcall("head_proj", "smes_gemm_ragged_m", ptr(self.O), self.d_out, R, ptr(self.head_w_bf), 1, T,
                  self.d_out, 0, ptr(self.seg_all if seg_one is None else seg_one), None, 0, None, None, 0, ptr(self.P),
                  self.ldp, 1, R, s)
            return
        tcall("fold_heads", "smes_fold_heads", E, T, self.ldg, self.d_out, di, ptr(self.head_w), ptr(self.w_bf[-1]),
             ptr(self.b32[-1]), ptr(self.G), ptr(self.c), ptr(self.work), s)
        if len(self.layers) == 1:
            tcall("fc1_fwd_folded", "smes_gemm_ragged_m", ptr(self.X), self.ld_in[0], R, ptr(self.G), E, self.ldg, di, 0, ptr(seg_pad),
                 ptr(self.c), 0, None, None, 0, ptr(self.P), self.ldp, 1, R, s)
            return
        if self.fuse:
            tcall("mlp_fwd", "smes_mlp_fwd", ptr(self.X), self.ld_in[0], R, ptr(self.w_bf[0]), ptr(self.b32[0]), ptr(self.G),
                 ptr(self.c), self.ldg, E, self.d, di, ptr(seg_pad), ptr(self.bits), R, ptr(self.H), self.ld_in[1],
                 ptr(self.P), self.ldp, s)
            return
        tcall("fc1_fwd", "smes_gemm_ragged_m", ptr(self.X), self.ld_in[0], R, ptr(self.w_bf[0]), E, di, self.d, 0, ptr(seg_pad),
             ptr(self.b32[0]), 1, ptr(self.bits), None, R, ptr(self.H), self.ld_in[1], 0, R, s)
        tcall("fc2_fwd_folded", "smes_gemm_ragged_m", ptr(self.H), self.ld_in[1], R, ptr(self.G), E, self.ldg, di, 0, ptr(seg_pad),
             ptr(self.c), 0, None, None, 0, ptr(self.P), self.ldp, 1, R, s)

    # ------------------------------------------------------------------ backward
    def backward(self, s, seg_pad, seg_one=None):
        """From C (row coefficients, pad rows zero): expert grads, dW_head share, dX."""
        E, R, T = self.E, self.R, self.T
        L = len(self.layers)
        di = self.dims[-2]
        if not self.folded:
            # d_packed = (C head_w) x relu mask; dW, db (ones column of X); dX; dW_head share = C^T O
            tcall("dpacked_gemm", "smes_gemm_ragged_m", ptr(self.Cm), self.ldc, R, ptr(self.head_wT_bf), 1,
                  self.d_out, self.ldc, 0, ptr(self.seg_all if seg_one is None else seg_one), None, 0, None,
                  ptr(self.bits), R, ptr(self.dO),
                  self.d_out, 0, R, s)
            gw, gb = self.g_layers[0]
            tcall("fc1_wgrad", "smes_gemm_ragged_k", ptr(self.dO), self.d_out, ptr(self.X), self.ld_in[0], R, E,
                  self.d_out, self.d, ptr(seg_pad), ptr(gw), ptr(gb), s)
            tcall("fc1_dgrad", "smes_gemm_ragged_m", ptr(self.dO), self.d_out, R, ptr(self.w_bf[0]), E, self.d,
                  self.d_out, 1, ptr(seg_pad), None, 0, None, None, R, ptr(self.dX), self.d, 0, R, s)
            tcall("head_wgrad", "smes_gemm_ragged_k", ptr(self.Cm), self.ldc, ptr(self.O), self.d_out, R, 1, T,
                  self.d_out, ptr(self.seg_all if seg_one is None else seg_one), ptr(self.g_head_w3), None, s)
            return
        inp = self.X if L == 1 else self.H
        if L == 2 and self.fuse:
            tcall("mlp_dgrad", "smes_mlp_dgrad", ptr(self.Cm), self.ldc, R, ptr(self.G), self.ldg, ptr(self.w_bf[0]), E, self.d, di,
                 ptr(seg_pad), ptr(self.bits), R, ptr(self.dX), self.d, None if self.fuse_wgrad else ptr(self.dH), di, s)
        else:
            dst = self.dX if L == 1 else self.dH
            tcall(f"fc{L}_dgrad_folded", "smes_gemm_ragged_m", ptr(self.Cm), self.ldc, R, ptr(self.G), E, di, self.ldg, 1, ptr(seg_pad), None,
                 0, None, ptr(self.bits) if L == 2 else None, R, ptr(dst), di, 0, R, s)
        tcall(f"fc{L}_wgrad_folded", "smes_gemm_ragged_k", ptr(self.Cm), self.ldc, ptr(inp), self.ld_in[L - 1], R, E,
              self.ldg, di, ptr(seg_pad), ptr(self.Qe), ptr(self.csum), s)
        gw, gb = self.g_layers[L - 1]
        tcall("unfold", "smes_unfold_grads", E, T, self.ldg, self.d_out, di, ptr(self.Qe), self.ldg * di, di, 1,
              ptr(self.csum), self.ldg, ptr(self.head_w), ptr(self.w_bf[-1]), ptr(self.b32[-1]), ptr(gw), ptr(gb),
              ptr(self.work), ptr(self.g_head_w), s)
        if L == 2 and self.fuse_wgrad:
            gw0, gb0 = self.g_layers[0]
            tcall("mlp_wgrad", "smes_mlp_wgrad", ptr(self.Cm), self.ldc, R, ptr(self.G), self.ldg, ptr(self.X),
                  self.ld_in[0], E, self.d, di, ptr(seg_pad), ptr(self.bits), R, ptr(gw0), ptr(gb0), s)
        elif L == 2:
            gw0, gb0 = self.g_layers[0]
            tcall("fc1_wgrad", "smes_gemm_ragged_k", ptr(self.dH), di, ptr(self.X), self.ld_in[0], R, E, di, self.d, ptr(seg_pad),
                 ptr(gw0), ptr(gb0), s)
            if not self.fuse:
                tcall("fc1_dgrad", "smes_gemm_ragged_m", ptr(self.dH), di, R, ptr(self.w_bf[0]), E, self.d, di, 1, ptr(seg_pad),
                     None, 0, None, None, R, ptr(self.dX), self.d, 0, R, s)
