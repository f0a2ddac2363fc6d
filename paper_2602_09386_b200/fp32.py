"""fp32 arithmetic mode of the SMES forward + loss (BASELINE c1; north star: fp32 within 1e-5).

The reference is float64 NumPy (taskmoe/linalg.py:3-8).  The bf16 engine (engine.py) stores
operands in bf16; this executor keeps every activation and weight in fp32 instead:

* dense contractions (router logits routing.py:101-103, the expert pools execution.py:126-158) run
  on the tcgen05 grouped GEMM as **bf16x3 products** (csrc/gemm.cu ``smes_gemm_ragged_m_x3``):
  each fp32 operand is stored as three bf16 planes (x = x0 + x1 + x2, 24 significant bits) and the
  six leading cross terms accumulate in the fp32 TMEM accumulator -- an fp32 GEMM on the tensor
  cores, six bf16 MMAs per fp32 MMA;
* routing is the same fused progressive router as the bf16 path (fp64 Stage I, exact Stage II) on
  the fp32 logits;
* plan and gather are the same stable counting sort, moving the bf16 planes of h;
* combine + heads + BCE run in fp32 (csrc/fp32.cu ``combine_fwd_f32``), loss sums in fp64.

Widths: every contraction dimension (d, hidden pool widths) must be a multiple of 64 -- the
``forward_sparse(..., precision="fp32")`` shim zero-pads.  Forward only (c1 is fwd + loss): the
backward of the layer runs in the bf16 engine.
"""
from __future__ import annotations

import torch

from ._lib import call, ptr
from ._lib import tcall as _tagged
from .engine import ACT, SMESParams, _require_cuda, _round
from .errors import ConfigError, NumericsError, ShapeError

__all__ = ["SMESForwardF32"]


class SMESForwardF32:
    """Fixed-shape fp32 forward (+ loss) of the SMES layer on one GPU."""

    def __init__(self, params: SMESParams, batch_size: int, k_shared: int, k_adaptive: int,
                 device: torch.device | str | None = None, lb_experts: int | None = None,
                 dense_probs_in_stats: bool = False):
        _require_cuda()
        self.dev = torch.device(device or "cuda")
        p = params
        T, E, d = p.num_tasks, p.num_experts, p.d_in
        B, ks, ka = int(batch_size), int(k_shared), int(k_adaptive)
        K = ks + ka
        if ks < 0 or ka < 0 or K < 1:
            raise ConfigError("budget must activate at least one expert per task")
        if K > E:
            raise ConfigError(f"budget k={K} exceeds expert count {E}")
        if B < 1:
            raise ShapeError("empty batch")
        dims = [d] + [l.d_out for l in p.layers]
        if (T * E) % 8 or any(x % 64 for x in dims[:-1]) or dims[-1] % 4:
            raise ShapeError(f"fp32 mode needs contraction widths % 64 == 0, d_out % 4 == 0 and T*E % 8 == 0 "
                             f"(dims={dims}, T*E={T * E})")
        for i, l in enumerate(p.layers):
            if l.d_in != dims[i] or l.weight.shape[0] != E:
                raise ShapeError(f"expert layer {i} has shape {tuple(l.weight.shape)}")
            if l.act not in ACT:
                raise ConfigError(f"unknown nonlinearity '{l.act}', expected one of {tuple(ACT)}")
        self.p = p
        self.T, self.E, self.d, self.B, self.ks, self.ka, self.K = T, E, d, B, ks, ka, K
        self.E_lb = int(lb_experts) if lb_experts else E
        self.dims, self.d_out = dims, dims[-1]
        self.dense = bool(dense_probs_in_stats)
        self.umax = min(E, ks + T * ka)
        self.rows_cap = _round(B * self.umax + E * 127, 128)
        self.B_pad = _round(B, 128)
        self.rpw = call("smes_route_rows_per_warp", B)
        self.C = call("smes_route_num_chunks", B, self.rpw)
        self.grid = call("smes_combine_fwd_f32_grid", B)
        self._alloc()
        self.refresh_weights()

    def _alloc(self):
        dev, T, E, B, K, d, R = self.dev, self.T, self.E, self.B, self.K, self.d, self.rows_cap
        i32, f32, f64, bf = torch.int32, torch.float32, torch.float64, torch.bfloat16
        z = lambda *s, dt=f32: torch.zeros(*s, dtype=dt, device=dev)
        self.h = z(B, d)                               # layer input, fp32
        self.h3 = z(B, 3 * d, dt=bf)                   # its bf16 planes
        self.z = z(B, T * E)                           # router logits, element (t,b,e) at b*T*E + t*E + e
        self.shared = z(B, self.ks, dt=i32)
        self.adaptive = z(T, B, self.ka, dt=i32)
        self.active = z(T, B, K, dt=i32)
        self.wsel = z(T, B, K)
        self.umask = z(B, (E + 31) // 32, dt=i32)
        self.usize = z(B, dt=i32)
        self.chunk_union = z(self.C, E, dt=i32)
        self.chunk_active = z(self.C, E, dt=i32)
        self.chunk_mass = z(self.C, E, dt=f64)
        self.chunk_dmass = z(self.C, E, dt=f64)
        self.chunk_base = z(self.C, E, dt=i32)
        self.loads = z(E, dt=i32)
        self.stats_raw = z(3 * E, dt=f64)
        self.seg_pad = z(E + 1, dt=i32)
        self.seg_log = z(E + 1, dt=i32)
        self.totals = z(3, dt=i32)
        self.ticket = z(call("smes_plan_reduce_work_ints", self.C, E), dt=i32)
        self.seg_half = z(2 * E + 1, dt=i32)
        self.flag = z(1, dt=i32)
        self.row_of = z(B, self.umax, dt=i32)
        self.gather_inst = z(R, dt=i32)
        self.gather_exp = z(R, dt=i32)
        self.X3 = z(R, 3 * d, dt=bf)                   # packed rows of h, bf16 planes
        self.outs = [z(R, w) for w in self.dims[1:]]   # fp32 pool outputs
        self.outs3 = [z(R, 3 * w, dt=bf) for w in self.dims[1:-1]]   # planes of the hidden pool outputs
        self.reps = z(T, B, self.d_out)
        self.logits = z(T, B)
        self.preds = z(T, B)
        self.labels = z(T, B)
        self.loss_part = z(self.grid, dt=f64)
        self.loss_out = z(3, dt=f64)
        self.ticket_loss = z(1, dt=i32)      # last-CTA ticket of the fused loss finalize
        self.stats_out = z(3 * E + 1, dt=f64)
        self.freq32 = z(E)
        self.seg_router = torch.tensor([0, self.B_pad], dtype=i32, device=dev)

    def _split(self, tag, src, rows, cols, dst, rows_dev=None, s=None):
        _tagged(tag, "smes_split_bf16x3", rows, cols, ptr(src), src.stride(0), ptr(dst), dst.stride(0),
                None if rows_dev is None else rows_dev, s if s is not None else self._stream())

    def refresh_weights(self):
        """fp32 master parameters -> the kernels' bf16 planes (buffers allocated once: a captured
        graph sees the refreshed weights)."""
        p, T, E, d, dev = self.p, self.T, self.E, self.d, self.dev
        if tuple(p.router_w.shape) != (T, E, d):
            raise ShapeError("refresh_weights: parameter shapes changed; build a new executor")
        first = not hasattr(self, "wr3")
        if first:
            self.wr32 = torch.empty(T * E, d, device=dev)
            self.wr3 = torch.empty(T * E, 3 * d, dtype=torch.bfloat16, device=dev)
            self.br = torch.empty(T * E, device=dev)
            self.w32 = [torch.empty(l.weight.shape, device=dev) for l in p.layers]
            self.w3 = [torch.empty(E, l.d_out, 3 * l.d_in, dtype=torch.bfloat16, device=dev) for l in p.layers]
            self.b32 = [torch.empty(l.bias.shape, device=dev) for l in p.layers]
            self.head_w = torch.empty(T, self.d_out, device=dev)
            self.head_b = torch.empty(T, device=dev)
            self.tw = torch.empty(T, dtype=torch.float64, device=dev)
            self.lam = torch.empty(T, device=dev)
        self.wr32.copy_(p.router_w.detach().reshape(T * E, d))
        self.br.copy_(p.router_b.detach().reshape(T * E))
        self._split("split_w", self.wr32, T * E, d, self.wr3)
        for w32, w3, b32, l in zip(self.w32, self.w3, self.b32, p.layers):
            w32.copy_(l.weight.detach())
            b32.copy_(l.bias.detach())
            self._split("split_w", w32.view(-1, l.d_in), E * l.d_out, l.d_in, w3.view(-1, 3 * l.d_in))
        self.head_w.copy_(p.head_w.detach())
        self.head_b.copy_(p.head_b.detach())
        tw = p.task_weights if p.task_weights is not None else torch.ones(T)
        lam = p.task_loss_weights if p.task_loss_weights is not None else torch.ones(T)
        self.tw.copy_(torch.as_tensor(tw))
        self.lam.copy_(torch.as_tensor(lam))
        self.beta = float(p.lb_strength)

    def _stream(self):
        return torch.cuda.current_stream(self.dev).cuda_stream

    def set_inputs(self, h: torch.Tensor, labels: torch.Tensor | None = None):
        if h.shape != (self.B, self.d):
            raise ShapeError(f"hidden has shape {tuple(h.shape)}, executor expects ({self.B}, {self.d})")
        self.h.copy_(h, non_blocking=True)
        if labels is not None:
            if labels.shape != (self.T, self.B):
                raise ShapeError(f"labels shape {tuple(labels.shape)} does not match ({self.T}, {self.B})")
            self.labels.copy_(labels, non_blocking=True)

    def forward(self, with_loss: bool = True, frozen: bool = False):
        """router logits -> progressive routing -> plan + gather -> expert pools -> combine, heads,
        BCE, LoadStats and the loss (model.py:267-324, training.py:60-94).  ``frozen``: reuse the
        selections already in ``shared``/``adaptive`` (model.py:284-300)."""
        s = self._stream()
        T, E, B, d, K = self.T, self.E, self.B, self.d, self.K
        R = self.rows_cap
        self._split("split_h", self.h, B, d, self.h3, s=s)
        _tagged("router_fwd_f32", "smes_gemm_ragged_m_x3", ptr(self.h3), 3 * d, B, ptr(self.wr3), 1, T * E, d,
                ptr(self.seg_router), ptr(self.br), 0, ptr(self.z), T * E, B, s)
        _tagged("route", "smes_route_batch", ptr(self.z), E, T * E, None, ptr(self.tw), T, B, E, self.ks, self.ka,
                self.rpw, ptr(self.shared), ptr(self.adaptive), ptr(self.active), ptr(self.wsel), ptr(self.umask),
                ptr(self.usize), ptr(self.chunk_union), ptr(self.chunk_active), ptr(self.chunk_mass),
                ptr(self.chunk_dmass), None, ptr(self.flag), int(frozen), s)
        _tagged("plan_reduce", "smes_plan_reduce_stats", self.C, E, ptr(self.chunk_union), ptr(self.chunk_active),
                ptr(self.chunk_mass), ptr(self.chunk_dmass), ptr(self.chunk_base), ptr(self.loads),
                ptr(self.stats_raw), ptr(self.seg_pad), ptr(self.seg_log), ptr(self.totals), ptr(self.ticket),
                ptr(self.seg_half), K, self.E_lb, float(B * T), int(self.dense), ptr(self.stats_out),
                ptr(self.freq32), s)
        _tagged("plan_scatter", "smes_plan_scatter", B, E, 3 * d, self.rpw, ptr(self.umask), ptr(self.chunk_base),
                ptr(self.seg_pad), ptr(self.loads), ptr(self.h3), 3 * d, ptr(self.X3), 3 * d, ptr(self.row_of),
                self.umax, ptr(self.gather_inst), ptr(self.gather_exp), None, 0, 0, s)
        inp, ld = self.X3, 3 * d
        padded_rows = self.totals.data_ptr() + 4          # totals[1]: rows of the padded segments
        for i, l in enumerate(self.p.layers):
            n, k = self.dims[i + 1], self.dims[i]
            _tagged(f"fc{i + 1}_fwd_f32", "smes_gemm_ragged_m_x3", ptr(inp), ld, R, ptr(self.w3[i]), E, n, k,
                    ptr(self.seg_pad), ptr(self.b32[i]), ACT[l.act], ptr(self.outs[i]), n, R, s)
            if i < len(self.p.layers) - 1:
                self._split(f"split_fc{i + 1}", self.outs[i], R, n, self.outs3[i], rows_dev=padded_rows, s=s)
                inp, ld = self.outs3[i], 3 * n
        if with_loss:
            # combine + heads + BCE, the loss finalize in the last CTA (one launch fewer)
            _tagged("combine_fwd_f32", "smes_combine_fwd_f32_loss", T, B, E, K, self.d_out, self.umax,
                    ptr(self.umask), ptr(self.usize), ptr(self.row_of), ptr(self.active), ptr(self.wsel),
                    ptr(self.outs[-1]), self.d_out, ptr(self.head_w), ptr(self.head_b), ptr(self.reps),
                    ptr(self.logits), ptr(self.preds), ptr(self.labels), ptr(self.lam), ptr(self.loss_part),
                    self.grid, ptr(self.ticket_loss), 1.0 / B, self.beta, self.stats_out[3 * E:].data_ptr(),
                    ptr(self.loss_out), s)
        else:
            _tagged("combine_fwd_f32", "smes_combine_fwd_f32", T, B, E, K, self.d_out, self.umax, ptr(self.umask),
                    ptr(self.usize), ptr(self.row_of), ptr(self.active), ptr(self.wsel), ptr(self.outs[-1]),
                    self.d_out, ptr(self.head_w), ptr(self.head_b), ptr(self.reps), ptr(self.logits),
                    ptr(self.preds), None, ptr(self.lam), None, self.grid, s)

    def check_finite(self):
        """Raise NumericsError if the router saw a non-finite logit (read after a forward)."""
        if int(self.flag.item()):
            raise NumericsError("routing logits must be finite")

    def n_act(self) -> int:
        return int(self.totals[2].item())

    def work_model(self, n_act: int, balance: float = 260.0) -> dict:
        """Algorithmic (flops, HBM bytes, bound) per launch tag (fp32 mode).  GEMM flops
        are the six bf16 MMAs of each fp32 product (the work the tensor pipe does: 6 * 2*M*N*K);
        bound = "tensor" when flops/bytes exceeds the machine balance."""
        T, E, B, d, K = self.T, self.E, self.B, self.d, self.K
        w = {"split_h": (0.0, B * d * (4 + 6)),
             "router_fwd_f32": (2.0 * B * d * T * E, B * (3 * d * 2 + T * E * 4)),
             "route": (0.0, B * T * E * 4 + B * T * K * 8 + B * (self.ks * 4 + 4)),
             "plan_scatter": (0.0, B * 3 * d * 2 + n_act * (3 * d * 2 + 12)),
             "combine_fwd_f32": (2.0 * T * B * K * self.d_out, n_act * self.d_out * 4 + T * B * self.d_out * 4)}
        for i in range(len(self.p.layers)):
            n, k = self.dims[i + 1], self.dims[i]
            w[f"fc{i + 1}_fwd_f32"] = (2.0 * n_act * n * k, n_act * (3 * k * 2 + n * 4) + E * n * 3 * k * 2)
            if i < len(self.p.layers) - 1:
                w[f"split_fc{i + 1}"] = (0.0, n_act * n * (4 + 6))
        out = {}
        for k, (fl, by) in w.items():
            if k.endswith("_f32") and k != "combine_fwd_f32":
                fl *= 6.0
            out[k] = (fl, by, "tensor" if by and fl / by > balance else "hbm")
        return out


def split_planes(x: torch.Tensor) -> torch.Tensor:
    """(rows, cols) fp32 -> (rows, 3 cols) bf16 planes [x0 | x1 | x2] on the device (split kernel)."""
    x = x.float().contiguous()
    rows, cols = x.shape
    out = torch.empty(rows, 3 * cols, dtype=torch.bfloat16, device=x.device)
    call("smes_split_bf16x3", rows, cols, ptr(x), cols, ptr(out), 3 * cols, None,
         torch.cuda.current_stream(x.device).cuda_stream)
    return out
