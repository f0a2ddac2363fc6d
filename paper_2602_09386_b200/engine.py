"""SMES layer engine: device workspaces + the kernel sequence of one step.

One :class:`SMESEngine` owns every buffer of the hot path for a fixed shape
(B, T, E, budget, expert stack).  ``forward`` / ``backward`` issue only
``_smes.so`` kernels on the current CUDA stream -- no host syncs, no torch
compute -- so a whole fwd+bwd step can be captured in one CUDA graph
(``capture_step``).

Kernel sequence (reference functions in taskmoe/ they replace):
  fwd: router GEMM (routing.py:101-103) -> route (routing.py:235-281)
       -> plan reduce + scatter/gather (execution.py:85-123, model.py:301)
       -> expert GEMMs (execution.py:126-158) -> stats finalize (balance.py:54-80)
       -> combine + heads + BCE (execution.py:161-191, model.py:202-208,
          training.py:54-57) -> loss finalize (training.py:90-94)
  bwd: combine/heads/LB backward (training.py:146-179, balance.py:83-99)
       -> expert dgrad/wgrad/bias (training.py:180-191) -> router dgrad/wgrad
          (training.py:209-212) -> un-permute (training.py:192) -> head grads
"""
from __future__ import annotations

import math
import os
from dataclasses import dataclass, field

import torch

from . import _lib
from ._lib import call, ptr
from .errors import ConfigError, CudaError, ShapeError

ACT = {"identity": 0, "relu": 1}


def _require_cuda():
    if not torch.cuda.is_available():
        raise CudaError("SMES kernels need a CUDA device (sm_100a); there is no CPU fallback")
    _lib.load()


@dataclass
class ExpertLayer:
    """One expert pool (experts.py:17-73): W (E, d_out, d_in), b (E, d_out), act."""
    weight: torch.Tensor
    bias: torch.Tensor
    act: str = "relu"

    @property
    def d_in(self):
        return self.weight.shape[2]

    @property
    def d_out(self):
        return self.weight.shape[1]


@dataclass
class SMESParams:
    """Parameters of the SMES layer in the reference layouts (model.py:36-111), fp32 masters."""
    router_w: torch.Tensor          # (T, E, d)
    router_b: torch.Tensor          # (T, E)
    layers: list                    # [ExpertLayer]
    head_w: torch.Tensor            # (T, d_out)
    head_b: torch.Tensor            # (T,)
    task_weights: torch.Tensor | None = None   # (T,) Stage-I pooling weights (routing.py:79-87)
    task_loss_weights: torch.Tensor | None = None  # (T,) lambda_t (training.py:138)
    lb_strength: float = 0.0        # beta (model.py:158)

    @property
    def num_tasks(self):
        return self.router_w.shape[0]

    @property
    def num_experts(self):
        return self.router_w.shape[1]

    @property
    def d_in(self):
        return self.router_w.shape[2]

    @property
    def d_out(self):
        return self.layers[-1].d_out


def _tagged(tag, name, *args):
    _lib.tag = tag
    try:
        return call(name, *args)
    finally:
        _lib.tag = None


def _round(x, m):
    return (x + m - 1) // m * m


def row_buffer_specs(T: int, E: int, B: int, k_shared: int, k_adaptive: int, dims, acts) -> list:
    """The engine's buffers sized by the packed-row capacity -- the per-batch part of its memory that
    a ``DeviceWorkspace`` block can back (workspace.py:42-57 sizes blocks by packed rows):
    (attribute, shape, dtype) in carve order.  ``dims`` = [d, widths of the pools], ``acts`` their
    nonlinearities."""
    umax = min(E, k_shared + T * k_adaptive)
    R = _round(B * umax + E * 127, 128)
    bf, i32, f32 = torch.bfloat16, torch.int32, torch.float32
    ld_in = [w + 64 for w in dims[:-1]]
    specs = [("gather_inst", (R,), i32), ("gather_exp", (R,), i32), ("X", (R, ld_in[0]), bf)]
    for i, w in enumerate(dims[1:]):
        last = i == len(dims) - 2
        specs.append((f"outs.{i}", (R, w if last else ld_in[i + 1]), bf))
    for i, (w, act) in enumerate(zip(dims[1:], acts)):
        if act == "relu":
            specs.append((f"bits.{i}", (w // 32, R), i32))
    specs += [("P", (R, _round(T, 8)), f32), ("Cm", (R, _round(T, 16)), bf)]
    for i, w in enumerate(dims[1:]):
        specs.append((f"d_outs.{i}", (R, w), bf))
    specs += [("dX", (R, dims[0]), bf), ("colsum_part", (R // 128, max(max(dims), T * E)), f32)]
    return specs


def workspace_bytes(params: "SMESParams", batch_size: int, k_shared: int, k_adaptive: int,
                    align: int = 256) -> int:
    """Bytes of one engine's packed-row buffers (carved 256-byte aligned): the block a
    ``WorkspacePool`` grants per concurrent stream (``DeviceWorkspace.carve``)."""
    dims = [params.d_in] + [l.d_out for l in params.layers]
    specs = row_buffer_specs(params.num_tasks, params.num_experts, int(batch_size), int(k_shared),
                             int(k_adaptive), dims, [l.act for l in params.layers])
    off = 0
    for _, shape, dt in specs:
        off = -(-off // align) * align + math.prod(shape) * torch.empty((), dtype=dt).element_size()
    return off


def router_wgrad_splits(B_pad: int, I: int, J: int, dev) -> int:
    """Split-K factor of the router weight gradient (dW_r = dz^T h, K = the batch): enough
    (split, tile) work units for ~2 rounds of the persistent grid, no more -- every split writes an I x J fp32
    partial that part_reduce reads back (at T*E = 8192, d = 1024 the former fixed 64 splits moved
    4.3 GB per step).  Tiles are 128 x 256 (x 128 for J < 256), csrc/gemm.cu."""
    try:
        n_sms = torch.cuda.get_device_properties(dev).multi_processor_count
    except Exception:
        n_sms = 148
    if os.environ.get("SMES_RW_SPLITS"):          # A/B measurements (tools/)
        return max(1, min(64, B_pad // 256, int(os.environ["SMES_RW_SPLITS"])))
    tiles = -(-I // 128) * (-(-J // 256) if J >= 256 else -(-J // 128))
    # whole rounds of the persistent GEMM grid: floor, so the last round is not nearly empty
    return max(1, min(64, B_pad // 256, 2 * n_sms // tiles))


class SMESEngine:
    """Fixed-shape executor of the SMES hot path on one GPU."""

    def __init__(self, params: SMESParams, batch_size: int, k_shared: int, k_adaptive: int,
                 dense_probs_in_stats: bool = False, keep_reps: bool = True,
                 device: torch.device | str | None = None, csum_from_gemm: bool = False,
                 fuse_mlp: bool = True, fuse_wgrad: bool = False, lb_experts: int | None = None,
                 workspace=None):
        """``workspace``: optional ``(DeviceWorkspace, PageBlock)``.  The packed-row buffers (the
        per-batch memory, ``row_buffer_specs``) are then carved from that block of the pool's HBM
        arena instead of being allocated, so concurrent serving streams share one provisioned pool
        (taskmoe/workspace.py:42-262); give the block back with ``pool.release(block, stream=s)``."""
        _require_cuda()
        self.dev = torch.device(device or "cuda")
        self._ws = workspace
        p = params
        self.p = p
        T, E, d = p.num_tasks, p.num_experts, p.d_in
        B = int(batch_size)
        ks, ka = int(k_shared), int(k_adaptive)
        K = ks + ka
        if ks < 0 or ka < 0:
            raise ConfigError("budget counts must be non-negative")
        if K < 1:
            raise ConfigError("budget must activate at least one expert per task")
        if K > E:
            raise ConfigError(f"budget k={K} exceeds expert count {E}: stage-II would have only "
                              f"{E - ks} candidates for {ka} adaptive picks")
        if B < 1:
            raise ShapeError("empty batch")
        if (T * E) % 8 or d % 32:
            raise ShapeError(f"kernel layout needs T*E % 8 == 0 and d % 32 == 0 (T*E={T * E}, d={d})")
        dims = [d] + [l.d_out for l in p.layers]
        if any(x % 32 for x in dims):
            raise ShapeError(f"expert widths must be multiples of 32, got {dims}")
        for i, l in enumerate(p.layers):
            if l.d_in != dims[i] or l.weight.shape[0] != E:
                raise ShapeError(f"expert layer {i} has shape {tuple(l.weight.shape)}")
            if l.act not in ACT:
                raise ConfigError(f"unknown nonlinearity '{l.act}', expected one of {tuple(ACT)}")
        self.T, self.E, self.d, self.B, self.ks, self.ka, self.K = T, E, d, B, ks, ka, K
        # E of the load-balancing coefficient E / K (balance.py:69-70, :97): the logical expert count
        # when the shim pads the pool with never-selected experts (model.py)
        self.E_lb = int(lb_experts) if lb_experts else E
        self.dims = dims
        self.d_out = dims[-1]
        self.grid = call("smes_combine_grid", B, T, self.d_out)
        self.dense = bool(dense_probs_in_stats)
        self._csum_from_gemm = bool(csum_from_gemm)
        self.keep_reps = keep_reps
        self.umax = min(E, ks + T * ka)
        self.rows_cap = _round(B * self.umax + E * 127, 128)
        self.B_pad = _round(B, 128)
        # head folding (csrc/fold.cu) for training steps: needs an identity last pool and the
        # sparse LB reading (the fused training combine produces the row coefficients C)
        self.can_fold = p.layers[-1].act == "identity" and not self.dense and T <= 32
        self._folded = False
        # fused expert MLP (csrc/mlp.cu) for folded training steps: relu fc1 + identity fc2
        lay = p.layers
        mlp_ok = bool(fuse_mlp and self.can_fold and len(lay) == 2 and lay[0].act == "relu"
                      and d % 64 == 0 and lay[0].d_out % 128 == 0 and T <= 16)
        # the fused kernels support d <= 512 (fwd) / 256 (dgrad); at d = 512 (c3) the fused forward
        # measured slower than the tensor-bound fc1 GEMM + folded P GEMM, so both use d <= 256
        self.fuse_mlp_fwd = mlp_ok and d <= 256
        self.fuse_mlp = mlp_ok and d <= 256
        self._fold_fresh = False            # G/c current for the loaded weights (inference scoring)
        # fc1 wgrad with dH recomputed per row block (csrc/mlp.cu mlp_wgrad) instead of storing dH:
        # measured slower at c2 (one CTA per (expert, d_ff chunk) re-streams X), so off by default
        self.fuse_wgrad = bool(fuse_wgrad and self.fuse_mlp)
        # SMES_GATHER_X=1: folded training steps read the layer input rows straight from h with
        # TMA gather4 (mlp_fwd and the fc1 weight gradient), so the packed copy X (the reference's
        # hidden[gather_instances], model.py:301) is never written.  Bit-identical, but measured
        # slower at c2 (0.776 vs 0.524 ms: gather4 ran at ~1 op / 75 cycles per SM whatever the
        # number of issuing lanes -- mlp_fwd 124 -> 181 us, fc1 wgrad 84 -> 351 us against the
        # scatter's 38 -> 15 us, tools/ab_gather.sh), so the packed copy stays the default.
        self.gather_x = os.environ.get("SMES_GATHER_X", "0") == "1"
        # SMES_FWD_PACK=1: mlp_fwd's own gather warp copies the X rows from h (LDGSTS) and writes the
        # packed X the weight gradient reads, so the plan scatter only places rows.  Bit-identical;
        # measured slower at c2 (mlp_fwd 125 -> 187 us against the scatter's 37 -> 15 us, step
        # 0.5225 -> 0.557 ms, tools/ab_pack.sh), so off by default
        self.fwd_pack = os.environ.get("SMES_FWD_PACK", "0") == "1"
        self._x_gathered = False
        self._x_packed_by_fwd = False
        self.rpw = call("smes_route_rows_per_warp", B)
        self.C = call("smes_route_num_chunks", B, self.rpw)
        # fused router front (csrc/front.cu): router GEMM -> routing straight from TMEM, so the
        # logits never round-trip HBM.  ``keep_logits`` still writes z (the API's router_logits,
        # the dense-reading backward and the parity checks read it); training steps turn it off.
        self.use_front = bool(call("smes_route_front_supported", T, E, d, ks, ka))
        self.keep_logits = True
        # serial: every launch on the caller's stream (no backward side stream) -- the bench's
        # per-kernel CUDA-event timing needs it, since events only see the stream they are on
        self.serial = False
        # measured 0.531 vs 0.529 ms at c2 with the fold on the side stream (tools/ab_fold.sh): off by default
        self.fold_side = os.environ.get("SMES_FOLD_SIDE", "0") == "1"
        self.fold_in_reduce = False        # set in _alloc once the fold buffers exist
        self.q_splits = 1
        self._alloc()
        self.refresh_weights()

    # ------------------------------------------------------------------ buffers
    def _alloc(self):
        dev, T, E, B, K, d = self.dev, self.T, self.E, self.B, self.K, self.d
        i32, f32, f64, bf = torch.int32, torch.float32, torch.float64, torch.bfloat16
        z = lambda *s, dt=f32: torch.zeros(*s, dtype=dt, device=dev)
        EW = (E + 31) // 32
        R = self.rows_cap
        # packed-row buffers: carved from the workspace block when one is bound, else allocated
        specs = row_buffer_specs(T, E, B, self.ks, self.ka, self.dims, [l.act for l in self.p.layers])
        if self._ws is not None:
            ws, block = self._ws
            bufs = ws.carve(block, [(shape, dt) for _, shape, dt in specs])
            for b_ in bufs:
                b_.zero_()
        else:
            bufs = [torch.zeros(shape, dtype=dt, device=dev) for _, shape, dt in specs]
        rows = dict(zip([n for n, _, _ in specs], bufs))
        self.workspace_nbytes = sum(b_.numel() * b_.element_size() for b_ in bufs)
        self.z = z(B, T * E)
        self.shared = z(B, self.ks, dt=i32)
        self.adaptive = z(T, B, self.ka, dt=i32)
        self.active = z(T, B, K, dt=i32)
        self.wsel = z(T, B, K)
        self.umask = z(B, EW, dt=torch.int32)
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
        self.totals = z(3, dt=i32)     # {0, padded rows, N_act}; [0:2] is the one-group segment table
        self.ticket = z(call("smes_plan_reduce_work_ints", self.C, E), dt=i32)
        self.flag = z(1, dt=i32)
        self.row_of = z(B, self.umax, dt=i32)
        self.gather_inst = rows["gather_inst"]
        self.gather_exp = rows["gather_exp"]
        # every wgrad Q operand (each layer's input and h) carries 64 extra columns whose first one
        # is 1.0: the wgrad GEMM's extra N=64 tile then yields the bias gradient (sum over rows)
        self.ld_in = [w + 64 for w in self.dims[:-1]]           # leading dims of layer inputs
        self.X = rows["X"]
        self.X[:, d] = 1.0
        self.outs = []
        for i, w in enumerate(self.dims[1:]):
            last = i == len(self.dims) - 2
            o = rows[f"outs.{i}"]
            if not last:
                o[:, w] = 1.0
            self.outs.append(o)
        self.ld_out = [o.shape[1] for o in self.outs]
        self.bits = [rows.get(f"bits.{i}") for i in range(len(self.p.layers))]
        self.reps = z(T, B, self.d_out, dt=bf)     # required by the backward (head grads)
        self.ldp = _round(T, 8)
        self.P = rows["P"]                          # head projections P = O head_W^T of every packed row
        self.ldc = _round(T, 16)
        self.Cm = rows["Cm"]                        # C[row, t] = w[row, t] * dlogit_t (training step)
        self.hw_part = z(2 * E, T, self.d_out)      # dW_head split-K partials (expert halves)
        # bias grads folded into the training combine: last (identity) pool via per-(expert, task)
        # sums of C, router via column sums of dz (per-warp smem accumulators, fixed-order reduce)
        fits = 8 * 4 * (E * T + T * E) <= 150 * 1024
        self.fuse_rb = fits
        # csum_from_gemm: take the per-(expert, task) sums of C from the folded wgrad's ones column
        # instead of the combine's smem partials (automatic when those do not fit)
        self.fuse_b_last = fits and self.p.layers[-1].act == "identity" and not self._csum_from_gemm
        self.part_csum = z(self.grid, E, T) if self.fuse_b_last else None
        self.part_rb = z(self.grid, T * E) if self.fuse_rb else None
        self.csum = z(E, T)
        if self.can_fold:
            di = self.dims[-2]
            self.ldg = _round(T, 8)
            self.G_fold = z(E, self.ldg, di, dt=bf)         # head_w W_last (per expert), rows >= T zero
            self.c_fold = z(E, self.ldg)                    # head_w b_last
            # folded pool's wgrad Q = C^T H per expert.  Small banks: Q^T = H^T C (I = d_in, N = T tile,
            # the grid covers the SMs) in (E, d_in(+1), ldg) layout; large banks (tensor-core unfold):
            # Q = C^T H in (E, ldg, d_in) with colsum(C) from the in-tile ones MMA
            self.q_swapped = bool(call("smes_fold_gemm_path", E, T, self.d_out, di))
            if self.q_swapped:
                self.Qe = z(E, self.ldg, di)
                self.q_strides = (self.ldg * di, di, 1)
            else:
                self.q_rows = di if self.fuse_b_last else di + 1   # + the ones column -> per-expert sums of C
                self.Qe = z(E, self.q_rows, self.ldg)
                self.q_strides = (self.q_rows * self.ldg, 1, self.ldg)
                tiles = E * ((self.q_rows + 127) // 128)
                # measured no faster at c2 (77 vs 75 us eager, tools/ab_split.sh): off unless SMES_WGRAD_SPLIT > 1
                self.q_splits = int(os.environ.get("SMES_WGRAD_SPLIT", 1))
                if self.q_splits > 1:
                    self.q_work = z(call("smes_gemm_ragged_k_split_work", E, self.q_rows, self.ldg, self.q_splits, 0))
            self.csum_q = z(E, self.ldg)                    # per-expert column sums of C
            self.fold_work = z(call("smes_fold_work_floats", E, T, self.d_out, di))
            self.fold_in_reduce = bool(call("smes_fold_full_supported", E, T, self.ldg, self.d_out, di)) and \
                os.environ.get("SMES_FOLD_IN_REDUCE", "1") == "1"
        self.seg_half = z(2 * E + 1, dt=i32)
        self.logits = z(T, B)
        self.preds = z(T, B)
        self.labels = z(T, B)
        self.loss_part = z(self.grid, dt=f64)
        self.loss_out = z(3, dt=f64)
        self.stats_out = z(3 * E + 1, dt=f64)
        self.freq32 = z(E)
        self.seg_router = torch.tensor([0, self.B_pad], dtype=i32, device=dev)
        # router wgrad reduces over B: split the batch into 256-row groups (split-K), reduce after
        self.rw_splits = router_wgrad_splits(self.B_pad, T * E, d, dev)
        edges = [min(self.B_pad, (self.B_pad // self.rw_splits) // 128 * 128 * i) for i in range(self.rw_splits)]
        self.seg_router_split = torch.tensor(edges + [self.B_pad], dtype=i32, device=dev)
        self.rw_part = z(self.rw_splits, T * E, d)
        self.rb_part = z(self.rw_splits, T * E)
        # backward
        self.d_outs = [rows[f"d_outs.{i}"] for i in range(len(self.dims) - 1)]   # grad w.r.t. each pool's output
        self.dX = rows["dX"]
        self.dz = z(self.B_pad, T * E, dt=bf)
        # all parameter gradients live in ONE flat fp32 buffer, laid out in the order the backward
        # finishes them so data parallelism can reduce contiguous buckets as they complete:
        #   [W_0, b_0, ..., W_{L-2}, b_{L-2}] [W_{L-1}, b_{L-1}, head_w, head_b] [router_w, router_b]
        nl = len(self.p.layers)
        shapes = []
        for l in self.p.layers:
            shapes += [(E, l.d_out, l.d_in), (E, l.d_out)]
        shapes += [(T, self.d_out), (T,), (T * E, d), (T * E,)]
        sizes = [int(torch.Size(sh).numel()) for sh in shapes]
        self.grad_flat = z(sum(sizes))
        views, off, offs = [], 0, []
        for sh, n in zip(shapes, sizes):
            offs.append(off)
            views.append(self.grad_flat[off:off + n].view(sh))
            off += n
        self.g_layers = [(views[2 * i], views[2 * i + 1]) for i in range(nl)]
        self.g_head_w, self.g_head_b, self.g_router_w, self.g_router_b = views[2 * nl:]
        last, router = offs[2 * (nl - 1)], offs[2 * nl + 2]
        # gradient buckets (name -> slice of grad_flat), in completion order of the backward
        self.grad_buckets = {"pools_first": slice(0, last), "last_pool_heads": slice(last, router),
                             "router": slice(router, off)}
        self.on_grads = None     # optional callback(bucket name, cuda stream) once a bucket is final
        self.colsum_part = rows["colsum_part"]
        self.dh_router = z(B, d)
        self.d_hidden = z(B, d)
        self.part_dw = z(self.grid, T, self.d_out)
        self.part_db = z(self.grid, T)
        self.ldh = d + 64
        self.h_full = z(B, self.ldh, dt=bf)
        self.h_full[:, d] = 1.0
        self.h = self.h_full[:, :d]                 # strided view; kernels get ptr + ldh

    def refresh_weights(self):
        """Copy the fp32 master parameters into the bf16 / fp32 kernel operands.

        The operand buffers are allocated once and refreshed with ``copy_``: a CUDA graph captured
        from ``step``/``score`` keeps reading the same addresses, so an optimizer update followed by
        ``refresh_weights`` is seen by the next replay (no re-capture needed)."""
        self._fold_fresh = False
        p, T, E, d = self.p, self.T, self.E, self.d
        dev = self.dev
        if tuple(p.router_w.shape) != (T, E, d) or len(p.layers) != len(self.dims) - 1:
            raise ShapeError("refresh_weights: parameter shapes changed; build a new engine")
        tw = p.task_weights if p.task_weights is not None else torch.ones(T)
        lam = p.task_loss_weights if p.task_loss_weights is not None else torch.ones(T)
        src = {
            "wr_bf": (p.router_w.detach().reshape(T * E, d), torch.bfloat16),
            "br": (p.router_b.detach().reshape(T * E), torch.float32),
            "head_w": (p.head_w.detach(), torch.float32),
            "head_b": (p.head_b.detach(), torch.float32),
            "tw": (torch.as_tensor(tw).detach(), torch.float64),
            "lam": (torch.as_tensor(lam).detach(), torch.float32),
        }
        first = not hasattr(self, "wr_bf")
        for name, (t, dt) in src.items():
            if first:
                setattr(self, name, torch.empty(t.shape, dtype=dt, device=dev))
            getattr(self, name).copy_(t.to(dev))
        if first:
            self.w_bf = [torch.empty(l.weight.shape, dtype=torch.bfloat16, device=dev) for l in p.layers]
            self.b32 = [torch.empty(l.bias.shape, dtype=torch.float32, device=dev) for l in p.layers]
            self.head_w_bf = torch.empty(1, T, self.head_w.shape[1], dtype=torch.bfloat16, device=dev)
            self.head_wT_bf = torch.zeros(1, self.head_w.shape[1], _round(T, 16), dtype=torch.bfloat16, device=dev)
        for dst, l in zip(self.w_bf, p.layers):
            dst.copy_(l.weight.detach().to(dev))
        for dst, l in zip(self.b32, p.layers):
            dst.copy_(l.bias.detach().to(dev))
        self.head_w_bf[0].copy_(self.head_w)
        self.head_wT_bf[0, :, :T].copy_(self.head_w.t())
        self.beta = float(p.lb_strength)

    # ------------------------------------------------------------------ steps
    def _stream(self):
        return torch.cuda.current_stream(self.dev).cuda_stream

    def set_inputs(self, h: torch.Tensor, labels: torch.Tensor | None = None):
        """Stage the layer input (and labels) into the engine's device buffers."""
        if h.shape != (self.B, self.d):
            raise ShapeError(f"hidden has shape {tuple(h.shape)}, engine expects ({self.B}, {self.d})")
        self.h.copy_(h, non_blocking=True)
        if labels is not None:
            if labels.shape != (self.T, self.B):
                raise ShapeError(f"labels shape {tuple(labels.shape)} does not match ({self.T}, {self.B})")
            self.labels.copy_(labels, non_blocking=True)

    def forward(self, with_loss: bool = True):
        self.forward_a()
        self.forward_b(with_loss=with_loss)

    def score(self):
        """Inference scoring (BASELINE c4: fwd only, no regularizer): predictions and logits.
        With an identity last pool the heads are folded into it (P = H G_e^T + c_e), so neither the
        hidden activations, the expert outputs O nor the task reps are written; otherwise this is
        the reference-shaped forward.  G/c are folded once per ``refresh_weights``: a CUDA graph
        captured from ``score`` must be re-captured after a weight refresh."""
        if not self.can_fold:
            self.forward(with_loss=False)
            return
        s = self._stream()
        T, E, B = self.T, self.E, self.B
        # the weights do not change between scoring calls: fold the heads once per weight refresh
        self.forward_a(fold=True, store_hidden=False, refold=not self._fold_fresh)
        self._fold_fresh = True
        _tagged("combine_score", "smes_combine_fwd", T, B, E, self.K, self.d_out, self.umax, ptr(self.umask),
                ptr(self.usize), ptr(self.row_of), ptr(self.active), ptr(self.wsel), None, self.d_out,
                ptr(self.head_w), ptr(self.head_b), ptr(self.P), self.ldp, None, ptr(self.logits), ptr(self.preds),
                None, ptr(self.lam), None, self.grid, s)

    def forward_a(self, frozen: bool = False, fold: bool = False, store_hidden: bool = True, refold: bool = True,
                  finalize_stats: bool = False, heads: bool = True):
        """Router GEMM -> routing -> plan -> expert GEMMs.  Ends with the per-expert
        LoadStats sums in ``stats_raw`` (the data-parallel exchange point).
        ``fold`` (training steps only, see csrc/fold.cu): the last identity pool is folded into
        the task heads, so its output O and the task reps are not materialised."""
        s = self._stream()
        T, E, B, d = self.T, self.E, self.B, self.d
        self._fold_ev = None
        if self.use_front and not frozen:
            # router GEMM + progressive router in one kernel (routing.py:101-103 + :235-281)
            # keep_logits off (training steps): neither z nor the dense mass (read only by the dense
            # LB reading and by the API's full_probs / compute_load_stats(dense_probs=True))
            full = self.keep_logits or self.dense
            _tagged("route_front", "smes_route_front", ptr(self.h), self.ldh, ptr(self.wr_bf), ptr(self.br),
                    ptr(self.tw), T, B, E, d, self.ks, self.ka, 4 * self.rpw, ptr(self.shared), ptr(self.adaptive),
                    ptr(self.active), ptr(self.wsel), ptr(self.umask), ptr(self.usize), ptr(self.chunk_union),
                    ptr(self.chunk_active), ptr(self.chunk_mass), ptr(self.chunk_dmass) if full else None,
                    ptr(self.flag), ptr(self.z) if full else None, s)
        else:
            # router logits z = h W_r^T + b_r  (B, T*E) fp32
            _tagged("router_fwd", "smes_gemm_ragged_m", ptr(self.h), self.ldh, B, ptr(self.wr_bf), 1, T * E, d, 0,
                    ptr(self.seg_router), ptr(self.br), 0, None, None, 0, ptr(self.z), T * E, 1, B, s)
            self.route(s, frozen=frozen)
        # the head fold (G_e = head_W W_last,e, c_e) depends on the weights only: it runs on the side
        # stream next to the plan reduce (32 CTAs) and the scatter, joined before the expert kernels
        # (forked after the router: the fused front wants every SM)
        if fold and refold and self.can_fold and not self.serial and self.fold_side:
            if not hasattr(self, "_side"):
                self._side = torch.cuda.Stream(self.dev)
            fork = torch.cuda.Event()
            fork.record(torch.cuda.current_stream(self.dev))
            self._side.wait_event(fork)
            self._fold(self._side.cuda_stream)
            self._fold_ev = torch.cuda.Event()
            self._fold_ev.record(self._side)
        fold_now = bool(fold and refold and self.can_fold and self._fold_ev is None and self.fold_in_reduce)
        self._folded_in_reduce = False
        if finalize_stats and fold_now:
            # plan reduce + LoadStats finalize + the head fold in one launch (the fold's blocks run in
            # the slack of the reduce's E column scans instead of as their own kernel)
            _tagged("plan_reduce", "smes_plan_reduce_stats_fold", self.C, E, ptr(self.chunk_union),
                    ptr(self.chunk_active), ptr(self.chunk_mass), ptr(self.chunk_dmass), ptr(self.chunk_base),
                    ptr(self.loads), ptr(self.stats_raw), ptr(self.seg_pad), ptr(self.seg_log), ptr(self.totals),
                    ptr(self.ticket), ptr(self.seg_half), self.K, self.E_lb, float(B * T), int(self.dense),
                    ptr(self.stats_out), ptr(self.freq32), T, self.ldg, self.d_out, self.dims[-2], ptr(self.head_w),
                    ptr(self.w_bf[-1]), ptr(self.b32[-1]), ptr(self.G_fold), ptr(self.c_fold), s)
            self._folded_in_reduce = True
        elif finalize_stats:
            # single device: LoadStats over the local B*T, finalized by the plan reduce's last block
            _tagged("plan_reduce", "smes_plan_reduce_stats", self.C, E, ptr(self.chunk_union), ptr(self.chunk_active),
                    ptr(self.chunk_mass), ptr(self.chunk_dmass), ptr(self.chunk_base), ptr(self.loads),
                    ptr(self.stats_raw), ptr(self.seg_pad), ptr(self.seg_log), ptr(self.totals), ptr(self.ticket),
                    ptr(self.seg_half), self.K, self.E_lb, float(B * T), int(self.dense), ptr(self.stats_out),
                    ptr(self.freq32), s)
        else:
            _tagged("plan_reduce", "smes_plan_reduce", self.C, E, ptr(self.chunk_union), ptr(self.chunk_active),
                    ptr(self.chunk_mass), ptr(self.chunk_dmass), ptr(self.chunk_base), ptr(self.loads),
                    ptr(self.stats_raw), ptr(self.seg_pad), ptr(self.seg_log), ptr(self.totals), ptr(self.ticket),
                    ptr(self.seg_half), s)
        # X is gathered by its consumers in folded training steps: the scatter only places rows
        self._x_gathered = bool(fold and self.fuse_mlp_fwd and self.gather_x and not self.fuse_wgrad)
        self._x_packed_by_fwd = bool(fold and self.fuse_mlp_fwd and self.fwd_pack and not self._x_gathered)
        xg = self._x_gathered or self._x_packed_by_fwd
        _tagged("plan_scatter", "smes_plan_scatter", B, E, d, self.rpw, ptr(self.umask), ptr(self.chunk_base), ptr(self.seg_pad),
             ptr(self.loads), None if xg else ptr(self.h), self.ldh, None if xg else ptr(self.X), self.ld_in[0],
             ptr(self.row_of), self.umax,
             ptr(self.gather_inst),
             ptr(self.gather_exp), ptr(self.Cm), self.ldc, self.ldc, s)
        if fold and not self.can_fold:
            raise ConfigError("head folding needs an identity last expert pool and sparse LB statistics")
        self.experts_forward(s, fold=fold, store_hidden=store_hidden, refold=refold, heads=heads)

    def forward_b(self, with_loss: bool = True, batch_times_tasks: float | None = None, train: bool = False,
                  batch_scale: int | None = None, lb_batch: int | None = None, stats_done: bool = False,
                  defer_reduce: bool = False):
        """LoadStats finalize (global B*T under data parallelism) -> combine + heads + loss.
        ``train`` (sparse LB reading) fuses the combine backward into the same pass.
        ``stats_done``: forward_a(finalize_stats=True) already finalized the local statistics.
        ``defer_reduce`` (training steps that call backward next): the post-combine reductions
        (loss, sums of C, bias grads) are issued by backward, on its side stream."""
        s = self._stream()
        T, E, B = self.T, self.E, self.B
        if not stats_done:
            self.stats_finalize(s, batch_times_tasks)
        self._fused_bwd = bool(train and not self.dense)
        if self._fused_bwd:
            bs = B if batch_scale is None else batch_scale
            lbb = B if lb_batch is None else lb_batch
            lb_coef = self.beta * self.E_lb / (self.K * lbb * T)
            _tagged("combine_train", "smes_combine_train", T, B, E, self.K, self.umax, ptr(self.umask),
                    ptr(self.usize), ptr(self.row_of), ptr(self.active), ptr(self.wsel), ptr(self.head_b),
                    ptr(self.P), self.ldp, ptr(self.logits), ptr(self.preds), ptr(self.labels), ptr(self.lam),
                    ptr(self.loss_part), 1.0 / bs, ptr(self.Cm), self.ldc, ptr(self.dz), ptr(self.freq32), lb_coef,
                    ptr(self.part_db), ptr(self.part_csum), ptr(self.part_rb), self.grid, s)
            self._post_pending = True
            if not defer_reduce:
                self._post_combine(s)
            return
        _tagged("combine_fwd", "smes_combine_fwd", T, B, E, self.K, self.d_out, self.umax, ptr(self.umask), ptr(self.usize),
             ptr(self.row_of), ptr(self.active), ptr(self.wsel), ptr(self.outs[-1]), self.d_out, ptr(self.head_w),
             ptr(self.head_b), ptr(self.P), self.ldp, ptr(self.reps), ptr(self.logits), ptr(self.preds),
             ptr(self.labels) if with_loss else None, ptr(self.lam), ptr(self.loss_part) if with_loss else None,
             self.grid, s)
        if with_loss:
            _tagged("loss_finalize", "smes_loss_finalize", self.grid, ptr(self.loss_part), 1.0 / B, self.beta,
                 self.stats_out[3 * E:].data_ptr(), ptr(self.loss_out), s)

    def route(self, s, probs_in=None, probs_out=None, frozen=False):
        T, E, B = self.T, self.E, self.B
        _tagged("route", "smes_route_batch", ptr(self.z), E, T * E, ptr(probs_in), ptr(self.tw), T, B, E, self.ks, self.ka,
             self.rpw, ptr(self.shared), ptr(self.adaptive), ptr(self.active), ptr(self.wsel), ptr(self.umask),
             ptr(self.usize), ptr(self.chunk_union), ptr(self.chunk_active), ptr(self.chunk_mass),
             # the dense mass only for the dense LB reading and the API (full_probs / dense stats)
             ptr(self.chunk_dmass) if (self.keep_logits or self.dense or frozen) else None, ptr(probs_out),
             ptr(self.flag), int(frozen), s)

    def experts_forward(self, s, fold: bool = False, store_hidden: bool = True, refold: bool = True,
                        heads: bool = True):
        R = self.rows_cap
        inp = self.X
        L = len(self.p.layers)
        pre = [] if (fold and self.fuse_mlp_fwd) else (self.p.layers[:L - 1] if fold else self.p.layers)
        for i, l in enumerate(pre):
            _tagged(f"fc{i + 1}_fwd", "smes_gemm_ragged_m", ptr(inp), self.ld_in[i], R, ptr(self.w_bf[i]), self.E,
                    self.dims[i + 1], self.dims[i], 0, ptr(self.seg_pad), ptr(self.b32[i]), ACT[l.act],
                    ptr(self.bits[i]), None, R, ptr(self.outs[i]), self.ld_out[i], 0, R, s)
            inp = self.outs[i]
        self._folded = fold
        if fold:
            # P = H G_e^T + c_e with G_e = head_W W_last,e: the last pool and the heads in one N = T GEMM
            di = self.dims[L - 1]
            if getattr(self, "_fold_ev", None) is not None:      # folded on the side stream (forward_a)
                torch.cuda.current_stream(self.dev).wait_event(self._fold_ev)
                self._fold_ev = None
            elif getattr(self, "_folded_in_reduce", False):      # folded by the plan reduce launch
                self._folded_in_reduce = False
            elif refold:   # training steps refold every step (the weights move between steps)
                self._fold(s)
            if self.fuse_mlp_fwd and self._x_packed_by_fwd:
                # the same, X rows gathered from h by the kernel's own warp and stored packed
                _tagged("mlp_fwd", "smes_mlp_fwd_pack", ptr(self.h), self.ldh, ptr(self.gather_inst), ptr(self.X),
                        self.ld_in[0], R, ptr(self.w_bf[0]), ptr(self.b32[0]), ptr(self.G_fold), ptr(self.c_fold),
                        self.ldg, self.E, self.d, di, ptr(self.seg_pad), ptr(self.bits[0]) if store_hidden else None,
                        R, ptr(self.outs[0]) if store_hidden else None, self.ld_out[0], ptr(self.P), self.ldp, s)
                return
            if self.fuse_mlp_fwd and self._x_gathered:
                # the same, X rows gathered from h (TMA gather4)
                _tagged("mlp_fwd", "smes_mlp_fwd_gather", ptr(self.h), self.ldh, self.B, ptr(self.gather_inst), R,
                        ptr(self.w_bf[0]), ptr(self.b32[0]), ptr(self.G_fold), ptr(self.c_fold), self.ldg, self.E,
                        self.d, di, ptr(self.seg_pad), ptr(self.bits[0]) if store_hidden else None, R,
                        ptr(self.outs[0]) if store_hidden else None, self.ld_out[0], ptr(self.P), self.ldp, s)
                return
            if self.fuse_mlp_fwd:
                # fc1 (+ relu mask, H kept for the weight gradients) and P in one chained kernel
                _tagged("mlp_fwd", "smes_mlp_fwd", ptr(self.X), self.ld_in[0], R, ptr(self.w_bf[0]),
                        ptr(self.b32[0]), ptr(self.G_fold), ptr(self.c_fold), self.ldg, self.E, self.d, di,
                        ptr(self.seg_pad), ptr(self.bits[0]) if store_hidden else None, R,
                        ptr(self.outs[0]) if store_hidden else None, self.ld_out[0], ptr(self.P), self.ldp, s)
                return
            _tagged(f"fc{L}_fwd_folded", "smes_gemm_ragged_m", ptr(inp), self.ld_in[L - 1], R, ptr(self.G_fold),
                    self.E, self.ldg, di, 0, ptr(self.seg_pad), ptr(self.c_fold), 0, None, None, 0, ptr(self.P),
                    self.ldp, 1, R, s)
            return
        if not heads:                    # the layer without its heads (SMESLayer): O is the output
            return
        # head projections of every packed row: P = O head_W^T (tcgen05 GEMM, N = T)
        _tagged("head_proj", "smes_gemm_ragged_m", ptr(self.outs[-1]), self.d_out, R, ptr(self.head_w_bf), 1, self.T,
                self.d_out, 0, ptr(self.totals), None, 0, None, None, 0, ptr(self.P), self.ldp, 1, R, s)

    def _fold(self, s):
        di = self.dims[-2]
        _tagged("fold_heads", "smes_fold_heads", self.E, self.T, self.ldg, self.d_out, di,
                ptr(self.head_w), ptr(self.w_bf[-1]), ptr(self.b32[-1]), ptr(self.G_fold), ptr(self.c_fold),
                ptr(self.fold_work), s)

    def stats_finalize(self, s, batch_times_tasks: float | None = None):
        bt = float(self.B * self.T) if batch_times_tasks is None else batch_times_tasks
        _tagged("stats_finalize", "smes_stats_finalize", self.E, self.K, self.E_lb, bt, int(self.dense), ptr(self.stats_raw), ptr(self.stats_out),
             ptr(self.freq32), s)

    def backward(self, batch_scale: int | None = None, lb_batch: int | None = None):
        """Reverse pass.  ``batch_scale`` is the B of lambda/B (training.py:148);
        ``lb_batch`` the B of the LB coefficient E/(K B T) (balance.py:97)."""
        s = self._stream()
        T, E, B, d, K = self.T, self.E, self.B, self.d, self.K
        R = self.rows_cap
        bs = B if batch_scale is None else batch_scale
        lbb = B if lb_batch is None else lb_batch
        lb_coef = self.beta * self.E_lb / (K * lbb * T)
        relu_last = int(self.p.layers[-1].act == "relu")
        n_layers = len(self.p.layers)
        side_hooks = False       # the side stream announced its gradient buckets itself
        fused = getattr(self, "_fused_bwd", False)
        folded = fused and self._folded
        # The router backward needs only dz and h: it runs on a side stream next to the expert
        # backward, whose wgrad GEMMs leave SMs idle (128 tiles on 148 SMs); joins before unpermute.
        side = fused and not self.serial
        unpermute_side = False
        if side:
            main = torch.cuda.current_stream(self.dev)
            if not hasattr(self, "_side"):
                self._side = torch.cuda.Stream(self.dev)
            if not hasattr(self, "_ev_fork"):
                self._ev_fork, self._ev_join = torch.cuda.Event(), torch.cuda.Event()
                self._ev_dx = torch.cuda.Event()
            self._ev_fork.record(main)
            self._side.wait_event(self._ev_fork)
            if getattr(self, "_post_pending", False):
                self._post_combine(self._side.cuda_stream)
            if not folded:
                self._router_backward(self._side.cuda_stream)
        elif getattr(self, "_post_pending", False):
            self._post_combine(s)
        top = n_layers - 1             # first pool handled by the generic dgrad/wgrad loop
        if folded:
            # the last (identity) pool through the folded heads (csrc/fold.cu):
            #   d_in_last = (C G_e) * relu-mask,  Qt_e = H_e^T C,  dW/db/dW_head from Qt and csum
            L = n_layers
            di = self.dims[L - 1]
            inp = self.X if L == 1 else self.outs[L - 2]
            dst = self.dX if L == 1 else self.d_outs[L - 2]
            mask = self.bits[L - 2] if L >= 2 else None
            if self.fuse_mlp:
                # dH = (C G_e) * mask and dX = dH W1 in one chained kernel; the fc1 weight gradient
                # recomputes dH per row block (mlp_wgrad), so dH never goes to HBM
                _tagged("mlp_dgrad", "smes_mlp_dgrad", ptr(self.Cm), self.ldc, R, ptr(self.G_fold), self.ldg,
                        ptr(self.w_bf[0]), E, d, di, ptr(self.seg_pad), ptr(mask), R, ptr(self.dX), d,
                        None if self.fuse_wgrad else ptr(dst), di, s)
                if side:      # dX is final here: the un-permute can run on the side stream
                    self._ev_dx.record(main)
                    unpermute_side = True
                if self.fuse_wgrad:
                    gw0, gb0 = self.g_layers[0]
                    _tagged("mlp_wgrad", "smes_mlp_wgrad", ptr(self.Cm), self.ldc, R, ptr(self.G_fold), self.ldg,
                            ptr(self.X), self.ld_in[0], E, d, di, ptr(self.seg_pad), ptr(mask), R, ptr(gw0),
                            ptr(gb0), s)
            else:
                _tagged(f"fc{L}_dgrad_folded", "smes_gemm_ragged_m", ptr(self.Cm), self.ldc, R, ptr(self.G_fold),
                        E, di, self.ldg, 1, ptr(self.seg_pad), None, 0, None, ptr(mask), R, ptr(dst), di, 0, R, s)
            if side:      # Q = C^T H and the unfold need only C and H: next to the dgrad chain
                self._last_pool_wgrad(self._side.cuda_stream, inp, di)
                if self.on_grads is not None:
                    self.on_grads("last_pool_heads", self._side)
                self._router_backward(self._side.cuda_stream, self._ev_dx if unpermute_side else None)
                if self.on_grads is not None:
                    self.on_grads("router", self._side)
                side_hooks = self.on_grads is not None
            else:
                self._last_pool_wgrad(s, inp, di)
            top = n_layers - 2
        elif fused:
            # d_packed = C head_W (K = T padded to 16), relu mask of O if the last pool is relu
            last = len(self.p.layers) - 1
            _tagged("dpacked_gemm", "smes_gemm_ragged_m", ptr(self.Cm), self.ldc, R, ptr(self.head_wT_bf), 1,
                    self.d_out, self.ldc, 0, ptr(self.totals), None, 0, None, ptr(self.bits[last]), R,
                    ptr(self.d_outs[-1]), self.d_out, 0, R, s)
            # dW_head = C^T O, split-K over expert halves, fixed-order reduce
            _tagged("head_wgrad", "smes_gemm_ragged_k", ptr(self.Cm), self.ldc, ptr(self.outs[-1]), self.d_out, R,
                    2 * E, T, self.d_out, ptr(self.seg_half), ptr(self.hw_part), None, s)
            _tagged("head_wgrad", "smes_part_reduce", ptr(self.hw_part), 2 * E, T * self.d_out, ptr(self.g_head_w), s)
        else:
            self.d_outs[-1].zero_()      # dense-reading path (API only): pad rows must be zero
            _tagged("combine_bwd", "smes_combine_bwd", T, B, E, K, self.d_out, self.umax, ptr(self.umask),
                    ptr(self.usize), ptr(self.row_of), ptr(self.active), ptr(self.wsel), ptr(self.outs[-1]),
                    self.d_out, ptr(self.head_w), ptr(self.P), self.ldp, ptr(self.reps), ptr(self.preds),
                    ptr(self.labels), ptr(self.lam), 1.0 / bs, relu_last, ptr(self.d_outs[-1]), ptr(self.dz),
                    ptr(self.freq32), lb_coef, int(self.dense), ptr(self.z), ptr(self.part_dw), ptr(self.part_db),
                    self.grid, s)
        if folded and self.fuse_wgrad:
            top = -1                   # fc1's dgrad and wgrad ran in the fused kernels
        for i in range(top, -1, -1):
            dout = self.d_outs[i]
            inp = self.X if i == 0 else self.outs[i - 1]
            gw, gb = self.g_layers[i]
            di, do = self.dims[i], self.dims[i + 1]
            if i > 0:   # dgrad into the previous layer's output, masked by its relu
                _tagged(f"fc{i + 1}_dgrad", "smes_gemm_ragged_m", ptr(dout), do, R, ptr(self.w_bf[i]), E, di, do, 1, ptr(self.seg_pad),
                     None, 0, None, ptr(self.bits[i - 1]), R, ptr(self.d_outs[i - 1]), di, 0, R, s)
            fused_last = i == n_layers - 1 and self.fuse_b_last and fused
            if fused_last:
                # db = (per-expert sums of C, reduced by post_combine) head_W: no bias tiles needed
                _tagged(f"fc{i + 1}_wgrad", "smes_gemm_ragged_k", ptr(dout), do, ptr(inp), self.ld_in[i], R, E, do,
                        di, ptr(self.seg_pad), ptr(gw), None, s)
                _tagged(f"fc{i + 1}_bias", "smes_bias_from_csum", E, T, do, ptr(self.csum), ptr(self.head_w), ptr(gb),
                        s)
            elif i == 0 and self._x_gathered:
                # wgrad + bias grad, the layer input rows gathered from h (TMA gather4)
                _tagged("fc1_wgrad", "smes_gemm_ragged_k_gather", ptr(dout), do, ptr(self.h), self.ldh, B,
                        ptr(self.gather_inst), R, E, do, di, ptr(self.seg_pad), ptr(gw), ptr(gb), s)
            else:
                # wgrad + bias grad in one launch (ones column of the layer input, see _alloc)
                _tagged(f"fc{i + 1}_wgrad", "smes_gemm_ragged_k", ptr(dout), do, ptr(inp), self.ld_in[i], R, E, do,
                        di, ptr(self.seg_pad), ptr(gw), ptr(gb), s)
        # dX = d_out0 W_0
        if not (folded and (n_layers == 1 or self.fuse_mlp)):
            _tagged("fc1_dgrad", "smes_gemm_ragged_m", ptr(self.d_outs[0]), self.dims[1], R, ptr(self.w_bf[0]), E, d, self.dims[1], 1,
                    ptr(self.seg_pad), None, 0, None, None, R, ptr(self.dX), d, 0, R, s)
        if side_hooks:
            self.on_grads("pools_first", main)    # every pool but the last: final on the main stream
        if side:
            self._ev_join.record(self._side)       # after every side-stream launch of this pass
            main.wait_event(self._ev_join)
        else:
            self._router_backward(s)
        if not unpermute_side:
            self._unpermute(s)
        if not getattr(self, "_fused_bwd", False):
            _tagged("head_reduce", "smes_part_reduce", ptr(self.part_dw), self.grid, T * self.d_out,
                    ptr(self.g_head_w), s)
        if not getattr(self, "_fused_bwd", False):
            _tagged("head_reduce", "smes_part_reduce", ptr(self.part_db), self.grid, T, ptr(self.g_head_b), s)
        if self.on_grads is not None and not side_hooks:
            cur = torch.cuda.current_stream(self.dev)
            for name in self.grad_buckets:
                self.on_grads(name, cur)

    def _post_combine(self, s):
        """Loss, per-(expert, task) sums of C, router / head bias grads: one reduction launch."""
        T, E, B = self.T, self.E, self.B
        _tagged("post_combine", "smes_post_combine", self.grid, ptr(self.part_csum), E * T, ptr(self.csum),
                ptr(self.part_rb), T * E, ptr(self.g_router_b), ptr(self.part_db), T, ptr(self.g_head_b),
                ptr(self.loss_part), 1.0 / B, self.beta, self.stats_out[3 * E:].data_ptr(), ptr(self.loss_out), s)
        self._post_pending = False

    def _last_pool_wgrad(self, s, inp, di):
        """Folded last pool's weight gradients: Q_e = H_e^T C_e (ragged-K), then dW / db / dW_head
        from Q and the per-(expert, task) sums of C (csrc/fold.cu)."""
        T, E, R, L = self.T, self.E, self.rows_cap, len(self.p.layers)
        if self.q_swapped:
            # Q_e = C_e^T H_e and csum_e = colsum(C_e) in one ragged-K GEMM (csum via the ones tile)
            _tagged(f"fc{L}_wgrad_folded", "smes_gemm_ragged_k", ptr(self.Cm), self.ldc, ptr(inp),
                    self.ld_in[L - 1], R, E, self.ldg, di, ptr(self.seg_pad), ptr(self.Qe), ptr(self.csum_q), s)
            cs, cs_es = self.csum_q, self.ldg
        else:
            if self.q_splits > 1:
                # few long groups (E x 4 tiles < the SMs): the K range split so every SM streams H
                _tagged(f"fc{L}_wgrad_folded", "smes_gemm_ragged_k_split", ptr(inp), self.ld_in[L - 1],
                        ptr(self.Cm), self.ldc, R, E, self.q_rows, self.ldg, ptr(self.seg_pad), ptr(self.Qe), None,
                        self.q_splits, ptr(self.q_work), s)
            else:
                _tagged(f"fc{L}_wgrad_folded", "smes_gemm_ragged_k", ptr(inp), self.ld_in[L - 1], ptr(self.Cm),
                        self.ldc, R, E, self.q_rows, self.ldg, ptr(self.seg_pad), ptr(self.Qe), None, s)
            if self.fuse_b_last:
                cs, cs_es = self.csum, T          # reduced by post_combine
            else:
                cs, cs_es = self.Qe[:, di, :], self.q_rows * self.ldg
        gw, gb = self.g_layers[L - 1]
        qes, qts, qks = self.q_strides
        _tagged("unfold", "smes_unfold_grads", E, T, self.ldg, self.d_out, di, ptr(self.Qe), qes, qts, qks,
                ptr(cs), cs_es, ptr(self.head_w), ptr(self.w_bf[-1]), ptr(self.b32[-1]), ptr(gw),
                ptr(gb), ptr(self.fold_work), ptr(self.g_head_w), s)

    def _unpermute(self, s):
        """d_hidden[b] = dh_router[b] + sum of the instance's packed dX rows (training.py:192, 209-212)."""
        _tagged("unpermute", "smes_unpermute", self.B, self.d, ptr(self.usize), ptr(self.row_of), self.umax,
                ptr(self.dX), self.d, ptr(self.dh_router), ptr(self.d_hidden), s)

    def _router_backward(self, s, dx_ready=None):
        """dh_r = dz W_r ; dW_r = dz^T h (split-K + fixed-order reduce) ; db_r = colsum(dz).
        ``dx_ready``: an event after which dX is final -- the un-permute then runs here, between
        the router dgrad and wgrad (side-stream schedule of backward)."""
        T, E, B, d = self.T, self.E, self.B, self.d
        _tagged("router_dgrad", "smes_gemm_ragged_m", ptr(self.dz), T * E, self.B_pad, ptr(self.wr_bf), 1, d, T * E, 1,
                ptr(self.seg_router), None, 0, None, None, 0, ptr(self.dh_router), d, 1, B, s)
        if dx_ready is not None:
            self._side.wait_event(dx_ready)
            self._unpermute(s)
        rb_fused = self.fuse_rb and getattr(self, "_fused_bwd", False)
        _tagged("router_wgrad", "smes_gemm_ragged_k", ptr(self.dz), T * E, ptr(self.h), self.ldh, B, self.rw_splits,
                T * E, d, ptr(self.seg_router_split), ptr(self.rw_part), None if rb_fused else ptr(self.rb_part), s)
        _tagged("router_wgrad", "smes_part_reduce", ptr(self.rw_part), self.rw_splits, T * E * d,
                ptr(self.g_router_w), s)
        if not rb_fused:                  # else reduced by post_combine
            _tagged("router_bias", "smes_part_reduce", ptr(self.rb_part), self.rw_splits, T * E,
                    ptr(self.g_router_b), s)

    # ------------------------------------------------------------------ layer form (no heads)
    def forward_layer(self):
        """Forward of the layer without its heads and loss (SMESLayer): routing, plan, every expert
        pool with O kept, LoadStats and the task reps (execution.py:161-191)."""
        s = self._stream()
        T, E, B = self.T, self.E, self.B
        self.forward_a(fold=False, heads=False)
        self.stats_finalize(s)
        _tagged("combine_fwd", "smes_combine_fwd", T, B, E, self.K, self.d_out, self.umax, ptr(self.umask),
                ptr(self.usize), ptr(self.row_of), ptr(self.active), ptr(self.wsel), ptr(self.outs[-1]), self.d_out,
                ptr(self.head_w), ptr(self.head_b), None, self.ldp, ptr(self.reps), ptr(self.logits),
                ptr(self.preds), None, ptr(self.lam), None, self.grid, s)

    def backward_reps(self, d_reps: torch.Tensor, d_lb: float):
        """Reverse of ``forward_layer`` for an upstream gradient d_reps (T, B, d_out) fp32 and the
        gradient d_lb of the returned L_lb: combine backward + LB term (csrc/layer.cu), then every
        pool's dgrad / wgrad, the router backward and the un-permute (training.py:160-212)."""
        s = self._stream()
        T, E, B, K = self.T, self.E, self.B, self.K
        R = self.rows_cap
        if d_reps.shape != (T, B, self.d_out) or d_reps.dtype != torch.float32 or not d_reps.is_contiguous():
            raise ShapeError(f"d_reps must be a contiguous fp32 ({T}, {B}, {self.d_out}) tensor")
        self._fused_bwd = False
        lb_coef = float(d_lb) * self.E_lb / (K * B * T)
        self.d_outs[-1].zero_()
        n_layers = len(self.p.layers)
        _tagged("combine_bwd", "smes_combine_bwd_reps", T, B, E, K, self.d_out, self.umax, ptr(self.umask),
                ptr(self.usize), ptr(self.row_of), ptr(self.active), ptr(self.wsel), ptr(self.outs[-1]),
                self.d_out, int(self.p.layers[-1].act == "relu"), ptr(d_reps), ptr(self.freq32), lb_coef,
                ptr(self.d_outs[-1]), ptr(self.dz), T * E, s)
        for i in range(n_layers - 1, -1, -1):
            dout = self.d_outs[i]
            inp = self.X if i == 0 else self.outs[i - 1]
            gw, gb = self.g_layers[i]
            di, do = self.dims[i], self.dims[i + 1]
            if i > 0:
                _tagged(f"fc{i + 1}_dgrad", "smes_gemm_ragged_m", ptr(dout), do, R, ptr(self.w_bf[i]), E, di, do, 1,
                        ptr(self.seg_pad), None, 0, None, ptr(self.bits[i - 1]), R, ptr(self.d_outs[i - 1]), di, 0,
                        R, s)
            _tagged(f"fc{i + 1}_wgrad", "smes_gemm_ragged_k", ptr(dout), do, ptr(inp), self.ld_in[i], R, E, do, di,
                    ptr(self.seg_pad), ptr(gw), ptr(gb), s)
        _tagged("fc1_dgrad", "smes_gemm_ragged_m", ptr(self.d_outs[0]), self.dims[1], R, ptr(self.w_bf[0]), E,
                self.d, self.dims[1], 1, ptr(self.seg_pad), None, 0, None, None, R, ptr(self.dX), self.d, 0, R, s)
        self._router_backward(s)
        self._unpermute(s)

    def step(self):
        self.forward_a(fold=self.can_fold, finalize_stats=True)
        self.forward_b(with_loss=True, train=True, stats_done=True, defer_reduce=True)
        self.backward()

    # ------------------------------------------------------------------ accounting
    def work_model(self, n_act: int, balance: float = 260.0) -> dict:
        """Algorithmic work per launch tag: (flops, bytes, bound).  SURVEY 8(d).
        ``bound`` is "tensor" when the kernel's arithmetic intensity exceeds the machine balance
        (FLOP/byte of the measured peaks), else "hbm"."""
        T, E, B, K, d, do = self.T, self.E, self.B, self.K, self.d, self.d_out
        U = n_act / B
        w = {"router_fwd": (2.0 * B * d * T * E, B * (d * 2 + T * E * 4)),
             "router_dgrad": (2.0 * B * d * T * E, B * (T * E * 2 + d * 4)),
             "router_wgrad": (2.0 * B * d * T * E, B * (T * E * 2 + d * 2)),
             "head_proj": (2.0 * n_act * do * T, n_act * (do * 2 + T * 4)),
             "combine_train": (0.0, B * (U * T * 4 + T * K * 8 + T * 16 + T * E * 2) + n_act * self.ldc * 2),
             "dpacked_gemm": (2.0 * n_act * do * T, n_act * (self.ldc * 2 + do * 2)),
             "head_wgrad": (2.0 * n_act * do * T, n_act * (self.ldc * 2 + do * 2)),
             "route": (0.0, B * (T * E * 4 + T * K * 8 + self.ks * 4 + (E + 31) // 32 * 4 + 4)),
             # fused front: h read once, selections/weights/union written; z only with keep_logits
             "route_front": (2.0 * B * d * T * E, B * (d * 2 + T * K * 8 + T * self.ka * 4 + self.ks * 4
                                                       + (E + 31) // 32 * 4 + 4
                                                       + (T * E * 4 if (self.keep_logits or self.dense) else 0))
                             + self.C * E * 24),
             "plan_scatter": (0.0, B * (d * 2 + U * d * 2 + U * 4) + n_act * 8),
             "combine_fwd": (0.0, B * (U * do * 2 + T * K * 8 + T * do * 2 * (self.reps is not None) + T * 12)),
             "combine_score": (0.0, B * (U * self.ldp * 4 + U * 4 + T * K * 8 + T * 8)),
             "plan_reduce": (0.0, self.C * E * 24 + E * 40),
             "combine_bwd": (0.0, B * (U * do * 2 * 2 + T * K * 8 + T * 8 + T * E * 2)),
             "unpermute": (0.0, B * (U * d * 2 + d * 8))}
        for i in range(len(self.dims) - 1):
            di, dn = self.dims[i], self.dims[i + 1]
            f = 2.0 * n_act * di * dn
            w[f"fc{i + 1}_fwd"] = (f, n_act * (di + dn) * 2)
            w[f"fc{i + 1}_wgrad"] = (f, n_act * (di + dn) * 2)
            w[f"fc{i + 1}_dgrad"] = (f, n_act * (di + dn) * 2)
            w[f"fc{i + 1}_bias"] = (0.0, n_act * dn * 2)
        if self.can_fold:
            L = len(self.dims) - 1
            di = self.dims[-2]
            lg = self.ldg
            # folded last pool: P = H G^T (N = T), dH = C G (K = T), Qt = H^T C
            w[f"fc{L}_fwd_folded"] = (2.0 * n_act * di * T, n_act * (di * 2 + self.ldp * 4))
            w[f"fc{L}_dgrad_folded"] = (2.0 * n_act * di * T, n_act * (self.ldc * 2 + di * 2 + di / 8))
            w[f"fc{L}_wgrad_folded"] = (2.0 * n_act * di * T, n_act * (di * 2 + self.ldc * 2))
            w["fold_heads"] = (2.0 * E * T * do * di, E * do * di * 2 + E * lg * di * 2)
            if self.fold_in_reduce:     # the training step folds inside the plan-reduce launch
                fl, by = w["fold_heads"]
                w["plan_reduce"] = (fl, w["plan_reduce"][1] + by)
            w["unfold"] = (4.0 * E * T * do * di, E * di * lg * 4 + E * do * di * (4 + 2))
            if self.fuse_mlp:
                dff = self.dims[1]
                # fused MLP: fc1 (+ relu mask, H kept) and P in one pass; dgrad dH (kept) + dX in one pass
                w["mlp_fwd"] = (2.0 * n_act * (d * dff + dff * T),
                                n_act * (d * 2 + dff * 2 + dff / 8 + self.ldp * 4))
                w["mlp_dgrad"] = (2.0 * n_act * (T * dff + dff * d),
                                  n_act * (self.ldc * 2 + dff / 8 + d * 2 + (0 if self.fuse_wgrad else dff * 2)))
                w["mlp_wgrad"] = (2.0 * n_act * (T * dff + dff * d), n_act * (self.ldc * 2 + dff / 8 + d * 2))
            if self._x_gathered:
                # X never written: the scatter places rows only; its consumers read h's B rows once
                # from HBM (the U-fold re-reads hit L2)
                dff = self.dims[1]
                w["plan_scatter"] = (0.0, B * U * 4 + n_act * 8)
                w["mlp_fwd"] = (w["mlp_fwd"][0], B * d * 2 + n_act * (dff * 2 + dff / 8 + self.ldp * 4))
                w["fc1_wgrad"] = (w["fc1_wgrad"][0], B * d * 2 + n_act * dff * 2)
        return {k: (f, b, "tensor" if b > 0 and f / b > balance else ("tensor" if b == 0 else "hbm"))
                for k, (f, b) in w.items()}

    # ------------------------------------------------------------------ graphs
    def capture_step(self, warmup: int = 1) -> torch.cuda.CUDAGraph:
        """Capture one fwd+bwd step (inputs read from ``self.h`` / ``self.labels``)."""
        st = torch.cuda.Stream(self.dev)
        st.wait_stream(torch.cuda.current_stream(self.dev))
        with torch.cuda.stream(st):
            for _ in range(warmup):
                self.step()
        torch.cuda.current_stream(self.dev).wait_stream(st)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.step()
        return g

    # ------------------------------------------------------------------ views
    def n_act(self) -> int:
        """Logical packed rows (reads the device counter: a host sync)."""
        return int(self.totals[2].item())

    def gradients(self) -> dict:
        """Gradient blocks with the reference's names (model.py:94-111), single-pool
        stacks use ``expert_{e}``; deeper stacks ``expert{l}_{e}``."""
        T, E = self.T, self.E
        g = {}
        single = len(self.p.layers) == 1
        for li, (gw, gb) in enumerate(self.g_layers):
            for e in range(E):
                pre = f"expert_{e}" if single else f"expert{li}_{e}"
                g[pre + ".weight"] = gw[e]
                g[pre + ".bias"] = gb[e]
        rw = self.g_router_w.view(T, E, self.d)
        rb = self.g_router_b.view(T, E)
        for t in range(T):
            g[f"router_{t}.weight"] = rw[t]
            g[f"router_{t}.bias"] = rb[t]
            g[f"head_{t}.weight"] = self.g_head_w[t:t + 1]
            g[f"head_{t}.bias"] = self.g_head_b[t:t + 1]
        return g
