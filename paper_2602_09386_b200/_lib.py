"""ctypes binding of the in-tree C-ABI library ``_smes.so`` (include/smes.h).

There is no fallback: if the library or a CUDA device is missing, the product
path raises.  Status codes map to the reference's exception classes
(taskmoe/errors.py:4-49).
"""
from __future__ import annotations

import ctypes as C
import os

from . import errors

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_smes.so")

P = C.c_void_p
I = C.c_int
L = C.c_long
F = C.c_float
D = C.c_double

# name -> argtypes (restype is int status unless listed in _RESTYPE)
SIGNATURES = {
    "smes_last_error": [],
    "smes_abi_version": [],
    "smes_route_rows_per_warp": [I],
    "smes_route_num_chunks": [I, I],
    "smes_route_batch": [P, L, L, P, P, I, I, I, I, I, I, P, P, P, P, P, P, P, P, P, P, P, P, I, P],
    "smes_route_front_supported": [I, I, I, I, I],
    "smes_route_front_count_exact": [P],
    "smes_route_count_exact": [P],
    "smes_plan_reduce_work_ints": [I, I],
    "smes_fold_full_supported": [I, I, I, I, I],
    "smes_gemm_ragged_k_split_work": [I, I, I, I, I],
    "smes_gemm_ragged_k_split": [P, L, P, L, L, I, I, I, P, P, P, I, P, P],
    "smes_plan_reduce_stats_fold": [I, I, P, P, P, P, P, P, P, P, P, P, P, P, I, I, D, I, P, P, I, I, I, I, P, P, P, P, P,
                                    P],
    "smes_route_rt_supported": [I, I, I, I],
    "smes_route_rt": [P, L, L, P, I, I, I, I, I, I, P, P, P, P, P, P, P, P, P, P, P, P],
    "smes_peer_allreduce_f64": [I, I, I, P, P, P, P, P, P, P, P],
    "smes_combine_bwd_reps": [I, I, I, I, I, I, P, P, P, P, P, P, L, I, P, P, F, P, P, L, P],
    "smes_route_front": [P, L, P, P, P, I, I, I, I, I, I, I, P, P, P, P, P, P, P, P, P, P, P, P, P],
    "smes_plan_reduce": [I, I, P, P, P, P, P, P, P, P, P, P, P, P, P],
    "smes_plan_reduce_stats": [I, I, P, P, P, P, P, P, P, P, P, P, P, P, I, I, D, I, P, P, P],
    "smes_plan_counts": [I, I, I, P, P, P, P],
    "smes_plan_scatter": [I, I, I, I, P, P, P, P, P, L, P, L, P, I, P, P, P, L, I, P],
    "smes_gemm_ragged_m": [P, L, L, P, I, I, I, I, P, P, I, P, P, L, P, L, I, L, P],
    "smes_gemm_ragged_k": [P, L, P, L, L, I, I, I, P, P, P, P],
    "smes_gemm_ragged_k_periodic": [P, L, L, P, L, L, I, I, I, P, P, P, I, P],
    "smes_gemm_ragged_k_gather": [P, L, P, L, L, P, L, I, I, I, P, P, P, P],
    "smes_combine_grid": [I, I, I],
    "smes_combine_fwd": [I, I, I, I, I, I, P, P, P, P, P, P, L, P, P, P, L, P, P, P, P, P, P, I, P],
    "smes_combine_bwd": [I, I, I, I, I, I, P, P, P, P, P, P, L, P, P, L, P, P, P, P, F, I, P, P, P, F, I, P, P, P, I, P],
    "smes_combine_train": [I, I, I, I, I, P, P, P, P, P, P, P, L, P, P, P, P, P, F, P, L, P, P, F, P, P, P, I, P],
    "smes_bias_from_csum": [I, I, I, P, P, P, P],
    "smes_fold_work_floats": [I, I, I, I],
    "smes_ep_pack": [I, I, P, I, I, P, L, I, P, P, P, P, P, P],
    "smes_ep_segments": [I, I, I, P, P, L, P, P],
    "smes_ep_copy_rows": [I, P, I, P, L, P, L, I, P],
    "smes_ep_combine_dh": [I, I, I, L, P, P, P, P, P],
    "smes_ep_capacity_guard": [I, L, P, P, P, P, L, P, L, P, P],
    "smes_ep_put_slots": [I, I, P, L, L, P, P, P],
    "smes_ep_pack_put": [I, I, P, I, I, P, L, I, I, P, P, P, P, P, P],
    "smes_ep_copy_rows_put": [I, P, I, L, I, P, L, P, L, I, P],
    "smes_ep_signal_wait": [I, I, P, P, I, P],
    "smes_ipc_handle": [P, P, P],
    "smes_ipc_open": [P, P],
    "smes_ipc_close": [P],
    "smes_mlp_fwd": [P, L, L, P, P, P, P, I, I, I, I, P, P, L, P, L, P, L, P],
    "smes_mlp_fwd_gather": [P, L, L, P, L, P, P, P, P, I, I, I, I, P, P, L, P, L, P, L, P],
    "smes_mlp_fwd_pack": [P, L, P, P, L, L, P, P, P, P, I, I, I, I, P, P, L, P, L, P, L, P],
    "smes_mlp_fwd2": [P, L, L, P, P, P, P, I, I, I, I, P, P, L, P, L, P, L, P],
    "smes_mlp_dgrad": [P, L, L, P, I, P, I, I, I, P, P, L, P, L, P, L, P],
    "smes_mlp_dgrad2": [P, L, L, P, I, P, I, I, I, P, P, L, P, L, P, L, P],
    "smes_mlp_wgrad": [P, L, L, P, I, P, L, I, I, I, P, P, L, P, P, P],
    "smes_fold_heads": [I, I, I, I, I, P, P, P, P, P, P, P],
    "smes_unfold_grads": [I, I, I, I, I, P, L, L, L, P, L, P, P, P, P, P, P, P, P],
    "smes_fold_gemm_path": [I, I, I, I],
    "smes_stats_finalize": [I, I, I, D, I, P, P, P, P],
    "smes_loss_finalize": [I, P, D, D, P, P, P],
    "smes_seg_colsum": [P, L, L, I, P, I, P, P, P],
    "smes_unpermute": [I, I, P, P, I, P, L, P, P, P],
    "smes_part_reduce": [P, I, I, P, P],
    "smes_post_combine": [I, P, I, P, P, I, P, P, I, P, P, D, D, P, P, P],
    "smes_lb_grad": [I, I, I, I, P, P, P, L, L, P, F, I, P, P],
    "smes_bce_loss": [I, I, P, P, P, P, I, P, P],
    "smes_gemm_ragged_m_x3": [P, L, L, P, I, I, I, P, P, I, P, L, L, P],
    "smes_split_bf16x3": [L, I, P, L, P, L, P, P],
    "smes_combine_fwd_f32_grid": [I],
    "smes_combine_fwd_f32": [I, I, I, I, I, I, P, P, P, P, P, P, L, P, P, P, P, P, P, P, P, I, P],
    "smes_combine_fwd_f32_loss": [I, I, I, I, I, I, P, P, P, P, P, P, L, P, P, P, P, P, P, P, P, I, P, D, D, P, P, P],
}
_RESTYPE = {"smes_last_error": C.c_char_p, "smes_gemm_ragged_k_split_work": C.c_long}
# entry points that return a value rather than a status
_VALUE_FNS = {"smes_abi_version", "smes_route_front_supported", "smes_fold_work_floats", "smes_fold_gemm_path", "smes_route_rows_per_warp", "smes_route_num_chunks", "smes_combine_grid",
              "smes_combine_fwd_f32_grid", "smes_last_error",
              "smes_route_front_count_exact", "smes_route_count_exact", "smes_route_rt_supported",
              "smes_plan_reduce_work_ints", "smes_fold_full_supported", "smes_gemm_ragged_k_split_work"}

# kernels launched per successful call (for the bench's gpu_launches count)
def _fold_gemm_path(E, T, d_out, d_in):      # csrc/fold.cu gemm_path()
    return E * d_out * d_in >= (1 << 24) and d_out % 64 == 0 and d_in % 64 == 0 and T <= 32


def _fold_launches(E, T, ldg, d_out, d_in, *_):
    if _fold_gemm_path(E, T, d_out, d_in) and ldg == (T + 7) // 8 * 8:
        return 4                              # prep, segments, ragged-K GEMM, convert
    tm = 8 if T <= 8 else 16 if T <= 16 else 32
    return 1 if d_out <= 256 and T <= 8 and ldg <= 8 else 2


def _unfold_launches(E, T, ldg, d_out, d_in, *_):
    return 7 if _fold_gemm_path(E, T, d_out, d_in) else 2


KERNELS_PER_CALL = {"smes_route_batch": 1, "smes_route_front": 1, "smes_peer_allreduce_f64": 1, "smes_combine_bwd_reps": 1, "smes_plan_reduce": 1, "smes_plan_reduce_stats": 1, "smes_plan_scatter": 1, "smes_gemm_ragged_m": 1,
                    "smes_gemm_ragged_k": 1, "smes_combine_fwd": 1, "smes_combine_bwd": 1, "smes_stats_finalize": 1,
                    "smes_loss_finalize": 1, "smes_seg_colsum": 2, "smes_unpermute": 1, "smes_part_reduce": 1,
                    "smes_plan_counts": 1, "smes_combine_train": 1, "smes_bias_from_csum": 1, "smes_lb_grad": 1, "smes_bce_loss": 1,
                    "smes_post_combine": 1, "smes_fold_heads": _fold_launches, "smes_unfold_grads": _unfold_launches, "smes_gemm_ragged_k_periodic": 1, "smes_gemm_ragged_k_gather": 1, "smes_mlp_fwd_gather": 1, "smes_mlp_fwd_pack": 1,
                    "smes_mlp_fwd": 1, "smes_mlp_fwd2": 1, "smes_mlp_dgrad": 1, "smes_mlp_dgrad2": 1, "smes_mlp_wgrad": 1, "smes_ep_pack": 2, "smes_ep_segments": 1,
                    "smes_ep_copy_rows": 1, "smes_ep_combine_dh": 1, "smes_ep_capacity_guard": 1,
                    "smes_ep_put_slots": 1, "smes_ep_signal_wait": 2, "smes_ep_pack_put": 2,
                    "smes_ep_copy_rows_put": 1, "smes_gemm_ragged_m_x3": 1, "smes_split_bf16x3": 1,
                    "smes_combine_fwd_f32": 1, "smes_combine_fwd_f32_loss": 1, "smes_route_rt": 1,
                    "smes_plan_reduce_stats_fold": 1,
                    "smes_gemm_ragged_k_split": lambda *a: 1 if a[11] <= 1 else 2}
launch_count = 0
_timer = None   # optional callable(name) -> context manager, used by the bench's per-kernel timing
trace = None    # optional list: every successful call appends (tag, kernels launched) -- ncu launch tags

_lib = None


def load(path: str = LIB_PATH) -> C.CDLL:
    """Load (once) and type the library; raises ImportError if it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(path):
            raise ImportError(f"SMES CUDA library not built: {path} (run paper_2602_09386_b200/build.py)")
        lib = C.CDLL(path)
        for name, argt in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = argt
            fn.restype = _RESTYPE.get(name, C.c_int)
        _lib = lib
    return _lib


_CODE_TO_EXC = {
    1: errors.ShapeError,
    2: errors.ConfigError,
    3: errors.NumericsError,
    4: errors.StateError,
    5: errors.CudaError,
}


tag = None   # label of the current launch site (set by the engine for per-kernel timing)


def call(name: str, *args):
    """Invoke an entry point; raise the mapped exception on a non-zero status."""
    global launch_count
    lib = load()
    if name in _VALUE_FNS:
        return getattr(lib, name)(*args)
    if _timer is not None:
        with _timer(tag or name):
            rc = getattr(lib, name)(*args)
    else:
        rc = getattr(lib, name)(*args)
    if rc != 0:
        msg = lib.smes_last_error().decode(errors="replace")
        raise _CODE_TO_EXC.get(rc, errors.TaskMoeError)(msg)
    k = KERNELS_PER_CALL.get(name, 0)
    k = k(*args) if callable(k) else k
    launch_count += k
    if trace is not None and k:
        trace.append((tag or name, k))
    return rc


def tcall(tag_: str, name: str, *args):
    """``call`` with a launch-site label (per-kernel timing in the bench)."""
    global tag
    tag = tag_
    try:
        return call(name, *args)
    finally:
        tag = None


def ptr(t) -> int | None:
    """Device pointer of a tensor (None -> NULL)."""
    return None if t is None else t.data_ptr()
