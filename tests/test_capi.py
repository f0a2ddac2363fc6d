"""CPU-side checks of the C ABI boundary: the in-tree library loads without a GPU,
exports every symbol include/smes.h declares, the ctypes signatures cover them, and
the product API fails loudly (no CPU fallback) when no CUDA device is present."""
import ctypes
import os
import re

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "smes.h")).read()
    return sorted(set(re.findall(r"\b(smes_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2602_09386_b200 import _lib
    lib = _lib.load()
    names = declared_symbols()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n
        assert n in _lib.SIGNATURES, f"{n} has no ctypes signature"
    assert lib.smes_abi_version() == 1


def test_error_codes_map_to_reference_exceptions():
    from paper_2602_09386_b200 import _lib, errors
    assert _lib._CODE_TO_EXC[1] is errors.ShapeError
    assert _lib._CODE_TO_EXC[2] is errors.ConfigError
    assert _lib._CODE_TO_EXC[3] is errors.NumericsError
    assert _lib._CODE_TO_EXC[4] is errors.StateError


def test_host_validation_without_gpu():
    """Shape/config validation happens host-side before any launch (same messages as
    the reference, routing.py:47-61)."""
    from paper_2602_09386_b200 import _lib, errors
    with pytest.raises(errors.ConfigError, match="candidates"):
        _lib.call("smes_route_batch", None, 0, 0, None, None, 2, 4, 4, 3, 2, 1, *([None] * 12), 0, None)
    with pytest.raises(errors.ShapeError):
        _lib.call("smes_gemm_ragged_m", None, 3, 128, None, 1, 64, 3, 0, None, None, 0, None, None, 0, None, 64, 0,
                  128, None)


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure mode")
def test_no_cpu_fallback():
    import paper_2602_09386_b200 as smes
    with pytest.raises(Exception):
        smes.route_batch(torch.zeros(2, 3, 8), smes.RoutingBudget(1, 1))
    p = smes.SMESParams(torch.zeros(2, 8, 32), torch.zeros(2, 8), [smes.ExpertLayer(torch.zeros(8, 32, 32),
                        torch.zeros(8, 32))], torch.zeros(2, 32), torch.zeros(2))
    with pytest.raises(smes.CudaError):
        smes.SMESEngine(p, 64, 1, 1)


def test_reference_api_surface():
    """Every hot-path name of taskmoe/__init__.py:12-80 that SURVEY 8(b) scopes is exported."""
    import paper_2602_09386_b200 as smes
    for name in ["RoutingBudget", "BatchRouting", "RoutingDecision", "route_batch", "progressive_route",
                 "naive_route_batch", "renormalized_weights", "ExecutionPlan", "build_execution_plan", "grouped_gemm",
                 "reconstruct_task_reps", "ExpertPool", "init_expert_pool", "LoadStats", "compute_load_stats",
                 "lb_loss_gradient", "skew_diagnostics", "MoeModel", "ForwardResult", "forward_sparse", "init_model",
                 "BackwardResult", "backward", "task_loss", "total_loss", "Affine", "FlopCounter",
                 "ShapeError", "ConfigError", "NumericsError", "StateError", "TaskMoeError"]:
        assert hasattr(smes, name), name
