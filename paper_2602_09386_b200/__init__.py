"""B200-native SMES layer (arXiv 2602.09386).

sm_100a CUDA kernels (csrc/, C ABI in include/smes.h) behind the reference
package's (taskmoe 0.1.0) Python module API: the same function names,
argument orders, result types and exception classes, on CUDA tensors.
There is no CPU fallback: every entry point raises CudaError without a GPU.
"""
from .errors import (ConfigError, CudaError, DataFormatError, NumericsError, PoolError, PoolTimeout, ShapeError,
                     StateError, TaskMoeError)
from .engine import ExpertLayer, SMESEngine, SMESParams
from .engine import workspace_bytes as engine_workspace_bytes
from .routing import (BatchRouting, RouterBank, RoutingBudget, RoutingDecision, compute_global_scores, dense_routing,
                      naive_route_batch, naive_sparse_route, progressive_route, renormalized_weights, route_batch,
                      stack_decisions)
from .execution import ExecutionPlan, build_execution_plan, grouped_gemm, reconstruct_task_reps
from .experts import ExpertPool, init_expert_pool
from .balance import LoadStats, SkewDiagnostics, compute_load_stats, lb_loss_gradient, skew_diagnostics
from .linalg import Affine, FlopCounter, init_affine, matmul, relu, sigmoid, softmax, top_k
from .model import ForwardResult, MoeModel, forward_sparse, heads_from_stacked, init_model
from .training import BackwardResult, backward, task_loss, total_loss
from .checkpoint import load_model, save_model
from .layer import SMESLayer
from .workspace import (DeviceWorkspace, LoadProfile, PageBlock, ReplayResult, WorkspacePool, provision,
                        required_pages, simulate_replay)

__version__ = "0.1.0"

__all__ = [
    "TaskMoeError", "ShapeError", "ConfigError", "NumericsError", "StateError", "CudaError", "DataFormatError",
    "PoolError", "PoolTimeout",
    "SMESEngine", "SMESParams", "ExpertLayer", "engine_workspace_bytes",
    "RoutingBudget", "RouterBank", "BatchRouting", "RoutingDecision", "route_batch", "progressive_route",
    "naive_route_batch", "naive_sparse_route", "renormalized_weights", "compute_global_scores", "dense_routing",
    "stack_decisions",
    "ExecutionPlan", "ExpertPool", "FlopCounter", "build_execution_plan", "grouped_gemm", "init_expert_pool",
    "reconstruct_task_reps",
    "LoadStats", "SkewDiagnostics", "compute_load_stats", "lb_loss_gradient", "skew_diagnostics",
    "Affine", "init_affine", "matmul", "relu", "sigmoid", "softmax", "top_k",
    "ForwardResult", "MoeModel", "forward_sparse", "heads_from_stacked", "init_model",
    "BackwardResult", "backward", "task_loss", "total_loss",
    "load_model", "save_model", "SMESLayer",
    "DeviceWorkspace", "LoadProfile", "PageBlock", "ReplayResult", "WorkspacePool", "provision", "required_pages",
    "simulate_replay",
]
