"""Exception types mirroring taskmoe.errors (errors.py:4-49).

When the reference package is importable the classes subclass its types, so
``except taskmoe.errors.ShapeError`` catches errors raised here too.
"""
from __future__ import annotations

try:  # pragma: no cover - depends on the environment
    from taskmoe import errors as _ref  # type: ignore
except Exception:  # the reference is not shipped to the GPU box
    _ref = None


def _base(name):
    return (getattr(_ref, name),) if _ref is not None else ()


class TaskMoeError(*(_base("TaskMoeError") or (Exception,))):
    """Base class for every error raised by this package."""


class ShapeError(TaskMoeError, *_base("ShapeError")):
    """Operands have incompatible or invalid shapes."""


class NumericsError(TaskMoeError, *_base("NumericsError")):
    """A numeric invariant was violated (NaN/Inf, invalid probability)."""


class ConfigError(TaskMoeError, *_base("ConfigError")):
    """Invalid configuration value or combination."""


class StateError(TaskMoeError, *_base("StateError")):
    """Operation requires state that is missing or inconsistent."""


class DataFormatError(TaskMoeError, *_base("DataFormatError")):
    """Malformed data file (checkpoint); the message names the offending field."""


class PoolError(TaskMoeError, *_base("PoolError")):
    """Invalid workspace-pool operation (infeasible request, double release)."""


class PoolTimeout(TaskMoeError, *_base("PoolTimeout")):
    """An allocation deadline expired before pages became available."""


class CudaError(TaskMoeError):
    """CUDA runtime/driver failure or missing device (no CPU fallback exists)."""
