"""B200-native SMES layer (arXiv 2602.09386): sm_100a CUDA kernels behind the
reference package's (taskmoe) Python module API."""
from .errors import ConfigError, CudaError, NumericsError, ShapeError, StateError, TaskMoeError
from .engine import ExpertLayer, SMESEngine, SMESParams

__version__ = "0.1.0"
