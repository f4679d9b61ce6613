"""B200-native OD-MoE decode hot path (arXiv 2512.03927): on-demand expert loading with an
INT8 shadow predictor, behind the C ABI of ``libodmoe.so`` (include/odmoe.h).

The package holds only the path: ``csrc/`` (sm_100a kernels + C++ runtime) and the ctypes
binding ``odmoe``. It never imports ``oracle/`` (test infrastructure)."""
from . import odmoe  # noqa: F401  (raises ImportError if libodmoe.so is missing)
from .odmoe import Engine, OdmoeError  # noqa: F401

__all__ = ["odmoe", "Engine", "OdmoeError"]
