"""B200-native restarted reflected-Halpern PDHG (cuPDLP+, arXiv 2507.14051).

The product is native code: a CUDA device library (lib/librhp_cuda.so, sources
in csrc/) behind the C ABI include/rhpdhg_cuda.h, and the C++ host solver
(lib/librhpdhg.so, sources in host/, API include/rhpdhg/*.hpp mirroring the
reference's proj/include/rhpdhg) behind the C ABI include/rhpdhg_c.h. This
Python package is a ctypes binding of those ABIs plus synthetic generators.
"""
from .lp import (  # noqa: F401
    DeviceError,
    InvalidProblemError,
    KktResiduals,
    LpProblem,
    NumericalBreakdownError,
    ParseError,
    RhpdhgError,
    Session,
    SolutionReport,
    SolverConfig,
    UsageError,
    kkt_residuals,
    set_device,
    set_device_options,
    solve,
)

__all__ = [
    "LpProblem", "SolverConfig", "SolutionReport", "KktResiduals", "Session", "solve",
    "kkt_residuals", "set_device", "set_device_options", "RhpdhgError", "UsageError",
    "InvalidProblemError", "ParseError", "NumericalBreakdownError", "DeviceError",
]
