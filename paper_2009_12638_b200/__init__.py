"""B200-native (sm_100a) engine for the block-Jacobi / Krylov 7-point stencil
path of arXiv 2009.12638's two-stage multisplitting method.

Drop-in mirror of the reference package ``blocksolve``'s solver entry points
for that path; every numerical step runs in the hand-written CUDA kernels of
``csrc/bs_engine.cu`` behind the C ABI of ``include/blocksolve_b200.h``.
"""

from .diagnostics import SpectralEstimate, iteration_operator, jacobi_iteration_operator, power_iteration
from .errors import (ConfigurationError, DeviceError, ProtocolError, SolverBreakdownError,
                     ZeroRhsError)
from .inner_solvers import InnerSolveReport, InnerSolverSpec, cg_solve, gmres_solve, jacobi_solve, solve
from .linalg import residual_norms, spmv
from .multisplit import (TRACE_HEADER, DelayModel, OuterConfig, ResidualTrace, SolveResult,
                         TraceRow, check_termination, combined_residual, outer_solve)
from .problems import (FACES, BlockDecomposition, BlockOperator, DirichletBoundary, Grid3D, LinearProblem,
                       StencilOperator, block_system, build_laplace_3d, decompose, seeded_rhs)

__version__ = "0.1.0"

__all__ = [
    "BlockDecomposition", "ConfigurationError", "DelayModel", "DeviceError", "DirichletBoundary",
    "FACES", "Grid3D", "InnerSolveReport", "InnerSolverSpec", "LinearProblem", "OuterConfig",
    "ProtocolError", "ResidualTrace", "SolveResult", "SolverBreakdownError", "StencilOperator",
    "TRACE_HEADER", "TraceRow", "ZeroRhsError", "build_laplace_3d", "cg_solve",
    "check_termination", "combined_residual", "decompose", "gmres_solve", "jacobi_solve", "outer_solve",
    "residual_norms", "seeded_rhs", "solve", "spmv", "SpectralEstimate", "iteration_operator",
    "jacobi_iteration_operator", "power_iteration", "BlockOperator", "block_system",
]
