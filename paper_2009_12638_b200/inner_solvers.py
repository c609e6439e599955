"""Inner solvers on the GPU (mirror of inner_solvers.py).

``cg_solve(a, b, x0, spec)`` keeps the reference signature and stopping
semantics (inner_solvers.py:102-146): relative to ||b|| (1 if b = 0), the
true residual is re-checked whenever the recurrence claims convergence, and
breakdown is reported, not raised.  The solve runs entirely on the device
(fused CG sweeps, device-side stop tests); the host polls once per batch.

``tolerance_basis="initial"`` (an addition; default keeps the reference
behaviour) measures the tolerance against ||b - A x0|| instead, which is
what fixed-count inner stages and PETSc's rtol mean.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from ._lib import STOP_NAMES
from .engine import torch
from .errors import ConfigurationError
from .engine import launch_bound
from .linalg import as_device_vector, put_vector, single_block_engine, take_vector
from .problems import StencilOperator

__all__ = [
    "InnerSolverSpec",
    "InnerSolveReport",
    "cg_solve",
    "gmres_solve",
    "jacobi_solve",
    "solve",
    "SOLVER_KINDS",
]

SOLVER_KINDS = ("jacobi", "cg", "gmres", "direct")
DEVICE_KINDS = ("jacobi", "cg", "gmres")
DEFAULT_RESTART = 30


@dataclass(frozen=True)
class InnerSolverSpec:
    """Which solver to run and when to stop it (inner_solvers.py:40-57)."""

    kind: str
    max_iterations: int
    tolerance: float = 0.0
    restart: int | None = None

    def __post_init__(self):
        if self.kind not in SOLVER_KINDS:
            raise ValueError(f"unknown solver kind {self.kind!r}")
        if self.max_iterations < 1:
            raise ValueError("max_iterations must be at least 1")
        if self.tolerance < 0:
            raise ValueError("tolerance must be non-negative")
        if self.restart is not None and self.restart < 1:
            raise ValueError("restart must be at least 1")


@dataclass
class InnerSolveReport:
    """Outcome of one solver invocation (inner_solvers.py:60-67)."""

    iterations_used: int
    final_relative_residual: float
    stop_reason: str  # tolerance_met | max_iterations | breakdown
    residual_history: list = field(default_factory=list)


def _check_basis(basis: str) -> None:
    if basis not in ("rhs", "initial"):
        raise ConfigurationError(f"tolerance_basis: unknown basis {basis!r}")


def cg_solve(a: StencilOperator, b, x0, spec: InnerSolverSpec, tolerance_basis: str = "rhs",
             batch: int = 8, out=None):
    """Conjugate gradients on the GPU; returns (x, InnerSolveReport).

    numpy in -> numpy out; CUDA tensor in -> CUDA tensor out (resident);
    host tensor in -> host tensor out (written into ``out`` when given, e.g.
    a pinned buffer, so the device->host copy runs at full PCIe speed).
    """
    return _fused_solve("cg", a, b, x0, spec, tolerance_basis, batch, out)


def jacobi_solve(a: StencilOperator, b, x0, spec: InnerSolverSpec, tolerance_basis: str = "rhs",
                 batch: int = 8, out=None):
    """Point-Jacobi sweeps x <- D^-1 (b - (A - D) x) on the GPU
    (inner_solvers.py:75-99): one fused sweep per iteration reads x_k once,
    yields ||b - A x_k|| / ||b|| and writes x_{k+1}; the first x_k meeting the
    tolerance is returned with k iterations, as in the reference.  Same
    argument / return conventions as ``cg_solve``."""
    return _fused_solve("jacobi", a, b, x0, spec, tolerance_basis, batch, out)


def _fused_solve(kind, a, b, x0, spec, tolerance_basis, batch, out):
    _check_basis(tolerance_basis)
    n = a.num_rows
    is_tensor = torch is not None and isinstance(b, torch.Tensor)
    on_device = is_tensor and b.is_cuda
    eng = single_block_engine(a, b.device if on_device else None, history_cap=spec.max_iterations)
    bd, host = as_device_vector(b, n, eng.device)
    xd, _ = as_device_vector(x0, n, eng.device)
    bb = eng.blocks[0]
    with torch.cuda.device(eng.device):
        put_vector(a, bb, "b", bd)
        put_vector(a, bb, "x", xd)
        begin = eng.cg_begin if kind == "cg" else eng.jacobi_begin
        begin(spec.max_iterations, spec.tolerance, tolerance_basis)
        eng.run(batch=batch, max_launches=launch_bound(spec.max_iterations, batch))
        eng.flush()
        rep = eng.reports()[0]
        its = int(rep.iterations_used)
        hist = bb.history[:its].tolist() if its else []
        x = take_vector(a, bb, "x")  # unpitched copy, never aliased to the engine
    report = InnerSolveReport(its, float(rep.final_relative_residual), STOP_NAMES[int(rep.stop_reason)],
                              hist)
    if host:
        return x.cpu().numpy(), report
    if is_tensor and not on_device:  # host tensor in, host tensor out
        if out is None:
            return x.cpu(), report
        out.copy_(x)
        return out, report
    if out is not None:
        out.copy_(x)
        return out, report
    return x, report


def gmres_solve(a: StencilOperator, b, x0, spec: InnerSolverSpec, tolerance_basis: str = "rhs",
                out=None):
    """Restarted GMRES(m) with MGS Arnoldi and Givens rotations on the GPU
    (inner_solvers.py:149-243): restart = min(spec.restart or 30, n); happy
    breakdown returns the exact iterate; a claimed convergence is verified
    against the true residual; a restart cycle without progress reports
    ``breakdown`` (stagnation)."""
    _check_basis(tolerance_basis)
    n = a.num_rows
    restart = min(spec.restart if spec.restart is not None else DEFAULT_RESTART, n)
    is_tensor = torch is not None and isinstance(b, torch.Tensor)
    on_device = is_tensor and b.is_cuda
    eng = single_block_engine(a, b.device if on_device else None, history_cap=spec.max_iterations)
    bd, host = as_device_vector(b, n, eng.device)
    xd, _ = as_device_vector(x0, n, eng.device)
    bb = eng.blocks[0]
    max_cycles = spec.max_iterations + 2  # every cycle consumes >= 1 iteration
    with torch.cuda.device(eng.device):
        eng.gmres_setup(restart)
        put_vector(a, bb, "b", bd)
        put_vector(a, bb, "x", xd)
        eng.gmres_begin(spec.max_iterations, spec.tolerance, tolerance_basis)
        eng.gmres_run(max_cycles=max_cycles)
        rep = eng.reports()[0]
        its = int(rep.iterations_used)
        hist = bb.history[:its].tolist() if its else []
        x = take_vector(a, bb, "x")
    report = InnerSolveReport(its, float(rep.final_relative_residual), STOP_NAMES[int(rep.stop_reason)],
                              hist)
    if host:
        return x.cpu().numpy(), report
    if out is not None:
        out.copy_(x)
        return out, report
    if is_tensor and not on_device:
        return x.cpu(), report
    return x, report


def solve(a: StencilOperator, b, x0, spec: InnerSolverSpec, tolerance_basis: str = "rhs"):
    """Dispatch on ``spec.kind`` (inner_solvers.py:264-276)."""
    if spec.kind == "cg":
        return cg_solve(a, b, x0, spec, tolerance_basis)
    if spec.kind == "jacobi":
        return jacobi_solve(a, b, x0, spec, tolerance_basis)
    if spec.kind == "gmres":
        return gmres_solve(a, b, x0, spec, tolerance_basis)
    raise ConfigurationError(
        f"inner: {spec.kind!r} is outside the accelerated path (device kinds: {DEVICE_KINDS})")
