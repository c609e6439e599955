"""Outer two-stage (block-Jacobi / multisplitting) driver on the GPU.

Mirror of the reference's ``multisplit.py`` API: ``OuterConfig``,
``outer_solve(problem, config) -> SolveResult``, ``ResidualTrace`` with the
fixed CSV schema, ``check_termination`` and ``combined_residual``.

Device schedule of one synchronous outer sweep k (multisplit.py:555-638):

  1. inner solve of every block at once (fused CG sweeps over all blocks
     resident on the GPU, device-side stop per block);
  2. halo pack: each block's boundary values (x + pending alpha*p) are stored
     straight into its neighbours' halo planes (comm.py:332-365 + merge
     multisplit.py:341-369, overlap 0: m = 1 copies);
  3. one residual sweep that is at once the sweep-k local residual
     (multisplit.py:372-396), the true residual of the gathered iterate on
     owned rows (404-406) and the rhs assembly + r0 of sweep k+1 (333-338);
  4. the per-block scalars come back to the host, which combines them in
     block order exactly like comm.py:442-445 and decides (409-426).

Sync results are deterministic and independent of how blocks are spread
over GPUs (fixed-order reductions, same tiles per block).
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .engine import BlockEngine, box_halo_plan, require_cuda, torch
from .errors import ConfigurationError
from .inner_solvers import InnerSolverSpec
from .problems import LinearProblem, decompose
from .sync_driver import run_sync

__all__ = [
    "OuterConfig",
    "TraceRow",
    "ResidualTrace",
    "SolveResult",
    "TRACE_HEADER",
    "check_termination",
    "combined_residual",
    "outer_solve",
]

TRACE_HEADER = (
    "outer_iteration,time,estimated_residual,true_residual,"
    "inner_iterations,max_halo_staleness"
)

DEFAULT_BUFFER_SLOTS = 100


@dataclass(frozen=True)
class DelayModel:
    """In-flight delay distribution in receiver outer iterations (comm.py:51-81).

    Async mode adds it on top of the device path's real asynchrony: halo posts
    and published residuals become visible k + d iterations after they were
    sent (see ``async_driver``).  Sync mode ignores it, as the reference's
    rendezvous exchanges do."""

    kind: str = "none"
    fixed: int = 0
    low: int = 0
    high: int = 0
    seed: int = 0

    def __post_init__(self):
        if self.kind not in ("none", "fixed", "uniform", "drop_free_jitter"):
            raise ConfigurationError(f"delay: unknown kind {self.kind!r}")
        if self.kind == "fixed" and self.fixed < 0:
            raise ConfigurationError("delay: fixed delay must be non-negative")
        if self.kind in ("uniform", "drop_free_jitter") and not (0 <= self.low <= self.high):
            raise ConfigurationError("delay: bounds must satisfy 0 <= low <= high")

    def draw(self, rng: np.random.Generator) -> int:
        """One delay (comm.py:76-81)."""
        if self.kind == "none":
            return 0
        if self.kind == "fixed":
            return self.fixed
        return int(rng.integers(self.low, self.high + 1))


@dataclass
class OuterConfig:
    """Tunables of the outer solve (multisplit.py:65-103) plus device knobs.

    Additions (defaults keep reference behaviour): ``device`` (CUDA device),
    ``tolerance_basis`` ("rhs" | "initial", see inner_solvers),
    ``batch`` (sweep cycles per host poll of the device stop counter).
    """

    block_grid: tuple = (1, 1, 1)
    overlap: int = 0
    inner: InnerSolverSpec = field(default_factory=lambda: InnerSolverSpec("gmres", 10))
    mode: str = "sync"
    buffer_slots: int = DEFAULT_BUFFER_SLOTS
    tol: float = 1e-6
    max_outer: int = 5000
    residual_check_mode: str = "paper"
    delay: DelayModel = field(default_factory=DelayModel)
    true_residual_interval: int = 10
    capture_iterates: bool = False
    execution: str = "replay"
    record_comm_events: bool = False
    device: str | None = None
    tolerance_basis: str = "rhs"
    batch: int = 4
    residual_check_every: int = 1

    def __post_init__(self):
        if self.mode not in ("sync", "async"):
            raise ConfigurationError(f"mode: unknown mode {self.mode!r}")
        if self.tol <= 0:
            raise ConfigurationError("tol: must be positive")
        if self.max_outer < 1:
            raise ConfigurationError("max_outer: must be at least 1")
        if self.residual_check_mode not in ("paper", "true"):
            raise ConfigurationError(f"residual_mode: unknown mode {self.residual_check_mode!r}")
        if self.execution not in ("replay", "threads"):
            raise ConfigurationError(f"exec: unknown execution {self.execution!r}")
        if self.execution != "replay" and (self.residual_check_mode == "true" or self.capture_iterates):
            raise ConfigurationError(
                "exec: true-residual termination and iterate capture need replay execution")
        if self.true_residual_interval < 1:
            raise ConfigurationError("true_res_every: must be at least 1")
        if self.tolerance_basis not in ("rhs", "initial"):
            raise ConfigurationError(f"tolerance_basis: unknown basis {self.tolerance_basis!r}")
        if self.batch < 1:
            raise ConfigurationError("batch: must be at least 1")
        if self.residual_check_every < 1:
            raise ConfigurationError("residual_check_every: must be at least 1")


@dataclass
class TraceRow:
    outer_iteration: int
    time: float
    estimated_residual: float
    true_residual: float | None
    inner_iterations: int
    max_halo_staleness: int


def _fmt(value: float) -> str:
    return format(value, ".17g")


@dataclass
class ResidualTrace:
    """Per-outer-iteration record with the fixed CSV schema (multisplit.py:443-484)."""

    rows: list = field(default_factory=list)

    def write_csv(self, path) -> None:
        lines = [TRACE_HEADER]
        for row in self.rows:
            true = "" if row.true_residual is None else _fmt(row.true_residual)
            lines.append(
                f"{row.outer_iteration},{_fmt(row.time)},{_fmt(row.estimated_residual)},{true},"
                f"{row.inner_iterations},{row.max_halo_staleness}")
        with open(path, "w") as fh:
            fh.write("\n".join(lines) + "\n")

    @classmethod
    def read_csv(cls, path) -> "ResidualTrace":
        with open(path) as fh:
            lines = [line.rstrip("\n") for line in fh]
        if not lines or lines[0] != TRACE_HEADER:
            raise ValueError(f"{path}: not a residual trace (unexpected header)")
        rows = []
        for line in lines[1:]:
            if not line:
                continue
            parts = line.split(",")
            if len(parts) != 6:
                raise ValueError(f"{path}: malformed trace row {line!r}")
            rows.append(TraceRow(int(parts[0]), float(parts[1]), float(parts[2]),
                                 None if parts[3] == "" else float(parts[3]), int(parts[4]),
                                 int(parts[5])))
        return cls(rows)


@dataclass
class SolveResult:
    solution: object
    trace: ResidualTrace
    converged: bool
    outer_iterations: int
    final_true_residual: float
    snapshots: list = field(default_factory=list)
    comm_events: list = field(default_factory=list)
    inner_iterations_per_block: list = field(default_factory=list)
    wall_seconds: float = 0.0


def combined_residual(local_residuals) -> float:
    """sqrt of the sum of squared block residues (multisplit.py:399-401)."""
    return math.sqrt(sum(float(r) ** 2 for r in local_residuals))


def check_termination(estimate: float, tol: float, completed: int, max_outer: int, mode: str) -> str:
    """{continue | confirm | stop} (multisplit.py:409-426)."""
    if mode == "sync":
        if estimate < tol or completed >= max_outer:
            return "stop"
        return "continue"
    if estimate < tol:
        return "confirm"
    if completed >= max_outer:
        return "stop"
    return "continue"


def _validate_device_path(config: OuterConfig) -> None:
    if config.mode == "async" and (config.inner.kind not in ("cg", "jacobi") or config.overlap != 0):
        raise ConfigurationError("mode: async runs CG or Jacobi inner solves on overlap-0 decompositions")
    if config.inner.kind not in ("jacobi", "cg", "gmres"):
        raise ConfigurationError(
            f"inner: {config.inner.kind!r} is outside the accelerated path (device kinds: jacobi, cg, gmres)")


def outer_solve(problem: LinearProblem, config: OuterConfig, probe=None, resume=None) -> SolveResult:
    """Run the two-stage solve on the GPU and gather the owned values.

    ``probe``: optional measurement hooks of the sync sweep loop (see
    ``sync_driver.run_sync``); results do not depend on it.  ``resume`` =
    (k, directory): continue a segmented synchronous run (overlap > 0) from
    the iterate ``BlockEngine.save_state`` wrote after sweep k; the trace of
    this call then starts at sweep k + 1."""
    _validate_device_path(config)
    if resume is not None and (config.overlap == 0 or config.mode != "sync"):
        raise ConfigurationError("resume: segmented runs are implemented for synchronous sweeps over "
                                 "overlapping decompositions")
    grid = problem.grid
    nx, ny, nz = grid.shape
    decomp = decompose(grid, config.block_grid, config.overlap)
    dev = require_cuda(config.device)
    rhs = problem.rhs
    on_device = torch is not None and isinstance(rhs, torch.Tensor)
    if on_device:
        b_dev = rhs.to(device=dev, dtype=torch.float64).reshape(nz, ny, nx)
        b_host = None
    else:
        b_host = np.asarray(rhs, dtype=np.float64)
        if b_host.shape != (grid.num_unknowns,):
            raise ValueError(f"expected a vector of length {grid.num_unknowns}, got {b_host.shape}")
        b_dev = torch.from_numpy(b_host.reshape(nz, ny, nx)).to(dev)

    # denominators of the local residual (multisplit.py:390-396) and ||b||
    if b_host is not None:
        b3h = b_host.reshape(nz, ny, nx)
        bnorm = float(np.linalg.norm(b_host))
        owned_norms = []
        for box in decomp.owned:
            sl = b3h[box.lo[2]:box.hi[2], box.lo[1]:box.hi[1], box.lo[0]:box.hi[0]]
            owned_norms.append(float(np.linalg.norm(sl.ravel())))
    else:
        bnorm = float(torch.linalg.vector_norm(b_dev))
        owned_norms = [float(torch.linalg.vector_norm(
            b_dev[box.lo[2]:box.hi[2], box.lo[1]:box.hi[1], box.lo[0]:box.hi[0]]))
            for box in decomp.owned]
    dens = [d if d != 0.0 else (bnorm if bnorm != 0.0 else 1.0) for d in owned_norms]

    t_start = time.perf_counter()
    spec = config.inner
    if config.mode == "async":
        return _outer_solve_async(problem, config, decomp, b_dev, dens, bnorm, dev, on_device, t_start)
    with torch.cuda.device(dev):
        overlap = config.overlap
        eng = BlockEngine(grid.shape, decomp.owned, overlap, dev, history_cap=1)
        eng.load_global("b", b_dev)
        if resume is not None:
            eng.load_state(resume[1])
        plan = box_halo_plan(decomp.owned, decomp.block_grid) if overlap == 0 else None
        snapshots = []

        def capture(k):
            if config.capture_iterates:
                snap = torch.empty(nz, ny, nx, dtype=torch.float64, device=dev)
                eng.flush()
                eng.gather_owned(snap)
                snapshots.append((k, snap.reshape(-1).cpu().numpy()))

        try:
            trace, per_block, converged, final_true = run_sync(
                eng, config, dens, bnorm, decomp.num_blocks, list(range(decomp.num_blocks)),
                lambda: eng.halo_pack(plan), lambda table: table, t_start, on_sweep=capture, probe=probe,
                resume_k=None if resume is None else resume[0])
            eng.flush()
            sol = torch.empty(nz, ny, nx, dtype=torch.float64, device=dev)
            eng.gather_owned(sol)
            torch.cuda.synchronize(dev)
        finally:
            eng.close()
    wall = time.perf_counter() - t_start
    rows = [TraceRow(k, t, est, tr, inner, 0) for k, t, est, tr, inner in trace]
    if rows and rows[-1].true_residual is None:
        rows[-1].true_residual = final_true
    solution = sol.reshape(-1) if on_device else sol.reshape(-1).cpu().numpy()
    return SolveResult(solution=solution, trace=ResidualTrace(rows), converged=converged,
                       outer_iterations=len(rows), final_true_residual=final_true,
                       snapshots=snapshots, inner_iterations_per_block=per_block, wall_seconds=wall)


def _outer_solve_async(problem, config, decomp, b_dev, dens, bnorm, dev, on_device, t_start):
    from .async_driver import outer_solve_async

    pieces = outer_solve_async(problem, config, decomp, b_dev, dens, bnorm, dev, config.inner)
    return async_result(problem, b_dev, on_device, t_start, pieces)


def async_result(problem, b_dev, on_device, t_start, pieces) -> SolveResult:
    """SolveResult of an asynchronous run: trace aggregated across blocks
    (multisplit.py:769-787) and the true residual of the gathered iterate."""
    from .linalg import residual_norms

    sol, records, converged, lapped, skipped = pieces
    flat = sol.reshape(-1)
    final_true = residual_norms(problem.matrix, flat, b_dev.reshape(-1))[1]
    # trace aggregation across blocks (multisplit.py:769-787)
    outer = max(len(r) for r in records)
    rows = []
    for k in range(outer):
        at_k = [r[k] for r in records if k < len(r)]
        est = records[0][k][2] if k < len(records[0]) else at_k[0][2]
        rows.append(TraceRow(k, max(a[1] for a in at_k), est, None, int(sum(a[3] for a in at_k)),
                             int(max(a[4] for a in at_k))))
    if rows:
        rows[-1].true_residual = final_true
    per_block = [[r[k][3] if k < len(r) else 0 for r in records] for k in range(outer)]
    solution = flat if on_device else flat.cpu().numpy()
    return SolveResult(solution=solution, trace=ResidualTrace(rows), converged=converged, outer_iterations=outer,
                       final_true_residual=final_true, inner_iterations_per_block=per_block,
                       wall_seconds=time.perf_counter() - t_start,
                       comm_events=[("lapped_reads", lapped), ("skipped_sends", skipped)])
