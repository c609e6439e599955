"""Spectral diagnostics on the device.

* ``power_iteration`` — the reference's power method (linalg.py:243-276):
  seeded start ``1 + U[0,1)`` (numpy's PCG64 stream, generated on the GPU
  bit-identically), radius = norm growth per step, converged when successive
  estimates differ by less than ``tol``.  Vectors stay resident in HBM; the
  norm is a fixed-order device reduction (bitwise repeatable).
* ``iteration_operator`` — the exact-inner-solve outer iteration as a linear
  map on the stacked per-block extended vectors (multisplit.py:800-830).  The
  reference factors every block densely (LU), which stops at a few thousand
  unknowns per block; here one application is one outer sweep of the engine
  with b = 0: halo exchange (overlap 0) or 1/m merge (overlap > 0), then a CG
  solve of every block to ``inner_tolerance`` from x0 = 0 — the same map to
  solver accuracy, at any size that fits in HBM.
* ``jacobi_iteration_operator`` — x -> D^-1 (D - A) x of the point-Jacobi
  iteration, one fused Jacobi sweep with b = 0.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .engine import BlockEngine, box_halo_plan, launch_bound, require_cuda, torch
from .linalg import as_device_vector
from .problems import Box, BlockDecomposition, LinearProblem, StencilOperator

__all__ = ["SpectralEstimate", "power_iteration", "iteration_operator", "jacobi_iteration_operator",
           "IterationOperator"]


@dataclass
class SpectralEstimate:
    """Dominant |eigenvalue| estimate from the power iteration (linalg.py:234-240)."""

    radius: float
    iterations_used: int
    converged: bool


def _stream(dev) -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def power_iteration(apply_map, dim: int, tol: float = 1e-10, max_iterations: int = 5000, seed: int = 0,
                    device=None, host_map: bool = False) -> SpectralEstimate:
    """Estimate the spectral radius of ``apply_map`` by the power method
    (linalg.py:243-276).  ``apply_map`` takes and returns a length-``dim``
    vector: a CUDA tensor (the device operators of this package,
    ``iteration_operator`` / ``jacobi_iteration_operator``, keep it resident
    end to end), or with ``host_map=True`` a numpy array (one host round trip
    per step, for reference-style callables)."""
    if dim < 1:
        raise ValueError("dim must be at least 1")
    if tol <= 0:
        raise ValueError("tol must be positive")
    dev = require_cuda(device if device is not None else getattr(apply_map, "device", None))
    lib = _lib.load()
    with torch.cuda.device(dev):
        st = np.random.default_rng(seed).bit_generator.state["state"]
        s, inc = int(st["state"]), int(st["inc"])
        m64 = (1 << 64) - 1
        x = torch.empty(dim, dtype=torch.float64, device=dev)
        # 1.0 + rng.random(dim) == uniform(1, 2): 1 + 1*u is exact
        _lib.check(lib.bs_uniform_pcg64(x.data_ptr(), dim, s >> 64, s & m64, inc >> 64, inc & m64, 1.0, 2.0,
                                        _stream(dev)))
        work = torch.zeros(_lib.VEC_WORK, dtype=torch.float64, device=dev)
        host = torch.zeros(1, dtype=torch.float64).pin_memory()

        def nrm2(v) -> float:
            _lib.check(lib.bs_vec_nrm2(v.data_ptr(), dim, work.data_ptr(), _stream(dev)))
            host.copy_(work[:1], non_blocking=True)
            torch.cuda.current_stream(dev).synchronize()
            return float(host[0])

        def scale(v, d, out):
            _lib.check(lib.bs_vec_scale(v.data_ptr(), dim, float(d), out.data_ptr(), _stream(dev)))

        scale(x, nrm2(x), x)
        previous = np.inf
        estimate = 0.0
        for it in range(1, max_iterations + 1):
            y = apply_map(x.cpu().numpy() if host_map else x)
            if not isinstance(y, torch.Tensor):
                y, _ = as_device_vector(y, dim, dev)
            y = y.to(device=dev, dtype=torch.float64).contiguous()
            if y.dim() != 1 or y.shape[0] != dim:
                raise ValueError(f"apply_map returned shape {tuple(y.shape)}, expected ({dim},)")
            estimate = nrm2(y)
            if estimate == 0.0:
                return SpectralEstimate(0.0, it, True)
            if abs(estimate - previous) < tol:
                return SpectralEstimate(estimate, it, True)
            previous = estimate
            x = torch.empty_like(y)
            scale(y, estimate, x)
        return SpectralEstimate(estimate, max_iterations, False)


class IterationOperator:
    """z -> M^-1 N z on the stacked extended vectors (multisplit.py:800-830),
    every block solve done by the device CG to ``inner_tolerance``.

    Callable on a CUDA tensor (result: CUDA tensor) or a numpy array (result:
    numpy).  ``close()`` frees the engine."""

    def __init__(self, problem: LinearProblem, decomp: BlockDecomposition, device=None,
                 inner_tolerance: float = 1e-13, inner_max_iterations: int | None = None):
        self.device = require_cuda(device)
        grid = problem.grid
        self.overlap = decomp.overlap
        self.eng = BlockEngine(grid.shape, decomp.owned, decomp.overlap, self.device, history_cap=1)
        self.plan = box_halo_plan(decomp.owned, decomp.block_grid) if decomp.overlap == 0 else None
        self.masks, sizes = [], []
        for b in range(decomp.num_blocks):
            if decomp.overlap == 0:
                self.masks.append(None)
                sizes.append(decomp.owned[b].size)
            else:
                m = decomp.region_mask(b)
                self.masks.append(torch.from_numpy(m).to(self.device))
                sizes.append(int(m.sum()))
        self.offsets = np.concatenate(([0], np.cumsum(sizes))).astype(np.int64)
        self.dim = int(self.offsets[-1])
        self.tol = float(inner_tolerance)
        largest = max(bb.padded.size for bb in self.eng.blocks)
        self.max_its = int(inner_max_iterations) if inner_max_iterations else max(100, 4 * largest)
        with torch.cuda.device(self.device):
            self.eng.zero("b")  # homogeneous system: rhs = -C * (averaged halo)

    def close(self) -> None:
        if self.eng is not None:
            self.eng.close()
            self.eng = None

    def _scatter(self, z) -> None:
        for b, bb in enumerate(self.eng.blocks):
            part = z[self.offsets[b]:self.offsets[b + 1]]
            x3 = bb.view3(bb.x)
            if self.masks[b] is None:
                x3.copy_(part.view(x3.shape))
            else:
                x3[self.masks[b]] = part

    def _gather(self, out) -> None:
        for b, bb in enumerate(self.eng.blocks):
            x3 = bb.view3(bb.x)
            out[self.offsets[b]:self.offsets[b + 1]] = x3.reshape(-1) if self.masks[b] is None \
                else x3[self.masks[b]]

    def __call__(self, z):
        zd, host = as_device_vector(z, self.dim, self.device)
        eng = self.eng
        with torch.cuda.device(self.device):
            self._scatter(zd)
            if self.overlap == 0:
                eng.halo_pack(self.plan)  # payload = neighbour's z, m = 1
                eng.zero("x")
            else:
                eng.overlap_merge()  # halo = (sum of neighbour payloads) / m_halo
                for b, bb in enumerate(eng.blocks):
                    bb.view3(bb.x)[self.masks[b]] = 0.0  # x0 = 0; the halo cells stay
            eng.cg_begin(self.max_its, self.tol, "rhs")
            eng.run(batch=8, max_launches=launch_bound(self.max_its, 8))
            eng.flush()
            for rep in eng.reports():
                if _lib.STOP_NAMES[int(rep.stop_reason)] not in ("tolerance_met", "max_iterations"):
                    raise ArithmeticError("iteration_operator: block solve broke down")
            out = torch.empty(self.dim, dtype=torch.float64, device=self.device)
            self._gather(out)
        return out.cpu().numpy() if host else out


def iteration_operator(problem: LinearProblem, decomp: BlockDecomposition, device=None,
                       inner_tolerance: float = 1e-13, inner_max_iterations: int | None = None):
    """(apply, dim) as the reference returns (multisplit.py:800-830)."""
    op = IterationOperator(problem, decomp, device, inner_tolerance, inner_max_iterations)
    return op, op.dim


class _JacobiMap:
    def __init__(self, a: StencilOperator, device=None):
        self.device = require_cuda(device)
        shape = (a.nx, a.ny, a.nz)
        self.dim = a.num_rows
        self.eng = BlockEngine(shape, [Box((0, 0, 0), shape)], 0, self.device, history_cap=2)
        with torch.cuda.device(self.device):
            self.eng.zero("b")

    def __call__(self, x):
        xd, host = as_device_vector(x, self.dim, self.device)
        bb = self.eng.blocks[0]
        with torch.cuda.device(self.device):
            bb.put("x", xd)
            self.eng.jacobi_begin(1, 0.0)  # x_1 = (0 - (A - D) x_0) / 6
            self.eng.run(batch=1, max_launches=8)
            self.eng.flush()
            out = bb.take("x")
        return out.cpu().numpy() if host else out

    def close(self) -> None:
        if self.eng is not None:
            self.eng.close()
            self.eng = None


def jacobi_iteration_operator(a: StencilOperator, device=None):
    """(apply, dim) of x -> D^-1 (D - A) x (the point-Jacobi iteration matrix
    the reference's tests build as ``x - spmv(a, x) / d``), on the device."""
    op = _JacobiMap(a, device)
    return op, op.dim
