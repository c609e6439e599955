"""Device SpMV and residual norms (mirror of linalg.py:178-205).

``spmv(a, x)`` applies the matrix-free 7-point operator on the GPU with the
reference's exact summation order (bit-identical to the CSR ``spmv``).
Inputs may be numpy arrays (copied to the device, result returned as numpy)
or CUDA tensors (kept resident).
"""

from __future__ import annotations

import numpy as np

from .engine import BlockEngine, require_cuda, torch
from .errors import ZeroRhsError
from .problems import BlockOperator, Box, StencilOperator

__all__ = ["spmv", "residual_norms", "as_device_vector", "single_block_engine", "put_vector", "take_vector"]

_ENGINES: dict = {}
_MASKS: dict = {}


def single_block_engine(a, device=None, history_cap: int = 1) -> BlockEngine:
    """Cached one-block engine: the whole grid for a ``StencilOperator``
    (overlap 0), the block's padded box and region for a ``BlockOperator``."""
    dev = require_cuda(device)
    if isinstance(a, BlockOperator):
        key = ("block", a.grid_shape, a.owned.lo, a.owned.hi, a.overlap, str(dev))
        make = lambda cap: BlockEngine(a.grid_shape, [a.owned], a.overlap, dev, history_cap=cap)  # noqa: E731
    else:
        shape = (a.nx, a.ny, a.nz)
        key = (shape, str(dev))
        make = lambda cap: BlockEngine(shape, [Box((0, 0, 0), shape)], 0, dev, history_cap=cap)  # noqa: E731
    eng = _ENGINES.get(key)
    if eng is None or eng.blocks[0].history.numel() < history_cap:
        if eng is not None:
            eng.close()
        if len(_ENGINES) >= 4:  # bounded cache: drop the oldest engine
            old = _ENGINES.pop(next(iter(_ENGINES)))
            old.close()
        eng = make(max(history_cap, 1))
        _ENGINES[key] = eng
    return eng


def _region_mask(a, device):
    if not isinstance(a, BlockOperator):
        return None
    key = (a, str(device))
    m = _MASKS.get(key)
    if m is None:
        m = _MASKS[key] = torch.from_numpy(a.mask).to(device)
    return m


def put_vector(a, bb, name: str, v) -> None:
    """Store an operator-ordered vector (whole grid, or a block's region in
    ascending global index) into the engine buffer ``name``."""
    m = _region_mask(a, v.device)
    if m is None:
        bb.put(name, v)
    else:
        bb.view3(getattr(bb, name))[m] = v


def take_vector(a, bb, name: str):
    """Operator-ordered copy of the engine buffer ``name``."""
    m = _region_mask(a, getattr(bb, name).device)
    return bb.take(name) if m is None else bb.view3(getattr(bb, name))[m]


def as_device_vector(v, n: int, device) -> tuple:
    """(device tensor view, was_numpy).  Mirrors ``as_vector`` checks (linalg.py:46-53)."""
    if torch is not None and isinstance(v, torch.Tensor):
        if v.dim() != 1:
            raise ValueError(f"expected a 1-D vector, got shape {tuple(v.shape)}")
        if v.shape[0] != n:
            raise ValueError(f"expected a vector of length {n}, got {v.shape[0]}")
        return v.to(device=device, dtype=torch.float64), False
    arr = np.asarray(v, dtype=np.float64)
    if arr.ndim != 1:
        raise ValueError(f"expected a 1-D vector, got shape {arr.shape}")
    if arr.shape[0] != n:
        raise ValueError(f"expected a vector of length {n}, got {arr.shape[0]}")
    return torch.from_numpy(np.ascontiguousarray(arr)).to(device), True


def spmv(a: StencilOperator, x):
    """y = A x (linalg.py:178-194), on the GPU."""
    n = a.num_cols
    if (torch is None or not isinstance(x, torch.Tensor)) and np.asarray(x).ndim == 1 \
            and np.asarray(x).shape[0] != n:
        raise ValueError(
            f"dimension mismatch: matrix has {n} columns, vector has {np.asarray(x).shape[0]}")
    eng = single_block_engine(a, None if not isinstance(x, getattr(torch, "Tensor", ())) or not x.is_cuda
                              else x.device)
    xd, host = as_device_vector(x, n, eng.device)
    bb = eng.blocks[0]
    with torch.cuda.device(eng.device):
        xp = bb.zeros_pitched()
        yp = bb.zeros_pitched()
        m = _region_mask(a, eng.device)
        if m is None:
            bb.view3(xp).copy_(xd.reshape(a.nz, a.ny, a.nx))
        else:
            bb.view3(xp)[m] = xd
        eng.apply(0, xp, yp)
        y = bb.view3(yp).contiguous().reshape(-1) if m is None else bb.view3(yp)[m]
    return y.cpu().numpy() if host else y


def residual_norms(a: StencilOperator, x, b) -> tuple:
    """(||b - Ax||, ||b - Ax|| / ||b||) (linalg.py:197-205)."""
    n = a.num_rows
    eng = single_block_engine(a)
    xd, _ = as_device_vector(x, n, eng.device)
    bd, _ = as_device_vector(b, n, eng.device)
    bb = eng.blocks[0]
    with torch.cuda.device(eng.device):
        put_vector(a, bb, "b", bd)
        put_vector(a, bb, "x", xd)
        eng.residual()
        rep = eng.reports()[0]
    absolute = float(np.sqrt(rep.r_sq))
    bnorm = float(np.sqrt(rep.rhs_sq))
    if bnorm == 0.0:
        raise ZeroRhsError("relative residual undefined for a zero right-hand side")
    return absolute, absolute / bnorm
