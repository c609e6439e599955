"""3D Laplace test problem and block decomposition (mirror of problems.py).

The operator is matrix-free: ``build_laplace_3d`` returns a ``LinearProblem``
whose ``matrix`` is a ``StencilOperator`` (the 7-point Laplacian of the grid)
instead of an assembled CSR.  Geometry is derived analytically (owned boxes,
L1-dilated extended regions, neighbor lists) so setup stays surface-sized at
512^3 and 1024^3, where the reference's full-grid masks are infeasible
(SURVEY §7 hard part 8).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, Union

import numpy as np

from .errors import ConfigurationError

__all__ = [
    "FACES",
    "DirichletBoundary",
    "Grid3D",
    "LinearProblem",
    "StencilOperator",
    "BlockDecomposition",
    "BlockOperator",
    "block_system",
    "build_laplace_3d",
    "decompose",
    "seeded_rhs",
]

FACES = ("x_lo", "x_hi", "y_lo", "y_hi", "z_lo", "z_hi")
_RHS_ORDER = ("z_lo", "y_lo", "x_lo", "x_hi", "y_hi", "z_hi")  # problems.py:143-167

FaceValue = Union[float, Callable[[int, int], float]]


class DirichletBoundary:
    """Per-face Dirichlet data (problems.py:42-85)."""

    def __init__(self, faces: dict | None = None, default: float = 0.0):
        faces = dict(faces or {})
        for name in faces:
            if name not in FACES:
                raise ConfigurationError(f"boundary: unknown face {name!r}")
        self._faces = {name: faces.get(name, float(default)) for name in FACES}

    @classmethod
    def constant(cls, value: float) -> "DirichletBoundary":
        return cls(default=float(value))

    @classmethod
    def zero(cls) -> "DirichletBoundary":
        return cls()

    def value(self, face: str, u: int, v: int) -> float:
        spec = self._faces[face]
        return float(spec(u, v)) if callable(spec) else spec

    def face_constants(self) -> dict:
        if any(callable(v) for v in self._faces.values()):
            raise ValueError("boundary with callable faces has no constant form")
        return {name: float(self._faces[name]) for name in FACES}

    def spec(self, face: str):
        return self._faces[face]

    def __eq__(self, other) -> bool:
        if not isinstance(other, DirichletBoundary):
            return NotImplemented
        return self._faces == other._faces

    def __repr__(self) -> str:
        return f"DirichletBoundary({self._faces!r})"


@dataclass(frozen=True)
class Grid3D:
    """Interior unknown counts plus boundary data (problems.py:88-111)."""

    nx: int
    ny: int
    nz: int
    boundary: DirichletBoundary = field(default_factory=DirichletBoundary.zero)

    def __post_init__(self):
        for name in ("nx", "ny", "nz"):
            if getattr(self, name) < 1:
                raise ConfigurationError(f"{name}: must be at least 1")

    @property
    def shape(self) -> tuple:
        return (self.nx, self.ny, self.nz)

    @property
    def num_unknowns(self) -> int:
        return self.nx * self.ny * self.nz

    def index(self, i: int, j: int, k: int) -> int:
        return i + self.nx * (j + self.ny * k)


@dataclass(frozen=True)
class StencilOperator:
    """Matrix-free 7-point Laplacian of a grid (diag 6, -1 per interior
    neighbor; problems.py:123-175).  Stands where the reference passes its
    assembled ``SparseMatrix``."""

    nx: int
    ny: int
    nz: int

    @property
    def shape(self) -> tuple:
        n = self.nx * self.ny * self.nz
        return (n, n)

    @property
    def num_rows(self) -> int:
        return self.nx * self.ny * self.nz

    num_cols = num_rows

    @property
    def nnz(self) -> int:
        nx, ny, nz = self.nx, self.ny, self.nz
        return 7 * nx * ny * nz - 2 * (ny * nz + nx * nz + nx * ny)


@dataclass
class LinearProblem:
    """Operator, right-hand side and generating grid (problems.py:114-120)."""

    matrix: StencilOperator
    rhs: np.ndarray
    grid: Grid3D


def _face_values(spec, a: np.ndarray, b: np.ndarray) -> np.ndarray:
    if callable(spec):
        return np.vectorize(lambda u, v: float(spec(int(u), int(v))), otypes=[float])(a, b)
    return np.full(a.shape, float(spec))


def build_laplace_3d(grid: Grid3D) -> LinearProblem:
    """Vectorised ``build_laplace_3d`` (problems.py:123-175).

    The rhs folds the Dirichlet data exactly as the reference does: every
    point starts at 0.0 and receives ``+=`` of each global face it touches in
    the order z_lo, y_lo, x_lo, x_hi, y_hi, z_hi, so the result is bitwise
    identical.  The operator stays implicit.
    """
    nx, ny, nz = grid.shape
    rhs = np.zeros((nz, ny, nx))
    bnd = grid.boundary
    for face in _RHS_ORDER:
        spec = bnd.spec(face)
        if not callable(spec) and spec == 0.0:
            continue  # += 0.0 never changes a value that started at +0.0
        if face in ("z_lo", "z_hi"):
            jj, ii = np.meshgrid(np.arange(ny), np.arange(nx), indexing="ij")
            rhs[0 if face == "z_lo" else nz - 1] += _face_values(spec, ii, jj)
        elif face in ("y_lo", "y_hi"):
            kk, ii = np.meshgrid(np.arange(nz), np.arange(nx), indexing="ij")
            rhs[:, 0 if face == "y_lo" else ny - 1, :] += _face_values(spec, ii, kk)
        else:
            kk, jj = np.meshgrid(np.arange(nz), np.arange(ny), indexing="ij")
            rhs[:, :, 0 if face == "x_lo" else nx - 1] += _face_values(spec, jj, kk)
    return LinearProblem(StencilOperator(nx, ny, nz), rhs.ravel(), grid)


def seeded_rhs(n: int, seed: int = 0, device=None):
    """Seeded rhs convention of SURVEY §8(d): uniform [-1, 1], x-fastest.

    With ``device`` the values are generated on the GPU (bit-identical to
    numpy's PCG64 stream; no host array, no upload)."""
    if device is None:
        return np.random.default_rng(seed).uniform(-1.0, 1.0, n)
    import ctypes

    from . import _lib
    from .engine import require_cuda, torch

    dev = require_cuda(device)
    st = np.random.default_rng(seed).bit_generator.state["state"]
    s, inc = int(st["state"]), int(st["inc"])
    out = torch.empty(n, dtype=torch.float64, device=dev)
    lib = _lib.load()
    m64 = (1 << 64) - 1
    with torch.cuda.device(dev):
        stream = ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
        _lib.check(lib.bs_uniform_pcg64(out.data_ptr(), n, s >> 64, s & m64, inc >> 64, inc & m64, -1.0, 1.0,
                                        stream))
    return out


def _split_ranges(n: int, g: int) -> list:
    """problems.py:216-225."""
    base, rem = divmod(n, g)
    out, start = [], 0
    for b in range(g):
        w = base + (1 if b < rem else 0)
        out.append((start, start + w))
        start += w
    return out


@dataclass(frozen=True)
class Box:
    """Half-open index box [lo, hi) in (x, y, z) (problems.py:193-213)."""

    lo: tuple
    hi: tuple

    @property
    def size(self) -> int:
        return (self.hi[0] - self.lo[0]) * (self.hi[1] - self.lo[1]) * (self.hi[2] - self.lo[2])

    @property
    def widths(self) -> tuple:
        return tuple(self.hi[d] - self.lo[d] for d in range(3))

    def contains(self, i: int, j: int, k: int) -> bool:
        return all(self.lo[d] <= p < self.hi[d] for d, p in enumerate((i, j, k)))


@dataclass
class BlockDecomposition:
    """Owned boxes and neighbor topology (problems.py:228-284), analytic."""

    grid: Grid3D
    block_grid: tuple
    overlap: int
    owned: list
    neighbors: list

    @property
    def num_blocks(self) -> int:
        return len(self.owned)

    def block_coords(self, block_id: int) -> tuple:
        gx, gy, gz = self.block_grid
        return (block_id % gx, (block_id // gx) % gy, block_id // (gx * gy))

    def padded_box(self, block_id: int) -> Box:
        """Bounding box of the extended region (owned box dilated by o)."""
        box = self.owned[block_id]
        shape = self.grid.shape
        lo = tuple(max(0, box.lo[d] - self.overlap) for d in range(3))
        hi = tuple(min(shape[d], box.hi[d] + self.overlap) for d in range(3))
        return Box(lo, hi)

    def region_mask(self, block_id: int) -> np.ndarray:
        """Extended-region mask over the padded box, (z, y, x) order."""
        box, pad = self.owned[block_id], self.padded_box(block_id)
        k, j, i = np.meshgrid(*(np.arange(pad.lo[d], pad.hi[d]) for d in (2, 1, 0)), indexing="ij")
        d = (np.maximum(0, np.maximum(box.lo[0] - i, i - (box.hi[0] - 1)))
             + np.maximum(0, np.maximum(box.lo[1] - j, j - (box.hi[1] - 1)))
             + np.maximum(0, np.maximum(box.lo[2] - k, k - (box.hi[2] - 1))))
        return d <= self.overlap

    def extended_indices(self, block_id: int) -> np.ndarray:
        nx, ny = self.grid.nx, self.grid.ny
        pad = self.padded_box(block_id)
        k, j, i = np.meshgrid(*(np.arange(pad.lo[d], pad.hi[d]) for d in (2, 1, 0)), indexing="ij")
        idx = i + nx * (j + ny * k)
        return idx[self.region_mask(block_id)].ravel()

    def owned_indices(self, block_id: int) -> np.ndarray:
        box = self.owned[block_id]
        nx, ny = self.grid.nx, self.grid.ny
        ii = np.arange(box.lo[0], box.hi[0])
        jj = np.arange(box.lo[1], box.hi[1])
        kk = np.arange(box.lo[2], box.hi[2])
        return (ii[None, None, :] + nx * (jj[None, :, None] + ny * kk[:, None, None])).ravel()


def _box_l1_gap(a: Box, b: Box) -> int:
    """L1 distance between two boxes (0 if they touch or overlap)."""
    gap = 0
    for d in range(3):
        gap += max(0, a.lo[d] - (b.hi[d] - 1), b.lo[d] - (a.hi[d] - 1))
    return gap


def region_size(grid_shape, owned: Box, overlap: int) -> int:
    """Points of a block's extended region — the owned box dilated ``overlap``
    times by the 7-point stencil (an L1 ball, problems.py:178-190) clipped to
    the grid — counted analytically: the rows of its block system A_ii."""
    counts = []
    for d in range(3):
        lo, hi, n = owned.lo[d], owned.hi[d], grid_shape[d]
        # coordinates at L1 distance exactly t outside [lo, hi) on this axis
        counts.append([hi - lo] + [int(lo - t >= 0) + int(hi - 1 + t < n) for t in range(1, overlap + 1)])
    cx, cy, cz = counts
    return sum(cx[a] * cy[b] * cz[c] for a in range(overlap + 1) for b in range(overlap + 1 - a)
               for c in range(overlap + 1 - a - b))


def decompose(grid: Grid3D, block_grid: tuple, overlap: int = 0) -> BlockDecomposition:
    """Analytic ``decompose`` (problems.py:287-359).

    Neighbors: the reference pairs blocks whose extended regions are within
    one stencil step (dilate(ext_a, 1) & ext_b).  Extended regions are L1
    balls of radius o around boxes, so that is L1-gap(box_a, box_b) <= 2o+1.
    """
    gx, gy, gz = block_grid
    nx, ny, nz = grid.shape
    for g, n, name in ((gx, nx, "gx"), (gy, ny, "gy"), (gz, nz, "gz")):
        if g < 1:
            raise ConfigurationError(f"{name}: must be at least 1")
        if g > n:
            raise ConfigurationError(f"{name}: {g} blocks exceed the {n} grid points of that dimension")
    if overlap < 0:
        raise ConfigurationError("overlap: must be non-negative")
    ranges = {"x": _split_ranges(nx, gx), "y": _split_ranges(ny, gy), "z": _split_ranges(nz, gz)}
    for axis, g, name in (("x", gx, "gx"), ("y", gy, "gy"), ("z", gz, "gz")):
        if g > 1:
            min_width = min(hi - lo for lo, hi in ranges[axis])
            if overlap >= min_width:
                raise ConfigurationError(
                    f"overlap: {overlap} is not smaller than the narrowest "
                    f"{axis}-range width {min_width} ({name}={g})")
    owned = []
    for bz in range(gz):
        for by in range(gy):
            for bx in range(gx):
                lo = (ranges["x"][bx][0], ranges["y"][by][0], ranges["z"][bz][0])
                hi = (ranges["x"][bx][1], ranges["y"][by][1], ranges["z"][bz][1])
                owned.append(Box(lo, hi))
    nb = len(owned)
    neighbors = [[] for _ in range(nb)]
    for a in range(nb):
        for b in range(a + 1, nb):
            if _box_l1_gap(owned[a], owned[b]) <= 2 * overlap + 1:
                neighbors[a].append(b)
                neighbors[b].append(a)
    return BlockDecomposition(grid, (gx, gy, gz), overlap, owned, neighbors)


class BlockOperator:
    """A block's local operator: the principal submatrix of the 7-point
    Laplacian on the block's extended region (problems.py:362-406), matrix-free.

    Unknowns are the region's points in ascending global index (the
    reference's ``extended_indices`` order).  ``spmv`` and the inner solvers
    accept it like a ``StencilOperator``; they run on a one-block engine of
    the decomposition's geometry, bit-identical to the reference's CSR
    ``spmv`` of the extracted ``SparseMatrix``."""

    def __init__(self, grid_shape, owned: Box, overlap: int, padded: Box, mask: np.ndarray, ext: np.ndarray):
        self.grid_shape = tuple(int(v) for v in grid_shape)
        self.owned = owned
        self.overlap = int(overlap)
        self.padded = padded
        self.mask = mask  # region mask over the padded box, (z, y, x)
        self.ext = ext

    @property
    def num_rows(self) -> int:
        return int(self.ext.shape[0])

    num_cols = num_rows

    @property
    def shape(self) -> tuple:
        return (self.num_rows, self.num_rows)

    @property
    def nnz(self) -> int:
        m = self.mask
        n = int(m.sum())
        for ax in range(3):
            sl_a = [slice(None)] * 3
            sl_b = [slice(None)] * 3
            sl_a[ax] = slice(1, None)
            sl_b[ax] = slice(None, -1)
            n += 2 * int((m[tuple(sl_a)] & m[tuple(sl_b)]).sum())
        return n

    def __eq__(self, other) -> bool:
        return (isinstance(other, BlockOperator) and self.grid_shape == other.grid_shape
                and self.owned == other.owned and self.overlap == other.overlap)

    def __hash__(self):
        return hash((self.grid_shape, self.owned, self.overlap))

    def __repr__(self) -> str:
        return (f"BlockOperator(grid={self.grid_shape}, owned={self.owned.lo}..{self.owned.hi}, "
                f"overlap={self.overlap}, n={self.num_rows})")


def block_system(problem: LinearProblem, decomp: BlockDecomposition, block_id: int):
    """(a_ii, coupling) of one block (problems.py:362-406).

    ``a_ii`` is the principal submatrix on the extended region (a
    ``BlockOperator``); ``coupling`` lists every (local_row, global_col,
    coefficient) linking the region to an outside column, by local row and
    ascending column — the reference's order and values (-1.0)."""
    if not 0 <= block_id < decomp.num_blocks:
        raise ValueError(f"block_id {block_id} out of range")
    nx, ny, nz = problem.grid.shape
    pad = decomp.padded_box(block_id)
    mask = decomp.region_mask(block_id)
    ext = decomp.extended_indices(block_id)
    k, j, i = np.meshgrid(*(np.arange(pad.lo[d], pad.hi[d]) for d in (2, 1, 0)), indexing="ij")
    local = np.full(mask.shape, -1, dtype=np.int64)
    local[mask] = np.arange(int(mask.sum()))
    rows, cols = [], []
    # ascending global column order within a row: z-1, y-1, x-1, x+1, y+1, z+1
    for di, dj, dk in ((0, 0, -1), (0, -1, 0), (-1, 0, 0), (1, 0, 0), (0, 1, 0), (0, 0, 1)):
        ni, nj, nk = i + di, j + dj, k + dk
        in_grid = (ni >= 0) & (nj >= 0) & (nk >= 0) & (ni < nx) & (nj < ny) & (nk < nz)
        li, lj, lk = ni - pad.lo[0], nj - pad.lo[1], nk - pad.lo[2]
        in_pad = (li >= 0) & (lj >= 0) & (lk >= 0) & (li < mask.shape[2]) & (lj < mask.shape[1]) & \
            (lk < mask.shape[0])
        in_region = np.zeros(mask.shape, dtype=bool)
        in_region[in_pad] = mask[lk[in_pad], lj[in_pad], li[in_pad]]
        sel = mask & in_grid & ~in_region
        rows.append(local[sel])
        cols.append((ni + nx * (nj + ny * nk))[sel])
    rows = np.concatenate(rows)
    cols = np.concatenate(cols)
    order = np.lexsort((cols, rows))
    coupling = [(int(r), int(c), -1.0) for r, c in zip(rows[order], cols[order])]
    op = BlockOperator(problem.grid.shape, decomp.owned[block_id], decomp.overlap, pad, mask, ext)
    return op, coupling
