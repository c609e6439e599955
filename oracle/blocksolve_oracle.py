"""CPU oracle for the block-Jacobi / Krylov 7-point stencil path.

TEST INFRASTRUCTURE ONLY.  This module is the *checker*: it restates, in
plain numpy, the algorithm of the reference package ``blocksolve``
(``/root/reference/pkg/src/blocksolve``) for the hot path this repository
accelerates.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import it.
The product path (``paper_2009_12638_b200``) never imports or calls it.

Pinning: ``tests/test_oracle_golden.py`` checks every function here against
golden vectors produced by running the unmodified reference in the build
container (``tests/golden/make_golden.py``) and against the reference's own
known-answer tests (restated).  Citations are ``file:line`` into
``/root/reference/pkg/src/blocksolve``.

Arithmetic notes (the parity contract):

* CSR SpMV (``linalg.py:178-194``) is ``np.add.reduceat`` over the per-row
  products.  numpy 2.x evaluates a segment as ``t_first + seq(t_rest)``
  (pairwise summation degenerates to a left-to-right loop below 8 terms);
  ``stencil_apply`` reproduces that association matrix-free.
* Dot products go through ``@`` (BLAS) exactly as the reference does, so the
  oracle's CG/GMRES iterates are bit-identical to the reference's on the same
  machine; the GPU uses fixed-order tree reductions and is compared within
  tolerance (iteration counts must match).
* The block-residual combiner uses Python's built-in ``sum`` (Neumaier
  compensated on CPython >= 3.12), as ``comm.py:442-445`` does.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Callable

import numpy as np

# --------------------------------------------------------------------------
# problem definition  (problems.py:37-175)
# --------------------------------------------------------------------------

FACES = ("x_lo", "x_hi", "y_lo", "y_hi", "z_lo", "z_hi")
# order in which Dirichlet face values are accumulated into the rhs
# (problems.py:143-167: z_lo, y_lo, x_lo, [diag], x_hi, y_hi, z_hi)
RHS_FACE_ORDER = ("z_lo", "y_lo", "x_lo", "x_hi", "y_hi", "z_hi")


def _face_values(spec, a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Evaluate a face spec (constant or callable (u, v)) on index grids."""
    if callable(spec):
        out = np.empty(a.shape)
        for idx in np.ndindex(a.shape):
            out[idx] = float(spec(int(a[idx]), int(b[idx])))
        return out
    return np.full(a.shape, float(spec))


def dirichlet_rhs(nx: int, ny: int, nz: int, faces: dict | None = None) -> np.ndarray:
    """Boundary-folded rhs of ``build_laplace_3d`` (problems.py:136-167).

    Each point starts at 0.0 and receives ``+= value`` for every global face
    it touches, in the order z_lo, y_lo, x_lo, x_hi, y_hi, z_hi.  Returned
    flat in x-fastest order (problems.py:110-111).
    """
    faces = dict(faces or {})
    rhs = np.zeros((nz, ny, nx))
    for face in RHS_FACE_ORDER:
        spec = faces.get(face, 0.0)
        if face == "z_lo":
            jj, ii = np.meshgrid(np.arange(ny), np.arange(nx), indexing="ij")
            rhs[0, :, :] += _face_values(spec, ii, jj)
        elif face == "z_hi":
            jj, ii = np.meshgrid(np.arange(ny), np.arange(nx), indexing="ij")
            rhs[nz - 1, :, :] += _face_values(spec, ii, jj)
        elif face == "y_lo":
            kk, ii = np.meshgrid(np.arange(nz), np.arange(nx), indexing="ij")
            rhs[:, 0, :] += _face_values(spec, ii, kk)
        elif face == "y_hi":
            kk, ii = np.meshgrid(np.arange(nz), np.arange(nx), indexing="ij")
            rhs[:, ny - 1, :] += _face_values(spec, ii, kk)
        elif face == "x_lo":
            kk, jj = np.meshgrid(np.arange(nz), np.arange(ny), indexing="ij")
            rhs[:, :, 0] += _face_values(spec, jj, kk)
        elif face == "x_hi":
            kk, jj = np.meshgrid(np.arange(nz), np.arange(ny), indexing="ij")
            rhs[:, :, nx - 1] += _face_values(spec, jj, kk)
    return rhs.ravel()


@dataclass
class CSR:
    """CSR matrix with strictly increasing columns per row (linalg.py:56-69)."""

    num_rows: int
    num_cols: int
    row_offsets: np.ndarray
    col_indices: np.ndarray
    values: np.ndarray

    def to_dense(self) -> np.ndarray:
        a = np.zeros((self.num_rows, self.num_cols))
        rows = np.repeat(np.arange(self.num_rows), np.diff(self.row_offsets))
        a[rows, self.col_indices] = self.values
        return a


def laplace_csr(nx: int, ny: int, nz: int) -> CSR:
    """The 7-point operator of ``build_laplace_3d`` (problems.py:123-175).

    Diagonal 6, -1 for every interior neighbor, entries per row in ascending
    column order z-1, y-1, x-1, diag, x+1, y+1, z+1.  Vectorised restatement
    of the reference's Python triple loop.
    """
    n = nx * ny * nz
    p = np.arange(n, dtype=np.int64)
    i = p % nx
    j = (p // nx) % ny
    k = p // (nx * ny)
    offs = (-nx * ny, -nx, -1, 0, 1, nx, nx * ny)
    valid = (k > 0, j > 0, i > 0, np.ones(n, bool), i < nx - 1, j < ny - 1, k < nz - 1)
    vals = (-1.0, -1.0, -1.0, 6.0, -1.0, -1.0, -1.0)
    cols = np.stack([p + o for o in offs], axis=1)
    ok = np.stack(valid, axis=1)
    v = np.broadcast_to(np.asarray(vals), (n, 7))
    counts = ok.sum(axis=1)
    offsets = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=offsets[1:])
    return CSR(n, n, offsets, cols[ok].astype(np.int64), np.ascontiguousarray(v[ok]))


def csr_spmv(a: CSR, x: np.ndarray) -> np.ndarray:
    """y = A x exactly as ``linalg.spmv`` evaluates it (linalg.py:178-194)."""
    x = np.asarray(x, dtype=np.float64)
    if x.ndim != 1 or x.shape[0] != a.num_cols:
        raise ValueError("dimension mismatch")
    out = np.zeros(a.num_rows)
    if a.values.shape[0] == 0:
        return out
    prod = a.values * x[a.col_indices]
    starts = a.row_offsets[:-1]
    nonempty = a.row_offsets[1:] > starts
    out[nonempty] = np.add.reduceat(prod, starts[nonempty])
    return out


def csr_diagonal(a: CSR) -> np.ndarray:
    """Stored diagonal entries, 0 where absent (linalg.py:134-142)."""
    d = np.zeros(min(a.num_rows, a.num_cols))
    rows = np.repeat(np.arange(a.num_rows), np.diff(a.row_offsets))
    hit = (rows == a.col_indices) & (rows < d.shape[0])
    d[rows[hit]] = a.values[hit]
    return d


def csr_without_diagonal(a: CSR) -> CSR:
    """Copy with the diagonal entries dropped, order kept (linalg.py:144-159)."""
    rows = np.repeat(np.arange(a.num_rows, dtype=np.int64), np.diff(a.row_offsets))
    keep = rows != a.col_indices
    counts = np.bincount(rows[keep], minlength=a.num_rows)
    offsets = np.zeros(a.num_rows + 1, dtype=np.int64)
    np.cumsum(counts, out=offsets[1:])
    return CSR(a.num_rows, a.num_cols, offsets, a.col_indices[keep].copy(), a.values[keep].copy())


class ThreadedCSR:
    """Row-partitioned ``csr_spmv`` on a thread pool (numpy releases the GIL in
    its gather, multiply and reduceat loops).  Rows are independent, so the
    result is bit-identical to ``csr_spmv``; used only as the host-CPU baseline
    with every core busy."""

    def __init__(self, a: CSR, threads: int):
        from concurrent.futures import ThreadPoolExecutor

        self.a = a
        self.threads = max(1, int(threads))
        self.pool = ThreadPoolExecutor(self.threads)
        bounds = np.linspace(0, a.num_rows, self.threads + 1).astype(np.int64)
        self.parts = []
        for r0, r1 in zip(bounds[:-1], bounds[1:]):
            e0, e1 = a.row_offsets[r0], a.row_offsets[r1]
            offs = a.row_offsets[r0:r1 + 1] - e0
            self.parts.append((int(r0), int(r1), a.col_indices[e0:e1], a.values[e0:e1], offs))

    def _chunk(self, part, x, out):
        r0, r1, cols, vals, offs = part
        if cols.shape[0] == 0:
            return
        prod = vals * x[cols]
        starts = offs[:-1]
        nonempty = offs[1:] > starts
        seg = out[r0:r1]
        seg[nonempty] = np.add.reduceat(prod, starts[nonempty])

    def __call__(self, x):
        out = np.zeros(self.a.num_rows)
        list(self.pool.map(lambda p: self._chunk(p, x, out), self.parts))
        return out


# --------------------------------------------------------------------------
# matrix-free restatement of the same SpMV on a (possibly non-box) region
# --------------------------------------------------------------------------


def _shift(a: np.ndarray, axis: int, step: int, fill) -> np.ndarray:
    """out[idx] = a[idx + step along axis] (fill outside)."""
    out = np.full_like(a, fill)
    src = [slice(None)] * 3
    dst = [slice(None)] * 3
    if step < 0:
        dst[axis] = slice(-step, None)
        src[axis] = slice(None, step)
    else:
        dst[axis] = slice(None, -step)
        src[axis] = slice(step, None)
    out[tuple(dst)] = a[tuple(src)]
    return out


def stencil_apply(u3: np.ndarray, region: np.ndarray | None = None) -> np.ndarray:
    """Principal-submatrix SpMV of the 7-point operator on ``region``.

    ``u3`` has shape (nz, ny, nx); ``region`` is a boolean mask of the rows
    and columns kept (default: the whole box, i.e. the global operator with
    zero Dirichlet data).  Reproduces ``csr_spmv`` bit for bit: the present
    terms t = [-u(z-1), -u(y-1), -u(x-1), 6u, -u(x+1), -u(y+1), -u(z+1)] are
    combined as ``t_first + (((t_a + t_b) + ...) + t_last)`` (numpy
    ``reduceat`` semantics); absent terms are exact zeros
    inside the left-to-right chain, which leaves every partial sum unchanged.
    Rows outside the region are returned as 0.
    """
    if region is None:
        region = np.ones(u3.shape, dtype=bool)
    u = np.where(region, u3, 0.0)
    zm = _shift(u, 0, -1, 0.0)
    ym = _shift(u, 1, -1, 0.0)
    xm = _shift(u, 2, -1, 0.0)
    xp = _shift(u, 2, 1, 0.0)
    yp = _shift(u, 1, 1, 0.0)
    zp = _shift(u, 0, 1, 0.0)
    pz = _shift(region, 0, -1, False)
    py = _shift(region, 1, -1, False)
    px = _shift(region, 2, -1, False)
    t = [-zm, -ym, -xm, 6.0 * u, -xp, -yp, -zp]

    def chain(first: int) -> np.ndarray:
        s = t[first]
        for q in range(first + 1, 7):
            s = s + t[q]
        return s

    y = np.where(
        pz,
        t[0] + chain(1),
        np.where(py, t[1] + chain(2), np.where(px, t[2] + chain(3), t[3] + chain(4))),
    )
    return np.where(region, y, 0.0)


def stencil_apply_box(u3: np.ndarray) -> np.ndarray:
    """``stencil_apply(u3)`` on a whole box, bit for bit, in a few in-place
    passes (the full-size fixtures at 512^3 need it to be fast).

    Every row with its z-1 neighbour present evaluates ``t0 + chain(1)``
    where ``chain(1) = ((((t1 + t2) + t3) + t4) + t5) + t6`` (absent terms are
    exact signed zeros, which leave a partial sum unchanged, so they are
    simply skipped); ``t0 + s`` is formed as ``s - u(z-1)`` (IEEE addition
    commutes, and ``a - b`` is ``a + (-b)``).  Plane 0 (no z-1 neighbour)
    takes the general ``stencil_apply`` on its two-plane slice.
    """
    u = np.asarray(u3, dtype=np.float64)
    nz = u.shape[0]
    s = np.empty_like(u)
    s[:, 0, :] = -0.0
    np.negative(u[:, :-1, :], out=s[:, 1:, :])  # t1 = -u(y-1)
    s[:, :, 1:] -= u[:, :, :-1]  # + t2
    s += 6.0 * u  # + t3
    s[:, :, :-1] -= u[:, :, 1:]  # + t4
    s[:, :-1, :] -= u[:, 1:, :]  # + t5
    s[:-1] -= u[1:]  # + t6
    s[1:] -= u[:-1]  # t0 + chain(1)
    s[0] = stencil_apply(u[:min(2, nz)])[0]
    return s


def outer_solve_slabs(shape, b: np.ndarray, nslabs: int, max_iterations: int, tolerance: float,
                      basis: str = "initial", sweeps: int = 1, pool=None, on_sweep=None):
    """Synchronous block Jacobi on z-slabs with overlap 0 and inner CG, matrix
    free — the same algorithm as ``outer_solve_sync`` (multisplit.py:544-707,
    paper residual mode) for ``block_grid=(1, 1, nslabs)``, for grids whose
    global CSR does not fit (configs 3/4 at 512^3).

    * block system A_ii = the slab's principal submatrix = ``stencil_apply_box``
      of the slab (problems.py:362-406); its coupling has one -1 per face row;
    * rhs = b - C halo (multisplit.py:333-338): a face row's coupling sum is
      ``-h`` (one term), so rhs = b - (-h);
    * payload = the neighbour's boundary plane (merge with m = 1, 341-369);
    * local residual r = (b - A_ii x) - C owner_halo on the slab rows, num =
      ||r||, den = ||b_owned|| else ||b|| else 1 (372-396); estimate =
      sqrt(sum(local^2)) in block order (comm.py:442-445).

    Runs exactly ``sweeps`` sweeps (no termination test) and returns one
    record per sweep: per-block iteration counts, local residuals, estimate
    and the iterates.  ``pool`` (a ``multiprocessing`` pool) solves the
    blocks of a sweep in parallel — they are independent in sync mode.
    """
    nx, ny, nz = shape
    b3 = np.asarray(b, dtype=np.float64).reshape(nz, ny, nx)
    ranges = split_ranges(nz, nslabs)
    bnorm = float(np.linalg.norm(b3.ravel()))
    dens = []
    for z0, z1 in ranges:
        d = float(np.linalg.norm(b3[z0:z1].ravel()))
        dens.append(d if d != 0.0 else (bnorm if bnorm != 0.0 else 1.0))
    xs = [np.zeros((z1 - z0, ny, nx)) for z0, z1 in ranges]
    halo_lo = [None] + [np.zeros((ny, nx)) for _ in range(nslabs - 1)]
    halo_hi = [np.zeros((ny, nx)) for _ in range(nslabs - 1)] + [None]
    records = []
    for k in range(sweeps):
        jobs = []
        for blk, (z0, z1) in enumerate(ranges):
            rhs = b3[z0:z1].copy()
            if halo_lo[blk] is not None:
                rhs[0] -= -halo_lo[blk]
            if halo_hi[blk] is not None:
                rhs[-1] -= -halo_hi[blk]
            jobs.append((rhs, xs[blk], max_iterations, tolerance, basis))
        outs = pool.map(_slab_cg, jobs) if pool is not None else [_slab_cg(j) for j in jobs]
        its = []
        for blk, (x_new, it) in enumerate(outs):
            xs[blk] = x_new
            its.append(it)
        for blk in range(nslabs):  # payloads of sweep k (multisplit.py:341-369, m = 1)
            if blk > 0:
                halo_lo[blk] = xs[blk - 1][-1].copy()
            if blk < nslabs - 1:
                halo_hi[blk] = xs[blk + 1][0].copy()
        locals_ = []
        for blk, (z0, z1) in enumerate(ranges):
            r = b3[z0:z1] - stencil_apply_box(xs[blk])
            if halo_lo[blk] is not None:
                r[0] -= -halo_lo[blk]
            if halo_hi[blk] is not None:
                r[-1] -= -halo_hi[blk]
            locals_.append(float(np.linalg.norm(r.ravel())) / dens[blk])
        estimate = math.sqrt(float(sum(locals_[w] ** 2 for w in range(nslabs))))
        rec = {"k": k, "its": its, "locals": locals_, "estimate": estimate, "x": xs}
        records.append(rec)
        if on_sweep is not None:
            on_sweep(rec)
    return records


class _Frame:
    """A block's working box for the matrix-free overlap sweep: its owned box
    grown by overlap + 1 on every side (region, halo and beyond), with the
    grid, region, owned, halo and shared masks over it, in (z, y, x) order."""

    def __init__(self, shape, box, overlap: int):
        nx, ny, nz = shape
        (x0, y0, z0), (x1, y1, z1) = box
        g = overlap + 1
        self.lo = (x0 - g, y0 - g, z0 - g)
        self.hi = (x1 + g, y1 + g, z1 + g)
        k, j, i = np.meshgrid(np.arange(self.lo[2], self.hi[2]), np.arange(self.lo[1], self.hi[1]),
                              np.arange(self.lo[0], self.hi[0]), indexing="ij")
        self.grid = (i >= 0) & (i < nx) & (j >= 0) & (j < ny) & (k >= 0) & (k < nz)
        d = (np.maximum(0, np.maximum(x0 - i, i - (x1 - 1))) + np.maximum(0, np.maximum(y0 - j, j - (y1 - 1)))
             + np.maximum(0, np.maximum(z0 - k, k - (z1 - 1))))
        self.region = self.grid & (d <= overlap)
        self.owned = self.grid & (d == 0)
        self.shared = self.region & ~self.owned
        # halo: in-grid cells outside the region next to it (the coupling columns)
        near = np.zeros_like(self.region)
        for axis in range(3):
            near |= _shift(self.region, axis, -1, False) | _shift(self.region, axis, 1, False)
        self.halo = self.grid & ~self.region & near
        self.shape = self.region.shape

    def overlap_slices(self, other: "_Frame"):
        """(slices into self, slices into other) of the two frames' intersection."""
        lo = [max(self.lo[d], other.lo[d]) for d in range(3)]
        hi = [min(self.hi[d], other.hi[d]) for d in range(3)]
        if any(lo[d] >= hi[d] for d in range(3)):
            return None
        mine = tuple(slice(lo[d] - self.lo[d], hi[d] - self.lo[d]) for d in (2, 1, 0))
        theirs = tuple(slice(lo[d] - other.lo[d], hi[d] - other.lo[d]) for d in (2, 1, 0))
        return mine, theirs

    def take(self, glob3: np.ndarray) -> np.ndarray:
        """A global (nz, ny, nx) array over the frame, 0 outside the grid."""
        nz, ny, nx = glob3.shape
        out = np.zeros(self.shape)
        lo = [max(0, self.lo[d]) for d in range(3)]
        hi = [min((nx, ny, nz)[d], self.hi[d]) for d in range(3)]
        out[tuple(slice(lo[d] - self.lo[d], hi[d] - self.lo[d]) for d in (2, 1, 0))] = \
            glob3[lo[2]:hi[2], lo[1]:hi[1], lo[0]:hi[0]]
        return out


def coupling_apply(h3: np.ndarray, region: np.ndarray, grid: np.ndarray) -> np.ndarray:
    """C h matrix-free: for each region row, the couplings to in-grid
    neighbours outside the region, -h(c), in ascending column order
    (z-1, y-1, x-1, x+1, y+1, z+1) combined as ``t_first + seq(t_rest)``
    (the reduceat rule of linalg.py:188-193 on the coupling CSR,
    multisplit.py:219-228); rows without couplings are 0."""
    outside = grid & ~region
    steps = ((0, -1), (1, -1), (2, -1), (2, 1), (1, 1), (0, 1))
    t = [-_shift(np.where(outside, h3, 0.0), ax, st, 0.0) for ax, st in steps]
    pres = [_shift(outside, ax, st, False) for ax, st in steps]
    y = np.zeros_like(h3)
    for lead in range(5, -1, -1):  # the first present term leads, absent later terms are exact zeros
        s = t[lead]
        if lead < 5:
            rest = t[lead + 1]
            for q in range(lead + 2, 6):
                rest = rest + t[q]
            s = s + rest
        y = np.where(pres[lead], s, y)
    return np.where(region, y, 0.0)


def outer_solve_boxes(shape, b: np.ndarray, block_grid, overlap: int, inner: dict, sweeps: int,
                      pool=None, on_sweep=None):
    """Synchronous two-stage sweep with overlapping box blocks, matrix free —
    ``outer_solve_sync`` (multisplit.py:544-707, paper mode) for grids whose
    global CSR does not fit (config 5 at 512^3 / 1024^3).

    Per block, over its frame (``_Frame``): A_ii = ``stencil_apply`` on the
    region; rhs = b - C halo (``coupling_apply``, multisplit.py:333-338);
    merge (341-369): halo(c) = (0 + sum of the neighbours' sweep-k values at c,
    ascending block order) / cover(c), shared(s) = (own + neighbours') /
    cover(s), owner copies for the residual; local residual (372-396) on the
    owned rows with shared values replaced by their owners'.  Inner solves
    see the region's points in ascending global order (the reference's
    extended ordering).  Runs ``sweeps`` sweeps; one record per sweep."""
    nx, ny, nz = shape
    b3 = np.asarray(b, dtype=np.float64).reshape(nz, ny, nx)
    bnorm = float(np.linalg.norm(b3.ravel()))
    boxes = owned_boxes(shape, block_grid)
    frames = [_Frame(shape, box, overlap) for box in boxes]
    nb = len(boxes)
    # cover counts over every frame; neighbours = blocks whose region meets
    # this block's region or halo (dilate(ext, 1) & ext_q, problems.py:343-349)
    cover = [np.zeros(f.shape) for f in frames]
    nbrs = [[] for _ in range(nb)]
    for p_, fp in enumerate(frames):
        for q, fq in enumerate(frames):
            sl = fp.overlap_slices(fq)
            if sl is None:
                continue
            mine, theirs = sl
            cover[p_][mine] += fq.region[theirs]
            if q != p_ and np.any(fq.region[theirs] & (fp.region[mine] | fp.halo[mine])):
                nbrs[p_].append(q)
    owner_of = []  # per frame: index of the block owning each in-grid cell
    for p_, fp in enumerate(frames):
        own = np.full(fp.shape, -1)
        for q, fq in enumerate(frames):
            sl = fp.overlap_slices(fq)
            if sl is not None:
                mine, theirs = sl
                own[mine] = np.where(fq.owned[theirs], q, own[mine])
        owner_of.append(own)
    bb = [f.take(b3) for f in frames]
    dens = []
    for p_, f in enumerate(frames):
        d = float(np.linalg.norm(bb[p_][f.owned]))
        dens.append(d if d != 0.0 else (bnorm if bnorm != 0.0 else 1.0))
    xs = [np.zeros(f.shape) for f in frames]
    halo = [np.zeros(f.shape) for f in frames]
    kind = inner["kind"]
    records = []
    for k in range(sweeps):
        jobs = []
        for p_, f in enumerate(frames):
            rhs = np.where(f.region, bb[p_] - coupling_apply(halo[p_], f.region, f.grid), 0.0)
            jobs.append((kind, rhs[f.region], xs[p_][f.region], f.region, inner))
        outs = pool.map(_region_solve, jobs) if pool is not None else [_region_solve(j) for j in jobs]
        its = []
        for p_, (xr, it) in enumerate(outs):
            xs[p_] = np.zeros(frames[p_].shape)
            xs[p_][frames[p_].region] = xr
            its.append(it)
        new_x, owner_halo, owner_shared = [], [], []
        for p_, f in enumerate(frames):
            acc_h = np.zeros(f.shape)
            acc_s = np.where(f.shared, xs[p_], 0.0)
            own_vals = np.zeros(f.shape)
            for q in nbrs[p_]:
                mine, theirs = f.overlap_slices(frames[q])
                inq = frames[q].region[theirs]
                xq = xs[q][theirs]
                sub = acc_h[mine]
                acc_h[mine] = np.where(inq & f.halo[mine], sub + xq, sub)
                sub = acc_s[mine]
                acc_s[mine] = np.where(inq & f.shared[mine], sub + xq, sub)
                ov = own_vals[mine]
                own_vals[mine] = np.where(frames[q].owned[theirs] & (f.halo[mine] | f.shared[mine]), xq, ov)
            halo_new = np.where(f.halo, acc_h / np.where(f.halo, cover[p_], 1.0), 0.0)
            xn = np.where(f.shared, acc_s / np.where(f.shared, cover[p_], 1.0), xs[p_])
            new_x.append((halo_new, xn))
            owner_halo.append(np.where(f.halo, own_vals, 0.0))
            owner_shared.append(np.where(f.shared, own_vals, 0.0))
        locals_ = []
        for p_, f in enumerate(frames):
            halo[p_], xs[p_] = new_x[p_]
            xv = np.where(f.shared, owner_shared[p_], xs[p_])
            r = np.where(f.region, bb[p_] - stencil_apply(xv, f.region), 0.0)
            r = r - coupling_apply(owner_halo[p_], f.region, f.grid)
            locals_.append(float(np.linalg.norm(r[f.owned])) / dens[p_])
        estimate = math.sqrt(float(sum(locals_[w] ** 2 for w in range(nb))))
        rec = {"k": k, "its": its, "locals": locals_, "estimate": estimate,
               "owned": [xs[p_][f.owned] for p_, f in enumerate(frames)], "boxes": boxes}
        records.append(rec)
        if on_sweep is not None:
            on_sweep(rec)
    return records


def _region_solve(job):
    kind, rhs, x0, region, inner = job

    def apply(v):
        u = np.zeros(region.shape)
        u[region] = v
        return stencil_apply(u, region)[region]

    its, tol, basis = inner["max_iterations"], inner.get("tolerance", 0.0), inner.get("basis", "rhs")
    if kind == "gmres":
        restart = inner.get("restart") or its
        x, rep = gmres(apply, rhs, x0, its, tol, restart, basis)
    else:
        x, rep = cg(apply, rhs, x0, its, tol, basis)
    if rep.stop_reason == "breakdown":
        raise RuntimeError("breakdown in a block solve")
    return x, rep.iterations_used


def _slab_cg(job):
    rhs, x0, max_iterations, tolerance, basis = job
    shape = rhs.shape
    x, rep = cg(lambda v: stencil_apply_box(v.reshape(shape)).ravel(), rhs.ravel(), x0.ravel(),
                max_iterations, tolerance, basis)
    if rep.stop_reason == "breakdown":
        raise RuntimeError("breakdown in a slab solve")
    return x.reshape(shape), rep.iterations_used


def offdiag_apply(u3: np.ndarray, region: np.ndarray | None = None) -> np.ndarray:
    """(A - D) u matrix-free on ``region``: ``csr_spmv`` of
    ``csr_without_diagonal`` bit for bit.  Present terms
    [-u(z-1), -u(y-1), -u(x-1), -u(x+1), -u(y+1), -u(z+1)] as
    ``t_first + seq(t_rest)``; unlike the full row no term is always present,
    so the upper neighbours can lead, and a row without neighbours is 0."""
    if region is None:
        region = np.ones(u3.shape, dtype=bool)
    u = np.where(region, u3, 0.0)
    t = [-_shift(u, 0, -1, 0.0), -_shift(u, 1, -1, 0.0), -_shift(u, 2, -1, 0.0),
         -_shift(u, 2, 1, 0.0), -_shift(u, 1, 1, 0.0), -_shift(u, 0, 1, 0.0)]
    pres = [_shift(region, 0, -1, False), _shift(region, 1, -1, False), _shift(region, 2, -1, False),
            _shift(region, 2, 1, False), _shift(region, 1, 1, False), _shift(region, 0, 1, False)]

    def chain(first: int) -> np.ndarray:
        s = t[first]
        for q in range(first + 1, 6):
            s = s + t[q]
        return s

    y = np.zeros_like(u)
    for lead in range(5, -1, -1):  # the first present term leads
        y = np.where(pres[lead], t[lead] + chain(lead + 1) if lead < 5 else t[5], y)
    return np.where(region, y, 0.0)


# --------------------------------------------------------------------------
# inner solvers  (inner_solvers.py)
# --------------------------------------------------------------------------

STAGNATION_RTOL = 1e-14  # inner_solvers.py:37


@dataclass
class Report:
    """Mirror of ``InnerSolveReport`` (inner_solvers.py:60-67)."""

    iterations_used: int
    final_relative_residual: float
    stop_reason: str
    residual_history: list = field(default_factory=list)


def _scale(b: np.ndarray) -> float:
    """inner_solvers.py:70-72."""
    bnorm = float(np.linalg.norm(b))
    return bnorm if bnorm > 0.0 else 1.0


def cg(apply: Callable, b, x0, max_iterations: int, tolerance: float = 0.0,
       basis: str = "rhs"):
    """Conjugate gradients, restating ``cg_solve`` (inner_solvers.py:102-146).

    ``basis="rhs"`` is the reference semantics (stop when ||r||/||b|| <= tol).
    ``basis="initial"`` is the r0-relative wrapper of SURVEY §8(c): the
    reference CG called with ``tol' = tol * ||b - A x0|| / ||b||``.
    """
    b = np.asarray(b, dtype=np.float64)
    x = np.array(x0, dtype=np.float64, copy=True)
    scale = _scale(b)
    r = b - apply(x)
    rel = float(np.linalg.norm(r)) / scale
    tol = tolerance if basis == "rhs" else tolerance * rel
    if rel <= tol:
        return x, Report(0, rel, "tolerance_met")
    p = r.copy()
    rr = float(r @ r)
    history = []
    it = 0
    while it < max_iterations:
        ap = apply(p)
        pap = float(p @ ap)
        if pap <= 0.0 or not np.isfinite(pap):
            return x, Report(it, rel, "breakdown", history)
        alpha = rr / pap
        x += alpha * p
        r -= alpha * ap
        it += 1
        rr_new = float(r @ r)
        rel = np.sqrt(rr_new) / scale
        history.append(rel)
        if not np.isfinite(rel):
            return x, Report(it, rel, "breakdown", history)
        if rel <= tol:
            r_true = b - apply(x)
            rel_true = float(np.linalg.norm(r_true)) / scale
            if rel_true <= tol:
                history[-1] = rel_true
                return x, Report(it, rel_true, "tolerance_met", history)
            r = r_true
            rr_new = float(r @ r)
            rel = np.sqrt(rr_new) / scale
            history[-1] = rel
        beta = rr_new / rr
        p = r + beta * p
        rr = rr_new
    return x, Report(it, rel, "max_iterations", history)


def jacobi(apply: Callable, apply_off: Callable, diag: np.ndarray, b, x0, max_iterations: int,
           tolerance: float = 0.0, basis: str = "rhs"):
    """Point Jacobi, restating ``jacobi_solve`` (inner_solvers.py:75-99):
    x <- (b - (A - D) x) / d, relative residual after every update, stop at
    the first iterate meeting ``tolerance`` (or non-finite: breakdown).
    ``basis="initial"`` scales the tolerance by the initial relative residual
    (the wrapper of SURVEY §8(c))."""
    b = np.asarray(b, dtype=np.float64)
    x = np.array(x0, dtype=np.float64, copy=True)
    d = np.asarray(diag, dtype=np.float64)
    if np.any(d == 0.0):
        return x, Report(0, np.inf, "breakdown")
    scale = _scale(b)
    rel = float(np.linalg.norm(b - apply(x))) / scale
    tol = tolerance if basis == "rhs" else tolerance * rel
    if rel <= tol:
        return x, Report(0, rel, "tolerance_met")
    history = []
    for it in range(1, max_iterations + 1):
        x = (b - apply_off(x)) / d
        rel = float(np.linalg.norm(b - apply(x))) / scale
        history.append(rel)
        if not np.isfinite(rel):
            return x, Report(it, rel, "breakdown", history)
        if rel <= tol:
            return x, Report(it, rel, "tolerance_met", history)
    return x, Report(max_iterations, rel, "max_iterations", history)


def _back_substitute(u: np.ndarray, rhs: np.ndarray) -> np.ndarray:
    """inner_solvers.py:246-251."""
    y = np.zeros_like(rhs)
    for i in range(rhs.shape[0] - 1, -1, -1):
        y[i] = (rhs[i] - u[i, i + 1:] @ y[i + 1:]) / u[i, i]
    return y


def gmres(apply: Callable, b, x0, max_iterations: int, tolerance: float = 0.0,
          restart: int | None = None, basis: str = "rhs"):
    """Restarted GMRES(m) with MGS Arnoldi + Givens, restating
    ``gmres_solve`` (inner_solvers.py:149-243)."""
    b = np.asarray(b, dtype=np.float64)
    x = np.array(x0, dtype=np.float64, copy=True)
    n = b.shape[0]
    m = min(restart if restart is not None else 30, n)
    scale = _scale(b)
    tol = tolerance
    if basis == "initial":
        tol = tolerance * (float(np.linalg.norm(b - apply(x))) / scale)
    history: list = []
    total = 0
    v = np.zeros((m + 1, n))
    h = np.zeros((m + 1, m))
    cs = np.zeros(m)
    sn = np.zeros(m)
    g = np.zeros(m + 1)

    def form(j: int) -> np.ndarray:
        y = _back_substitute(h[: j + 1, : j + 1], g[: j + 1])
        return x + v[: j + 1].T @ y

    while True:
        r = b - apply(x)
        beta = float(np.linalg.norm(r))
        rel = beta / scale
        if total == 0 and rel <= tol:
            return x, Report(0, rel, "tolerance_met")
        cycle_start = rel
        h[:] = 0.0
        g[:] = 0.0
        g[0] = beta
        v[0] = r / beta
        for j in range(m):
            w = apply(v[j])
            for i in range(j + 1):
                h[i, j] = float(v[i] @ w)
                w -= h[i, j] * v[i]
            wnorm = float(np.linalg.norm(w))
            h[j + 1, j] = wnorm
            happy = wnorm <= 1e-14 * max(float(np.linalg.norm(h[: j + 2, j])), 1e-300)
            for i in range(j):
                hij = cs[i] * h[i, j] + sn[i] * h[i + 1, j]
                h[i + 1, j] = -sn[i] * h[i, j] + cs[i] * h[i + 1, j]
                h[i, j] = hij
            denom = float(np.hypot(h[j, j], h[j + 1, j]))
            cs[j] = h[j, j] / denom
            sn[j] = h[j + 1, j] / denom
            h[j, j] = denom
            h[j + 1, j] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            total += 1
            rel = abs(g[j + 1]) / scale
            history.append(rel)
            if happy:
                x = form(j)
                rel = float(np.linalg.norm(b - apply(x))) / scale
                history[-1] = rel
                return x, Report(total, rel, "tolerance_met", history)
            if rel <= tol or total >= max_iterations:
                x = form(j)
                rel_true = float(np.linalg.norm(b - apply(x))) / scale
                if rel_true <= tol:
                    history[-1] = rel_true
                    return x, Report(total, rel_true, "tolerance_met", history)
                if total >= max_iterations:
                    return x, Report(total, rel_true, "max_iterations", history)
                break
            if j == m - 1:
                x = form(j)
                break
            v[j + 1] = w / wnorm
        rel_true = float(np.linalg.norm(b - apply(x))) / scale
        if not np.isfinite(rel_true):
            return x, Report(total, rel_true, "breakdown", history)
        if cycle_start - rel_true < STAGNATION_RTOL * cycle_start:
            return x, Report(total, rel_true, "breakdown", history)


# --------------------------------------------------------------------------
# decomposition  (problems.py:178-359)
# --------------------------------------------------------------------------


def split_ranges(n: int, g: int) -> list:
    """problems.py:216-225: near-equal ranges, remainder to the low blocks."""
    base, rem = divmod(n, g)
    out, start = [], 0
    for b in range(g):
        w = base + (1 if b < rem else 0)
        out.append((start, start + w))
        start += w
    return out


def owned_boxes(shape, block_grid) -> list:
    """Owned boxes in block-id order bx fastest (problems.py:322-328).

    Each box is ((x0, y0, z0), (x1, y1, z1)), half open.
    """
    nx, ny, nz = shape
    gx, gy, gz = block_grid
    rx, ry, rz = split_ranges(nx, gx), split_ranges(ny, gy), split_ranges(nz, gz)
    boxes = []
    for bz in range(gz):
        for by in range(gy):
            for bx in range(gx):
                boxes.append(((rx[bx][0], ry[by][0], rz[bz][0]),
                              (rx[bx][1], ry[by][1], rz[bz][1])))
    return boxes


def dilate(mask: np.ndarray, steps: int) -> np.ndarray:
    """7-point dilation of a (nz, ny, nx) mask (problems.py:178-190)."""
    out = mask.copy()
    for _ in range(steps):
        grown = out.copy()
        for axis in range(3):
            grown |= _shift(out, axis, -1, False)
            grown |= _shift(out, axis, 1, False)
        out = grown
    return out


def region_mask(shape, box, overlap: int) -> np.ndarray:
    """Extended region = owned box dilated ``overlap`` times, computed
    analytically as the L1 ball {p : dist_1(p, box) <= overlap} (equal to
    ``_dilate`` of the box mask, problems.py:330-340)."""
    nx, ny, nz = shape
    (x0, y0, z0), (x1, y1, z1) = box
    k, j, i = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    d = (np.maximum(0, np.maximum(x0 - i, i - (x1 - 1)))
         + np.maximum(0, np.maximum(y0 - j, j - (y1 - 1)))
         + np.maximum(0, np.maximum(z0 - k, k - (z1 - 1))))
    return d <= overlap


@dataclass
class Workspace:
    """Per-block geometry and payload maps (multisplit.py:122-163, 198-330)."""

    block_id: int
    ext: np.ndarray
    a_ii: CSR
    coupling: CSR
    halo_cols: np.ndarray
    b_ext: np.ndarray
    b_owned_norm: float
    b_global_norm: float
    owned_global: np.ndarray
    owned_local: np.ndarray
    shared_local: np.ndarray
    m_halo: np.ndarray
    m_shared: np.ndarray
    neighbors: list
    send_idx: dict = field(default_factory=dict)
    recv_halo: dict = field(default_factory=dict)
    recv_shared: dict = field(default_factory=dict)
    owner_halo_map: dict = field(default_factory=dict)
    owner_shared_map: dict = field(default_factory=dict)
    payload_len: dict = field(default_factory=dict)


def _sub_csr(a: CSR, rows: np.ndarray, col_map: np.ndarray, keep_cols) -> tuple:
    """Rows ``rows`` of ``a`` split into (kept, dropped) column sets."""
    counts = a.row_offsets[rows + 1] - a.row_offsets[rows]
    total = int(counts.sum())
    pos = np.repeat(a.row_offsets[rows], counts) + (
        np.arange(total) - np.repeat(np.cumsum(counts) - counts, counts))
    local_rows = np.repeat(np.arange(rows.shape[0]), counts)
    cols = a.col_indices[pos]
    vals = a.values[pos]
    inside = keep_cols[cols]
    return local_rows, cols, vals, inside


def _csr_from_rows(m: int, ncols: int, rows, cols, vals) -> CSR:
    order = np.lexsort((cols, rows))
    rows, cols, vals = rows[order], cols[order], vals[order]
    off = np.zeros(m + 1, dtype=np.int64)
    np.add.at(off, rows + 1, 1)
    np.cumsum(off, out=off)
    return CSR(m, ncols, off, cols.astype(np.int64), vals.astype(np.float64))


def build_workspaces(shape, b: np.ndarray, block_grid, overlap: int,
                     a: CSR | None = None) -> tuple:
    """Restates ``decompose`` + ``build_workspaces``
    (problems.py:287-406, multisplit.py:198-330) for small grids."""
    nx, ny, nz = shape
    n = nx * ny * nz
    if a is None:
        a = laplace_csr(nx, ny, nz)
    boxes = owned_boxes(shape, block_grid)
    masks = [region_mask(shape, box, overlap) for box in boxes]
    exts = [np.nonzero(mk.ravel())[0] for mk in masks]
    cover = np.zeros(n, dtype=np.int64)
    for mk in masks:
        cover += mk.ravel()
    reach = [dilate(mk, 1) for mk in masks]
    nb = len(boxes)
    neighbors = [[] for _ in range(nb)]
    for p in range(nb):
        for q in range(p + 1, nb):
            if np.any(reach[p] & masks[q]):
                neighbors[p].append(q)
                neighbors[q].append(p)
    b_global_norm = float(np.linalg.norm(b))
    wss = []
    for blk in range(nb):
        ext = exts[blk]
        in_ext = np.zeros(n, dtype=bool)
        in_ext[ext] = True
        local_of = np.full(n, -1, dtype=np.int64)
        local_of[ext] = np.arange(ext.shape[0])
        rows, cols, vals, inside = _sub_csr(a, ext, local_of, in_ext)
        a_ii = _csr_from_rows(ext.shape[0], ext.shape[0], rows[inside],
                              local_of[cols[inside]], vals[inside])
        halo_cols = np.unique(cols[~inside])
        coupling = _csr_from_rows(ext.shape[0], halo_cols.shape[0], rows[~inside],
                                  np.searchsorted(halo_cols, cols[~inside]), vals[~inside])
        (x0, y0, z0), (x1, y1, z1) = boxes[blk]
        owned = (np.arange(x0, x1)[None, None, :]
                 + nx * (np.arange(y0, y1)[None, :, None]
                         + ny * np.arange(z0, z1)[:, None, None])).ravel()
        owned_local = np.searchsorted(ext, owned)
        mask = np.zeros(ext.shape[0], bool)
        mask[owned_local] = True
        shared_local = np.nonzero(~mask)[0]
        wss.append(Workspace(
            block_id=blk, ext=ext, a_ii=a_ii, coupling=coupling, halo_cols=halo_cols,
            b_ext=b[ext].copy(), b_owned_norm=float(np.linalg.norm(b[owned])),
            b_global_norm=b_global_norm, owned_global=owned, owned_local=owned_local,
            shared_local=shared_local, m_halo=cover[halo_cols].astype(float),
            m_shared=cover[ext[shared_local]].astype(float),
            neighbors=list(neighbors[blk])))

    def owned_by(q, pts):
        (qx0, qy0, qz0), (qx1, qy1, qz1) = boxes[q]
        i, j, k = pts % nx, (pts // nx) % ny, pts // (nx * ny)
        return (qx0 <= i) & (i < qx1) & (qy0 <= j) & (j < qy1) & (qz0 <= k) & (k < qz1)

    for blk, ws in enumerate(wss):
        shared_global = ws.ext[ws.shared_local]
        need = np.union1d(shared_global, ws.halo_cols)
        for q in ws.neighbors:
            shipped = np.intersect1d(exts[q], need, assume_unique=True)
            wss[q].send_idx[blk] = np.searchsorted(exts[q], shipped)
            ws.payload_len[q] = int(shipped.shape[0])
            own_q = owned_by(q, shipped)
            in_halo = np.isin(shipped, ws.halo_cols)
            ws.recv_halo[q] = (np.nonzero(in_halo)[0],
                               np.searchsorted(ws.halo_cols, shipped[in_halo]))
            sel = in_halo & own_q
            ws.owner_halo_map[q] = (np.nonzero(sel)[0],
                                    np.searchsorted(ws.halo_cols, shipped[sel]))
            in_sh = np.isin(shipped, shared_global)
            ws.recv_shared[q] = (np.nonzero(in_sh)[0],
                                 np.searchsorted(shared_global, shipped[in_sh]))
            sel = in_sh & own_q
            ws.owner_shared_map[q] = (np.nonzero(sel)[0],
                                      np.searchsorted(shared_global, shipped[sel]))
    return boxes, wss, neighbors, cover


# --------------------------------------------------------------------------
# outer sweep  (multisplit.py:333-426, 544-797) — synchronous replay
# --------------------------------------------------------------------------


@dataclass
class OracleTraceRow:
    outer_iteration: int
    estimated_residual: float
    true_residual: float | None
    inner_iterations: int


@dataclass
class OracleResult:
    solution: np.ndarray
    rows: list
    converged: bool
    outer_iterations: int
    final_true_residual: float
    per_block_inner: list  # [k][block] inner iterations
    snapshots: list = field(default_factory=list)


def true_relative_residual(a: CSR, b: np.ndarray, x: np.ndarray) -> float:
    """multisplit.py:404-406 -> linalg.residual_norms (linalg.py:197-205)."""
    r = b - csr_spmv(a, x)
    bnorm = float(np.linalg.norm(b))
    if bnorm == 0.0:
        raise ZeroDivisionError("relative residual undefined for a zero rhs")
    return float(np.linalg.norm(r)) / bnorm


def outer_solve_sync(shape, b: np.ndarray, block_grid, overlap: int, inner: dict,
                     tol: float = 1e-6, max_outer: int = 5000,
                     residual_check_mode: str = "paper",
                     true_residual_interval: int = 10,
                     capture_iterates: bool = False) -> OracleResult:
    """Synchronous two-stage solve (multisplit.py:544-797, replay execution).

    ``inner`` = dict(kind="jacobi"|"cg"|"gmres", max_iterations, tolerance, restart,
    basis="rhs"|"initial").  Sync exchanges deliver every neighbor's
    iteration-k payload, so the schedule is plain block Jacobi and the
    result does not depend on worker order.
    """
    nx, ny, nz = shape
    a = laplace_csr(nx, ny, nz)
    boxes, wss, neighbors, cover = build_workspaces(shape, b, block_grid, overlap, a)
    kind = inner["kind"]
    max_its = inner["max_iterations"]
    itol = inner.get("tolerance", 0.0)
    basis = inner.get("basis", "rhs")
    restart = inner.get("restart")
    if kind == "gmres" and restart is None:
        restart = max_its  # multisplit.py:532-536
    nb = len(wss)
    # per-block state (multisplit.py:151-163)
    xs = [np.zeros(ws.ext.shape[0]) for ws in wss]
    halo = [np.zeros(ws.halo_cols.shape[0]) for ws in wss]
    own_shared = [np.zeros(ws.shared_local.shape[0]) for ws in wss]
    owner_halo = [np.zeros(ws.halo_cols.shape[0]) for ws in wss]
    owner_shared = [np.zeros(ws.shared_local.shape[0]) for ws in wss]
    rows, per_block_inner, snapshots = [], [], []
    converged = False
    k = 0
    solution = np.zeros(a.num_rows)
    last_true = {}
    while True:
        its_k = []
        for blk, ws in enumerate(wss):
            rhs = ws.b_ext.copy()
            if ws.halo_cols.size:
                rhs -= csr_spmv(ws.coupling, halo[blk])
            ap = (lambda v, m=ws.a_ii: csr_spmv(m, v))
            if kind == "cg":
                x_new, rep = cg(ap, rhs, xs[blk], max_its, itol, basis)
            elif kind == "jacobi":
                off = (lambda v, m=csr_without_diagonal(ws.a_ii): csr_spmv(m, v))
                x_new, rep = jacobi(ap, off, csr_diagonal(ws.a_ii), rhs, xs[blk], max_its, itol, basis)
            else:
                x_new, rep = gmres(ap, rhs, xs[blk], max_its, itol, restart, basis)
            if rep.stop_reason == "breakdown":
                raise RuntimeError(f"breakdown in block {blk} at outer iteration {k}")
            xs[blk] = x_new
            own_shared[blk] = x_new[ws.shared_local].copy()
            its_k.append(rep.iterations_used)
        payloads = [{q: xs[blk][wss[blk].send_idx[q]] for q in wss[blk].neighbors}
                    for blk in range(nb)]
        locals_ = []
        for blk, ws in enumerate(wss):
            # merge_overlap (multisplit.py:341-369)
            if ws.halo_cols.size:
                acc = np.zeros(ws.halo_cols.shape[0])
                for q in ws.neighbors:
                    pl = payloads[q][blk]
                    sel, slots = ws.recv_halo[q]
                    if sel.size:
                        acc[slots] += pl[sel]
                    sel, slots = ws.owner_halo_map[q]
                    if sel.size:
                        owner_halo[blk][slots] = pl[sel]
                halo[blk] = acc / ws.m_halo
            if ws.shared_local.size:
                acc = own_shared[blk].copy()
                for q in ws.neighbors:
                    pl = payloads[q][blk]
                    sel, slots = ws.recv_shared[q]
                    if sel.size:
                        acc[slots] += pl[sel]
                    sel, slots = ws.owner_shared_map[q]
                    if sel.size:
                        owner_shared[blk][slots] = pl[sel]
                xs[blk][ws.shared_local] = acc / ws.m_shared
            # local_relative_residual (multisplit.py:372-396)
            if ws.shared_local.size:
                xv = xs[blk].copy()
                xv[ws.shared_local] = owner_shared[blk]
            else:
                xv = xs[blk]
            r = ws.b_ext - csr_spmv(ws.a_ii, xv)
            if ws.halo_cols.size:
                r -= csr_spmv(ws.coupling, owner_halo[blk])
            num = float(np.linalg.norm(r[ws.owned_local]))
            den = ws.b_owned_norm or ws.b_global_norm or 1.0
            locals_.append(num / den)
        total = float(sum(locals_[w] ** 2 for w in range(nb)))  # comm.py:442-445
        estimate = math.sqrt(total)
        for ws in wss:
            solution[ws.owned_global] = xs[ws.block_id][ws.owned_local]
        want_true = residual_check_mode == "true" or k % true_residual_interval == 0
        sample = true_relative_residual(a, b, solution) if want_true else None
        if capture_iterates:
            snapshots.append((k, solution.copy()))
        rows.append(OracleTraceRow(k, estimate, sample, int(sum(its_k))))
        per_block_inner.append(its_k)
        if sample is not None:
            last_true[k] = sample
        # check_termination (multisplit.py:409-426) then the driver's
        # true-mode stop request (multisplit.py:685-686)
        if estimate < tol or k + 1 >= max_outer:
            converged = estimate < tol
            break
        if residual_check_mode == "true" and sample is not None and sample < tol:
            converged = True
            break
        k += 1
    final_true = true_relative_residual(a, b, solution)
    if rows and rows[-1].true_residual is None:
        rows[-1].true_residual = final_true
    return OracleResult(solution, rows, converged, len(rows), final_true,
                        per_block_inner, snapshots)


def seeded_rhs(n: int, seed: int = 0) -> np.ndarray:
    """SURVEY §8(d) convention: default_rng(seed).uniform(-1, 1, n), x-fastest."""
    return np.random.default_rng(seed).uniform(-1.0, 1.0, n)


# --------------------------------------------------------------------------
# spectral diagnostics  (linalg.py:234-276, multisplit.py:800-830)
# --------------------------------------------------------------------------


@dataclass
class Spectral:
    """Mirror of ``SpectralEstimate`` (linalg.py:234-240)."""

    radius: float
    iterations_used: int
    converged: bool


def power_iteration(apply_map: Callable, dim: int, tol: float = 1e-10, max_iterations: int = 5000,
                    seed: int = 0) -> Spectral:
    """Power method restating ``power_iteration`` (linalg.py:243-276)."""
    if dim < 1:
        raise ValueError("dim must be at least 1")
    if tol <= 0:
        raise ValueError("tol must be positive")
    x = 1.0 + np.random.default_rng(seed).random(dim)
    x /= np.linalg.norm(x)
    previous = np.inf
    estimate = 0.0
    for it in range(1, max_iterations + 1):
        y = np.asarray(apply_map(x), dtype=np.float64)
        estimate = float(np.linalg.norm(y))
        if estimate == 0.0:
            return Spectral(0.0, it, True)
        if abs(estimate - previous) < tol:
            return Spectral(estimate, it, True)
        previous = estimate
        x = y / estimate
    return Spectral(estimate, max_iterations, False)


def iteration_operator(shape, block_grid, overlap: int):
    """The exact-inner-solve outer iteration z -> M^-1 N z on stacked extended
    vectors, restating ``iteration_operator`` (multisplit.py:800-830) with
    dense block solves (small grids only)."""
    n = shape[0] * shape[1] * shape[2]
    _, wss, _, _ = build_workspaces(shape, np.zeros(n), block_grid, overlap)
    dense = [ws.a_ii.to_dense() for ws in wss]
    offsets = np.concatenate(([0], np.cumsum([ws.ext.shape[0] for ws in wss])))

    def apply(z):
        parts = [z[offsets[i]:offsets[i + 1]] for i in range(len(wss))]
        out = np.empty_like(z)
        for i, ws in enumerate(wss):
            if ws.halo_cols.size:
                acc = np.zeros(ws.halo_cols.shape[0])
                for q in ws.neighbors:
                    payload = parts[q][wss[q].send_idx[i]]
                    sel, slots = ws.recv_halo[q]
                    if sel.size:
                        acc[slots] += payload[sel]
                rhs = -csr_spmv(ws.coupling, acc / ws.m_halo)
            else:
                rhs = np.zeros(ws.ext.shape[0])
            out[offsets[i]:offsets[i + 1]] = np.linalg.solve(dense[i], rhs)
        return out

    return apply, int(offsets[-1])
