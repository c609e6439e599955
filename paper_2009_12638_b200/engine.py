"""Device-side block set: buffers in HBM + the libbsgpu.so context.

A ``BlockEngine`` owns, for every block resident on one GPU, the padded-box
vectors x, r, p0, p1, b (fp64, x-fastest), the halo planes just outside the
padded box, and a device residual-history buffer.  Tensors are torch-owned
(PyTorch is plumbing here: allocation and streams); all arithmetic runs in
the hand-written sm_100a kernels of ``csrc/bs_engine.cu``.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import DeviceError
from .problems import Box

try:  # torch is the buffer/stream plumbing; absence is a hard error on use
    import torch
except Exception:  # pragma: no cover
    torch = None


def require_cuda(device) -> "torch.device":
    if torch is None or not torch.cuda.is_available():
        raise DeviceError("the B200 engine needs a CUDA device (no CPU fallback)")
    dev = torch.device(device if device is not None else "cuda")
    if dev.type != "cuda":
        raise DeviceError(f"device must be a CUDA device, got {dev}")
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    return dev


PITCH_ALIGN = 4  # doubles; must match csrc/bs_engine.cu


def row_pitch(nx: int) -> int:
    return (nx + PITCH_ALIGN - 1) // PITCH_ALIGN * PITCH_ALIGN


@dataclass
class BlockBuffers:
    """Padded-box vectors of one block, x-fastest with a row pitch."""

    owned: Box
    padded: Box
    pitch: int
    x: "torch.Tensor"
    r: "torch.Tensor"
    p0: "torch.Tensor"
    p1: "torch.Tensor"
    b: "torch.Tensor"
    ghost: list
    history: "torch.Tensor"

    @property
    def dims(self) -> tuple:
        return tuple(self.padded.hi[d] - self.padded.lo[d] for d in range(3))

    def view3(self, t: "torch.Tensor") -> "torch.Tensor":
        """(nz, ny, nx) view of a pitched padded-box vector (non-contiguous)."""
        nx, ny, nz = self.dims
        return t.view(nz, ny, self.pitch)[:, :, :nx]

    def put(self, name: str, flat: "torch.Tensor") -> None:
        """Store an unpitched x-fastest padded-box vector into ``name``."""
        nx, ny, nz = self.dims
        self.view3(getattr(self, name)).copy_(flat.reshape(nz, ny, nx))

    def take(self, name: str) -> "torch.Tensor":
        """Unpitched contiguous copy of ``name``."""
        return self.view3(getattr(self, name)).contiguous().reshape(-1)

    def zeros_pitched(self) -> "torch.Tensor":
        nx, ny, nz = self.dims
        return torch.zeros(nz * ny * self.pitch, dtype=torch.float64, device=self.x.device)

    def owned_slices(self) -> tuple:
        lo, plo = self.owned.lo, self.padded.lo
        return tuple(slice(self.owned.lo[d] - plo[d], self.owned.hi[d] - plo[d]) for d in (2, 1, 0))


class BlockEngine:
    """All blocks of one decomposition that live on one device."""

    def __init__(self, grid_shape, owned: list, overlap: int, device=None,
                 history_cap: int = 0, z_chunk: int = 0, block_ids=None, remote=None, resolve_remote=None):
        """``remote``: indices of ``owned`` that another process owns (overlap
        > 0 only).  They become phantom descriptors — geometry plus the
        owner's snapshot buffer, peer-mapped — that the overlap merge reads;
        ``resolve_remote(engine)`` is called once the local buffers exist and
        returns {index: device pointer of that block's snapshot}."""
        self.lib = _lib.load()
        self.device = require_cuda(device)
        self.grid_shape = tuple(int(v) for v in grid_shape)
        self.overlap = int(overlap)
        self.block_ids = list(block_ids) if block_ids is not None else list(range(len(owned)))
        self.remote = set(int(i) for i in (remote or ()))
        if self.remote and self.overlap == 0:
            raise DeviceError("phantom blocks are only used by the overlap > 0 merge")
        self.blocks: list = []
        nx, ny, nz = self.grid_shape
        descs = (_lib.BlockDesc * len(owned))()
        opts = dict(dtype=torch.float64, device=self.device)
        cap = max(1, int(history_cap))
        for i, box in enumerate(owned):
            d = descs[i]
            d.global_dims[:] = [nx, ny, nz]
            d.owned_lo[:] = list(box.lo)
            d.owned_hi[:] = list(box.hi)
            d.overlap = overlap
            if i in self.remote:
                self.blocks.append(None)
                d.remote = 1
                continue
            lo = tuple(max(0, box.lo[d] - overlap) for d in range(3))
            hi = tuple(min(self.grid_shape[d], box.hi[d] + overlap) for d in range(3))
            pad = Box(lo, hi)
            px, py, pz = (hi[d] - lo[d] for d in range(3))
            pitch = row_pitch(px)
            n = pitch * py * pz
            ghosts = []
            faces = (  # dir -> (exists, plane size)
                (lo[2] > 0, px * py), (lo[1] > 0, px * pz), (lo[0] > 0, py * pz),
                (hi[0] < nx, py * pz), (hi[1] < ny, px * pz), (hi[2] < nz, px * py))
            for exists, size in faces:
                ghosts.append(torch.zeros(size, **opts) if exists else None)
            bb = BlockBuffers(
                owned=box, padded=pad, pitch=pitch, x=torch.zeros(n, **opts), r=torch.zeros(n, **opts),
                p0=torch.zeros(n, **opts), p1=torch.zeros(n, **opts), b=torch.zeros(n, **opts),
                ghost=ghosts, history=torch.zeros(cap, **opts))
            self.blocks.append(bb)
            d.x, d.r, d.p0, d.p1, d.b = (bb.x.data_ptr(), bb.r.data_ptr(), bb.p0.data_ptr(),
                                         bb.p1.data_ptr(), bb.b.data_ptr())
            for q in range(_lib.NDIR):
                d.ghost[q] = ghosts[q].data_ptr() if ghosts[q] is not None else None
            d.history = bb.history.data_ptr()
            d.history_cap = cap
        if self.remote:
            ptrs = resolve_remote(self)
            for i in self.remote:
                descs[i].r = int(ptrs[i])
        self._descs = descs
        if not z_chunk:
            z_chunk = int(os.environ.get("BS_ZCHUNK", "0"))
        ctx = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            _lib.check(self.lib.bs_ctx_create(self.device.index, len(owned), descs, int(z_chunk),
                                              ctypes.byref(ctx)))
        self.ctx = ctx
        self.nblocks = len(owned)
        for i, bb in enumerate(self.blocks):
            if bb is not None and self.lib.bs_block_pitch(ctx, i) != bb.pitch:
                raise DeviceError("row pitch mismatch between host and engine")
        self._reports = (_lib.BlockReport * self.nblocks)()

    # -- plumbing ---------------------------------------------------------
    def close(self) -> None:
        if getattr(self, "ctx", None):
            self.lib.bs_ctx_destroy(self.ctx)
            self.ctx = None

    def __del__(self):  # pragma: no cover - best effort
        try:
            self.close()
        except Exception:
            pass

    @property
    def stream(self) -> ctypes.c_void_p:
        return ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    @property
    def local_indices(self) -> list:
        return [i for i, bb in enumerate(self.blocks) if bb is not None]

    def _mask(self, active):
        if active is None and self.remote:
            active = [bb is not None for bb in self.blocks]  # phantoms are never armed
        if active is None:
            return None
        arr = (ctypes.c_int32 * self.nblocks)(*[1 if a else 0 for a in active])
        return ctypes.cast(arr, ctypes.c_void_p), arr

    @property
    def num_ctas(self) -> int:
        return self.lib.bs_ctx_num_ctas(self.ctx)

    RUN_PATHS = {-1: "none", 0: "graph", 1: "persistent", 2: "stream", 3: "launch", 4: "jacobi-graph"}

    @property
    def run_path(self) -> str:
        """How the last ``run`` drove its solves (bs_ctx_run_path)."""
        return self.RUN_PATHS.get(self.lib.bs_ctx_run_path(self.ctx), "?")

    # -- data movement ----------------------------------------------------
    def load_global(self, name: str, g3: "torch.Tensor") -> None:
        """Scatter a global (nz, ny, nx) device tensor into every block's padded box."""
        for bb in self.blocks:
            if bb is None:
                continue
            (x0, y0, z0), (x1, y1, z1) = bb.padded.lo, bb.padded.hi
            bb.view3(getattr(bb, name)).copy_(g3[z0:z1, y0:y1, x0:x1])

    def load_host(self, name: str, g3: np.ndarray) -> None:
        """Scatter a global (nz, ny, nx) host array into every block's padded box."""
        for bb in self.blocks:
            if bb is None:
                continue
            (x0, y0, z0), (x1, y1, z1) = bb.padded.lo, bb.padded.hi
            src = torch.from_numpy(np.ascontiguousarray(g3[z0:z1, y0:y1, x0:x1])).to(self.device)
            bb.view3(getattr(bb, name)).copy_(src)

    # -- halo planes across processes (distributed.py) --------------------
    @property
    def comm_device(self):
        return self.device

    def plane_len(self, block: int, direction: int) -> int:
        px, py, pz = self.blocks[block].dims
        return {0: px * py, 5: px * py, 1: px * pz, 4: px * pz}.get(direction, py * pz)

    def new_plane(self, n: int) -> "torch.Tensor":
        return torch.zeros(n, dtype=torch.float64, device=self.device)

    def ghost(self, block: int, direction: int) -> "torch.Tensor":
        return self.blocks[block].ghost[direction]

    def post_plane(self, block: int, direction: int, buf: "torch.Tensor") -> None:
        """Block's own boundary plane facing `direction` (x + pending alpha p) -> buf."""
        if not hasattr(self, "_seq1"):
            self._seq1 = torch.zeros(1, dtype=torch.int64, device=self.device)
        _lib.check(self.lib.bs_async_post(self.ctx, block, direction, buf.data_ptr(), self._seq1.data_ptr(), 1, 0,
                                          self.stream))

    def post_plane_ptr(self, block: int, direction: int, dst_ptr: int) -> None:
        """Block's boundary plane facing `direction` stored at a raw (possibly
        peer-mapped) device address."""
        if not hasattr(self, "_seq1"):
            self._seq1 = torch.zeros(1, dtype=torch.int64, device=self.device)
        _lib.check(self.lib.bs_async_post(self.ctx, block, direction, ctypes.c_void_p(dst_ptr),
                                          self._seq1.data_ptr(), 1, 0, self.stream))

    def synchronize(self) -> None:
        torch.cuda.current_stream(self.device).synchronize()

    def save_state(self, directory: str) -> None:
        """Write the outer iterate — every local block's x (pending updates
        applied) and halo planes — as raw fp64 files: all a synchronous sweep
        needs to continue (``outer_solve(resume=...)``)."""
        self.flush()
        self.synchronize()
        os.makedirs(directory, exist_ok=True)
        for i, bb in enumerate(self.blocks):
            if bb is None:
                continue
            gid = self.block_ids[i]
            bb.x.cpu().numpy().tofile(os.path.join(directory, f"x_{gid}.f64"))
            for q, g in enumerate(bb.ghost):
                if g is not None:
                    g.cpu().numpy().tofile(os.path.join(directory, f"halo_{gid}_{q}.f64"))

    def load_state(self, directory: str) -> None:
        """Restore what ``save_state`` wrote (same decomposition)."""
        def read(name, t):
            a = np.fromfile(os.path.join(directory, name), dtype=np.float64)
            if a.size != t.numel():
                raise DeviceError(f"checkpoint {name}: {a.size} values, the block holds {t.numel()}")
            t.copy_(torch.from_numpy(a))

        for i, bb in enumerate(self.blocks):
            if bb is None:
                continue
            gid = self.block_ids[i]
            read(f"x_{gid}.f64", bb.x)
            for q, g in enumerate(bb.ghost):
                if g is not None:
                    read(f"halo_{gid}_{q}.f64", g)
        self.synchronize()

    def gather_owned(self, out3: "torch.Tensor", name: str = "x") -> None:
        """Write every block's owned values of ``name`` into a global (nz, ny, nx) tensor."""
        for bb in self.blocks:
            if bb is None:
                continue
            (x0, y0, z0), (x1, y1, z1) = bb.owned.lo, bb.owned.hi
            out3[z0:z1, y0:y1, x0:x1].copy_(bb.view3(getattr(bb, name))[bb.owned_slices()])

    def zero(self, *names) -> None:
        for bb in self.blocks:
            if bb is None:
                continue
            for name in names:
                getattr(bb, name).zero_()
            if "ghost" in names:
                for g in bb.ghost:
                    if g is not None:
                        g.zero_()

    # -- engine calls -----------------------------------------------------
    def apply(self, block: int, x: "torch.Tensor", y: "torch.Tensor") -> None:
        _lib.check(self.lib.bs_stencil_apply(self.ctx, block, x.data_ptr(), y.data_ptr(), self.stream))

    def cg_begin(self, max_iterations: int, tolerance: float, basis: str = "rhs", active=None) -> None:
        m = self._mask(active)
        _lib.check(self.lib.bs_cg_begin(self.ctx, int(max_iterations), float(tolerance),
                                        _lib.BASIS[basis], m[0] if m else None, self.stream))

    def jacobi_begin(self, max_iterations: int, tolerance: float, basis: str = "rhs", active=None) -> None:
        m = self._mask(active)
        _lib.check(self.lib.bs_jacobi_begin(self.ctx, int(max_iterations), float(tolerance),
                                            _lib.BASIS[basis], m[0] if m else None, self.stream))

    def sweep_resid(self) -> None:
        _lib.check(self.lib.bs_sweep_resid(self.ctx, self.stream))

    def cancel(self, active=None) -> None:
        m = self._mask(active)
        _lib.check(self.lib.bs_cancel(self.ctx, m[0] if m else None, self.stream))

    def run(self, batch: int = 4, max_launches: int = 0) -> int:
        n = ctypes.c_int64(0)
        _lib.check(self.lib.bs_run(self.ctx, int(batch), int(max_launches), self.stream, ctypes.byref(n)))
        return n.value

    def residual(self, active=None) -> None:
        m = self._mask(active)
        _lib.check(self.lib.bs_residual(self.ctx, m[0] if m else None, self.stream))

    def flush(self) -> None:
        _lib.check(self.lib.bs_flush(self.ctx, self.stream))

    # -- GMRES(m) workspace ----------------------------------------------
    def gmres_setup(self, m: int, shared=None) -> None:
        """Allocate the GMRES(m) workspace: m Krylov vectors + the work vector.

        Per block by default.  ``shared=True`` (or automatically, when the
        per-block bases would take more than half of the free device memory)
        allocates ONE basis for all blocks; ``gmres_run`` then solves the
        blocks one after another (``bs_gmres_run_block``), which gives the
        same numbers — a block's passes only touch its own state — and is what
        lets config 5 at 1024^3 (eight 514^3 padded blocks, 31 vectors each)
        run on one GPU.  Idempotent.
        """
        live = [bb for bb in self.blocks if bb is not None]
        n_max = max(bb.x.numel() for bb in live)
        if shared is None:
            env = os.environ.get("BS_GMRES_SHARED")
            if env is not None:
                shared = env == "1"
            else:
                per_block = sum((m + 1) * bb.x.numel() * 8 for bb in live)
                free, _ = torch.cuda.mem_get_info(self.device)
                shared = len(live) > 1 and per_block > free // 2
        shared = bool(shared) and len(live) > 1
        if getattr(self, "_gm", 0) == m and getattr(self, "_gshared", False) == shared:
            return
        self._gbufs = []  # release an earlier workspace before allocating the new one
        descs = (_lib.GmresDesc * self.nblocks)()
        if shared:
            V = torch.zeros(m, n_max, dtype=torch.float64, device=self.device)
            W = torch.zeros(n_max, dtype=torch.float64, device=self.device)
            self._gbufs.append((V, W))
        for i, bb in enumerate(self.blocks):
            if bb is None:  # phantom: no workspace (the C side skips it)
                continue
            if not shared:
                n = bb.x.numel()
                V = torch.zeros(m, n, dtype=torch.float64, device=self.device)
                W = torch.zeros(n, dtype=torch.float64, device=self.device)
                self._gbufs.append((V, W))
            descs[i].V = V.data_ptr()
            descs[i].vstride = V.shape[1]
            descs[i].W = W.data_ptr()
        _lib.check(self.lib.bs_gmres_setup(self.ctx, int(m), descs))
        self._gm = m
        self._gshared = shared

    @property
    def gmres_shared(self) -> bool:
        return bool(getattr(self, "_gshared", False))

    def gmres_begin(self, max_iterations: int, tolerance: float, basis: str = "rhs", active=None) -> None:
        m = self._mask(active)
        _lib.check(self.lib.bs_gmres_begin(self.ctx, int(max_iterations), float(tolerance),
                                           _lib.BASIS[basis], m[0] if m else None, self.stream))

    def gmres_run(self, max_cycles: int = 0) -> int:
        """Run the armed GMRES solves; one block at a time with a shared basis."""
        n = ctypes.c_int64(0)
        if not self.gmres_shared:
            _lib.check(self.lib.bs_gmres_run(self.ctx, int(max_cycles), self.stream, ctypes.byref(n)))
            return n.value
        total = 0
        for b in self.local_indices:
            _lib.check(self.lib.bs_gmres_run_block(self.ctx, b, int(max_cycles), self.stream, ctypes.byref(n)))
            total += n.value
        return total

    def halo_pack(self, plan: np.ndarray) -> None:
        plan = np.ascontiguousarray(plan, dtype=np.int32)
        if plan.size == 0:
            return
        _lib.check(self.lib.bs_halo_pack(self.ctx, plan.shape[0], plan.ctypes.data_as(ctypes.c_void_p),
                                         self.stream))

    def overlap_merge(self) -> None:
        _lib.check(self.lib.bs_overlap_merge(self.ctx, self.stream))

    def overlap_snapshot(self) -> None:
        _lib.check(self.lib.bs_overlap_snapshot(self.ctx, self.stream))

    def overlap_combine(self) -> None:
        _lib.check(self.lib.bs_overlap_combine(self.ctx, self.stream))

    def owner_residual(self) -> None:
        _lib.check(self.lib.bs_owner_residual(self.ctx, self.stream))

    def reports(self) -> list:
        _lib.check(self.lib.bs_read_reports(self.ctx, self._reports, self.stream))
        # copies: the next read reuses the staging array
        return [_lib.BlockReport.from_buffer_copy(self._reports[i]) for i in range(self.nblocks)]


def launch_bound(max_iterations: int, batch: int) -> int:
    """Safety cap on sweep launches of one armed solve: every CG iteration takes
    at most two RESID/S1/S2 cycles (a failed convergence check adds one)."""
    return 3 * (2 * int(max_iterations) + 4 + int(batch))


def box_halo_plan(decomp_owned: list, block_grid: tuple) -> np.ndarray:
    """(dst, dir, src) triples of the overlap-0 face exchange for a box grid.

    Direction order = ascending column order (0 z-1, 1 y-1, 2 x-1, 3 x+1,
    4 y+1, 5 z+1); block ids are bx-fastest (problems.py:322-328).
    """
    gx, gy, gz = block_grid
    plan = []
    for bid in range(len(decomp_owned)):
        bx, by, bz = bid % gx, (bid // gx) % gy, bid // (gx * gy)
        cand = ((0, bz > 0, bid - gx * gy), (1, by > 0, bid - gx), (2, bx > 0, bid - 1),
                (3, bx < gx - 1, bid + 1), (4, by < gy - 1, bid + gx), (5, bz < gz - 1, bid + gx * gy))
        for d, ok, src in cand:
            if ok:
                plan.append((bid, d, src))
    return np.asarray(plan, dtype=np.int32).reshape(-1, 3)
