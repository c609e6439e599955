"""One process per GPU: the synchronous outer sweep sharded by block.

Launch with ``torchrun`` (one rank per GPU, NCCL) and call
``outer_solve_distributed(problem, config)`` on every rank.  Blocks are
split into contiguous id ranges (z-slabs of configs 3/4: rank r holds slabs
[r*B/N, (r+1)*B/N)), so a rank exchanges at most two halo planes per sweep.

Per sweep there is exactly one exchange step and one reduction, as in the
reference (comm.py:332-365 and 422-453):

* halo planes: pairs on the same rank are packed device-side
  (``bs_halo_pack``); a plane crossing ranks is packed by ``bs_async_post``
  into a send buffer (x + pending alpha p, the reference payload) and moved
  with one batched NCCL send/recv into the receiver's halo plane;
* per-block scalars: one all-reduce of an (nblocks x 4) fp64 table in which
  each block's row is filled only by its owner — exact, so every rank sees
  the same numbers and combines them in block order exactly as
  ``comm.py:442-445``; iteration counts are therefore identical at 1/2/4/8
  GPUs (the fixed-order per-block reductions do not depend on the GPU count).

Overlap > 0 (config 5: 2x2x2 cubes with a 2-plane overlap, one per GPU):
every rank's engine holds all blocks — its own, plus *phantoms* of the others
whose only buffer is the owner's snapshot vector, opened once through CUDA
IPC.  Per sweep: flush, snapshot, host barrier, then the merge and the
owner-canonical residual read the neighbours' snapshots straight from their
GPUs' memory (NVLink loads inside the merge kernels — no packing, no staging
copy, the reference's index-list payloads are the kernels' reads), and the
scalar all-reduce is the barrier before the next inner solve overwrites them.

``engine_factory`` lets CPU tests (gloo, world_size 2) drive the same host
logic with an oracle-backed stand-in engine; production uses ``BlockEngine``
on ``cuda:LOCAL_RANK``.
"""

from __future__ import annotations

import math
import os
import time

import numpy as np

from . import _lib
from .engine import BlockEngine, box_halo_plan, require_cuda, torch
from .errors import ConfigurationError
from .multisplit import OuterConfig, ResidualTrace, SolveResult, TraceRow
from .problems import LinearProblem, decompose
from .sync_driver import run_sync


def block_range(nblocks: int, rank: int, world: int) -> list:
    """Contiguous share of block ids for `rank` (remainder to the low ranks)."""
    base, rem = divmod(nblocks, world)
    lo = rank * base + min(rank, rem)
    return list(range(lo, lo + base + (1 if rank < rem else 0)))


def rank_of_block(nblocks: int, world: int) -> list:
    owner = [0] * nblocks
    for r in range(world):
        for g in block_range(nblocks, r, world):
            owner[g] = r
    return owner


class HaloExchange:
    """Routing of the overlap-0 halo plan across ranks.

    transport "nccl": the boundary plane is packed into a send buffer and moved
    by one batched NCCL isend/irecv into the neighbour's halo plane.
    transport "p2p": every rank exports its halo planes as CUDA IPC handles
    once; each sweep the sender's pack kernel stores its boundary plane
    straight into the peer's halo plane over NVLink (one-sided put, no
    staging copy), bracketed by two host barriers (nobody reads a halo plane
    while it is overwritten; every put landed before the next residual sweep).
    """

    def __init__(self, eng, plan: np.ndarray, local_ids: list, owner: list, rank: int, group=None,
                 transport: str = "nccl"):
        if transport not in ("nccl", "p2p"):
            raise ConfigurationError(f"transport: unknown halo transport {transport!r}")
        self.eng = eng
        self.group = group
        self.rank = rank
        self.transport = transport
        loc = {g: i for i, g in enumerate(local_ids)}
        self.local_plan = np.asarray([(loc[d], dr, loc[s]) for d, dr, s in plan.tolist()
                                      if owner[d] == rank and owner[s] == rank], dtype=np.int32).reshape(-1, 3)
        self.ops = []  # global plan order: identical op order on both ends of every pair
        for d, dr, s in plan.tolist():
            if owner[d] == rank and owner[s] != rank:
                self.ops.append(("recv", owner[s], loc[d], dr, None))
            elif owner[s] == rank and owner[d] != rank:
                li = loc[s]
                ghost_len = eng.plane_len(li, 5 - dr)
                buf = eng.new_plane(ghost_len) if transport == "nccl" else None
                self.ops.append(("send", owner[d], li, 5 - dr, buf, (d, dr)))
        self.ops = [op if len(op) == 6 else op + (None,) for op in self.ops]
        self._opened = []
        if transport == "p2p":
            self._open_peer_planes(plan, owner, local_ids)

    def _open_peer_planes(self, plan, owner, local_ids):
        import ctypes

        lib = _lib.load()
        loc = {g: i for i, g in enumerate(local_ids)}
        mine = {}
        try:
            for d, dr, s in plan.tolist():
                if owner[d] == self.rank and owner[s] != self.rank:
                    handle = (ctypes.c_ubyte * 64)()
                    off = ctypes.c_uint64(0)
                    _lib.check(lib.bs_ipc_export(ctypes.c_void_p(self.eng.ghost(loc[d], dr).data_ptr()), handle,
                                                 ctypes.byref(off)))
                    mine[(d, dr)] = (bytes(handle), off.value)
        except Exception as exc:  # every rank must still reach the collective below
            mine = {"error": f"rank {self.rank}: {exc}"}
        gathered = [None] * torch.distributed.get_world_size(self.group)
        torch.distributed.all_gather_object(gathered, mine, group=self.group)
        errors = [part["error"] for part in gathered if "error" in part]
        if errors:
            raise RuntimeError("p2p halo transport: exporting halo planes failed: " + "; ".join(errors))
        table = {k: v for part in gathered for k, v in part.items()}
        ops = []
        for kind, peer, li, dr, buf, key in self.ops:
            if kind == "send":
                handle, off = table[key]
                ptr = ctypes.c_void_p()
                _lib.check(lib.bs_ipc_open((ctypes.c_ubyte * 64).from_buffer_copy(handle), off, ctypes.byref(ptr)))
                self._opened.append(ptr.value - off)
                buf = ptr.value  # the peer's halo plane itself
            ops.append((kind, peer, li, dr, buf, key))
        self.ops = ops

    def close(self) -> None:
        if self._opened:
            lib = _lib.load()
            for base in self._opened:
                lib.bs_ipc_close(base)
            self._opened = []

    def __call__(self) -> None:
        if self.local_plan.size:
            self.eng.halo_pack(self.local_plan)
        if not self.ops:
            return
        if self.transport == "p2p":
            self.eng.synchronize()
            torch.distributed.barrier(group=self.group)  # every rank is done reading its halo planes
            for kind, peer, li, dr, ptr, key in self.ops:
                if kind == "send":
                    self.eng.post_plane_ptr(li, dr, ptr)
            self.eng.synchronize()
            torch.distributed.barrier(group=self.group)  # every put has landed
            return
        for kind, peer, li, dr, buf, key in self.ops:
            if kind == "send":
                self.eng.post_plane(li, dr, buf)
        self.eng.synchronize()
        p2p = []
        for kind, peer, li, dr, buf, key in self.ops:
            if kind == "send":
                p2p.append(torch.distributed.P2POp(torch.distributed.isend, buf, peer, self.group))
            else:
                p2p.append(torch.distributed.P2POp(torch.distributed.irecv, self.eng.ghost(li, dr), peer,
                                                   self.group))
        for req in torch.distributed.batch_isend_irecv(p2p):
            req.wait()
        self.eng.synchronize()


def _auto_transport(group=None) -> str:
    """"p2p" when every rank's GPU can map every other rank's memory (NVLink /
    NVSwitch peers), else "nccl".  Decided from the gathered device list, so
    every rank picks the same transport."""
    dist = torch.distributed
    if dist.get_backend(group) == "gloo" or not torch.cuda.is_available():
        return "nccl"
    dev = torch.cuda.current_device()
    devs = [None] * dist.get_world_size(group)
    dist.all_gather_object(devs, dev, group=group)
    ok = all(a == b or torch.cuda.can_device_access_peer(a, b) for a in devs for b in devs)
    flags = [None] * len(devs)
    dist.all_gather_object(flags, bool(ok), group=group)
    return "p2p" if all(flags) else "nccl"


def _default_factory(grid_shape, owned, overlap, local_ids):
    dev = require_cuda(f"cuda:{int(os.environ.get('LOCAL_RANK', torch.cuda.current_device()))}")
    return BlockEngine(grid_shape, owned, overlap, dev, history_cap=1, block_ids=local_ids)


def outer_solve_distributed(problem: LinearProblem, config: OuterConfig, group=None,
                            engine_factory=None, transport: str = "auto", probe=None) -> SolveResult:
    """Sharded synchronous two-stage solve; every rank returns the same result
    (solution gathered on every rank).  ``transport``: "nccl", "p2p" or
    "auto" (p2p when every pair of the ranks' GPUs has peer access, else
    nccl).  ``probe``: measurement hooks (``sync_driver.run_sync``)."""
    dist = torch.distributed
    if not dist.is_initialized():
        raise ConfigurationError("distributed: torch.distributed is not initialised")
    if config.mode == "async" and (config.inner.kind not in ("cg", "jacobi") or config.overlap != 0):
        raise ConfigurationError("mode: async runs CG or Jacobi inner solves on overlap-0 decompositions")
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    grid = problem.grid
    nx, ny, nz = grid.shape
    decomp = decompose(grid, config.block_grid, config.overlap)
    nb = decomp.num_blocks
    if world > nb:
        raise ConfigurationError(f"distributed: {world} ranks for {nb} blocks")
    local_ids = block_range(nb, rank, world)
    owner = rank_of_block(nb, world)
    b_host = np.asarray(problem.rhs if not isinstance(problem.rhs, torch.Tensor) else problem.rhs.cpu().numpy(),
                        dtype=np.float64)
    b3 = b_host.reshape(nz, ny, nx)
    bnorm = float(np.linalg.norm(b_host))
    dens = []
    for box in decomp.owned:
        d = float(np.linalg.norm(b3[box.lo[2]:box.hi[2], box.lo[1]:box.hi[1], box.lo[0]:box.hi[0]].ravel()))
        dens.append(d if d != 0.0 else (bnorm if bnorm != 0.0 else 1.0))
    if config.mode == "async":
        if engine_factory is not None:
            raise ConfigurationError("distributed: async runs on the device engine")
        return _solve_async(problem, config, group, decomp, local_ids, b_host, bnorm, dens)
    if config.overlap != 0:
        if engine_factory is not None:
            raise ConfigurationError("distributed: overlap > 0 runs on the device engine")
        return _solve_overlap(config, group, grid, decomp, local_ids, owner, rank, world, b3, bnorm, dens)
    auto = transport == "auto"
    if auto:
        transport = _auto_transport(group)
    factory = engine_factory or _default_factory
    eng = factory(grid.shape, [decomp.owned[g] for g in local_ids], config.overlap, local_ids)
    eng.load_host("b", b3)
    host_comm = dist.get_backend(group) == "gloo"
    comm_dev = torch.device("cpu") if host_comm else eng.comm_device
    plan = box_halo_plan(decomp.owned, decomp.block_grid)
    if auto and transport == "p2p":
        # "auto" never fails a solve over the transport: if any rank cannot map a
        # peer's halo planes (every collective of the set-up has completed by
        # then), all ranks agree to fall back to the batched NCCL exchange
        exchange, err = None, None
        try:
            exchange = HaloExchange(eng, plan, local_ids, owner, rank, group, "p2p")
        except Exception as exc:
            err = exc
        ok = torch.tensor([0 if err is not None else 1], dtype=torch.int32, device=comm_dev)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=group)
        if int(ok.item()) == 0:
            if exchange is not None:
                exchange.close()
            if rank == 0:
                import warnings

                warnings.warn(f"p2p halo transport unavailable ({err or 'failed on another rank'}); using nccl")
            exchange = HaloExchange(eng, plan, local_ids, owner, rank, group, "nccl")
    else:
        exchange = HaloExchange(eng, plan, local_ids, owner, rank, group, transport)

    def allreduce_rows(table: np.ndarray) -> np.ndarray:
        t = torch.from_numpy(table).to(comm_dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
        return t.cpu().numpy()

    t_start = time.perf_counter()
    try:
        trace, per_block, converged, final_true = run_sync(eng, config, dens, bnorm, nb, local_ids, exchange,
                                                          allreduce_rows, t_start, probe=probe)
        eng.flush()
        sol = torch.zeros(nz, ny, nx, dtype=torch.float64, device=eng.comm_device)
        eng.gather_owned(sol)
        sol = sol.to(comm_dev)
        dist.all_reduce(sol, op=dist.ReduceOp.SUM, group=group)  # disjoint owned boxes: exact
    finally:
        exchange.close()
        eng.close()
    rows = [TraceRow(k, t, est, tr, inner, 0) for k, t, est, tr, inner in trace]
    if rows and rows[-1].true_residual is None:
        rows[-1].true_residual = final_true
    return SolveResult(solution=sol.reshape(-1).cpu().numpy(), trace=ResidualTrace(rows), converged=converged,
                       outer_iterations=len(rows), final_true_residual=final_true,
                       inner_iterations_per_block=per_block, wall_seconds=time.perf_counter() - t_start)


def _open_snapshots(eng, group, world, opened):
    """resolve_remote for the phantom engine: export every local block's
    snapshot buffer (its r) as a CUDA IPC handle, gather all ranks' handles,
    open the ones of the phantoms (once per solve)."""
    import ctypes

    lib = _lib.load()
    mine = {}
    for i in eng.local_indices:
        handle = (ctypes.c_ubyte * 64)()
        off = ctypes.c_uint64(0)
        _lib.check(lib.bs_ipc_export(ctypes.c_void_p(eng.blocks[i].r.data_ptr()), handle, ctypes.byref(off)))
        mine[i] = (bytes(handle), off.value)
    gathered = [None] * world
    torch.distributed.all_gather_object(gathered, mine, group=group)
    table = {k: v for part in gathered for k, v in part.items()}
    ptrs = {}
    for i in sorted(eng.remote):
        handle, off = table[i]
        ptr = ctypes.c_void_p()
        _lib.check(lib.bs_ipc_open((ctypes.c_ubyte * 64).from_buffer_copy(handle), off, ctypes.byref(ptr)))
        opened.append(ptr.value - off)
        ptrs[i] = ptr.value
    return ptrs


def _solve_overlap(config, group, grid, decomp, local_ids, owner, rank, world, b3, bnorm, dens):
    """Sharded sync sweep with overlap > 0 over peer-mapped snapshots (module doc)."""
    dist = torch.distributed
    nx, ny, nz = grid.shape
    nb = decomp.num_blocks
    dev = require_cuda(f"cuda:{int(os.environ.get('LOCAL_RANK', torch.cuda.current_device()))}")
    opened = []
    remote = [g for g in range(nb) if owner[g] != rank]
    with torch.cuda.device(dev):
        eng = BlockEngine(grid.shape, decomp.owned, config.overlap, dev, history_cap=1, remote=remote,
                          resolve_remote=lambda e: _open_snapshots(e, group, world, opened))
        host_comm = dist.get_backend(group) == "gloo"
        comm_dev = torch.device("cpu") if host_comm else dev

        def merge():
            eng.overlap_snapshot()
            eng.synchronize()
            dist.barrier(group=group)  # every snapshot of this sweep is complete before any read
            eng.overlap_combine()

        def allreduce_rows(table: np.ndarray) -> np.ndarray:
            t = torch.from_numpy(table).to(comm_dev)
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)  # also: nobody still reads a snapshot
            return t.cpu().numpy()

        t_start = time.perf_counter()
        try:
            eng.load_host("b", b3)
            trace, per_block, converged, final_true = run_sync(
                eng, config, dens, bnorm, nb, local_ids, lambda: None, allreduce_rows, t_start,
                merge=merge, eng_index=local_ids)
            eng.flush()
            sol = torch.zeros(nz, ny, nx, dtype=torch.float64, device=dev)
            eng.gather_owned(sol)
            sol = sol.to(comm_dev)
            dist.all_reduce(sol, op=dist.ReduceOp.SUM, group=group)  # disjoint owned boxes: exact
        finally:
            eng.synchronize()
            dist.barrier(group=group)  # no peer reads our snapshots any more
            eng.close()
            lib = _lib.load()
            for base in opened:
                lib.bs_ipc_close(base)
    rows = [TraceRow(k, t, est, tr, inner, 0) for k, t, est, tr, inner in trace]
    if rows and rows[-1].true_residual is None:
        rows[-1].true_residual = final_true
    return SolveResult(solution=sol.reshape(-1).cpu().numpy(), trace=ResidualTrace(rows), converged=converged,
                       outer_iterations=len(rows), final_true_residual=final_true,
                       inner_iterations_per_block=per_block, wall_seconds=time.perf_counter() - t_start)


def _solve_async(problem, config, group, decomp, local_ids, b_host, bnorm, dens):
    """Asynchronous block Jacobi, one process per GPU: each rank drives its
    blocks with the single-process async driver; halo posts to blocks of
    other ranks are one-sided puts into their IPC-mapped mailbox rings, the
    residual board is node-shared memory, and only the confirmation round
    synchronises (a gloo barrier) — no per-sweep barrier anywhere."""
    from .async_driver import outer_solve_async
    from .multisplit import async_result

    dist = torch.distributed
    nx, ny, nz = problem.grid.shape
    dev = require_cuda(f"cuda:{int(os.environ.get('LOCAL_RANK', torch.cuda.current_device()))}")
    host_group = group if dist.get_backend(group) == "gloo" else dist.new_group(
        ranks=dist.get_process_group_ranks(group) if group is not None else None, backend="gloo")
    t_start = time.perf_counter()
    with torch.cuda.device(dev):
        b_dev = torch.from_numpy(b_host.reshape(nz, ny, nx)).to(dev)
        pieces = outer_solve_async(problem, config, decomp, b_dev, dens, bnorm, dev, config.inner,
                                   local=local_ids, group=host_group, distributed=True)
        res = async_result(problem, b_dev, False, t_start, pieces)
    return res
