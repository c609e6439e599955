"""Asynchronous block Jacobi on the GPU (mode="async").

Reference semantics: ``comm.py:367-418`` (non-blocking R-slot halo swap:
post if a slot is free, apply only the freshest delivered payload, keep the
old halo otherwise), ``comm.py:455-527`` (stale residual estimate) and
``comm.py:531-598`` + ``multisplit.py:608-632`` (a confirmation round — a
synchronous halo flush followed by an exact reduction — before stopping).

The reference *simulates* asynchrony with a delay model inside one Python
process.  Here it is real: every block has its own engine context and CUDA
stream, driven by its own host thread, and never waits for a neighbour.
After each inner solve a block posts its boundary planes one-sidedly into
the neighbours' mailbox rings (``bs_async_post``: payload, then a
system-scope release of the slot's sequence number); before each solve it
installs the freshest payload newer than the one it applied
(``bs_async_receive``, seqlock-validated).  Rings live in the receiver's
memory, so the same kernels work on peer-mapped NVLink memory.

The global estimate is the square root of the sum of every block's latest
published local residual squared (+inf until all blocks published once),
refreshed every ``residual_check_every`` sweeps; when it drops below ``tol``
the blocks meet in a confirmation round whose exact sum decides.
"""

from __future__ import annotations

import math
import threading
import time

import numpy as np

from . import _lib
from .engine import BlockEngine, box_halo_plan, launch_bound, torch
from .errors import SolverBreakdownError

RING_SLOTS_MAX = 8  # real hardware has no injected delays: deeper rings only hold stale planes


class _Mailbox:
    """Directed channel src -> dst, memory owned by dst."""

    def __init__(self, dst: int, ghost_dir: int, src: int, plane: int, slots: int, device):
        self.dst, self.ghost_dir, self.src = dst, ghost_dir, src
        self.post_dir = 5 - ghost_dir  # the sender's own boundary plane facing the receiver
        self.R = slots
        self.ring = torch.zeros(slots, plane, dtype=torch.float64, device=device)
        self.seqs = torch.zeros(slots, dtype=torch.int64, device=device)
        self.applied = torch.zeros(1, dtype=torch.int64, device=device)
        self.stage = torch.zeros(plane, dtype=torch.float64, device=device)
        self.torn = torch.zeros(1, dtype=torch.int32, device=device)


class _Board:
    """Host-side residual board + confirmation rendezvous (the fabric's role)."""

    def __init__(self, nb: int):
        self.nb = nb
        self.lock = threading.Lock()
        self.local_sq = [math.inf] * nb
        self.confirm_requested = False
        self.stop = False
        self.converged = False
        self.error: BaseException | None = None
        self.barrier = threading.Barrier(nb)
        self.confirm_sq = [0.0] * nb

    def estimate(self) -> float:
        with self.lock:
            total = float(sum(self.local_sq[w] for w in range(self.nb)))  # block order (comm.py:443-445)
        return math.sqrt(total) if math.isfinite(total) else math.inf


def outer_solve_async(problem, config, decomp, b_dev, dens, bnorm, dev, spec):
    """Run the asynchronous two-stage solve; returns the pieces of a SolveResult."""
    grid = problem.grid
    nx, ny, nz = grid.shape
    nb = decomp.num_blocks
    every = max(1, int(getattr(config, "residual_check_every", 1)))
    slots = max(1, min(int(config.buffer_slots), RING_SLOTS_MAX))
    engines, streams = [], []
    with torch.cuda.device(dev):
        for i in range(nb):
            eng = BlockEngine(grid.shape, [decomp.owned[i]], 0, dev, history_cap=1)
            eng.load_global("b", b_dev)
            engines.append(eng)
            streams.append(torch.cuda.Stream(dev))
        torch.cuda.synchronize(dev)
        plan = box_halo_plan(decomp.owned, decomp.block_grid)
        incoming = [[] for _ in range(nb)]
        outgoing = [[] for _ in range(nb)]
        for dst, gdir, src in plan.tolist():
            plane = engines[dst].blocks[0].ghost[gdir].numel()
            mb = _Mailbox(dst, gdir, src, plane, slots, dev)
            incoming[dst].append(mb)
            outgoing[src].append(mb)
    board = _Board(nb)
    records = [[] for _ in range(nb)]
    t0 = time.perf_counter()

    def local_residual(b: int) -> float:
        eng = engines[b]
        eng.residual()
        rep = eng.reports()[0]
        return (math.sqrt(rep.r_owned_sq) / dens[b]) ** 2

    def worker(b: int):
        eng = engines[b]
        lib = eng.lib
        try:
            with torch.cuda.device(dev), torch.cuda.stream(streams[b]):
                st = eng.stream
                estimate = math.inf
                k = 0
                while True:
                    for mb in incoming[b]:  # freshest delivered payloads (comm.py:401-416)
                        _lib.check(lib.bs_async_receive(eng.ctx, 0, mb.ghost_dir, mb.ring.data_ptr(),
                                                        mb.seqs.data_ptr(), mb.R, mb.applied.data_ptr(),
                                                        mb.stage.data_ptr(), mb.torn.data_ptr(), st))
                    begin = eng.cg_begin if spec.kind == "cg" else eng.jacobi_begin
                    begin(spec.max_iterations, spec.tolerance, config.tolerance_basis)
                    eng.run(batch=config.batch, max_launches=launch_bound(spec.max_iterations, config.batch))
                    rep = eng.reports()[0]
                    if int(rep.stop_reason) == 3:
                        raise SolverBreakdownError(b, k, f"{spec.kind} reported breakdown")
                    its = int(rep.iterations_used)
                    for mb in outgoing[b]:  # one-sided puts, never blocking (comm.py:380-400)
                        _lib.check(lib.bs_async_post(eng.ctx, 0, mb.post_dir, mb.ring.data_ptr(),
                                                     mb.seqs.data_ptr(), mb.R, 2 * k, st))
                    # seq = 2k (sweep post) or 2k+1 (confirm flush): monotonic per channel
                    applied = [(int(mb.applied.item()) - 1) // 2 for mb in incoming[b]]
                    staleness = max([k - a for a in applied if a >= 0] + [0])
                    if (k + 1) % every == 0:
                        val = local_residual(b)
                        with board.lock:
                            board.local_sq[b] = val
                        estimate = board.estimate()
                        if estimate < config.tol:
                            board.confirm_requested = True
                    if k + 1 >= config.max_outer:
                        board.stop = True
                    records[b].append((k, time.perf_counter() - t0, estimate, its, staleness))
                    if board.confirm_requested or board.stop:
                        if _confirm(b, k):
                            return
                    k += 1
        except BaseException as exc:  # propagate after join; release the others
            board.error = exc
            board.stop = True
            board.barrier.abort()

    def _confirm(b: int, k: int) -> bool:
        """Confirmation round (comm.py:542-598): flush current payloads, recompute
        the local residues on that consistent snapshot, exact sum.  Also the
        common exit point when the sweep budget is exhausted."""
        eng = engines[b]
        st = eng.stream
        try:
            board.barrier.wait()
            if board.stop and not board.confirm_requested:
                return True
            for mb in outgoing[b]:
                _lib.check(eng.lib.bs_async_post(eng.ctx, 0, mb.post_dir, mb.ring.data_ptr(), mb.seqs.data_ptr(),
                                                 mb.R, 2 * k + 1, st))
            torch.cuda.current_stream(dev).synchronize()
            board.barrier.wait()
            for mb in incoming[b]:
                _lib.check(eng.lib.bs_async_receive(eng.ctx, 0, mb.ghost_dir, mb.ring.data_ptr(), mb.seqs.data_ptr(),
                                                    mb.R, mb.applied.data_ptr(), mb.stage.data_ptr(),
                                                    mb.torn.data_ptr(), st))
            board.confirm_sq[b] = local_residual(b)
            with board.lock:
                board.local_sq[b] = board.confirm_sq[b]
            board.barrier.wait()
            total = float(sum(board.confirm_sq[w] for w in range(nb)))
            done = math.sqrt(total) < config.tol
            board.barrier.wait()
            if b == 0:
                board.confirm_requested = False
                if done:
                    board.converged = True
                    board.stop = True
            board.barrier.wait()
            return board.stop
        except threading.BrokenBarrierError:
            return True

    threads = [threading.Thread(target=worker, args=(b,), name=f"block-{b}") for b in range(nb)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if board.error is not None:
        for eng in engines:
            eng.close()
        raise board.error
    with torch.cuda.device(dev):
        sol = torch.empty(nz, ny, nx, dtype=torch.float64, device=dev)
        for eng in engines:
            eng.flush()
            eng.gather_owned(sol)
        torch.cuda.synchronize(dev)
        torn = int(sum(int(mb.torn.item()) for lst in incoming for mb in lst))
        for eng in engines:
            eng.close()
    # a lapped read (sender overwrote the slot mid-copy) kept the old halo,
    # i.e. behaved like "no fresh payload delivered"; reported, not an error
    return sol, records, board.converged, torn
