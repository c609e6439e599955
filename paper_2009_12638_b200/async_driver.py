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

Injected latency (``OuterConfig.delay``, comm.py:51-81): on top of the real
asynchrony, every halo post and every published residual carries a delivery
iteration ``k + d`` (d drawn from the seeded DelayModel; drop_free_jitter
clamps it to be non-decreasing per channel).  A receiver that has begun
sweep s only accepts payloads with delivery <= s - 1 (its exchange at the
end of sweep s - 1 in the reference's schedule), and a sender keeps the
reference's R-slot pool (``SendPool``): a slot is in flight until the
receiver has begun its delivery iteration, a post finding no free slot is
skipped (comm.py:376-400).  Each ring has one
extra slot reserved for the confirmation round's flush, which is never
delayed (comm.py:542-598).
"""

from __future__ import annotations

import math
import threading
import time

import numpy as np

from . import _lib
from .engine import BlockEngine, box_halo_plan, launch_bound, torch
from .errors import ConfigurationError, SolverBreakdownError

RING_SLOTS_MAX = 8  # without injected delays deeper rings only hold stale planes
NO_FILTER = (1 << 63) - 1  # receiver_k that accepts every published slot
# Test hook: called as SWEEP_HOOK(block, k) by a block's thread before it
# begins sweep k (e.g. to suspend one block for a while; tests only).
SWEEP_HOOK = None


class SendPool:
    """Sender-side R-slot pool of one directed channel under injected latency
    (HaloBufferPool, comm.py:94-132, and the post rule of comm.py:376-393).

    A post stamped with delivery iteration t occupies its slot until the
    receiver's last exchange iteration reaches t (then it is reclaimed); a
    post finding every slot in flight is skipped, never blocks.
    drop_free_jitter clamps delivery times to be non-decreasing (FIFO).
    Slots rotate so a just-delivered payload is not overwritten first."""

    def __init__(self, capacity: int, delay):
        self.capacity = int(capacity)
        self.delay = delay
        self.in_flight: dict = {}  # slot -> delivery iteration
        self.last_delivery = -1
        self.next_slot = 0
        self.skipped = 0

    def reclaim(self, receiver_reached: int) -> None:
        self.in_flight = {s: t for s, t in self.in_flight.items() if t > receiver_reached}

    @property
    def free_slots(self) -> int:
        return self.capacity - len(self.in_flight)

    def post(self, k: int, drawn_delay: int):
        """(slot, delivery iteration) for sender iteration k, or None (skipped)."""
        free = [s for s in range(self.capacity) if s not in self.in_flight]
        if not free:
            self.skipped += 1
            return None
        deliver_at = k + int(drawn_delay)
        if self.delay.kind == "drop_free_jitter":
            deliver_at = max(deliver_at, self.last_delivery)
        self.last_delivery = deliver_at
        slot = min(free, key=lambda s: (s - self.next_slot) % self.capacity)
        self.next_slot = (slot + 1) % self.capacity
        self.in_flight[slot] = deliver_at
        return slot, deliver_at


class _Mailbox:
    """Directed channel src -> dst, memory owned by dst.  Slots 0..R-1 carry
    sweep posts, slot R the (never delayed) confirmation flush."""

    def __init__(self, dst: int, ghost_dir: int, src: int, plane: int, slots: int, device):
        self.dst, self.ghost_dir, self.src = dst, ghost_dir, src
        self.post_dir = 5 - ghost_dir  # the sender's own boundary plane facing the receiver
        self.R = slots
        self.ring = torch.zeros(slots + 1, plane, dtype=torch.float64, device=device)
        self.seqs = torch.zeros(slots + 1, dtype=torch.int64, device=device)
        self.deliver = torch.zeros(slots + 1, dtype=torch.int64, device=device)
        self.applied = torch.zeros(1, dtype=torch.int64, device=device)
        self.stage = torch.zeros(plane, dtype=torch.float64, device=device)
        self.torn = torch.zeros(1, dtype=torch.int32, device=device)
        self.pool = None  # SendPool under injected latency
        # where the sender writes: this process's tensors, or (sender in
        # another process) the receiver's, opened through CUDA IPC
        self.ring_ptr, self.seqs_ptr, self.deliver_ptr = (self.ring.data_ptr(), self.seqs.data_ptr(),
                                                          self.deliver.data_ptr())


class _RemoteMailbox:
    """Sender-side view of a mailbox owned by a receiver in another process:
    the ring, sequence and delivery words are the receiver's device memory,
    peer-mapped (one-sided NVLink puts)."""

    def __init__(self, dst: int, ghost_dir: int, src: int, slots: int, ptrs):
        self.dst, self.ghost_dir, self.src = dst, ghost_dir, src
        self.post_dir = 5 - ghost_dir
        self.R = slots
        self.ring_ptr, self.seqs_ptr, self.deliver_ptr = ptrs
        self.pool = None


class _Rendezvous:
    """Barrier of every block of the solve: the block threads of this process
    (threading.Barrier), and across processes one gloo barrier taken by the
    thread the local barrier elects."""

    def __init__(self, n_local: int, group=None, multi: bool = False):
        # a generous timeout: a block reaches the round at most one sweep
        # after the request, but a lost peer must not hang the node
        self.local = threading.Barrier(n_local, timeout=600.0)
        self.group = group
        self.multi = multi

    def wait(self):
        if self.local.wait() == 0 and self.multi:
            try:
                torch.distributed.barrier(group=self.group)
            except Exception:
                self.local.abort()
                raise
        self.local.wait()

    def abort(self):
        self.local.abort()


class _Board:
    """Host-side residual board + confirmation rendezvous (the fabric's role).

    ``store`` holds the cross-block words: float64 local_sq[nb],
    confirm_sq[nb] and four flags (confirm requested, stop, converged,
    failed).  One process: a private array.  Several processes (one per
    GPU, same node): a POSIX shared-memory segment every rank maps, written
    one-sidedly (aligned 8-byte stores) — the board is an estimate by
    design (comm.py:455-527); the confirmation round's barrier orders it."""

    FLAGS = ("confirm_requested", "stop", "converged", "failed")

    def __init__(self, nb: int, n_local: int = None, store=None, group=None, multi: bool = False):
        self.nb = nb
        self.lock = threading.Lock()
        self.store = store if store is not None else np.zeros(2 * nb + 4)
        if store is None:
            self.local_sq[:] = math.inf
        self.progress = [0] * nb        # sweep each block has begun
        self.pub = [[] for _ in range(nb)]  # delayed model: (deliver_at, value) per publisher
        self.error: BaseException | None = None
        self.barrier = _Rendezvous(nb if n_local is None else n_local, group, multi)

    @property
    def local_sq(self):
        return self.store[:self.nb]

    @property
    def confirm_sq(self):
        return self.store[self.nb:2 * self.nb]

    def _flag(i):
        def get(self):
            return bool(self.store[2 * self.nb + i] != 0.0)

        def put(self, v):
            self.store[2 * self.nb + i] = 1.0 if v else 0.0
        return property(get, put)

    confirm_requested = _flag(0)
    stop = _flag(1)
    converged = _flag(2)
    failed = _flag(3)
    del _flag

    def estimate(self) -> float:
        with self.lock:
            total = 0.0
            for w in range(self.nb):  # block order (comm.py:443-445)
                total += float(self.local_sq[w])
        return math.sqrt(total) if math.isfinite(total) else math.inf

    def estimate_delayed(self, reader: int, k: int) -> float:
        """Reader's view under injected latency: its own latest value, and for
        every other block the freshest one whose delivery iteration <= k."""
        with self.lock:
            vals = []
            for w in range(self.nb):
                if w == reader:
                    vals.append(self.local_sq[w])
                    continue
                seen = [v for t, v in self.pub[w] if t <= k]
                vals.append(seen[-1] if seen else math.inf)
            total = float(sum(vals))
        return math.sqrt(total) if math.isfinite(total) else math.inf


def outer_solve_async(problem, config, decomp, b_dev, dens, bnorm, dev, spec, local=None, group=None,
                      distributed=False):
    """Run the asynchronous two-stage solve; returns the pieces of a SolveResult.

    ``distributed`` (one process per GPU; ``group`` a gloo group, None = the
    default one): this process drives the blocks in ``local``; mailboxes of cross-process channels live in the
    receiver's process and the sender puts into them through CUDA IPC; the
    board is a shared-memory segment and the confirmation round adds a gloo
    barrier (``group``).  Every rank returns the full solution and records."""
    grid = problem.grid
    nx, ny, nz = grid.shape
    nb = decomp.num_blocks
    local = list(range(nb)) if local is None else list(local)
    multi = bool(distributed)
    every = max(1, int(getattr(config, "residual_check_every", 1)))
    delay = config.delay
    delayed = delay.kind != "none"
    # with injected delays the reference's pool depth matters (sends are
    # skipped when R are in flight), so keep it; otherwise a short ring
    slots = max(1, int(config.buffer_slots) if delayed else min(int(config.buffer_slots), RING_SLOTS_MAX))
    rng = np.random.default_rng(delay.seed)
    rng_lock = threading.Lock()
    if multi and delayed:
        raise ConfigurationError("delay: injected latency is a single-process experiment (one GPU)")
    engines, streams = {}, {}
    opened, shm = [], None
    with torch.cuda.device(dev):
        for i in local:
            eng = BlockEngine(grid.shape, [decomp.owned[i]], 0, dev, history_cap=1)
            eng.load_global("b", b_dev)
            engines[i] = eng
            streams[i] = torch.cuda.Stream(dev)
        torch.cuda.synchronize(dev)
        plan = box_halo_plan(decomp.owned, decomp.block_grid)
        incoming = {i: [] for i in local}
        outgoing = {i: [] for i in local}
        for dst, gdir, src in plan.tolist():
            if dst not in engines:
                continue
            plane = engines[dst].blocks[0].ghost[gdir].numel()
            mb = _Mailbox(dst, gdir, src, plane, slots, dev)
            if delayed:
                mb.pool = SendPool(slots, delay)
            incoming[dst].append(mb)
            if src in engines:
                outgoing[src].append(mb)
        if multi:
            for mb in _open_remote_mailboxes(plan, incoming, engines, slots, group, opened):
                outgoing[mb.src].append(mb)
            for lst in outgoing.values():  # post order as in one process: plan order
                lst.sort(key=lambda m: (m.dst, m.ghost_dir))
            store, shm = _shared_store(nb, group)
            board = _Board(nb, len(local), store, group, multi=True)
        else:
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
                    if SWEEP_HOOK is not None:
                        SWEEP_HOOK(b, k)
                    with board.lock:
                        board.progress[b] = k
                    begin = eng.cg_begin if spec.kind == "cg" else eng.jacobi_begin
                    begin(spec.max_iterations, spec.tolerance, config.tolerance_basis)
                    eng.run(batch=config.batch, max_launches=launch_bound(spec.max_iterations, config.batch))
                    rep = eng.reports()[0]
                    if int(rep.stop_reason) == 3:
                        raise SolverBreakdownError(b, k, f"{spec.kind} reported breakdown")
                    its = int(rep.iterations_used)
                    for mb in outgoing[b]:  # one-sided puts, never blocking (comm.py:380-400)
                        _post(eng, mb, k, st)
                    # the exchange's receive half, after the solve and the posts as in the reference's
                    # loop (multisplit.py:575-586): the freshest delivered payloads (comm.py:401-416; under
                    # injected latency those due by this iteration k) land in the halo planes, so the local
                    # residual below sees them — evaluated on the halos the solve itself used it would only
                    # measure the inner solve's accuracy and request confirmation rounds far too early
                    limit = k if delayed else NO_FILTER
                    for mb in incoming[b]:
                        _lib.check(lib.bs_async_receive_at(eng.ctx, 0, mb.ghost_dir, mb.ring.data_ptr(),
                                                           mb.seqs.data_ptr(), mb.deliver.data_ptr(), mb.R + 1,
                                                           limit, mb.applied.data_ptr(), mb.stage.data_ptr(),
                                                           mb.torn.data_ptr(), st))
                    # seq = 2k (sweep post) or 2k+1 (confirm flush): monotonic per channel
                    applied = [(int(mb.applied.item()) - 1) // 2 for mb in incoming[b]]
                    staleness = max([k - a for a in applied if a >= 0] + [0])
                    if (k + 1) % every == 0:
                        val = local_residual(b)
                        with board.lock:
                            board.local_sq[b] = val
                            if delayed:
                                board.pub[b].append((k + _draw(), val))
                                _prune(board.pub[b], min(board.progress))
                        estimate = board.estimate_delayed(b, k) if delayed else board.estimate()
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
            board.failed = True
            board.barrier.abort()

    def _draw() -> int:
        with rng_lock:  # one seeded stream shared by every channel (comm.py:236)
            return delay.draw(rng)

    def _prune(entries: list, floor: int) -> None:
        """Drop publications superseded by a newer one every reader already sees."""
        while len(entries) > 1 and entries[1][0] <= floor:
            entries.pop(0)

    def _post(eng, mb, k: int, st) -> None:
        if not delayed:
            slot = k % mb.R
            _lib.check(eng.lib.bs_async_post_slot(eng.ctx, 0, mb.post_dir, mb.ring_ptr, mb.seqs_ptr,
                                                  mb.deliver_ptr, slot, 2 * k, 0, st))
            return
        with board.lock:
            reached = board.progress[mb.dst]  # the receiver's begun iteration (comm.py:383)
        mb.pool.reclaim(reached)
        got = mb.pool.post(k, _draw() if mb.pool.free_slots else 0)
        if got is None:
            return  # exhausted pool: skip, never block (comm.py:392-393)
        slot, deliver_at = got
        _lib.check(eng.lib.bs_async_post_slot(eng.ctx, 0, mb.post_dir, mb.ring_ptr, mb.seqs_ptr,
                                              mb.deliver_ptr, slot, 2 * k, deliver_at, st))

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
            for mb in outgoing[b]:  # the reserved slot R: a synchronous, undelayed flush
                _lib.check(eng.lib.bs_async_post_slot(eng.ctx, 0, mb.post_dir, mb.ring_ptr,
                                                      mb.seqs_ptr, mb.deliver_ptr, mb.R, 2 * k + 1,
                                                      0, st))
            torch.cuda.current_stream(dev).synchronize()
            board.barrier.wait()
            for mb in incoming[b]:
                _lib.check(eng.lib.bs_async_receive_at(eng.ctx, 0, mb.ghost_dir, mb.ring.data_ptr(),
                                                       mb.seqs.data_ptr(), mb.deliver.data_ptr(), mb.R + 1,
                                                       NO_FILTER, mb.applied.data_ptr(), mb.stage.data_ptr(),
                                                       mb.torn.data_ptr(), st))
            board.confirm_sq[b] = local_residual(b)
            with board.lock:
                board.local_sq[b] = board.confirm_sq[b]
                if delayed:
                    board.pub[b].append((-1, board.confirm_sq[b]))  # the flush is seen by everyone
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

    threads = [threading.Thread(target=worker, args=(b,), name=f"block-{b}") for b in local]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if board.error is not None:
        for eng in engines.values():
            eng.close()
        _close_fabric(opened, shm, multi)
        raise board.error
    with torch.cuda.device(dev):
        sol = torch.zeros(nz, ny, nx, dtype=torch.float64, device=dev)
        for eng in engines.values():
            eng.flush()
            eng.gather_owned(sol)
        torch.cuda.synchronize(dev)
        torn = int(sum(int(mb.torn.item()) for lst in incoming.values() for mb in lst))
        skipped = int(sum(mb.pool.skipped for lst in incoming.values() for mb in lst if mb.pool is not None))
        converged = board.converged
        recs = {b: records[b] for b in local}
        if multi:
            # disjoint owned boxes: the sum is exact; every rank gets everything
            cpu = torch.distributed.get_backend(group) == "gloo"
            t = sol.cpu() if cpu else sol
            torch.distributed.all_reduce(t, group=group)
            sol = t.to(dev)
            counts = torch.tensor([torn, skipped], dtype=torch.int64)
            torch.distributed.all_reduce(counts, group=group)
            torn, skipped = int(counts[0]), int(counts[1])
            parts = [None] * torch.distributed.get_world_size(group)
            torch.distributed.all_gather_object(parts, recs, group=group)
            recs = {b: r for part in parts for b, r in part.items()}
            torch.distributed.barrier(group=group)  # nobody posts into our rings any more
        for eng in engines.values():
            eng.close()
    _close_fabric(opened, shm, multi)
    # a lapped read (sender overwrote the slot mid-copy) kept the old halo,
    # i.e. behaved like "no fresh payload delivered"; reported, not an error
    return sol, [recs[b] for b in range(nb)], converged, torn, skipped


def _open_remote_mailboxes(plan, incoming, engines, slots, group, opened):
    """Export the rings this process receives on (their ring, sequence and
    delivery buffers) as CUDA IPC handles, gather every rank's, and open the
    ones this process sends into.  Returns the sender-side views."""
    import ctypes

    lib = _lib.load()
    mine = {}
    for dst, lst in incoming.items():
        for mb in lst:
            if mb.src in engines:
                continue
            hs = []
            for t in (mb.ring, mb.seqs, mb.deliver):
                handle = (ctypes.c_ubyte * 64)()
                off = ctypes.c_uint64(0)
                _lib.check(lib.bs_ipc_export(ctypes.c_void_p(t.data_ptr()), handle, ctypes.byref(off)))
                hs.append((bytes(handle), off.value))
            mine[(mb.dst, mb.ghost_dir, mb.src)] = hs
    parts = [None] * torch.distributed.get_world_size(group)
    torch.distributed.all_gather_object(parts, mine, group=group)
    table = {k: v for part in parts for k, v in part.items()}
    out = []
    for dst, gdir, src in plan.tolist():
        if src not in engines or dst in engines:
            continue
        ptrs = []
        for handle, off in table[(dst, gdir, src)]:
            ptr = ctypes.c_void_p()
            _lib.check(lib.bs_ipc_open((ctypes.c_ubyte * 64).from_buffer_copy(handle), off, ctypes.byref(ptr)))
            opened.append(ptr.value - off)
            ptrs.append(ptr.value)
        out.append(_RemoteMailbox(dst, gdir, src, slots, ptrs))
    return out


def _shared_store(nb: int, group):
    """The board's float64[2 nb + 4] in a POSIX shared-memory segment created
    by rank 0 and mapped by every rank of the node (``_Board``)."""
    from multiprocessing import shared_memory

    n = 2 * nb + 4
    rank = torch.distributed.get_rank(group)
    name = [None]
    if rank == 0:
        shm = shared_memory.SharedMemory(create=True, size=8 * n)
        name[0] = shm.name
    src = torch.distributed.get_global_rank(group, 0) if group is not None else 0
    torch.distributed.broadcast_object_list(name, src=src, group=group)
    if rank != 0:
        shm = shared_memory.SharedMemory(name=name[0])
    store = np.ndarray((n,), dtype=np.float64, buffer=shm.buf)
    if rank == 0:
        store[:] = 0.0
        store[:nb] = math.inf  # local_sq: +inf until every block published
    torch.distributed.barrier(group=group)
    return store, shm


def _close_fabric(opened, shm, multi):
    if opened:
        lib = _lib.load()
        for base in opened:
            lib.bs_ipc_close(base)
    if shm is not None:
        try:
            shm.close()
            if torch.distributed.get_rank() == 0:
                shm.unlink()
        except Exception:
            pass
