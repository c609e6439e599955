"""The synchronous outer sweep (multisplit.py:544-707, replay semantics) over a
set of engine blocks — all blocks of the problem (one GPU) or this rank's
share of them (one process per GPU, see ``distributed.py``).

Schedule of sweep k (every block at once, device-side):

  1. inner solve (fused CG or point-Jacobi sweeps, or GMRES(m) Arnoldi passes);
  2. overlap 0: halo exchange — neighbours' boundary planes (x + pending
     alpha p) land in this block's halo planes (comm.py:332-365, merge with
     m = 1), locally by ``k_halo_pack`` or across ranks by P2P; then one
     residual sweep that is at once the sweep-k local residual
     (multisplit.py:372-396), the true residual on owned rows (404-406) and
     the rhs/r0 assembly of sweep k+1 (333-338).
     overlap > 0: flush, snapshot + 1/m merge, owner-canonical residual;
  3. per-block scalars are combined across blocks (and ranks) into one array
     ordered by block id; every rank evaluates the same estimate exactly as
     comm.py:442-445 does and takes the same decision (409-426).
"""

from __future__ import annotations

import math
import time

import numpy as np

from .engine import launch_bound
from .errors import ConfigurationError, SolverBreakdownError
from .problems import region_size


def make_inner(eng, spec, config):
    """(arm, solve) callables for the configured inner solver."""
    if spec.kind == "gmres":
        # _make_inner_solver (multisplit.py:532-536): one cycle of the configured
        # length unless a restart is given; gmres_solve caps it at n (162)
        restart = spec.restart if spec.restart is not None else spec.max_iterations
        # gmres_solve caps the restart at the block's row count (inner_solvers.py:162)
        caps = sorted({min(restart, region_size(eng.grid_shape, bb.owned, eng.overlap))
                       for bb in eng.blocks if bb is not None})
        if len(caps) > 1:
            raise ConfigurationError(
                f"restart: blocks with fewer than {restart} unknowns would restart after {caps[0]} steps while "
                f"others use {caps[-1]}; the device GMRES runs one restart length per engine")
        eng.gmres_setup(caps[0])

        def arm():
            eng.gmres_begin(spec.max_iterations, spec.tolerance, config.tolerance_basis)

        def solve():
            eng.gmres_run(max_cycles=spec.max_iterations + 2)
    else:  # fused stencil-sweep solvers: CG (two sweeps per iteration) or point Jacobi (one)
        begin = eng.cg_begin if spec.kind == "cg" else eng.jacobi_begin

        def arm():
            begin(spec.max_iterations, spec.tolerance, config.tolerance_basis)

        def solve():
            eng.run(batch=config.batch, max_launches=launch_bound(spec.max_iterations, config.batch))
    return arm, solve


def run_sync(eng, config, dens, bnorm, nblocks, local_ids, exchange, allreduce_rows, t_start,
             on_sweep=None, merge=None, eng_index=None, probe=None, resume_k=None):
    """Run sweeps until the reference's termination rule fires.

    ``exchange()`` performs the overlap-0 halo exchange; ``allreduce_rows(a)``
    sums an (nblocks, 4) array whose rows only the owning rank fills (exact:
    every entry is nonzero on one rank).  ``merge()`` performs the overlap > 0
    merge (default: ``eng.overlap_merge``); ``eng_index[li]`` is the engine
    slot of ``local_ids[li]`` (default: li).  Returns (rows, per_block, converged,
    final_true) with rows = (k, time, estimate, true_or_None, inner_total).

    ``probe`` (measurement only, e.g. ``bench.py``): an object whose
    ``begin(phase, k)`` / ``end(phase, k)`` bracket the inner solve
    (phase "solve", sweep k), the halo exchange ("exchange") and the residual
    sweep with its re-arm ("resid", overlap 0) on the host
    thread that launches them, and whose ``sweep(k, its)`` is called once per
    completed sweep with the global per-block inner iteration counts (and
    ``trace(k, estimate, true_residual, inner_total)``, if it has one).

    Segmented runs (overlap > 0): a probe with ``pause(k) -> bool`` is asked
    after every sweep that decided to continue; True ends this call there
    (``probe.paused_at = k``; the outer iterate is the blocks' x and halo
    planes, ``BlockEngine.save_state``).  ``resume_k`` continues such a run:
    the engine holds the restored iterate of sweep ``resume_k`` and the next
    inner solve starts from it, exactly as the uninterrupted loop would.
    """
    spec = config.inner
    overlap = eng.overlap
    if merge is None and overlap:
        merge = eng.overlap_merge
    eng_index = list(eng_index) if eng_index is not None else list(range(len(local_ids)))
    arm, solve = make_inner(eng, spec, config)
    if probe is None:
        probe = _NoProbe()
    if hasattr(probe, "attach"):
        probe.attach(eng)
    k = 0
    if resume_k is not None:
        if not overlap:
            raise ConfigurationError("resume: segmented runs are implemented for overlapping decompositions")
        k = int(resume_k) + 1
    arm()
    probe.begin("solve", k)
    solve()  # sweep 0: rhs = b (zero halos), x0 = 0
    probe.end("solve", k)
    rows, per_block = [], []
    converged = False
    final_true = math.nan
    while True:
        if overlap == 0:
            # one device -> host read per sweep: arm() (k_arm) keeps the solve's
            # count and stop reason as last_* while it re-arms the blocks
            probe.begin("exchange", k)
            exchange()
            probe.end("exchange", k)
            probe.begin("resid", k)
            arm()
            eng.sweep_resid()
            probe.end("resid", k)
            reps = eng.reports()
            its_stop = [(r.last_iterations, r.last_stop_reason) for r in reps]
        else:
            eng.flush()
            merge()
            eng.owner_residual()
            reps = eng.reports()
            its_stop = [(r.iterations_used, r.stop_reason) for r in reps]
        table = np.zeros((nblocks, 4))
        for li, gid in enumerate(local_ids):
            e = eng_index[li]
            table[gid] = (its_stop[e][0], 1.0 if int(its_stop[e][1]) == 3 else 0.0,
                          reps[e].r_owned_sq, reps[e].rglob_owned_sq)
        table = allreduce_rows(table)
        broken = np.nonzero(table[:, 1])[0]
        if broken.size:
            raise SolverBreakdownError(int(broken[0]), k, f"{spec.kind} reported breakdown")
        its = [int(v) for v in table[:, 0]]
        per_block.append(its)
        locals_ = [math.sqrt(table[g, 2]) / dens[g] for g in range(nblocks)]
        estimate = math.sqrt(sum(v ** 2 for v in locals_))  # comm.py:442-445 order
        true_res = math.sqrt(sum(float(table[g, 3]) for g in range(nblocks))) / bnorm if bnorm else math.inf
        want_true = config.residual_check_mode == "true" or k % config.true_residual_interval == 0
        now = float(k) if config.execution == "replay" else time.perf_counter() - t_start
        rows.append((k, now, estimate, true_res if want_true else None, int(sum(its))))
        if hasattr(probe, "trace"):
            probe.trace(k, estimate, true_res, int(sum(its)))
        if on_sweep is not None:
            on_sweep(k)
        probe.sweep(k, its)
        final_true = true_res
        if estimate < config.tol or k + 1 >= config.max_outer:  # check_termination (409-426)
            converged = estimate < config.tol
            eng.cancel()
            break
        if config.residual_check_mode == "true" and true_res < config.tol:  # 685-686
            converged = True
            eng.cancel()
            break
        if overlap and hasattr(probe, "pause") and probe.pause(k):
            probe.paused_at = k
            break
        if overlap:
            arm()
        probe.begin("solve", k + 1)
        solve()
        probe.end("solve", k + 1)
        k += 1
    return rows, per_block, converged, final_true


class _NoProbe:
    def begin(self, phase, k):
        pass

    def end(self, phase, k):
        pass

    def sweep(self, k, its):
        pass
