"""Multi-rank host logic on CPU: world_size 1 and 2 over gloo (127.0.0.1).

The sharded synchronous driver (``distributed.outer_solve_distributed``) runs
with the oracle-backed stand-in engine; results must be identical for 1 and
2 ranks (block routing + exact block-row reductions) and match the oracle's
own synchronous replay of the reference algorithm.
"""

import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from oracle import blocksolve_oracle as O
from paper_2009_12638_b200.distributed import block_range, rank_of_block


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_dir, case):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import paper_2009_12638_b200 as bs
    from fake_engine import FakeEngine
    from paper_2009_12638_b200.distributed import outer_solve_distributed

    torch.distributed.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                                         world_size=world)
    n, bg, its, tol = case[:4]
    b = O.seeded_rhs(n ** 3, 0)
    prob = bs.LinearProblem(bs.StencilOperator(n, n, n), b, bs.Grid3D(n, n, n))
    cfg = bs.OuterConfig(block_grid=bg, inner=bs.InnerSolverSpec("cg", its), tol=tol, max_outer=500)
    if len(case) > 4 and case[4] == "p2p_unavailable":
        # "auto" picked p2p (as it would on NVLink peers) but no rank can export its halo planes (no CUDA
        # memory here): every rank must agree on the NCCL-style exchange instead of failing or hanging
        import warnings

        import paper_2009_12638_b200.distributed as D

        D._auto_transport = lambda group=None: "p2p"
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            res = outer_solve_distributed(prob, cfg, engine_factory=FakeEngine, transport="auto")
    else:
        res = outer_solve_distributed(prob, cfg, engine_factory=FakeEngine)
    np.savez(os.path.join(out_dir, f"r{world}_{rank}.npz"), solution=res.solution,
             counts=np.asarray(res.inner_iterations_per_block),
             est=np.asarray([r.estimated_residual for r in res.trace.rows]),
             converged=res.converged, outer=res.outer_iterations)
    torch.distributed.destroy_process_group()


def test_block_ownership_is_contiguous_and_complete():
    for nb in (1, 5, 8):
        for world in range(1, nb + 1):
            ids = [g for r in range(world) for g in block_range(nb, r, world)]
            assert ids == list(range(nb))
            owner = rank_of_block(nb, world)
            assert all(owner[g] == r for r in range(world) for g in block_range(nb, r, world))


@pytest.mark.timeout(300)
def test_two_ranks_match_one_rank_and_the_oracle():
    case = (12, (1, 1, 4), 8, 1e-7)
    with tempfile.TemporaryDirectory() as tmp:
        for world in (1, 2):
            mp.spawn(_worker, args=(world, _free_port(), tmp, case), nprocs=world, join=True)
        one = np.load(os.path.join(tmp, "r1_0.npz"))
        for rank in (0, 1):
            two = np.load(os.path.join(tmp, f"r2_{rank}.npz"))
            assert int(two["outer"]) == int(one["outer"])
            assert np.array_equal(two["counts"], one["counts"])
            assert np.array_equal(two["est"], one["est"])
            assert np.array_equal(two["solution"], one["solution"])
    n, bg, its, tol = case
    ro = O.outer_solve_sync((n, n, n), O.seeded_rhs(n ** 3, 0), bg, 0, dict(kind="cg", max_iterations=its),
                            tol=tol, max_outer=500)
    assert int(one["outer"]) == ro.outer_iterations and bool(one["converged"]) == ro.converged
    assert np.array_equal(one["counts"], np.asarray(ro.per_block_inner))
    assert np.allclose(one["est"], [r.estimated_residual for r in ro.rows], rtol=1e-10)
    assert np.linalg.norm(one["solution"] - ro.solution) <= 1e-12 * np.linalg.norm(ro.solution)


@pytest.mark.timeout(300)
def test_auto_transport_falls_back_when_p2p_setup_fails():
    """transport="auto" with p2p selected but unavailable on every rank: the ranks agree (one all-reduce
    after the set-up's collectives) to use the batched send/recv exchange; results equal the one-rank run."""
    case = (12, (1, 1, 4), 8, 1e-7)
    with tempfile.TemporaryDirectory() as tmp:
        mp.spawn(_worker, args=(1, _free_port(), tmp, case), nprocs=1, join=True)
        mp.spawn(_worker, args=(2, _free_port(), tmp, case + ("p2p_unavailable",)), nprocs=2, join=True)
        one = np.load(os.path.join(tmp, "r1_0.npz"))
        for rank in (0, 1):
            two = np.load(os.path.join(tmp, f"r2_{rank}.npz"))
            assert int(two["outer"]) == int(one["outer"])
            assert np.array_equal(two["counts"], one["counts"])
            assert np.array_equal(two["est"], one["est"])
            assert np.array_equal(two["solution"], one["solution"])
