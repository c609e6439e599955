"""The persistent cooperative CG kernels and the CUDA-graph launch path are
the same computation: identical tile partials summed in the same order, so
their results must be bitwise identical — for up to four blocks (every CTA
reduces the tile partials itself after the local-decision barrier), for
many blocks (per-block last tile, last-arriver barrier), and for the
streaming kernel ``k_cg_stream`` (BS_PERSIST=3 forces it; by default it runs
whenever the tiles outnumber the co-resident CTAs)."""

import os

import numpy as np
import pytest

from oracle import blocksolve_oracle as O

pytestmark = pytest.mark.gpu

import paper_2009_12638_b200 as bs  # noqa: E402


def _with_persist(mode, fn):
    old = os.environ.get("BS_PERSIST")
    os.environ["BS_PERSIST"] = mode
    try:
        return fn()
    finally:
        if old is None:
            del os.environ["BS_PERSIST"]
        else:
            os.environ["BS_PERSIST"] = old


@pytest.mark.parametrize("mode", ["1", "3"])
def test_single_block_persistent_equals_graph(mode):
    n = 64
    b = O.seeded_rhs(n ** 3, 0)
    op = bs.StencilOperator(n, n, n)
    spec = bs.InnerSolverSpec("cg", 2000, 1e-8)
    xa, ra = _with_persist("0", lambda: bs.cg_solve(op, b, np.zeros(n ** 3), spec))
    xb, rb = _with_persist(mode, lambda: bs.cg_solve(op, b, np.zeros(n ** 3), spec))
    assert ra.iterations_used == rb.iterations_used == 231
    assert ra.residual_history == rb.residual_history
    assert np.array_equal(xa, xb)


@pytest.mark.parametrize("mode", ["1", "3"])
def test_capped_and_warm_start_persistent_equals_graph(mode):
    n = 40
    b = O.seeded_rhs(n ** 3, 3)
    x0 = np.random.default_rng(1).uniform(-1, 1, n ** 3)
    op = bs.StencilOperator(n, n, n)
    for spec in (bs.InnerSolverSpec("cg", 17, 0.0), bs.InnerSolverSpec("cg", 500, 1e-6)):
        xa, ra = _with_persist("0", lambda: bs.cg_solve(op, b, x0, spec, tolerance_basis="initial"))
        xb, rb = _with_persist(mode, lambda: bs.cg_solve(op, b, x0, spec, tolerance_basis="initial"))
        assert (ra.iterations_used, ra.stop_reason) == (rb.iterations_used, rb.stop_reason)
        assert ra.residual_history == rb.residual_history
        assert np.array_equal(xa, xb)


@pytest.mark.parametrize("mode", ["1", "3"])
@pytest.mark.parametrize("bg", [(1, 1, 2), (1, 1, 8), (2, 2, 2)])
def test_outer_sync_persistent_equals_graph(bg, mode):
    """2 blocks (central reduction) and 8 blocks (per-block last tile)."""
    n = 24
    b = O.seeded_rhs(n ** 3, 0)
    prob = bs.LinearProblem(bs.StencilOperator(n, n, n), b, bs.Grid3D(n, n, n))
    cfg = bs.OuterConfig(block_grid=bg, inner=bs.InnerSolverSpec("cg", 15, 1e-2), tol=1e-8,
                         tolerance_basis="initial", residual_check_mode="true")
    ra = _with_persist("0", lambda: bs.outer_solve(prob, cfg))
    rb = _with_persist(mode, lambda: bs.outer_solve(prob, cfg))
    assert ra.outer_iterations == rb.outer_iterations
    assert ra.inner_iterations_per_block == rb.inner_iterations_per_block
    assert [r.estimated_residual for r in ra.trace.rows] == [r.estimated_residual for r in rb.trace.rows]
    assert np.array_equal(ra.solution, rb.solution)


def test_streaming_kernel_many_tiles_equals_graph():
    """128^3 in 8 z-slabs: 512 tiles, more than the co-resident CTAs, so the
    default path is k_cg_stream (several tiles per CTA per sweep)."""
    n = 128
    b = O.seeded_rhs(n ** 3, 0)
    prob = bs.LinearProblem(bs.StencilOperator(n, n, n), b, bs.Grid3D(n, n, n))
    cfg = bs.OuterConfig(block_grid=(1, 1, 8), inner=bs.InnerSolverSpec("cg", 40, 1e-3), tol=1e-30,
                         max_outer=6, tolerance_basis="initial")
    ra = _with_persist("0", lambda: bs.outer_solve(prob, cfg))
    rb = _with_persist("1", lambda: bs.outer_solve(prob, cfg))
    assert ra.inner_iterations_per_block == rb.inner_iterations_per_block
    assert [r.estimated_residual for r in ra.trace.rows] == [r.estimated_residual for r in rb.trace.rows]
    assert np.array_equal(ra.solution, rb.solution)
