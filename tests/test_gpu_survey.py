"""Reference numbers measured by running the unmodified reference (SURVEY
Appendix B, P6/P9/P13/P14/P15), reproduced through the public API.

Sweep counts and true residuals must match; per-block inner counts can move
by one iteration late in a long solve when dot products are reassociated
(the reference itself does that, tests/test_oracle_envelope.py), so the P9
inner totals are compared within 0.05%."""

import numpy as np
import pytest

from oracle import blocksolve_oracle as O

pytestmark = pytest.mark.gpu

import paper_2009_12638_b200 as bs  # noqa: E402


def seeded(n, seed=0):
    return bs.LinearProblem(bs.StencilOperator(n, n, n), O.seeded_rhs(n ** 3, seed), bs.Grid3D(n, n, n))


def solve(prob, **kw):
    r = bs.outer_solve(prob, bs.OuterConfig(**kw))
    return r, sum(row.inner_iterations for row in r.trace.rows)


def test_p6_config2_at_128():
    x, rep = bs.cg_solve(bs.StencilOperator(128, 128, 128), O.seeded_rhs(128 ** 3, 0), np.zeros(128 ** 3),
                         bs.InnerSolverSpec("cg", 5000, 1e-8))
    assert (rep.iterations_used, rep.stop_reason) == (446, "tolerance_met")
    assert rep.final_relative_residual == pytest.approx(9.877e-9, rel=1e-3)


@pytest.mark.parametrize("mode,sweeps,inner,true", [("true", 478, 63981, 9.885e-9), ("paper", 517, 68659, 3.444e-9)])
def test_p9_config3_analogue_64(mode, sweeps, inner, true):
    r, tot = solve(seeded(64), block_grid=(1, 1, 8), inner=bs.InnerSolverSpec("cg", 100, 1e-3), tol=1e-8,
                   tolerance_basis="initial", residual_check_mode=mode)
    assert r.converged and r.outer_iterations == sweeps
    assert abs(tot - inner) <= 5e-4 * inner
    assert r.final_true_residual == pytest.approx(true, rel=1e-3)


@pytest.mark.parametrize("mode,sweeps", [("true", 260), ("paper", 280)])
def test_p13_fixed_cg20_slabs_32(mode, sweeps):
    r, tot = solve(seeded(32), block_grid=(1, 1, 8), inner=bs.InnerSolverSpec("cg", 20), tol=1e-8,
                   residual_check_mode=mode)
    assert r.converged and r.outer_iterations == sweeps and tot == 20 * 8 * sweeps


@pytest.mark.parametrize("mode,sweeps,inner,true", [("paper", 66, 15720, 5.376e-9), ("true", 64, 15240, 8.561e-9)])
def test_p14_config5_analogue_32(mode, sweeps, inner, true):
    prob = bs.build_laplace_3d(bs.Grid3D(32, 32, 32, bs.DirichletBoundary({"z_lo": 1.0})))
    r, tot = solve(prob, block_grid=(2, 2, 2), overlap=2, inner=bs.InnerSolverSpec("gmres", 30, 1e-3, 30), tol=1e-8,
                   tolerance_basis="initial", residual_check_mode=mode)
    assert r.converged and r.outer_iterations == sweeps and tot == inner
    assert r.trace.rows[0].inner_iterations == 120  # the 4 upper blocks have b = 0 (0 its)
    assert r.final_true_residual == pytest.approx(true, rel=1e-3)


@pytest.mark.parametrize("mode,sweeps", [("true", 84), ("paper", 88)])
def test_p15_stop_timing_16(mode, sweeps):
    r, _ = solve(seeded(16), block_grid=(1, 1, 4), inner=bs.InnerSolverSpec("cg", 10), tol=1e-8,
                 residual_check_mode=mode)
    assert r.converged and r.outer_iterations == sweeps


def test_degeneration_single_block_equals_plain_gmres():
    """test_acceptance.py:104-125 (a): one block + inner GMRES == plain GMRES."""
    prob = bs.build_laplace_3d(bs.Grid3D(6, 6, 6, bs.DirichletBoundary({"x_lo": 1.0, "y_hi": 0.5, "z_lo": 2.0})))
    spec = bs.InnerSolverSpec("gmres", 500, 1e-8, restart=30)
    x_plain, rep = bs.gmres_solve(prob.matrix, prob.rhs, np.zeros(216), spec)
    r = bs.outer_solve(prob, bs.OuterConfig(block_grid=(1, 1, 1), inner=spec, tol=1e-6, max_outer=10))
    assert r.outer_iterations == 1
    assert np.array_equal(r.solution, x_plain)
    assert r.trace.rows[0].inner_iterations == rep.iterations_used


def test_degeneration_point_blocks_equal_point_jacobi():
    """test_acceptance.py (b) restated for the device kinds: one-unknown blocks
    with one point-Jacobi inner sweep are point Jacobi on the global system,
    iterate for iterate (same reduceat order for the coupling sum)."""
    n = 3
    prob = bs.build_laplace_3d(bs.Grid3D(n, n, n, bs.DirichletBoundary({"z_lo": 1.0, "x_hi": 0.5})))
    r = bs.outer_solve(prob, bs.OuterConfig(block_grid=(n, n, n), inner=bs.InnerSolverSpec("jacobi", 1), tol=1e-300,
                                            max_outer=8, capture_iterates=True))
    a = O.laplace_csr(n, n, n)
    off = O.csr_without_diagonal(a)
    x = np.zeros(n ** 3)
    assert len(r.snapshots) == 8
    for _, snap in r.snapshots:
        x = (prob.rhs - O.csr_spmv(off, x)) / 6.0
        assert np.array_equal(snap, x)


@pytest.mark.parametrize("overlap,block_grid", [(2, (2, 2, 2)), (0, (1, 1, 4))])
def test_shared_gmres_basis_equals_per_block(monkeypatch, overlap, block_grid):
    """One Krylov basis shared by all blocks, solved one block at a time
    (bs_gmres_run_block: how config 5 at 1024^3 fits one GPU) gives the
    per-block-basis run's numbers bit for bit."""
    prob = bs.LinearProblem(bs.StencilOperator(24, 24, 24), O.seeded_rhs(24 ** 3, 1), bs.Grid3D(24, 24, 24))
    cfg = dict(block_grid=block_grid, overlap=overlap, inner=bs.InnerSolverSpec("gmres", 30, 1e-3, 30), tol=1e-8,
               tolerance_basis="initial", max_outer=40)
    runs = []
    for shared in ("0", "1"):
        monkeypatch.setenv("BS_GMRES_SHARED", shared)
        r = bs.outer_solve(prob, bs.OuterConfig(**cfg))
        runs.append((r, [(row.inner_iterations, row.estimated_residual) for row in r.trace.rows]))
    (a, ta), (b, tb) = runs
    assert a.outer_iterations == b.outer_iterations and ta == tb
    assert np.array_equal(a.solution, b.solution)
