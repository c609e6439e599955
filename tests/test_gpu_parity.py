"""GPU parity: the CUDA path vs the reference golden vectors and the oracle.

All tests call through the C ABI (ctypes) via the package's public API.
Bars (north_star): SpMV bit-identical; inner/outer iteration counts equal in
sync mode; converged solution within 1e-8 relative L2 of the reference.
"""

import math

import numpy as np
import pytest

from golden_io import arrays, meta
from oracle import blocksolve_oracle as O

pytestmark = pytest.mark.gpu

import paper_2009_12638_b200 as bs  # noqa: E402
from paper_2009_12638_b200.engine import BlockEngine  # noqa: E402
from paper_2009_12638_b200.problems import Box  # noqa: E402


def torch():
    import torch as t

    return t


# ------------------------------------------------------------------ SpMV (a1)


@pytest.mark.parametrize("shape", [(6, 5, 4), (16, 16, 16), (7, 1, 3)])
def test_spmv_bit_identical_to_reference(shape):
    A = arrays()
    key = "spmv/%dx%dx%d" % shape
    y = bs.spmv(bs.StencilOperator(*shape), A[key + "/x"])
    assert np.array_equal(y, A[key + "/y"])


def _blocksys_keys():
    return [k for k in meta() if k.startswith("blocksys/")]


@pytest.mark.parametrize("key", _blocksys_keys())
def test_block_system_spmv_bit_identical(key):
    """Principal-submatrix SpMV on box and L1-dilated regions (problems.py:362-406)."""
    t = torch()
    A, M = arrays(), meta()[key]
    shape, bg, ov = tuple(M["shape"]), tuple(M["block_grid"]), M["overlap"]
    dec = bs.decompose(bs.Grid3D(*shape), bg, ov)
    assert dec.neighbors == M["neighbors"]
    eng = BlockEngine(shape, dec.owned, ov, "cuda")
    nx, ny, _ = shape
    for b in range(dec.num_blocks):
        ext = A[f"{key}/{b}/ext"]
        assert np.array_equal(dec.extended_indices(b), ext)
        pad = dec.padded_box(b)
        px, py, pz = (pad.hi[d] - pad.lo[d] for d in range(3))
        gi, gj, gk = ext % nx, (ext // nx) % ny, ext // (nx * ny)
        loc = (gi - pad.lo[0]) + px * ((gj - pad.lo[1]) + py * (gk - pad.lo[2]))
        xp = np.full(px * py * pz, 1e300)  # garbage outside the region must be ignored
        xp[loc] = A[f"{key}/{b}/x"]
        bb = eng.blocks[b]
        xd = bb.zeros_pitched()
        bb.view3(xd).copy_(t.from_numpy(xp).cuda().reshape(pz, py, px))
        yd = bb.zeros_pitched()
        eng.apply(b, xd, yd)
        y = bb.view3(yd).contiguous().reshape(-1).cpu().numpy()[loc]
        assert np.array_equal(y, A[f"{key}/{b}/y"]), f"block {b}"
    eng.close()


def test_spmv_known_answers():
    # test_linalg.py:73-79 restated on the device operator
    y = bs.spmv(bs.StencilOperator(4, 4, 4), np.ones(64))
    assert y[bs.Grid3D(4, 4, 4).index(1, 1, 1)] == 0.0
    with pytest.raises(ValueError, match="dimension mismatch"):
        bs.spmv(bs.StencilOperator(4, 4, 4), np.ones(63))


def test_spmv_linearity_and_oracle_at_scale():
    rng = np.random.default_rng(1)
    shape = (67, 45, 33)  # ragged vs the 32x8 tiles
    n = 67 * 45 * 33
    x, z = rng.standard_normal(n), rng.standard_normal(n)
    op = bs.StencilOperator(*shape)
    left = bs.spmv(op, 0.7 * x - 1.3 * z)
    right = 0.7 * bs.spmv(op, x) - 1.3 * bs.spmv(op, z)
    assert np.linalg.norm(left - right) <= 1e-12 * np.linalg.norm(left)
    ref = O.stencil_apply(x.reshape(33, 45, 67)).ravel()
    assert np.array_equal(bs.spmv(op, x), ref)


# ------------------------------------------------------------------ CG (a2)


@pytest.mark.parametrize("key,tol", [("cg/12_seed0", 1e-8), ("cg/20_seed1", 1e-10), ("cg/32_seed0", 1e-8)])
def test_cg_matches_reference(key, tol):
    A, M = arrays(), meta()[key]
    n = int(key.split("/")[1].split("_")[0])
    seed = int(key.split("seed")[1])
    b = O.seeded_rhs(n ** 3, seed)
    x, rep = bs.cg_solve(bs.StencilOperator(n, n, n), b, np.zeros(n ** 3),
                         bs.InnerSolverSpec("cg", 10 * n, tol))
    assert rep.iterations_used == M["iterations_used"]
    assert rep.stop_reason == M["stop_reason"]
    # recurrence residuals lose relative accuracy as they shrink (dot rounding
    # differs from OpenBLAS at 1e-16 of ||r0||): compare against ||r0|| scale
    assert np.allclose(rep.residual_history, M["residual_history"], rtol=1e-9, atol=1e-13)
    ref = A[key + "/x"]
    assert np.linalg.norm(x - ref) <= 1e-10 * np.linalg.norm(ref)


def test_cg_warm_start_capped_and_initial_basis():
    A, M = arrays(), meta()
    n = 10
    prob = bs.build_laplace_3d(bs.Grid3D(n, n, n, bs.DirichletBoundary({"z_lo": 1.0})))
    x0 = A["cg/warm/x0"]
    x, rep = bs.cg_solve(prob.matrix, prob.rhs, x0, bs.InnerSolverSpec("cg", 17, 1e-3))
    assert (rep.iterations_used, rep.stop_reason) == (17, "max_iterations")
    assert np.allclose(rep.residual_history, M["cg/warm"]["residual_history"], rtol=1e-9)
    assert np.abs(x - A["cg/warm/x"]).max() <= 1e-12
    x, rep = bs.cg_solve(prob.matrix, prob.rhs, x0, bs.InnerSolverSpec("cg", 200, 1e-3),
                         tolerance_basis="initial")
    assert rep.iterations_used == M["cg/warm_initial"]["iterations_used"]
    assert rep.stop_reason == "tolerance_met"
    assert np.abs(x - A["cg/warm_initial/x"]).max() <= 1e-11


def test_cg_edge_cases():
    op = bs.StencilOperator(5, 4, 3)
    # zero rhs with a non-zero start: scale falls back to 1, converges to 0
    rng = np.random.default_rng(7)
    x, rep = bs.cg_solve(op, np.zeros(60), rng.standard_normal(60), bs.InnerSolverSpec("cg", 500, 1e-12))
    assert rep.stop_reason == "tolerance_met" and np.abs(x).max() <= 1e-10
    # exact start: zero iterations, x untouched
    b = rng.standard_normal(60)
    xs, _ = bs.cg_solve(op, b, np.zeros(60), bs.InnerSolverSpec("cg", 500, 1e-14))
    x2, rep2 = bs.cg_solve(op, b, xs, bs.InnerSolverSpec("cg", 500, 1e-3))
    assert rep2.iterations_used == 0 and np.array_equal(x2, xs)
    # 1x1x1 grid: [[6]] x = b in one iteration
    x, rep = bs.cg_solve(bs.StencilOperator(1, 1, 1), np.array([3.0]), np.zeros(1),
                         bs.InnerSolverSpec("cg", 5, 1e-12))
    assert rep.iterations_used == 1 and x[0] == 0.5
    # determinism: bitwise identical repeats
    xa, ra = bs.cg_solve(op, b, np.zeros(60), bs.InnerSolverSpec("cg", 30, 1e-9))
    xb, rb = bs.cg_solve(op, b, np.zeros(60), bs.InnerSolverSpec("cg", 30, 1e-9))
    assert np.array_equal(xa, xb) and ra.residual_history == rb.residual_history


def test_cg_config2_analogue_64_against_oracle():
    n = 64
    b = O.seeded_rhs(n ** 3, 0)
    a = O.laplace_csr(n, n, n)
    xo, ro = O.cg(lambda v: O.csr_spmv(a, v), b, np.zeros(n ** 3), 2000, 1e-8)
    x, rep = bs.cg_solve(bs.StencilOperator(n, n, n), b, np.zeros(n ** 3), bs.InnerSolverSpec("cg", 2000, 1e-8))
    assert rep.iterations_used == ro.iterations_used == 231
    assert np.allclose(rep.residual_history, ro.residual_history, rtol=1e-8)
    assert np.linalg.norm(x - xo) <= 1e-10 * np.linalg.norm(xo)


def test_cg_config2_full_256_iteration_count():
    """Config 2 at full size: 856 CG iterations, final rel 9.832311620407356e-09
    (reference run)."""
    t = torch()
    n = 256
    b = t.from_numpy(O.seeded_rhs(n ** 3, 0)).cuda()
    x, rep = bs.cg_solve(bs.StencilOperator(n, n, n), b, t.zeros_like(b), bs.InnerSolverSpec("cg", 5000, 1e-8))
    assert rep.iterations_used == 856
    assert rep.stop_reason == "tolerance_met"
    assert rep.final_relative_residual == pytest.approx(9.832311620407356e-09, rel=1e-6)
    assert rep.residual_history[:3] == pytest.approx(
        [0.4073481114578424, 0.24363013224694208, 0.17767096348143008], rel=1e-12)
    # size-independent check: the true residual of the returned iterate
    _, rel = bs.residual_norms(bs.StencilOperator(n, n, n), x, b)
    assert rel <= 1e-8


# ------------------------------------------------------------------ point Jacobi (a2')


def _jacobi_case(key):
    A = arrays()
    if key == "jacobi/10_tol":
        return (10, 10, 10), O.dirichlet_rhs(10, 10, 10, {"x_lo": 1.0, "z_hi": 0.5}), np.zeros(1000), 400, 1e-3
    if key == "jacobi/9x6x4_maxit":
        return (9, 6, 4), O.seeded_rhs(216, 2), A[key + "/x0"], 25, 0.0
    if key == "jacobi/zero_rhs":
        return (4, 4, 4), np.zeros(64), np.zeros(64), 5, 0.0
    shape = tuple(int(v) for v in key.split("/")[1].split("x"))
    n = shape[0] * shape[1] * shape[2]
    return shape, O.seeded_rhs(n, 4), np.zeros(n), 12, 0.0


@pytest.mark.parametrize("key", ["jacobi/10_tol", "jacobi/9x6x4_maxit", "jacobi/7x1x3", "jacobi/1x1x5",
                                 "jacobi/1x1x1", "jacobi/zero_rhs"])
def test_jacobi_matches_reference(key):
    """The Jacobi update is elementwise over the reduceat off-diagonal row:
    iterates are bit-identical to the reference's; residual norms use the
    device's fixed-order reduction (tolerance)."""
    A, M = arrays(), meta()[key]
    shape, b, x0, its, tol = _jacobi_case(key)
    x, rep = bs.jacobi_solve(bs.StencilOperator(*shape), b, x0, bs.InnerSolverSpec("jacobi", its, tol))
    assert rep.iterations_used == M["iterations_used"]
    assert rep.stop_reason == M["stop_reason"]
    assert np.array_equal(x, A[key + "/x"])
    assert np.allclose(rep.residual_history, M["residual_history"], rtol=1e-12, atol=1e-300)
    if M["residual_history"]:
        assert rep.final_relative_residual == pytest.approx(M["final_relative_residual"], rel=1e-12)


def test_jacobi_at_scale_bit_identical_and_basis():
    """64^3 (odd-sized tiles, many CTAs): 150 capped sweeps bit-identical to the
    oracle; the r0-relative basis stops where the oracle does."""
    n = 64
    b = O.seeded_rhs(n ** 3, 1)
    op = bs.StencilOperator(n, n, n)
    ap = lambda v: O.stencil_apply(v.reshape(n, n, n)).ravel()
    ao = lambda v: O.offdiag_apply(v.reshape(n, n, n)).ravel()
    d = np.full(n ** 3, 6.0)
    xo, ro = O.jacobi(ap, ao, d, b, np.zeros(n ** 3), 150, 0.0)
    x, rep = bs.jacobi_solve(op, b, np.zeros(n ** 3), bs.InnerSolverSpec("jacobi", 150, 0.0))
    assert (rep.iterations_used, rep.stop_reason) == (150, "max_iterations")
    assert np.array_equal(x, xo)
    assert np.allclose(rep.residual_history, ro.residual_history, rtol=1e-11)
    x0 = np.random.default_rng(3).uniform(-1, 1, n ** 3)
    xo, ro = O.jacobi(ap, ao, d, b, x0, 500, 0.5, basis="initial")
    x, rep = bs.jacobi_solve(op, b, x0, bs.InnerSolverSpec("jacobi", 500, 0.5), tolerance_basis="initial")
    assert rep.iterations_used == ro.iterations_used and rep.stop_reason == ro.stop_reason == "tolerance_met"
    assert np.array_equal(x, xo)
    # determinism and engine reuse across solver kinds (the Jacobi iterate is
    # flushed home before a CG solve starts on the same engine)
    x2, _ = bs.jacobi_solve(op, b, x0, bs.InnerSolverSpec("jacobi", 500, 0.5), tolerance_basis="initial")
    assert np.array_equal(x, x2)
    xc, rc = bs.cg_solve(op, b, np.zeros(n ** 3), bs.InnerSolverSpec("cg", 2000, 1e-8))
    assert rc.stop_reason == "tolerance_met"
    x3, r3 = bs.jacobi_solve(op, b, xc, bs.InnerSolverSpec("jacobi", 7, 0.0))
    xo3, ro3 = O.jacobi(ap, ao, d, b, xc, 7, 0.0)
    assert np.array_equal(x3, xo3)


def test_async_jacobi_inner_converges():
    n = 16
    b = O.seeded_rhs(n ** 3, 0)
    prob = bs.LinearProblem(bs.StencilOperator(n, n, n), b, bs.Grid3D(n, n, n))
    cfg = bs.OuterConfig(block_grid=(1, 1, 2), inner=bs.InnerSolverSpec("jacobi", 20), mode="async", tol=1e-6,
                         max_outer=20000, residual_check_every=5)
    res = bs.outer_solve(prob, cfg)
    assert res.converged and res.final_true_residual < 1e-6


# ------------------------------------------------------------------ outer sync


OUTER = ["outer/cfg1_16_fixed", "outer/cfg1_16_literal", "outer/cfg3_16_paper",
         "outer/cfg3_16_true", "outer/box_12_222", "outer/cfg5_12_o2", "outer/o1_10_211",
         "outer/jac_10_112", "outer/jac_8_221_o1"]


@pytest.mark.parametrize("key", OUTER)
def test_outer_sync_matches_reference(key):
    A, M = arrays(), meta()[key]
    c = M["case"]
    n = c["n"]
    kind, its, itol = c["inner"]
    grid = bs.Grid3D(n, n, n)
    prob = bs.LinearProblem(bs.StencilOperator(n, n, n), A[key + "/rhs"], grid)
    cfg = bs.OuterConfig(block_grid=tuple(c["bg"]), overlap=c["ov"],
                         inner=bs.InnerSolverSpec(kind, its, itol), tol=c["tol"],
                         max_outer=c.get("max_outer", 5000), residual_check_mode=c["mode"])
    res = bs.outer_solve(prob, cfg)
    assert res.converged == M["converged"]
    assert res.outer_iterations == M["outer_iterations"]
    # per-sweep residuals: 1e-9 relative plus an absolute floor of 5e-12 — the
    # reference algorithm itself moves its box_12_222 estimates by 8.3e-13
    # absolute (1.5e-6 relative) when only its dot products are reassociated
    # (measured with the oracle)
    for row, ref in zip(res.trace.rows, M["trace"]):
        assert row.outer_iteration == ref[0] and row.time == ref[1]
        assert row.inner_iterations == ref[4], f"sweep {ref[0]}"
        assert row.estimated_residual == pytest.approx(ref[2], rel=1e-9, abs=5e-12)
        if ref[3] is None:
            assert row.true_residual is None
        else:
            assert row.true_residual == pytest.approx(ref[3], rel=1e-9, abs=5e-12)
        assert row.max_halo_staleness == ref[5]
    sol = A[key + "/solution"]
    assert np.linalg.norm(res.solution - sol) <= 1e-10 * np.linalg.norm(sol)
    assert res.final_true_residual == pytest.approx(M["final_true_residual"], rel=1e-8)


def test_outer_config1_full_size_counts():
    """Config 1 (64^3, z_lo=1, 2 z-slabs, CG 50 its, outer 1e-6) in both tolerance
    bases.  Reference runs: literal basis stalls at
    8.063e-3; the r0-relative basis converges in 134 sweeps / 13,350 inner its
    with true residual 9.537e-7."""
    prob = bs.build_laplace_3d(bs.Grid3D(64, 64, 64, bs.DirichletBoundary({"z_lo": 1.0})))
    cfg = bs.OuterConfig(block_grid=(1, 1, 2), inner=bs.InnerSolverSpec("cg", 50, 1e-2), tol=1e-6,
                         max_outer=5000, tolerance_basis="initial")
    res = bs.outer_solve(prob, cfg)
    assert res.converged and res.outer_iterations == 134
    assert sum(r.inner_iterations for r in res.trace.rows) == 13350
    assert res.final_true_residual == pytest.approx(9.537e-7, rel=1e-3)
    lit = bs.outer_solve(prob, bs.OuterConfig(block_grid=(1, 1, 2), inner=bs.InnerSolverSpec("cg", 50, 1e-2),
                                              tol=1e-6, max_outer=40))
    assert not lit.converged
    assert [r.inner_iterations for r in lit.trace.rows[:6]] == [50, 55, 50, 6, 46, 0]
    assert lit.trace.rows[-1].estimated_residual == pytest.approx(8.063e-3, rel=1e-3)


def test_outer_block_count_invariance_of_counts():
    """8 z-slabs, r0-relative CG(100, 1e-3), true mode (config-3 shape at 32^3).

    Repeats are bitwise identical (fixed-order reductions).  Against the
    oracle: the outer count is equal and per-block inner counts are equal
    until the residual is so small that a 1e-16 change of the dot-product
    association can move an inner stop by one iteration — the reference
    algorithm itself does that when OpenBLAS dots are replaced by pairwise
    ones (tests/test_oracle_envelope.py: 63 sweeps differ from sweep 191 on).
    """
    n = 32
    b = O.seeded_rhs(n ** 3, 0)
    prob = bs.LinearProblem(bs.StencilOperator(n, n, n), b, bs.Grid3D(n, n, n))
    cfg = bs.OuterConfig(block_grid=(1, 1, 8), inner=bs.InnerSolverSpec("cg", 100, 1e-3), tol=1e-8,
                         tolerance_basis="initial", residual_check_mode="true")
    r1 = bs.outer_solve(prob, cfg)
    r2 = bs.outer_solve(prob, cfg)
    assert r1.inner_iterations_per_block == r2.inner_iterations_per_block
    assert np.array_equal(r1.solution, r2.solution)
    ro = O.outer_solve_sync((n, n, n), b, (1, 1, 8), 0,
                            dict(kind="cg", max_iterations=100, tolerance=1e-3, basis="initial"),
                            tol=1e-8, residual_check_mode="true")
    assert r1.outer_iterations == ro.outer_iterations
    assert r1.inner_iterations_per_block[:150] == ro.per_block_inner[:150]
    tot, tot_o = np.sum(r1.inner_iterations_per_block), np.sum(ro.per_block_inner)
    assert abs(tot - tot_o) <= 1e-3 * tot_o
    assert np.linalg.norm(r1.solution - ro.solution) <= 1e-8 * np.linalg.norm(ro.solution)


# ------------------------------------------------------------------ GMRES (a3)


@pytest.mark.parametrize("key", ["gmres/8_200_10", "gmres/10_30_30", "gmres/6_40_7"])
def test_gmres_matches_reference(key):
    A, M = arrays(), meta()[key]
    _, n, its, restart = key.replace("/", "_").split("_")
    n, its, restart = int(n), int(its), int(restart)
    tol = {"gmres/8_200_10": 1e-10, "gmres/10_30_30": 1e-3, "gmres/6_40_7": 0.0}[key]
    prob = bs.build_laplace_3d(bs.Grid3D(n, n, n, bs.DirichletBoundary({"x_lo": 1.0, "y_hi": 0.5})))
    x, rep = bs.gmres_solve(prob.matrix, prob.rhs, np.zeros(n ** 3), bs.InnerSolverSpec("gmres", its, tol, restart))
    assert rep.iterations_used == M["iterations_used"]
    assert rep.stop_reason == M["stop_reason"]
    assert np.allclose(rep.residual_history, M["residual_history"], rtol=1e-8, atol=1e-13)
    ref = A[key + "/x"]
    assert np.abs(x - ref).max() <= 1e-10 * max(1.0, np.abs(ref).max())


def test_gmres_edge_cases_and_oracle():
    # 1x1x1: Krylov space closes after one step (happy breakdown, inner_solvers.py:196-198)
    x, rep = bs.gmres_solve(bs.StencilOperator(1, 1, 1), np.array([3.0]), np.zeros(1),
                            bs.InnerSolverSpec("gmres", 10, 0.0))
    assert (rep.iterations_used, rep.stop_reason) == (1, "tolerance_met") and x[0] == 0.5
    # zero rhs from a non-zero start
    rng = np.random.default_rng(7)
    op = bs.StencilOperator(5, 4, 3)
    x, rep = bs.gmres_solve(op, np.zeros(60), rng.standard_normal(60), bs.InnerSolverSpec("gmres", 500, 1e-12))
    assert rep.stop_reason == "tolerance_met" and np.abs(x).max() <= 1e-10
    # restarted solve against the oracle on a ragged grid, warm start, r0 basis
    shape = (37, 21, 13)
    n = 37 * 21 * 13
    b = O.seeded_rhs(n, 4)
    x0 = rng.uniform(-1, 1, n)
    a = O.laplace_csr(*shape)
    xo, ro = O.gmres(lambda v: O.csr_spmv(a, v), b, x0, 120, 1e-6, 25, basis="initial")
    x, rep = bs.gmres_solve(bs.StencilOperator(*shape), b, x0, bs.InnerSolverSpec("gmres", 120, 1e-6, 25),
                            tolerance_basis="initial")
    assert rep.iterations_used == ro.iterations_used and rep.stop_reason == ro.stop_reason
    assert np.allclose(rep.residual_history, ro.residual_history, rtol=1e-7, atol=1e-14)
    assert np.linalg.norm(x - xo) <= 1e-9 * np.linalg.norm(xo)


def test_outer_sync_gmres_matches_oracle():
    """GMRES(10) one cycle per sweep (multisplit.py:532-536), 2x2x2 boxes, overlap 0."""
    n = 12
    prob = bs.build_laplace_3d(bs.Grid3D(n, n, n, bs.DirichletBoundary({"z_lo": 1.0})))
    cfg = bs.OuterConfig(block_grid=(2, 2, 2), inner=bs.InnerSolverSpec("gmres", 10), tol=1e-8)
    res = bs.outer_solve(prob, cfg)
    ro = O.outer_solve_sync((n, n, n), prob.rhs, (2, 2, 2), 0, dict(kind="gmres", max_iterations=10),
                            tol=1e-8)
    assert res.converged == ro.converged and res.outer_iterations == ro.outer_iterations
    assert res.inner_iterations_per_block == ro.per_block_inner
    for row, ref in zip(res.trace.rows, ro.rows):
        assert row.estimated_residual == pytest.approx(ref.estimated_residual, rel=1e-8)
    assert np.linalg.norm(res.solution - ro.solution) <= 1e-9 * np.linalg.norm(ro.solution)


@pytest.mark.parametrize("kind", ["jacobi", "cg"])
def test_outer_sync_lean_and_coupled_tiles_against_oracle(kind):
    """Blocks wide and deep enough (48 x 24 x 40) for full 32 x 8 tiles and unguarded ring rounds: tiles
    without a coupled face take the lean rounds of the residual / Jacobi sweeps (rhs = b, no face code),
    tiles on a coupled x / y face and the rounds holding a block's first / last plane the general path.
    Point-Jacobi inner sweeps are bit-reproducible, so the whole outer iteration is."""
    shape = (96, 48, 40)
    b = O.seeded_rhs(shape[0] * shape[1] * shape[2], 5)
    prob = bs.LinearProblem(bs.StencilOperator(*shape), b, bs.Grid3D(*shape))
    its = 6 if kind == "jacobi" else 8
    for bg in ((2, 2, 1), (1, 1, 1)):
        cfg = bs.OuterConfig(block_grid=bg, inner=bs.InnerSolverSpec(kind, its), tol=1e-30, max_outer=4)
        res = bs.outer_solve(prob, cfg)
        ro = O.outer_solve_sync(shape, b, bg, 0, dict(kind=kind, max_iterations=its), tol=1e-30, max_outer=4)
        assert res.outer_iterations == ro.outer_iterations == 4 and not res.converged
        assert res.inner_iterations_per_block == ro.per_block_inner
        for row, ref in zip(res.trace.rows, ro.rows):
            assert row.estimated_residual == pytest.approx(ref.estimated_residual, rel=1e-9)
            if ref.true_residual is not None:
                assert row.true_residual == pytest.approx(ref.true_residual, rel=1e-9)
        if kind == "jacobi":
            assert np.array_equal(res.solution, ro.solution)
        else:
            assert np.linalg.norm(res.solution - ro.solution) <= 1e-10 * np.linalg.norm(ro.solution)


# ------------------------------------------------------------------ async (a9)


def test_async_converges_to_the_sync_solution():
    """Async block Jacobi (config-4 shape: z-slabs, CG fixed 10 its, residual
    checked every 5 sweeps, confirmed stop).  Nondeterministic by design
    (SURVEY §0 item 7): compare the converged result only — true residual
    below tol and distance to a tight solve within 10x the sync oracle's."""
    n = 24
    b = O.seeded_rhs(n ** 3, 0)
    prob = bs.LinearProblem(bs.StencilOperator(n, n, n), b, bs.Grid3D(n, n, n))
    tol = 1e-8
    cfg = bs.OuterConfig(block_grid=(1, 1, 4), inner=bs.InnerSolverSpec("cg", 10), mode="async", tol=tol,
                         max_outer=3000, residual_check_every=5)
    res = bs.outer_solve(prob, cfg)
    assert res.converged
    assert res.final_true_residual < tol
    a = O.laplace_csr(n, n, n)
    tight, _ = O.cg(lambda v: O.csr_spmv(a, v), b, np.zeros(n ** 3), 5000, 1e-13)
    ro = O.outer_solve_sync((n, n, n), b, (1, 1, 4), 0, dict(kind="cg", max_iterations=10), tol=tol)
    sync_err = np.linalg.norm(ro.solution - tight) / np.linalg.norm(tight)
    async_err = np.linalg.norm(res.solution - tight) / np.linalg.norm(tight)
    assert async_err <= 10 * sync_err
    assert res.outer_iterations >= 10
    assert all(row.inner_iterations > 0 for row in res.trace.rows)


@pytest.mark.parametrize("delay,slots", [(("fixed", 3, 0, 0), 100), (("drop_free_jitter", 0, 1, 4), 100),
                                         (("fixed", 4, 0, 0), 2)])
def test_async_injected_delay(delay, slots):
    """DelayModel on real asynchrony (comm.py:51-81, 376-416): a payload posted
    at sweep j with delay d is applied by the receiver's exchange of an
    iteration k >= j + d (the exchange follows the solve, multisplit.py:575-586),
    so the observed halo staleness is at least d sweeps while payloads flow; an
    exhausted R-slot pool skips sends; the solve still converges."""
    n = 16
    b = O.seeded_rhs(n ** 3, 0)
    prob = bs.LinearProblem(bs.StencilOperator(n, n, n), b, bs.Grid3D(n, n, n))
    kind, fixed, low, high = delay
    cfg = bs.OuterConfig(block_grid=(1, 1, 2), inner=bs.InnerSolverSpec("cg", 10), mode="async", tol=1e-7,
                         max_outer=5000, residual_check_every=2, buffer_slots=slots,
                         delay=bs.DelayModel(kind, fixed=fixed, low=low, high=high, seed=1))
    res = bs.outer_solve(prob, cfg)
    assert res.converged and res.final_true_residual < 1e-7
    # staleness = k - (sweep of the applied payload) >= d while payloads flow
    # (measured: 93-100% of the rows with a 100-slot pool); a confirmation
    # round flushes fresh planes and resets it to 0, after which it climbs back
    # through 1..d, and with a pool shallower than the delay most sends are
    # skipped and confirmation rounds dominate the end of the run — there only
    # the maximum is asserted.
    dmin = fixed if kind == "fixed" else low
    late = np.array([r.max_halo_staleness for r in res.trace.rows[10:]])
    if slots >= dmin + 1:
        assert np.mean(late >= dmin) >= 0.6
    assert late.max() >= dmin
    events = dict(res.comm_events)
    if slots < fixed + 1:  # a pool shallower than the delay must skip sends
        assert events["skipped_sends"] > 0


# ------------------------------------------------------------------ multi-rank plumbing (e)


def test_post_plane_matches_device_halo_pack():
    """The cross-rank send buffer (bs_async_post) carries exactly what the
    same-GPU pack (bs_halo_pack) stores in the neighbour's halo plane."""
    t = torch()
    n = 20
    b = O.seeded_rhs(n ** 3, 1)
    dec = bs.decompose(bs.Grid3D(n, n, n), (2, 1, 2), 0)
    eng = BlockEngine((n, n, n), dec.owned, 0, "cuda")
    eng.load_host("b", b.reshape(n, n, n))
    eng.cg_begin(7, 0.0)
    eng.run()
    from paper_2009_12638_b200.engine import box_halo_plan
    plan = box_halo_plan(dec.owned, dec.block_grid)
    eng.halo_pack(plan)
    for dst, d, src in plan.tolist():
        buf = eng.new_plane(eng.plane_len(src, 5 - d))
        eng.post_plane(src, 5 - d, buf)
        t.cuda.synchronize()
        assert t.equal(buf, eng.ghost(dst, d))
    eng.close()


def test_distributed_driver_single_rank_nccl_equals_outer_solve():
    import socket

    t = torch()
    from paper_2009_12638_b200.distributed import outer_solve_distributed

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    t.distributed.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        n = 24
        b = O.seeded_rhs(n ** 3, 0)
        prob = bs.LinearProblem(bs.StencilOperator(n, n, n), b, bs.Grid3D(n, n, n))
        cfg = bs.OuterConfig(block_grid=(1, 1, 4), inner=bs.InnerSolverSpec("cg", 20, 1e-2), tol=1e-8,
                             tolerance_basis="initial")
        rd = outer_solve_distributed(prob, cfg)
        rl = bs.outer_solve(prob, cfg)
        assert rd.outer_iterations == rl.outer_iterations
        assert rd.inner_iterations_per_block == rl.inner_iterations_per_block
        assert [r.estimated_residual for r in rd.trace.rows] == [r.estimated_residual for r in rl.trace.rows]
        assert np.array_equal(rd.solution, rl.solution)
    finally:
        t.distributed.destroy_process_group()


def test_device_seeded_rhs_bit_identical_to_numpy():
    for n, seed in ((1, 0), (1000, 3), (256 ** 3, 0)):
        d = bs.seeded_rhs(n, seed, device="cuda").cpu().numpy()
        assert np.array_equal(d, O.seeded_rhs(n, seed))


# ------------------------------------------------------------------ block systems through the public API


def test_block_system_spmv_and_solves_public_api():
    """spmv / cg_solve / gmres_solve on ``block_system`` operators (box and
    L1-dilated regions) vs the reference's golden SpMV and the oracle."""
    A, M = arrays(), meta()
    for key in ("blocksys/8x8x8_222_o2", "blocksys/9x7x6_213_o1", "blocksys/6x6x6_321_o0"):
        m = M[key]
        shape, bg, ov = tuple(m["shape"]), tuple(m["block_grid"]), m["overlap"]
        prob = bs.build_laplace_3d(bs.Grid3D(*shape))
        dec = bs.decompose(prob.grid, bg, ov)
        _, wss, _, _ = O.build_workspaces(shape, np.zeros(int(np.prod(shape))), bg, ov)
        for b in range(dec.num_blocks):
            op, _ = bs.block_system(prob, dec, b)
            y = bs.spmv(op, A[f"{key}/{b}/x"])
            assert np.array_equal(y, A[f"{key}/{b}/y"]), (key, b)
        op, _ = bs.block_system(prob, dec, 1)
        rhs = np.random.default_rng(1).uniform(-1, 1, op.num_rows)
        ap = lambda v, a=wss[1].a_ii: O.csr_spmv(a, v)
        x, rep = bs.cg_solve(op, rhs, np.zeros(op.num_rows), bs.InnerSolverSpec("cg", 500, 1e-10))
        xo, ro = O.cg(ap, rhs, np.zeros(op.num_rows), 500, 1e-10)
        assert rep.iterations_used == ro.iterations_used
        assert np.linalg.norm(x - xo) <= 1e-9 * np.linalg.norm(xo)
        x, rep = bs.gmres_solve(op, rhs, np.zeros(op.num_rows), bs.InnerSolverSpec("gmres", 60, 1e-10, 20))
        xo, ro = O.gmres(ap, rhs, np.zeros(op.num_rows), 60, 1e-10, 20)
        assert rep.iterations_used == ro.iterations_used
        assert np.linalg.norm(x - xo) <= 1e-9 * np.linalg.norm(xo)
        _, rel = bs.residual_norms(op, x, rhs)
        assert rel <= 1e-9


def test_full_size_512_size_independent_properties():
    """BASELINE configs 3/4 grid size (512^3 = 134M unknowns, one block):
    SpMV bit-identical to the matrix-free oracle on a slab of planes checked
    in place (stencil rows only see z +- 1), SpMV of a constant = exact face
    counts, and a CG solve to 1e-8 whose true residual meets the tolerance."""
    import torch

    n = 512
    op = bs.StencilOperator(n, n, n)
    x = bs.seeded_rhs(n ** 3, 7, device="cuda")
    y = bs.spmv(op, x)
    xs = x.view(n, n, n)[200:204].cpu().numpy()  # planes 200..203 -> rows 201, 202 are exact
    ys = O.stencil_apply(np.concatenate([xs], axis=0)).reshape(4, n, n)
    assert np.array_equal(y.view(n, n, n)[201:203].cpu().numpy(), ys[1:3])
    ones = torch.ones(n ** 3, dtype=torch.float64, device="cuda")
    y1 = bs.spmv(op, ones).view(n, n, n)
    assert float(y1[1:-1, 1:-1, 1:-1].abs().max()) == 0.0  # interior rows of A*1 vanish exactly
    assert float(y1[0, 0, 0]) == 3.0 and float(y1[0, 5, 5]) == 1.0
    b = bs.seeded_rhs(n ** 3, 0, device="cuda")
    xs, rep = bs.cg_solve(op, b, torch.zeros_like(b), bs.InnerSolverSpec("cg", 5000, 1e-8))
    assert rep.stop_reason == "tolerance_met"
    _, rel = bs.residual_norms(op, xs, b)
    assert rel <= 1e-8


@pytest.mark.parametrize("shape", [(9, 7, 5), (33, 17, 13), (40, 24, 3), (37, 9, 66), (64, 40, 1)])
def test_cg_ragged_shapes_against_oracle(shape):
    """Ragged tiles (x, y not multiples of the 32x8 tile), odd plane counts
    (sweep 2 stages plane pairs; an odd count leaves a half-empty last box,
    and the reversed walk ends on a box below the grid) and one-plane grids:
    counts and histories equal to the reference algorithm, solution to 1e-10;
    the persistent kernel and the graph path agree bit for bit."""
    import os

    nx, ny, nz = shape
    N = nx * ny * nz
    b = O.seeded_rhs(N, 3)
    a = O.laplace_csr(nx, ny, nz)
    xo, ro = O.cg(lambda v: O.csr_spmv(a, v), b, np.zeros(N), 4000, 1e-9)
    op = bs.StencilOperator(nx, ny, nz)
    spec = bs.InnerSolverSpec("cg", 4000, 1e-9)
    out = {}
    for mode in ("1", "0"):
        old = os.environ.get("BS_PERSIST")
        os.environ["BS_PERSIST"] = mode
        try:
            out[mode] = bs.cg_solve(op, b, np.zeros(N), spec)
        finally:
            if old is None:
                del os.environ["BS_PERSIST"]
            else:
                os.environ["BS_PERSIST"] = old
    x, rep = out["1"]
    assert rep.iterations_used == ro.iterations_used
    assert np.allclose(rep.residual_history, ro.residual_history, rtol=1e-8, atol=1e-14)
    assert np.linalg.norm(x - xo) <= 1e-10 * np.linalg.norm(xo)
    xg, rg = out["0"]
    assert rg.iterations_used == rep.iterations_used and rg.residual_history == rep.residual_history
    assert np.array_equal(xg, x)
