"""Host-side API parity with the reference (CPU): validation messages, error
types, decomposition geometry vs the oracle, trace CSV round trip, combiner."""

import math

import numpy as np
import pytest

import paper_2009_12638_b200 as bs
from oracle import blocksolve_oracle as O


def test_spec_validation():
    # inner_solvers.py:49-57
    with pytest.raises(ValueError):
        bs.InnerSolverSpec("sor", 10)
    with pytest.raises(ValueError):
        bs.InnerSolverSpec("cg", 0)
    with pytest.raises(ValueError):
        bs.InnerSolverSpec("cg", 10, tolerance=-1.0)
    with pytest.raises(ValueError):
        bs.InnerSolverSpec("gmres", 10, restart=0)


@pytest.mark.parametrize("kwargs,field", [
    (dict(mode="warp"), "mode"), (dict(tol=0.0), "tol"), (dict(max_outer=0), "max_outer"),
    (dict(residual_check_mode="x"), "residual_mode"), (dict(execution="gpu"), "exec"),
    (dict(execution="threads", residual_check_mode="true"), "exec"), (dict(true_residual_interval=0), "true_res_every"),
    (dict(tolerance_basis="r0"), "tolerance_basis"), (dict(residual_check_every=0), "residual_check_every"),
])
def test_outer_config_validation_names_the_field(kwargs, field):
    # multisplit.py:83-103: ConfigurationError (a ValueError) naming the field
    with pytest.raises(bs.ConfigurationError, match=field):
        bs.OuterConfig(**kwargs)


def test_errors_taxonomy():
    assert issubclass(bs.ConfigurationError, ValueError)
    assert issubclass(bs.ProtocolError, RuntimeError)
    e = bs.SolverBreakdownError(3, 7, "cg reported breakdown")
    assert e.block_id == 3 and e.outer_iteration == 7 and "block 3" in str(e)


def test_boundary_and_grid_validation():
    with pytest.raises(bs.ConfigurationError, match="boundary"):
        bs.DirichletBoundary({"w_lo": 1.0})
    with pytest.raises(bs.ConfigurationError, match="nx"):
        bs.Grid3D(0, 1, 1)


@pytest.mark.parametrize("shape,bg,ov", [((8, 8, 8), (2, 2, 2), 2), ((9, 7, 6), (2, 1, 3), 1), ((13, 11, 9), (2, 3, 2), 1),
                                         ((16, 16, 16), (1, 1, 4), 0), ((6, 6, 6), (3, 2, 1), 0)])
def test_analytic_decomposition_equals_oracle_masks(shape, bg, ov):
    """problems.py:287-359 via full-grid masks (oracle) == analytic geometry."""
    dec = bs.decompose(bs.Grid3D(*shape), bg, ov)
    boxes, wss, nbrs, cover = O.build_workspaces(shape, np.zeros(np.prod(shape)), bg, ov)
    assert [(b.lo, b.hi) for b in dec.owned] == [tuple(map(tuple, b)) for b in boxes]
    assert dec.neighbors == nbrs
    for blk in range(dec.num_blocks):
        assert np.array_equal(dec.extended_indices(blk), wss[blk].ext)
        assert np.array_equal(dec.owned_indices(blk), wss[blk].owned_global)


def test_decompose_preconditions():
    with pytest.raises(bs.ConfigurationError, match="gx"):
        bs.decompose(bs.Grid3D(4, 4, 4), (5, 1, 1))
    with pytest.raises(bs.ConfigurationError, match="overlap"):
        bs.decompose(bs.Grid3D(4, 4, 4), (2, 1, 1), 2)
    with pytest.raises(bs.ConfigurationError, match="overlap"):
        bs.decompose(bs.Grid3D(4, 4, 4), (1, 1, 1), -1)


def test_build_laplace_rhs_bitwise_vs_oracle():
    faces = {"x_lo": 1.0, "y_hi": 0.5, "z_lo": 2.0, "x_hi": -0.25}
    p = bs.build_laplace_3d(bs.Grid3D(5, 4, 3, bs.DirichletBoundary(faces)))
    assert np.array_equal(p.rhs, O.dirichlet_rhs(5, 4, 3, faces))
    assert p.matrix.nnz == O.laplace_csr(5, 4, 3).values.shape[0]


def test_combiner_and_termination():
    # multisplit.py:399-426
    assert bs.combined_residual([3.0, 4.0]) == 5.0 and bs.combined_residual([]) == 0.0
    assert bs.check_termination(5e-7, 1e-6, 10, 100, "sync") == "stop"
    assert bs.check_termination(1.0, 1e-6, 100, 100, "async") == "stop"
    assert bs.check_termination(5e-7, 1e-6, 10, 100, "async") == "confirm"
    assert bs.check_termination(1e-3, 1e-6, 10, 100, "sync") == "continue"


def test_trace_csv_round_trip(tmp_path):
    rows = [bs.TraceRow(0, 0.0, 0.5, 0.25, 10, 0), bs.TraceRow(1, 1.0, 1e-7, None, 8, 2)]
    tr = bs.ResidualTrace(rows)
    path = tmp_path / "t.csv"
    tr.write_csv(path)
    assert path.read_text().splitlines()[0] == bs.TRACE_HEADER
    assert bs.ResidualTrace.read_csv(path) == tr
    bad = tmp_path / "bad.csv"
    bad.write_text("time,residual\n0,1\n")
    with pytest.raises(ValueError, match="bad.csv"):
        bs.ResidualTrace.read_csv(bad)


def test_no_cpu_fallback():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(bs.DeviceError):
        bs.spmv(bs.StencilOperator(4, 4, 4), np.ones(64))
    with pytest.raises(bs.DeviceError):
        bs.cg_solve(bs.StencilOperator(4, 4, 4), np.ones(64), np.zeros(64), bs.InnerSolverSpec("cg", 5))
    with pytest.raises(bs.DeviceError):
        bs.jacobi_solve(bs.StencilOperator(4, 4, 4), np.ones(64), np.zeros(64), bs.InnerSolverSpec("jacobi", 5))


def test_solver_kind_routing():
    """Device kinds: jacobi, cg, gmres; 'direct' is a reference-only dense solve."""
    from paper_2009_12638_b200.inner_solvers import DEVICE_KINDS, SOLVER_KINDS

    assert DEVICE_KINDS == ("jacobi", "cg", "gmres")
    assert set(DEVICE_KINDS) < set(SOLVER_KINDS)
    with pytest.raises(bs.ConfigurationError, match="outside the accelerated path"):
        bs.solve(bs.StencilOperator(2, 2, 2), np.ones(8), np.zeros(8), bs.InnerSolverSpec("direct", 1))


def test_delay_model_draws_like_the_reference():
    """DelayModel.draw (comm.py:76-81) and the CLI spelling (cli.py:82-100)."""
    from paper_2009_12638_b200.cli import parse_delay

    rng = np.random.default_rng(3)
    assert bs.DelayModel().draw(rng) == 0
    assert bs.DelayModel("fixed", fixed=4).draw(rng) == 4
    m = bs.DelayModel("uniform", low=1, high=3, seed=7)
    r1, r2 = np.random.default_rng(7), np.random.default_rng(7)
    assert [m.draw(r1) for _ in range(50)] == [int(r2.integers(1, 4)) for _ in range(50)]
    assert parse_delay("jitter:2:5", 9) == bs.DelayModel("drop_free_jitter", low=2, high=5, seed=9)
    assert parse_delay("fixed:3", 0) == bs.DelayModel("fixed", fixed=3)
    with pytest.raises(bs.ConfigurationError, match="delay"):
        parse_delay("fixed", 0)
    with pytest.raises(bs.ConfigurationError, match="delay"):
        parse_delay("uniform:a:b", 0)
    with pytest.raises(bs.ConfigurationError, match="delay"):
        bs.DelayModel("uniform", low=3, high=1)


def test_send_pool_mirrors_the_reference_halo_buffer_pool():
    """SendPool (async_driver) against the reference pool semantics
    (comm.py:94-132, 376-393; test_comm.py TestAsyncExchange restated)."""
    from paper_2009_12638_b200.async_driver import SendPool

    # one slot, fixed delay 3: a post lands every 3 iterations, the rest skip
    pool = SendPool(1, bs.DelayModel("fixed", fixed=3))
    landed = []
    for k in range(31):
        pool.reclaim(k)  # the receiver (in lockstep) has begun iteration k
        got = pool.post(k, 3 if pool.free_slots else 0)
        if got is not None:
            landed.append(got[1] - 3)
    assert landed == list(range(0, 31, 3))  # sends at 0, 3, 6, ... (test_comm.py:149-157)
    assert pool.skipped == 31 - len(landed) > 0
    # conservation: in flight + free == capacity at every step
    rng = np.random.default_rng(13)
    m = bs.DelayModel("uniform", low=0, high=3, seed=13)
    pool = SendPool(4, m)
    for k in range(500):
        pool.reclaim(k)
        if pool.free_slots:
            pool.post(k, m.draw(rng))
        else:
            assert pool.post(k, 0) is None
        assert len(pool.in_flight) + pool.free_slots == pool.capacity == 4
    # drop_free_jitter: delivery times never regress (FIFO, no stale discards)
    m = bs.DelayModel("drop_free_jitter", low=0, high=4, seed=21)
    rng = np.random.default_rng(21)
    pool = SendPool(100, m)
    times = []
    for k in range(300):
        pool.reclaim(k)
        got = pool.post(k, m.draw(rng))
        times.append(got[1])
    assert all(b >= a for a, b in zip(times, times[1:]))
    assert all(t >= k for k, t in enumerate(times))


def _blocksys_keys():
    from golden_io import meta

    return sorted(k for k in meta() if k.startswith("blocksys/"))


@pytest.mark.parametrize("key", _blocksys_keys())
def test_block_system_matches_reference(key):
    """block_system (problems.py:362-406): region, couplings and size equal the
    reference's extraction (golden vectors from the unmodified reference)."""
    from golden_io import arrays, meta
    from oracle import blocksolve_oracle as O

    A, m = arrays(), meta()[key]
    shape, bg, ov = tuple(m["shape"]), tuple(m["block_grid"]), m["overlap"]
    prob = bs.build_laplace_3d(bs.Grid3D(*shape))
    dec = bs.decompose(prob.grid, bg, ov)
    _, wss, _, _ = O.build_workspaces(shape, np.zeros(int(np.prod(shape))), bg, ov)
    for b in range(dec.num_blocks):
        op, coupling = bs.block_system(prob, dec, b)
        assert np.array_equal(op.ext, A[f"{key}/{b}/ext"])
        assert np.array_equal(np.asarray(coupling, dtype=np.float64).reshape(-1, 3), A[f"{key}/{b}/coupling"])
        assert op.num_rows == op.shape[0] == wss[b].a_ii.num_rows
        assert op.nnz == wss[b].a_ii.values.shape[0]
    with pytest.raises(ValueError, match="out of range"):
        bs.block_system(prob, dec, dec.num_blocks)


def test_region_size_counts_the_dilated_region():
    """problems.region_size (rows of a block system, the GMRES restart cap of
    inner_solvers.py:162) == the oracle's L1-ball mask (= the reference's
    repeated dilation, pinned in test_oracle_golden)."""
    from oracle import blocksolve_oracle as O
    from paper_2009_12638_b200.problems import Grid3D, decompose, region_size

    for n, bg, o in [(12, (2, 2, 2), 2), (16, (2, 2, 2), 2), (10, (2, 1, 1), 1), (13, (3, 1, 2), 3), (6, (1, 1, 1), 0)]:
        d = decompose(Grid3D(n, n, n), bg, o)
        for box in d.owned:
            assert region_size((n, n, n), box, o) == int(O.region_mask((n, n, n), (box.lo, box.hi), o).sum())
