"""Pin the CPU oracle against the reference's golden vectors and its own
known-answer tests (restated).  CPU only."""

import numpy as np
import pytest

from golden_io import arrays, meta
from oracle import blocksolve_oracle as O


def lap(shape):
    return O.laplace_csr(*shape)


# ---------------------------------------------------------------- assembly


def test_assembly_bit_equal_to_reference():
    A, M = arrays(), meta()["assembly"]
    a = lap(M["shape"])
    assert np.array_equal(a.row_offsets, A["assembly/offsets"])
    assert np.array_equal(a.col_indices, A["assembly/cols"])
    assert np.array_equal(a.values, A["assembly/vals"])
    rhs = O.dirichlet_rhs(*M["shape"], M["faces"])
    assert np.array_equal(rhs, A["assembly/rhs"])


def test_callable_face_rhs():
    rhs = O.dirichlet_rhs(3, 4, 2, {"y_lo": lambda i, k: 0.5 * i + k, "z_hi": 1.5})
    assert np.array_equal(rhs, arrays()["assembly_callable/rhs"])


def test_known_answers_assembly():
    # test_problems.py:41-76 restated: [[6]]/[6]; 3x1x1 chain; mixed faces
    a = lap((1, 1, 1))
    assert np.array_equal(a.to_dense(), [[6.0]])
    assert np.array_equal(O.dirichlet_rhs(1, 1, 1, {f: 1.0 for f in O.FACES}), [6.0])
    chain = lap((3, 1, 1)).to_dense()
    assert np.array_equal(chain[1], [-1.0, 6.0, -1.0])
    rhs = O.dirichlet_rhs(2, 1, 1, {"x_lo": 2.0, "x_hi": 0.0, "y_lo": 0.25, "y_hi": 0.25})
    assert np.array_equal(rhs, [2.5, 0.5])


# ---------------------------------------------------------------- spmv


@pytest.mark.parametrize("shape", [(6, 5, 4), (16, 16, 16), (7, 1, 3)])
def test_csr_spmv_bit_equal(shape):
    A = arrays()
    key = "spmv/%dx%dx%d" % shape
    y = O.csr_spmv(lap(shape), A[key + "/x"])
    assert np.array_equal(y, A[key + "/y"])


@pytest.mark.parametrize("shape", [(6, 5, 4), (16, 16, 16), (7, 1, 3)])
def test_matrix_free_stencil_bit_equal(shape):
    A = arrays()
    key = "spmv/%dx%dx%d" % shape
    nx, ny, nz = shape
    y = O.stencil_apply(A[key + "/x"].reshape(nz, ny, nx)).ravel()
    assert np.array_equal(y, A[key + "/y"])


def _blocksys_keys():
    return [k for k in meta() if k.startswith("blocksys/")]


@pytest.mark.parametrize("key", _blocksys_keys())
def test_block_regions_and_block_spmv(key):
    """decompose (extended = L1 ball) + principal-submatrix SpMV, bitwise."""
    A, M = arrays(), meta()[key]
    shape, bg, ov = tuple(M["shape"]), tuple(M["block_grid"]), M["overlap"]
    nx, ny, nz = shape
    boxes = O.owned_boxes(shape, bg)
    cover = np.zeros(nx * ny * nz, dtype=np.int64)
    for b, box in enumerate(boxes):
        mask = O.region_mask(shape, box, ov)
        # analytic L1 ball == the reference's repeated 7-point dilation
        seed = np.zeros((nz, ny, nx), bool)
        (x0, y0, z0), (x1, y1, z1) = box
        seed[z0:z1, y0:y1, x0:x1] = True
        assert np.array_equal(mask, O.dilate(seed, ov))
        ext = np.nonzero(mask.ravel())[0]
        assert np.array_equal(ext, A[f"{key}/{b}/ext"])
        cover += mask.ravel()
        x = A[f"{key}/{b}/x"]
        u = np.zeros(nx * ny * nz)
        u[ext] = x
        y = O.stencil_apply(u.reshape(nz, ny, nx), mask).ravel()[ext]
        assert np.array_equal(y, A[f"{key}/{b}/y"])
    assert np.array_equal(cover, A[key + "/cover"])
    _, wss, nbrs, _ = O.build_workspaces(shape, np.zeros(nx * ny * nz), bg, ov)
    assert nbrs == M["neighbors"]


def test_spmv_known_answers():
    # test_linalg.py:62-93 restated on the stencil
    y = O.csr_spmv(lap((4, 4, 4)), np.ones(64))
    assert y[1 + 4 * (1 + 4 * 1)] == 0.0
    assert np.array_equal(O.csr_spmv(lap((3, 1, 1)), np.ones(3)), [5.0, 4.0, 5.0])


# ---------------------------------------------------------------- CG / GMRES


def _cg_case(key):
    n = int(key.split("/")[1].split("_")[0])
    seed = int(key.split("seed")[1])
    b = O.seeded_rhs(n ** 3, seed)
    a = lap((n, n, n))
    return a, b, n


@pytest.mark.parametrize("key", ["cg/12_seed0", "cg/20_seed1", "cg/32_seed0"])
def test_cg_matches_reference(key):
    A, M = arrays(), meta()[key]
    a, b, n = _cg_case(key)
    tol = {"cg/12_seed0": 1e-8, "cg/20_seed1": 1e-10, "cg/32_seed0": 1e-8}[key]
    x, rep = O.cg(lambda v: O.csr_spmv(a, v), b, np.zeros(n ** 3), 10 * n, tol)
    assert rep.iterations_used == M["iterations_used"]
    assert rep.stop_reason == M["stop_reason"]
    assert np.allclose(rep.residual_history, M["residual_history"], rtol=1e-12, atol=0)
    assert np.abs(x - A[key + "/x"]).max() <= 1e-13 * np.abs(A[key + "/x"]).max()


def test_cg_warm_start_and_initial_basis():
    A, M = arrays(), meta()
    n = 10
    a = lap((n, n, n))
    b = O.dirichlet_rhs(n, n, n, {"z_lo": 1.0})
    x0 = A["cg/warm/x0"]
    ap = lambda v: O.csr_spmv(a, v)
    x, rep = O.cg(ap, b, x0, 17, 1e-3)
    assert rep.iterations_used == M["cg/warm"]["iterations_used"] == 17
    assert rep.stop_reason == "max_iterations"
    assert np.allclose(x, A["cg/warm/x"], rtol=0, atol=1e-13)
    x, rep = O.cg(ap, b, x0, 200, 1e-3, basis="initial")
    assert rep.iterations_used == M["cg/warm_initial"]["iterations_used"]
    assert np.allclose(x, A["cg/warm_initial/x"], rtol=0, atol=1e-12)


@pytest.mark.parametrize("key", ["gmres/8_200_10", "gmres/10_30_30", "gmres/6_40_7"])
def test_gmres_matches_reference(key):
    A, M = arrays(), meta()[key]
    _, n, its, restart = key.replace("/", "_").split("_")
    n, its, restart = int(n), int(its), int(restart)
    tol = {"gmres/8_200_10": 1e-10, "gmres/10_30_30": 1e-3, "gmres/6_40_7": 0.0}[key]
    a = lap((n, n, n))
    b = O.dirichlet_rhs(n, n, n, {"x_lo": 1.0, "y_hi": 0.5})
    x, rep = O.gmres(lambda v: O.csr_spmv(a, v), b, np.zeros(n ** 3), its, tol, restart)
    assert rep.iterations_used == M["iterations_used"]
    assert rep.stop_reason == M["stop_reason"]
    assert np.allclose(rep.residual_history, M["residual_history"], rtol=1e-10, atol=1e-300)
    assert np.abs(x - A[key + "/x"]).max() <= 1e-12 * max(1.0, np.abs(x).max())


def test_cg_known_answers():
    # test_inner_solvers.py:91-130 restated
    ident = lambda v: v.copy()
    b = np.array([2.0, -1.0, 0.5])
    x, rep = O.cg(ident, b, np.zeros(3), 5, 1e-12)
    assert rep.iterations_used == 1 and np.allclose(x, b, atol=1e-15)
    x, rep = O.cg(lambda v: np.array([1.0, -1.0]) * v, np.ones(2), np.zeros(2), 10, 1e-10)
    assert rep.stop_reason == "breakdown"


# ---------------------------------------------------------------- point Jacobi


def _jacobi_case(key):
    """(shape, b, x0, max_its, tol) of a golden Jacobi case (make_golden.py)."""
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


JACOBI = ["jacobi/10_tol", "jacobi/9x6x4_maxit", "jacobi/7x1x3", "jacobi/1x1x5", "jacobi/1x1x1",
          "jacobi/zero_rhs"]


@pytest.mark.parametrize("key", JACOBI)
@pytest.mark.parametrize("form", ["csr", "matrix_free"])
def test_jacobi_matches_reference(key, form):
    A, M = arrays(), meta()[key]
    shape, b, x0, its, tol = _jacobi_case(key)
    a = lap(shape)
    if form == "csr":
        off = O.csr_without_diagonal(a)
        ap, ao, d = (lambda v: O.csr_spmv(a, v)), (lambda v: O.csr_spmv(off, v)), O.csr_diagonal(a)
    else:
        nx, ny, nz = shape
        ap = lambda v: O.stencil_apply(v.reshape(nz, ny, nx)).ravel()
        ao = lambda v: O.offdiag_apply(v.reshape(nz, ny, nx)).ravel()
        d = np.full(a.num_rows, 6.0)
    x, rep = O.jacobi(ap, ao, d, b, x0, its, tol)
    assert rep.iterations_used == M["iterations_used"]
    assert rep.stop_reason == M["stop_reason"]
    assert np.array_equal(x, A[key + "/x"])  # the update is elementwise: bit-exact
    assert np.allclose(rep.residual_history, M["residual_history"], rtol=1e-13, atol=0)


@pytest.mark.parametrize("shape", [(6, 5, 4), (16, 16, 16), (7, 1, 3)])
def test_offdiag_matrix_free_bit_equal(shape):
    A = arrays()
    x = A["spmv/%dx%dx%d/x" % shape]
    a = lap(shape)
    off = O.csr_without_diagonal(a)
    assert off.values.shape[0] == a.values.shape[0] - a.num_rows
    assert np.array_equal(O.csr_diagonal(a), np.full(a.num_rows, 6.0))
    nx, ny, nz = shape
    y = O.offdiag_apply(x.reshape(nz, ny, nx)).ravel()
    assert np.array_equal(y, O.csr_spmv(off, x))
    # the full row = offdiag + the diagonal's place in the chain: cross-check the
    # region form on an L1 ball (rows whose leading term is an upper neighbour)
    reg = O.region_mask((nx, ny, nz), O.owned_boxes((nx, ny, nz), (2, 1, 1))[0], 1)
    u = x.reshape(nz, ny, nx)
    rows = np.flatnonzero(reg.ravel())
    sub = O.csr_without_diagonal(_principal(a, rows))
    assert np.array_equal(O.offdiag_apply(u, reg).ravel()[rows], O.csr_spmv(sub, x[rows]))


def _principal(a, rows):
    """Principal submatrix of CSR `a` on sorted `rows` (entries kept in order)."""
    pos = -np.ones(a.num_cols, dtype=np.int64)
    pos[rows] = np.arange(rows.shape[0])
    offs, cols, vals = [0], [], []
    for r in rows:
        s, e = a.row_offsets[r], a.row_offsets[r + 1]
        c = pos[a.col_indices[s:e]]
        keep = c >= 0
        cols.append(c[keep])
        vals.append(a.values[s:e][keep])
        offs.append(offs[-1] + int(keep.sum()))
    return O.CSR(rows.shape[0], rows.shape[0], np.asarray(offs, dtype=np.int64), np.concatenate(cols),
                 np.concatenate(vals))


# ---------------------------------------------------------------- outer sync


OUTER = ["outer/cfg1_16_fixed", "outer/cfg1_16_literal", "outer/cfg3_16_paper",
         "outer/cfg3_16_true", "outer/box_12_222", "outer/cfg5_12_o2", "outer/o1_10_211",
         "outer/jac_10_112", "outer/jac_8_221_o1"]


@pytest.mark.parametrize("key", OUTER)
def test_outer_sync_matches_reference_trace(key):
    A, M = arrays(), meta()[key]
    c = M["case"]
    n = c["n"]
    kind, its, itol = c["inner"]
    res = O.outer_solve_sync((n, n, n), A[key + "/rhs"], tuple(c["bg"]), c["ov"],
                             dict(kind=kind, max_iterations=its, tolerance=itol),
                             tol=c["tol"], max_outer=c.get("max_outer", 5000),
                             residual_check_mode=c["mode"])
    assert res.converged == M["converged"]
    assert res.outer_iterations == M["outer_iterations"]
    ref_rows = M["trace"]
    assert len(res.rows) == len(ref_rows)
    for row, ref in zip(res.rows, ref_rows):
        assert row.outer_iteration == ref[0]
        assert row.inner_iterations == ref[4]
        assert row.estimated_residual == pytest.approx(ref[2], rel=1e-10)
        if ref[3] is None:
            assert row.true_residual is None
        else:
            assert row.true_residual == pytest.approx(ref[3], rel=1e-10)
    assert res.final_true_residual == pytest.approx(M["final_true_residual"], rel=1e-10)
    sol = A[key + "/solution"]
    assert np.linalg.norm(res.solution - sol) <= 1e-12 * np.linalg.norm(sol)


def test_threaded_csr_bit_identical():
    A = arrays()
    a = lap((16, 16, 16))
    x = A["spmv/16x16x16/x"]
    assert np.array_equal(O.ThreadedCSR(a, 3)(x), A["spmv/16x16x16/y"])


# ---------------------------------------------------------------- spectral diagnostics


def test_power_iteration_matches_reference():
    M = meta()
    e = O.power_iteration(lambda v: np.array([1.0, 2.0, 3.0]) * v, 3, tol=1e-12, seed=1)
    ref = M["power/diag123"]
    assert (e.iterations_used, e.converged) == (ref["iterations_used"], ref["converged"])
    assert e.radius == ref["radius"]
    a = lap((8, 8, 8))
    e = O.power_iteration(lambda v: v - O.csr_spmv(a, v) / 6.0, 512, tol=1e-10, seed=1)
    ref = M["power/jacobi_8"]
    assert (e.iterations_used, e.converged, e.radius) == (ref["iterations_used"], ref["converged"], ref["radius"])
    # known answers (test_linalg.py:163-195 restated)
    assert O.power_iteration(lambda v: np.zeros_like(v), 5, seed=0) == O.Spectral(0.0, 1, True)
    with pytest.raises(ValueError):
        O.power_iteration(lambda v: v, 0)
    with pytest.raises(ValueError):
        O.power_iteration(lambda v: v, 3, tol=0.0)


def test_iteration_operator_matrix_matches_reference():
    A = arrays()
    apply, dim = O.iteration_operator((4, 4, 4), (2, 1, 1), 0)
    assert dim == 64
    mat = np.stack([apply(e) for e in np.eye(dim)], axis=1)
    assert np.abs(mat - A["itop/4_211_o0/matrix"]).max() <= 1e-14


@pytest.mark.parametrize("key", ["itop/4_211_o0", "itop/4_221_o1", "itop/8_211_o0", "itop/8_411_o0",
                                 "itop/6_113_o0", "itop/6_222_o1"])
def test_iteration_operator_radius_matches_reference(key):
    ref = meta()[key]
    n, bg, ov = key.split("/")[1].split("_")
    n, bg, ov = int(n), tuple(int(c) for c in bg), int(ov[1:])
    apply, dim = O.iteration_operator((n, n, n), bg, ov)
    assert dim == ref["dim"]
    e = O.power_iteration(apply, dim, tol=1e-10, seed=0)
    assert e.converged == ref["converged"]
    if ref["converged"]:
        assert abs(e.iterations_used - ref["iterations_used"]) <= 1
    assert e.radius == pytest.approx(ref["radius"], rel=1e-9)


# ---------------------------------------------------------------- full-size slab oracle (config 3 fixture)


@pytest.mark.parametrize("shape", [(1, 1, 1), (5, 1, 7), (7, 5, 1), (9, 11, 13), (16, 16, 16), (3, 2, 2)])
def test_box_stencil_bit_equal(shape):
    """stencil_apply_box (the fast whole-box path of the 512^3 fixture) ==
    stencil_apply bit for bit, signed zeros included."""
    nx, ny, nz = shape
    rng = np.random.default_rng(7)
    u = rng.standard_normal((nz, ny, nx)) * np.exp(rng.uniform(-20, 20, (nz, ny, nx)))
    a, b = O.stencil_apply(u), O.stencil_apply_box(u)
    assert np.array_equal(a, b) and np.array_equal(np.signbit(a), np.signbit(b))


def test_box_stencil_matches_reference_spmv():
    A = arrays()
    for shape in [(6, 5, 4), (16, 16, 16), (7, 1, 3)]:
        key = "spmv/%dx%dx%d" % shape
        nx, ny, nz = shape
        assert np.array_equal(O.stencil_apply_box(A[key + "/x"].reshape(nz, ny, nx)).ravel(), A[key + "/y"])


def test_slab_oracle_matches_reference_trace():
    """The matrix-free z-slab outer sweep against the reference's own trace
    (outer/cfg3_16_paper: 16^3, 4 slabs, fixed 10 CG its, paper mode)."""
    A, M = arrays(), meta()["outer/cfg3_16_paper"]
    n = M["case"]["n"]
    recs = O.outer_solve_slabs((n, n, n), A["outer/cfg3_16_paper/rhs"], 4, 10, 0.0, "rhs",
                               sweeps=M["outer_iterations"])
    for rec, ref in zip(recs, M["trace"]):
        assert sum(rec["its"]) == ref[4]
        assert rec["estimate"] == pytest.approx(ref[2], rel=1e-10)
    x = np.concatenate([xx.ravel() for xx in recs[-1]["x"]])
    sol = A["outer/cfg3_16_paper/solution"]
    assert np.linalg.norm(x - sol) <= 1e-12 * np.linalg.norm(sol)


def test_slab_oracle_equals_csr_oracle():
    """outer_solve_slabs == outer_solve_sync bit for bit (counts, estimates,
    iterates) on the config-3 analogue with the r0-relative basis."""
    n = 16
    b = O.seeded_rhs(n ** 3, 0)
    res = O.outer_solve_sync((n, n, n), b, (1, 1, 4), 0,
                             dict(kind="cg", max_iterations=30, tolerance=1e-3, basis="initial"),
                             tol=1e-30, max_outer=6)
    recs = O.outer_solve_slabs((n, n, n), b, 4, 30, 1e-3, "initial", sweeps=6)
    for rec, row, its in zip(recs, res.rows, res.per_block_inner):
        assert rec["its"] == its
        assert rec["estimate"] == row.estimated_residual
    assert np.array_equal(np.concatenate([xx.ravel() for xx in recs[-1]["x"]]), res.solution)


def test_cfg3_fixture_is_consistent():
    """The committed 512^3 fixture: 8 slabs x 3 sweeps, estimates = the
    block-order combiner of its local residuals (comm.py:442-445)."""
    import json
    import math
    import os

    with open(os.path.join(os.path.dirname(__file__), "golden", "cfg3_512.json")) as fh:
        m = json.load(fh)
    assert m["n"] == 512 and m["nslabs"] == 8 and len(m["sweeps"]) == 3
    for s in m["sweeps"]:
        assert len(s["its"]) == 8 and all(1 <= i <= 100 for i in s["its"])
        assert s["estimate"] == math.sqrt(float(sum(v ** 2 for v in s["locals"])))
    est = [s["estimate"] for s in m["sweeps"]]
    assert est == sorted(est, reverse=True)


# ---------------------------------------------------------------- full-size overlap oracle (config 5 fixture)


@pytest.mark.parametrize("case", [
    (12, (2, 2, 2), 2, dict(kind="gmres", max_iterations=10), {"z_lo": 1.0}),
    (10, (2, 1, 1), 1, dict(kind="cg", max_iterations=6), None),
    (12, (2, 2, 2), 0, dict(kind="cg", max_iterations=8), None),
    (16, (2, 2, 2), 2, dict(kind="gmres", max_iterations=30, tolerance=1e-3, basis="initial"), {"z_lo": 1.0}),
])
def test_box_oracle_equals_csr_oracle(case):
    """outer_solve_boxes (matrix-free frames, coupling_apply) == the CSR
    outer_solve_sync bit for bit: counts, estimates and iterates."""
    n, bg, ov, inner, faces = case
    b = O.dirichlet_rhs(n, n, n, faces) if faces else O.seeded_rhs(n ** 3, 3)
    res = O.outer_solve_sync((n, n, n), b, bg, ov, inner, tol=1e-30, max_outer=4)
    recs = O.outer_solve_boxes((n, n, n), b, bg, ov, inner, sweeps=4)
    for rec, row, its in zip(recs, res.rows, res.per_block_inner):
        assert rec["its"] == its
        assert rec["estimate"] == row.estimated_residual
    sol = np.zeros((n, n, n))
    for box, xo in zip(recs[-1]["boxes"], recs[-1]["owned"]):
        (x0, y0, z0), (x1, y1, z1) = box
        sol[z0:z1, y0:y1, x0:x1] = xo.reshape(z1 - z0, y1 - y0, x1 - x0)
    assert np.array_equal(sol.ravel(), res.solution)


def test_box_oracle_matches_reference_trace():
    """The matrix-free overlap sweep against the reference's own trace
    (outer/cfg5_12_o2: 12^3, 2x2x2, overlap 2, fixed GMRES 10 its)."""
    A, M = arrays(), meta()["outer/cfg5_12_o2"]
    c = M["case"]
    n = c["n"]
    b = O.dirichlet_rhs(n, n, n, c["faces"])
    recs = O.outer_solve_boxes((n, n, n), b, tuple(c["bg"]), c["ov"],
                               dict(kind="gmres", max_iterations=c["inner"][1]), sweeps=min(6, M["outer_iterations"]))
    for rec, ref in zip(recs, M["trace"]):
        assert sum(rec["its"]) == ref[4]
        assert rec["estimate"] == pytest.approx(ref[2], rel=1e-10)


def test_coupling_apply_is_the_coupling_csr():
    """coupling_apply == the reference's coupling CSR (oracle build_workspaces,
    pinned) applied to a wide-range halo vector, bit for bit."""
    n, bg, ov = 12, (2, 2, 2), 2
    rng = np.random.default_rng(4)
    boxes, wss, _, _ = O.build_workspaces((n, n, n), np.zeros(n ** 3), bg, ov)
    for ws, box in zip(wss, boxes):
        f = O._Frame((n, n, n), box, ov)
        h = rng.standard_normal(ws.halo_cols.shape[0]) * np.exp(rng.uniform(-15, 15, ws.halo_cols.shape[0]))
        ref = O.csr_spmv(ws.coupling, h)
        glob = np.zeros(n ** 3)
        glob[ws.halo_cols] = h
        got = O.coupling_apply(f.take(glob.reshape(n, n, n)), f.region, f.grid)[f.region]
        assert np.array_equal(got, ref)
