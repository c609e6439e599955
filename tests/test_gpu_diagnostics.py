"""Spectral diagnostics on the GPU vs the reference's
golden values (tests/golden/make_golden.py) and the oracle."""

import numpy as np
import pytest

from golden_io import arrays, meta
from oracle import blocksolve_oracle as O

pytestmark = pytest.mark.gpu

import paper_2009_12638_b200 as bs  # noqa: E402
from paper_2009_12638_b200 import diagnostics as D  # noqa: E402


def _problem(n):
    return bs.build_laplace_3d(bs.Grid3D(n, n, n, bs.DirichletBoundary({"x_lo": 1.0, "y_hi": 0.5})))


def test_power_iteration_known_answers():
    import torch

    w = torch.tensor([1.0, 2.0, 3.0], dtype=torch.float64, device="cuda")
    e = D.power_iteration(lambda v: v * w, 3, tol=1e-12, seed=1)
    ref = meta()["power/diag123"]
    assert e.converged and e.radius == pytest.approx(ref["radius"], abs=1e-12)
    assert abs(e.iterations_used - ref["iterations_used"]) <= 1
    z = D.power_iteration(lambda v: torch.zeros_like(v), 5, seed=0)
    assert (z.radius, z.iterations_used, z.converged) == (0.0, 1, True)
    # host (numpy) callables work too
    e2 = D.power_iteration(lambda v: np.array([1.0, 2.0, 3.0]) * v, 3, tol=1e-12, seed=1, device="cuda",
                            host_map=True)
    assert e2.radius == pytest.approx(3.0, abs=1e-10)
    with pytest.raises(ValueError):
        D.power_iteration(lambda v: v, 0, device="cuda")
    with pytest.raises(ValueError):
        D.power_iteration(lambda v: v, 3, tol=0.0, device="cuda")


def test_jacobi_iteration_radius():
    ref = meta()["power/jacobi_8"]
    op, dim = D.jacobi_iteration_operator(bs.StencilOperator(8, 8, 8))
    try:
        e = D.power_iteration(op, dim, tol=1e-10, seed=1)
        e2 = D.power_iteration(op, dim, tol=1e-10, seed=1)
    finally:
        op.close()
    assert e.converged and e.radius == pytest.approx(ref["radius"], rel=1e-9)
    assert abs(e.iterations_used - ref["iterations_used"]) <= 2
    assert (e.radius, e.iterations_used) == (e2.radius, e2.iterations_used)  # fixed-order reductions
    assert e.radius < np.cos(np.pi / 9) + 1e-12  # analytic rho(I - A/6) = cos(pi/(n+1))


def test_iteration_operator_matrix_matches_reference():
    A = arrays()
    pr = _problem(4)
    op, dim = D.iteration_operator(pr, bs.decompose(pr.grid, (2, 1, 1), 0))
    try:
        mat = np.stack([op(e) for e in np.eye(dim)], axis=1)
    finally:
        op.close()
    assert dim == 64
    assert np.abs(mat - A["itop/4_211_o0/matrix"]).max() <= 1e-11


@pytest.mark.parametrize("key", ["itop/4_211_o0", "itop/4_221_o1", "itop/8_211_o0", "itop/8_411_o0",
                                 "itop/6_113_o0", "itop/6_222_o1"])
def test_iteration_operator_radius_matches_reference(key):
    ref = meta()[key]
    n, bg, ov = key.split("/")[1].split("_")
    n, bg, ov = int(n), tuple(int(c) for c in bg), int(ov[1:])
    pr = _problem(n)
    op, dim = D.iteration_operator(pr, bs.decompose(pr.grid, bg, ov))
    try:
        assert dim == ref["dim"]
        e = D.power_iteration(op, dim, tol=1e-10, seed=0, max_iterations=5000)
    finally:
        op.close()
    assert e.converged == ref["converged"]
    if ref["converged"]:
        assert abs(e.iterations_used - ref["iterations_used"]) <= 2
        assert e.radius == pytest.approx(ref["radius"], rel=1e-8)
    else:  # the reference's own estimate after 5000 steps (its stopping test never fires)
        assert e.radius == pytest.approx(ref["radius"], rel=1e-6)


def test_iteration_operator_at_scale():
    """64^3 slabs: beyond what dense LU reaches.  More blocks -> larger radius
    (test_multisplit.py:415-422), all below one."""
    n = 64
    pr = _problem(n)
    radii = []
    for gz in (2, 4):
        op, dim = D.iteration_operator(pr, bs.decompose(pr.grid, (1, 1, gz), 0), inner_tolerance=1e-12)
        try:
            assert dim == n ** 3
            radii.append(D.power_iteration(op, dim, tol=1e-7, seed=0, max_iterations=400).radius)
        finally:
            op.close()
    assert radii[0] < radii[1] < 1.0
    # oracle cross-check at a size dense solves still handle
    pr = _problem(10)
    op, dim = D.iteration_operator(pr, bs.decompose(pr.grid, (1, 1, 2), 0))
    try:
        apply_o, dim_o = O.iteration_operator((10, 10, 10), (1, 1, 2), 0)
        z = np.random.default_rng(5).standard_normal(dim)
        assert np.abs(op(z) - apply_o(z)).max() <= 1e-10 * np.abs(apply_o(z)).max()
    finally:
        op.close()
