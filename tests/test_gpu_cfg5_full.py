"""Config 5's weak-scaling companion at full size (BASELINE.json configs[4],
SURVEY §8(d)): 512^3, u = 1 on z_lo, block_grid (2, 2, 2), overlap 2,
GMRES(30) to 1e-3 relative to ||r0||, sync, paper residual — the first two
sweeps through the public ``outer_solve`` compared with the full-size
oracle fixture (tests/golden/make_cfg5_fixture.py: the matrix-free overlap
restatement, pinned bit for bit to the CSR oracle, which is pinned to the
reference).

Bar (north_star): identical inner iteration counts per block; estimates
within 1e-9 relative (dots reassociated: OpenBLAS vs fixed-order trees);
iterates within 1e-9 of their max norm."""

import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
FIX = os.path.join(HERE, "golden", "cfg5_512.json")


@pytest.mark.skipif(not os.path.exists(FIX), reason="fixture not generated")
def test_config5_companion_first_sweeps_match_full_size_oracle():
    import paper_2009_12638_b200 as bs

    with open(FIX) as fh:
        meta = json.load(fh)
    with np.load(FIX.replace(".json", ".npz")) as z:
        idx, samples = z["idx"], z["samples"]
    n = meta["n"]
    grid = bs.Grid3D(n, n, n, bs.DirichletBoundary(meta["faces"]))
    prob = bs.build_laplace_3d(grid)
    kind, its, tol = meta["inner"]
    sweeps = len(meta["sweeps"])
    cfg = bs.OuterConfig(block_grid=tuple(meta["block_grid"]), overlap=meta["overlap"],
                         inner=bs.InnerSolverSpec(kind, its, tol, meta["restart"]), mode="sync", tol=1e-8,
                         max_outer=sweeps, tolerance_basis=meta["basis"],
                         residual_check_mode=meta["residual_check_mode"], capture_iterates=True)
    res = bs.outer_solve(prob, cfg)
    assert res.outer_iterations == sweeps
    assert res.inner_iterations_per_block == [s["its"] for s in meta["sweeps"]]
    for row, s in zip(res.trace.rows, meta["sweeps"]):
        assert abs(row.estimated_residual - s["estimate"]) <= 1e-9 * s["estimate"], (row, s["estimate"])
    for (k, x), s, ref in zip(res.snapshots, meta["sweeps"], samples):
        assert k == s["k"]
        assert np.max(np.abs(x[idx] - ref)) <= 1e-9 * np.max(np.abs(ref)), k
