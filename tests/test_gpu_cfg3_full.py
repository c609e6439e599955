"""Config 3 at its full size (BASELINE.json configs[2]): 512^3, seeded rhs,
eight z-slabs of 64 planes, inner CG(100, 1e-3 relative to ||r0||), sync,
paper residual mode — the first three sweeps through the public
``outer_solve`` compared with the full-size oracle fixture
(``tests/golden/make_cfg3_fixture.py``: the matrix-free slab restatement,
pinned bit for bit to the CSR oracle, which is pinned to the reference).

Bar (north_star): identical inner iteration counts; per-sweep estimates
within 1e-9 relative (the dots are reassociated: the oracle's are OpenBLAS,
the device's fixed-order trees); iterates within 1e-9 of their max norm."""

import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def _fixture():
    with open(os.path.join(HERE, "golden", "cfg3_512.json")) as fh:
        meta = json.load(fh)
    with np.load(os.path.join(HERE, "golden", "cfg3_512.npz")) as z:
        return meta, z["idx"], z["samples"]


def test_config3_first_sweeps_match_full_size_oracle():
    import paper_2009_12638_b200 as bs

    meta, idx, samples = _fixture()
    n = meta["n"]
    b = np.random.default_rng(meta["seed"]).uniform(-1.0, 1.0, n ** 3)
    prob = bs.LinearProblem(bs.StencilOperator(n, n, n), b, bs.Grid3D(n, n, n))
    kind, its, tol = meta["inner"]
    sweeps = len(meta["sweeps"])
    cfg = bs.OuterConfig(block_grid=(1, 1, meta["nslabs"]), inner=bs.InnerSolverSpec(kind, its, tol),
                         mode="sync", tol=1e-8, max_outer=sweeps, tolerance_basis=meta["basis"],
                         residual_check_mode=meta["residual_check_mode"], capture_iterates=True)
    res = bs.outer_solve(prob, cfg)
    assert res.outer_iterations == sweeps and not res.converged
    assert res.inner_iterations_per_block == [s["its"] for s in meta["sweeps"]]
    for row, s in zip(res.trace.rows, meta["sweeps"]):
        assert abs(row.estimated_residual - s["estimate"]) <= 1e-9 * s["estimate"], (row, s["estimate"])
    nz = n // meta["nslabs"]
    for (k, x), s, ref in zip(res.snapshots, meta["sweeps"], samples):
        assert k == s["k"]
        scale = np.max(np.abs(ref))
        assert np.max(np.abs(x[idx] - ref)) <= 1e-9 * scale, k
        x3 = x.reshape(n, n, n)
        for blk in range(meta["nslabs"]):
            slab = x3[blk * nz:(blk + 1) * nz]
            assert abs(float(np.sum(slab)) - s["slab_sum"][blk]) <= 1e-9 * float(np.sum(np.abs(slab)))
            assert abs(float(np.sum(slab * slab)) - s["slab_sumsq"][blk]) <= 1e-9 * s["slab_sumsq"][blk]
