"""Segmented synchronous runs (overlap > 0): pausing after sweep k, writing the outer iterate
(BlockEngine.save_state) and resuming in a fresh engine continues bit for bit — the long config-5
solve at 1024^3 is run this way, one GPU call per segment (scripts/run_cfg5.py)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_2009_12638_b200 as bs  # noqa: E402
from paper_2009_12638_b200.errors import ConfigurationError  # noqa: E402


class Pauser:
    def __init__(self, at, directory):
        self.at, self.directory, self.eng, self.paused_at = at, directory, None, None

    def attach(self, eng):
        self.eng = eng

    def begin(self, phase, k):
        pass

    def end(self, phase, k):
        pass

    def sweep(self, k, its):
        pass

    def pause(self, k):
        if k == self.at:
            self.eng.save_state(self.directory)
            return True
        return False


def _rows(res):
    return [(r.outer_iteration, r.estimated_residual, r.true_residual, r.inner_iterations) for r in res.trace.rows]


@pytest.mark.parametrize("inner", [bs.InnerSolverSpec("gmres", 10, 1e-3, 10), bs.InnerSolverSpec("cg", 6)])
def test_paused_and_resumed_run_equals_the_uninterrupted_one(tmp_path, inner):
    n = 24
    prob = bs.build_laplace_3d(bs.Grid3D(n, n, n, bs.DirichletBoundary({"z_lo": 1.0})))
    cfg = bs.OuterConfig(block_grid=(2, 2, 2), overlap=2, inner=inner, tol=1e-8, max_outer=400,
                         tolerance_basis="initial", true_residual_interval=1)
    full = bs.outer_solve(prob, cfg)
    assert full.converged and full.outer_iterations > 20
    first = Pauser(7, str(tmp_path / "ckpt"))
    a = bs.outer_solve(prob, cfg, probe=first)
    assert first.paused_at == 7 and not a.converged and a.outer_iterations == 8
    second = Pauser(15, str(tmp_path / "ckpt"))
    b = bs.outer_solve(prob, cfg, probe=second, resume=(7, str(tmp_path / "ckpt")))
    assert second.paused_at == 15 and b.trace.rows[0].outer_iteration == 8
    c = bs.outer_solve(prob, cfg, resume=(15, str(tmp_path / "ckpt")))
    assert c.converged
    assert _rows(a) + _rows(b) + _rows(c) == _rows(full)
    assert (a.inner_iterations_per_block + b.inner_iterations_per_block + c.inner_iterations_per_block
            == full.inner_iterations_per_block)
    assert np.array_equal(c.solution, full.solution)
    assert c.final_true_residual == full.final_true_residual


def test_resume_needs_an_overlapping_decomposition(tmp_path):
    n = 16
    prob = bs.build_laplace_3d(bs.Grid3D(n, n, n, bs.DirichletBoundary({"z_lo": 1.0})))
    cfg = bs.OuterConfig(block_grid=(1, 1, 2), inner=bs.InnerSolverSpec("cg", 5), max_outer=3)
    p = Pauser(1, str(tmp_path / "c"))
    res = bs.outer_solve(prob, cfg, probe=p)  # overlap 0: never asked to pause
    assert p.paused_at is None and res.outer_iterations == 3
    p.eng = None
    with pytest.raises(ConfigurationError):
        bs.outer_solve(prob, cfg, resume=(1, str(tmp_path / "c")))
