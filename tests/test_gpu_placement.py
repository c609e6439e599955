"""Placement invariance on real kernels: the same 8-slab problem solved with
all blocks in one engine, or split over 2/4/8 engines (as 2/4/8 GPUs would
hold them) whose halo planes cross through the same send-buffer path the
NCCL exchange uses, gives bitwise-identical iteration counts, estimates and
solutions."""

import numpy as np
import pytest

from oracle import blocksolve_oracle as O

pytestmark = pytest.mark.gpu

import paper_2009_12638_b200 as bs  # noqa: E402
from paper_2009_12638_b200.engine import BlockEngine, box_halo_plan  # noqa: E402
from paper_2009_12638_b200.sync_driver import run_sync  # noqa: E402


class SplitEngines:
    """The engine interface of run_sync over several engines (one per 'GPU')."""

    def __init__(self, grid_shape, owned, groups):
        self.groups = groups
        self.engs = [BlockEngine(grid_shape, [owned[g] for g in grp], 0, "cuda", history_cap=1) for grp in groups]
        self.where = {g: (e, i) for e, grp in enumerate(groups) for i, g in enumerate(grp)}
        self.overlap = 0
        self.blocks = [bb for e in self.engs for bb in e.blocks]

    def _all(self, name, *a, **k):
        for e in self.engs:
            getattr(e, name)(*a, **k)

    def load_host(self, name, g3):
        self._all("load_host", name, g3)

    def cg_begin(self, *a, **k):
        self._all("cg_begin", *a, **k)

    def run(self, *a, **k):
        self._all("run", *a, **k)

    def sweep_resid(self):
        self._all("sweep_resid")

    def cancel(self):
        self._all("cancel")

    def flush(self):
        self._all("flush")

    def close(self):
        self._all("close")

    def reports(self):
        return [r for e in self.engs for r in e.reports()]

    def gather_owned(self, out3):
        self._all("gather_owned", out3)

    def exchange(self, plan):
        import torch

        for dst, d, src in plan.tolist():
            (ed, ld), (es, ls) = self.where[dst], self.where[src]
            if ed is es:
                self.engs[ed].halo_pack(np.asarray([(ld, d, ls)], dtype=np.int32))
            else:  # cross-"GPU": pack into a send buffer, deliver into the halo plane
                buf = self.engs[es].new_plane(self.engs[es].plane_len(ls, 5 - d))
                self.engs[es].post_plane(ls, 5 - d, buf)
                self.engs[ed].ghost(ld, d).copy_(buf)
        torch.cuda.synchronize()


@pytest.mark.parametrize("split", [1, 2, 4, 8])
def test_counts_and_solution_identical_for_every_placement(split):
    import torch

    n = 32
    b = O.seeded_rhs(n ** 3, 0)
    grid = bs.Grid3D(n, n, n)
    dec = bs.decompose(grid, (1, 1, 8), 0)
    cfg = bs.OuterConfig(block_grid=(1, 1, 8), inner=bs.InnerSolverSpec("cg", 100, 1e-3), tol=1e-8,
                         tolerance_basis="initial")
    prob = bs.LinearProblem(bs.StencilOperator(n, n, n), b, grid)
    ref = bs.outer_solve(prob, cfg)
    per = 8 // split
    eng = SplitEngines((n, n, n), dec.owned, [list(range(g * per, (g + 1) * per)) for g in range(split)])
    eng.load_host("b", b.reshape(n, n, n))
    plan = box_halo_plan(dec.owned, dec.block_grid)
    bnorm = float(np.linalg.norm(b))
    dens = []
    for box in dec.owned:
        d = float(np.linalg.norm(b.reshape(n, n, n)[box.lo[2]:box.hi[2], :, :].ravel()))
        dens.append(d or bnorm)
    rows, per_block, converged, final_true = run_sync(eng, cfg, dens, bnorm, 8, list(range(8)),
                                                      lambda: eng.exchange(plan), lambda t: t, 0.0)
    eng.flush()
    sol = torch.empty(n, n, n, dtype=torch.float64, device="cuda")
    eng.gather_owned(sol)
    eng.close()
    assert per_block == ref.inner_iterations_per_block
    assert [r[2] for r in rows] == [r.estimated_residual for r in ref.trace.rows]
    assert converged == ref.converged
    assert np.array_equal(sol.reshape(-1).cpu().numpy(), ref.solution)


def test_uneven_boxes_with_overlap_match_oracle():
    """Ragged split (13 = 7 + 6 ...) in all three directions, overlap 1, CG, true mode."""
    shape = (13, 11, 9)
    n = 13 * 11 * 9
    b = O.seeded_rhs(n, 2)
    grid = bs.Grid3D(*shape)
    prob = bs.LinearProblem(bs.StencilOperator(*shape), b, grid)
    cfg = bs.OuterConfig(block_grid=(2, 3, 2), overlap=1, inner=bs.InnerSolverSpec("cg", 6), tol=1e-7,
                         residual_check_mode="true")
    res = bs.outer_solve(prob, cfg)
    ro = O.outer_solve_sync(shape, b, (2, 3, 2), 1, dict(kind="cg", max_iterations=6), tol=1e-7,
                            residual_check_mode="true")
    assert res.outer_iterations == ro.outer_iterations and res.converged == ro.converged
    assert res.inner_iterations_per_block == ro.per_block_inner
    assert np.linalg.norm(res.solution - ro.solution) <= 1e-10 * np.linalg.norm(ro.solution)
