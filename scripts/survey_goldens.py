"""Run the SURVEY Appendix B reference numbers (P6, P9, P13, P14, P15) on the GPU."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2009_12638_b200 as bs  # noqa: E402
from oracle import blocksolve_oracle as O  # noqa: E402


def seeded(n, seed=0):
    b = O.seeded_rhs(n ** 3, seed)
    return bs.LinearProblem(bs.StencilOperator(n, n, n), b, bs.Grid3D(n, n, n))


def faces(n, f):
    return bs.build_laplace_3d(bs.Grid3D(n, n, n, bs.DirichletBoundary(f)))


def run(label, prob, **kw):
    t0 = time.perf_counter()
    r = bs.outer_solve(prob, bs.OuterConfig(**kw))
    inner = sum(row.inner_iterations for row in r.trace.rows)
    print(f"{label}: sweeps {r.outer_iterations} inner {inner} true {r.final_true_residual:.4e} "
          f"converged {r.converged} ({time.perf_counter() - t0:.1f}s)", flush=True)


x, rep = bs.cg_solve(bs.StencilOperator(128, 128, 128), O.seeded_rhs(128 ** 3, 0), np.zeros(128 ** 3),
                     bs.InnerSolverSpec("cg", 5000, 1e-8))
print(f"P6 128^3 CG: its {rep.iterations_used} rel {rep.final_relative_residual:.4e}")
for mode in ("true", "paper"):
    run(f"P9 64^3 8 slabs cg(100,1e-3,initial) {mode}", seeded(64), block_grid=(1, 1, 8),
        inner=bs.InnerSolverSpec("cg", 100, 1e-3), tol=1e-8, tolerance_basis="initial", residual_check_mode=mode)
for mode in ("true", "paper"):
    run(f"P13 32^3 8 slabs cg(20,0) {mode}", seeded(32), block_grid=(1, 1, 8), inner=bs.InnerSolverSpec("cg", 20),
        tol=1e-8, residual_check_mode=mode)
for mode in ("paper", "true"):
    run(f"P14 32^3 2x2x2 o2 gmres(30,1e-3,initial) {mode}", faces(32, {"z_lo": 1.0}), block_grid=(2, 2, 2),
        overlap=2, inner=bs.InnerSolverSpec("gmres", 30, 1e-3, 30), tol=1e-8, tolerance_basis="initial",
        residual_check_mode=mode)
for mode in ("true", "paper"):
    run(f"P15 16^3 4 slabs cg(10,0) {mode}", seeded(16), block_grid=(1, 1, 4), inner=bs.InnerSolverSpec("cg", 10),
        tol=1e-8, residual_check_mode=mode)
