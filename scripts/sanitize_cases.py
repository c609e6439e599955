"""Small solves for compute-sanitizer (memcheck / racecheck / synccheck):
CG (graph path and persistent kernels), the streaming kernel, GMRES(10) with
overlap, point Jacobi, and an asynchronous solve (mailbox rings, seqlock)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_12638_b200 as bs  # noqa: E402

n = 12
b = np.random.default_rng(0).uniform(-1.0, 1.0, n ** 3)
prob = bs.LinearProblem(bs.StencilOperator(n, n, n), b, bs.Grid3D(n, n, n))
for mode in ("0", "1", "3"):
    os.environ["BS_PERSIST"] = mode
    r = bs.outer_solve(prob, bs.OuterConfig(block_grid=(1, 1, 2), inner=bs.InnerSolverSpec("cg", 8), tol=1e-6,
                                            max_outer=6))
    print("cg path", mode, r.outer_iterations, flush=True)
os.environ["BS_PERSIST"] = "1"
fprob = bs.build_laplace_3d(bs.Grid3D(n, n, n, bs.DirichletBoundary({"z_lo": 1.0})))
r = bs.outer_solve(fprob, bs.OuterConfig(block_grid=(2, 2, 2), overlap=2, inner=bs.InnerSolverSpec("gmres", 10),
                                         tol=1e-6, max_outer=4))
print("gmres overlap", r.outer_iterations, flush=True)
x, rep = bs.jacobi_solve(bs.StencilOperator(n, n, n), b, np.zeros(n ** 3), bs.InnerSolverSpec("jacobi", 20))
print("jacobi", rep.iterations_used, flush=True)
r = bs.outer_solve(prob, bs.OuterConfig(block_grid=(1, 1, 2), inner=bs.InnerSolverSpec("cg", 8), mode="async",
                                        tol=1e-6, max_outer=60, residual_check_every=2))
print("async", r.outer_iterations, r.converged, flush=True)
