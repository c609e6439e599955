"""Per-sweep estimate deviation of the device solve from the oracle on the
CLI golden configuration (12^3, 2 z-slabs, CG 10 fixed, z_lo=1, x_hi=0.5)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_12638_b200 as bs  # noqa: E402
from oracle import blocksolve_oracle as O  # noqa: E402

n = 12
faces = {"z_lo": 1.0, "x_hi": 0.5}
b = O.dirichlet_rhs(n, n, n, faces)
ro = O.outer_solve_sync((n, n, n), b, (1, 1, 2), 0, dict(kind="cg", max_iterations=10), tol=1e-6)
prob = bs.build_laplace_3d(bs.Grid3D(n, n, n, bs.DirichletBoundary(faces)))
print("rhs equal:", np.array_equal(np.asarray(prob.rhs), b))
for mode in ("0", "1"):
    os.environ["BS_PERSIST"] = mode
    res = bs.outer_solve(prob, bs.OuterConfig(block_grid=(1, 1, 2), inner=bs.InnerSolverSpec("cg", 10), tol=1e-6))
    dev = [abs(a.estimated_residual - c.estimated_residual) / c.estimated_residual for a, c in zip(res.trace.rows, ro.rows)]
    print("BS_PERSIST", mode, "sweeps", res.outer_iterations, ro.outer_iterations, "max rel dev", max(dev),
          ["%.1e" % d for d in dev[:20]])
# CG alone on one slab (the first inner solve) vs the oracle
a = O.laplace_csr(n, n, n // 2)
rhs = b[: n * n * n // 2]
xo, rep_o = O.cg(lambda v: O.csr_spmv(a, v), rhs, np.zeros(rhs.size), 10, 0.0)
x, rep = bs.cg_solve(bs.StencilOperator(n, n, n // 2), rhs, np.zeros(rhs.size), bs.InnerSolverSpec("cg", 10))
print("slab CG: rel diff", np.linalg.norm(x - xo) / np.linalg.norm(xo), "hist",
      [f"{abs(p - q) / q:.1e}" for p, q in zip(rep.residual_history, rep_o.residual_history)])
