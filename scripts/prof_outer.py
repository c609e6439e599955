"""A few sweeps of an outer workload (for ncu launch lists / per-sweep timing).

usage: prof_outer.py config5 N SWEEPS   (config3 / config5 shapes of bench.py)
Prints the per-sweep wall time from the trace (execution="threads" stamps
wall-clock times in the trace's time column)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2009_12638_b200 as bs  # noqa: E402
from bench import WORKLOADS as OUTER_WORKLOADS  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "config5"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 256
sweeps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
w = OUTER_WORKLOADS[name]
grid = bs.Grid3D(n, n, n, bs.DirichletBoundary(w["faces"] or {}))
prob = (bs.build_laplace_3d(grid) if w["faces"] else
        bs.LinearProblem(bs.StencilOperator(n, n, n), np.random.default_rng(0).uniform(-1.0, 1.0, n ** 3), grid))
kind, its, itol = w["inner"]
cfg = bs.OuterConfig(block_grid=w["block_grid"], overlap=w["overlap"], inner=bs.InnerSolverSpec(kind, its, itol),
                     mode="sync", tol=w["tol"], max_outer=sweeps, tolerance_basis=w["basis"], execution="threads")
t0 = time.perf_counter()
res = bs.outer_solve(prob, cfg)
torch.cuda.synchronize()
t = [row.time for row in res.trace.rows]
its = [sum(r) for r in res.inner_iterations_per_block]
print(f"{name} n={n}: {res.outer_iterations} sweeps in {time.perf_counter() - t0:.2f} s (incl. setup)")
for k in range(1, len(t)):
    print(f"  sweep {k}: {1e3 * (t[k] - t[k - 1]):.1f} ms, inner its {its[k]} per block {res.inner_iterations_per_block[k]}")
