"""Config 4 (BASELINE.json configs[3]) at full size, the converged-result bar
of SURVEY §8(d) for asynchronous runs (nondeterministic by design): 512^3,
seeded rhs, eight z-slabs, CG fixed 20 iterations, residual checked every 10
sweeps, tol 1e-8.  Checks (a) converged with final true residual < tol and
(b) relative L2 distance to a tight solve (single-block CG to 1e-13) <= 10x
the synchronous twin's (same config, mode sync: the oracle-matching path).
Prints one JSON line."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_12638_b200 as bs  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
N = n ** 3
b = np.random.default_rng(0).uniform(-1.0, 1.0, N)
prob = bs.LinearProblem(bs.StencilOperator(n, n, n), b, bs.Grid3D(n, n, n))
out = {"n": n}
t0 = time.perf_counter()
ra = bs.outer_solve(prob, bs.OuterConfig(block_grid=(1, 1, 8), inner=bs.InnerSolverSpec("cg", 20), mode="async",
                                         tol=1e-8, max_outer=100000, residual_check_every=10, execution="threads"))
out["async"] = {"seconds": time.perf_counter() - t0, "converged": ra.converged, "outer_sweeps": ra.outer_iterations,
                "final_true_residual": ra.final_true_residual,
                "comm_events": dict(ra.comm_events)}
t0 = time.perf_counter()
rs = bs.outer_solve(prob, bs.OuterConfig(block_grid=(1, 1, 8), inner=bs.InnerSolverSpec("cg", 20), mode="sync",
                                         tol=1e-8, max_outer=100000))
out["sync"] = {"seconds": time.perf_counter() - t0, "converged": rs.converged, "outer_sweeps": rs.outer_iterations,
               "final_true_residual": rs.final_true_residual}
t0 = time.perf_counter()
bt = torch.from_numpy(b).cuda()
xt, rep = bs.cg_solve(bs.StencilOperator(n, n, n), bt, torch.zeros_like(bt), bs.InnerSolverSpec("cg", 100000, 1e-13))
xt = xt.cpu().numpy()
out["tight"] = {"seconds": time.perf_counter() - t0, "iterations": rep.iterations_used,
                "relative_residual": rep.final_relative_residual}
nt = np.linalg.norm(xt)
out["async_err"] = float(np.linalg.norm(ra.solution - xt) / nt)
out["sync_err"] = float(np.linalg.norm(rs.solution - xt) / nt)
out["bar"] = {"converged_below_tol": bool(ra.converged and ra.final_true_residual < 1e-8),
              "within_10x_sync_error": bool(out["async_err"] <= 10 * out["sync_err"])}
print(json.dumps(out), flush=True)
