"""Config 5 (BASELINE.json configs[4]) to convergence on one GPU: n^3 grid
(default 1024), u = 1 on z_lo, block_grid (2, 2, 2), overlap 2, GMRES(30)
to 1e-3 relative to ||r0||, sync, paper residual, tol 1e-8.  At 1024^3 the
eight 514^3-point blocks share one Krylov basis (solved one after another,
bitwise the per-block numbers).  Progress (sweep, estimate, true residual,
inner its, elapsed) is flushed to stdout every LOG_EVERY sweeps, so a run cut
short still leaves its trace."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_12638_b200 as bs  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
max_outer = int(sys.argv[2]) if len(sys.argv) > 2 else 100000
every = int(os.environ.get("LOG_EVERY", "50"))
t0 = time.perf_counter()


class Log:
    def begin(self, phase, k):
        pass

    def end(self, phase, k):
        pass

    def sweep(self, k, its):
        pass

    def trace(self, k, est, true_res, inner):
        if k % every == 0:
            print(json.dumps({"k": k, "estimate": est, "true": true_res, "inner": inner,
                              "elapsed_s": round(time.perf_counter() - t0, 2)}), flush=True)


grid = bs.Grid3D(n, n, n, bs.DirichletBoundary({"z_lo": 1.0}))
prob = bs.build_laplace_3d(grid)
cfg = bs.OuterConfig(block_grid=(2, 2, 2), overlap=2, inner=bs.InnerSolverSpec("gmres", 30, 1e-3, 30), mode="sync",
                     tol=1e-8, max_outer=max_outer, tolerance_basis="initial", residual_check_mode="paper")
print(json.dumps({"config": "config5", "n": n, "setup_s": round(time.perf_counter() - t0, 2)}), flush=True)
res = bs.outer_solve(prob, cfg, probe=Log())
total = time.perf_counter() - t0
its = sum(sum(r) for r in res.inner_iterations_per_block)
print(json.dumps({"done": True, "n": n, "converged": res.converged, "outer_sweeps": res.outer_iterations,
                  "inner_iterations_total": its, "final_estimate": res.trace.rows[-1].estimated_residual,
                  "final_true_residual": res.final_true_residual, "time_to_solution_s": total,
                  "seconds_per_sweep": total / res.outer_iterations}), flush=True)
