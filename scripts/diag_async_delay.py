"""Staleness distribution of the injected-latency configs of tests/test_gpu_parity.py::test_async_injected_delay."""
import sys
from collections import Counter

import numpy as np

sys.path.insert(0, ".")
import paper_2009_12638_b200 as bs  # noqa: E402

n = 16
b = bs.seeded_rhs(n ** 3, 0)
prob = bs.LinearProblem(bs.StencilOperator(n, n, n), b, bs.Grid3D(n, n, n))
for (kind, fixed, low, high), slots in [(("fixed", 3, 0, 0), 100), (("drop_free_jitter", 0, 1, 4), 100),
                                        (("fixed", 4, 0, 0), 2)]:
    for rep in range(3):
        cfg = bs.OuterConfig(block_grid=(1, 1, 2), inner=bs.InnerSolverSpec("cg", 10), mode="async", tol=1e-7,
                             max_outer=5000, residual_check_every=2, buffer_slots=slots,
                             delay=bs.DelayModel(kind, fixed=fixed, low=low, high=high, seed=1))
        res = bs.outer_solve(prob, cfg)
        late = np.array([r.max_halo_staleness for r in res.trace.rows[10:]])
        dmin = fixed if kind == "fixed" else low
        print(kind, fixed, low, high, "slots", slots, "sweeps", res.outer_iterations, "converged", res.converged,
              "true", f"{res.final_true_residual:.2e}", "staleness", sorted(Counter(late.tolist()).items()),
              f"share >= d+1: {np.mean(late >= dmin + 1):.2f}  share >= d: {np.mean(late >= dmin):.2f}",
              dict(res.comm_events), flush=True)
