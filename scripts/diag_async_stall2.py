"""Why do the other blocks sometimes stop while one block's host thread sleeps?  Same scenario as
diag_async_stall.py with per-sweep timestamps per block and a log of every board estimate below tol."""
import sys
import threading
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2009_12638_b200 as bs  # noqa: E402
from paper_2009_12638_b200 import async_driver  # noqa: E402

n = 32
b = bs.seeded_rhs(n ** 3, 0)
prob = bs.LinearProblem(bs.StencilOperator(n, n, n), b, bs.Grid3D(n, n, n))
stamps, low, lock = {}, [], threading.Lock()
orig = async_driver._Board.estimate


def estimate(self):
    v = orig(self)
    if v < 1e-8:
        with lock:
            low.append((time.perf_counter(), threading.current_thread().name, v, np.array(self.local_sq).copy(),
                        list(self.progress)))
    return v


async_driver._Board.estimate = estimate


def hook(blk, k):
    with lock:
        stamps.setdefault(blk, []).append(time.perf_counter())
    if blk == 3 and k == 5:
        time.sleep(2.0)


for rep in range(4):
    stamps.clear()
    low.clear()
    async_driver.SWEEP_HOOK = hook
    cfg = bs.OuterConfig(block_grid=(1, 1, 8), inner=bs.InnerSolverSpec("cg", 20), mode="async", tol=1e-8,
                         max_outer=200000, residual_check_every=1)
    t0 = time.perf_counter()
    res = bs.outer_solve(prob, cfg)
    wake = stamps[3][5] + 2.0
    others = max(sum(1 for t in stamps[q] if t < wake) for q in stamps if q != 3)
    print(f"rep {rep}: others_during_stall={others} sweeps={res.outer_iterations} solve={time.perf_counter() - t0:.2f}s")
    for q in sorted(stamps):
        ts = np.array(stamps[q])
        gaps = np.diff(ts)
        i = int(np.argmax(gaps)) if len(gaps) else 0
        print(f"   block {q}: {len(ts)} sweeps, longest gap {gaps[i]:.3f}s after sweep {i} (t={ts[i] - t0:.3f}s)")
    for t, name, v, sq, prog in low[:3]:
        print(f"   estimate {v:.3e} < tol at t={t - t0:.3f}s by {name}: progress {prog} local_sq {np.array2string(sq, precision=2)}")
    print(f"   {len(low)} estimates below tol; first at t={low[0][0] - t0:.3f}s" if low else "   no estimate below tol", flush=True)
