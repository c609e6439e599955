"""How many sweeps the other blocks of an asynchronous solve complete while one block is suspended for 2 s
(tests/test_gpu_async_protocol.py::test_suspended_block_in_async_solve), and the async sweep rate."""
import sys
import threading
import time

sys.path.insert(0, ".")
import paper_2009_12638_b200 as bs  # noqa: E402
from paper_2009_12638_b200 import async_driver  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
b = bs.seeded_rhs(n ** 3, 0)
prob = bs.LinearProblem(bs.StencilOperator(n, n, n), b, bs.Grid3D(n, n, n))
progress, lock = {}, threading.Lock()


def hook(blk, k):
    with lock:
        progress[blk] = k
    if blk == 3 and k == 5:
        time.sleep(2.0)
        with lock:
            progress["others"] = max(v for key, v in progress.items() if isinstance(key, int) and key != 3)


for rep in range(3):
    progress.clear()
    async_driver.SWEEP_HOOK = hook
    cfg = bs.OuterConfig(block_grid=(1, 1, 8), inner=bs.InnerSolverSpec("cg", 20), mode="async", tol=1e-8,
                         max_outer=200000, residual_check_every=1)
    t = time.perf_counter()
    res = bs.outer_solve(prob, cfg)
    dt = time.perf_counter() - t
    print(time.strftime("%Y/%m/%d %H:%M:%S"), f"n={n} others_during_stall={progress.get('others')} sweeps={res.outer_iterations} converged={res.converged} "
          f"solve={dt:.2f}s", flush=True)
