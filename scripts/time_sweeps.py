"""CUDA-event times of single sweeps at n^3 (or nx ny nz; one block): the residual sweep
(bs_residual), a point-Jacobi solve of K sweeps, and the GMRES cycle."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2009_12638_b200 as bs  # noqa: E402
from paper_2009_12638_b200.linalg import single_block_engine  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
shape = (n, int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (n, n, n)  # nx ny nz
N = shape[0] * shape[1] * shape[2]
op = bs.StencilOperator(*shape)
b = bs.seeded_rhs(N, 0, device="cuda")
eng = single_block_engine(op, b.device, history_cap=256)
bb = eng.blocks[0]
bb.put("b", b)
bb.put("x", torch.zeros_like(b))
s = torch.cuda.current_stream()


def ev_time(fn, reps):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


t = ev_time(lambda: eng.residual(), 20)
print(f"residual sweep: {t:.1f} us  ({24 * N / t / 1e3:.0f} GB/s at 24 B/pt)")
K = 100


def jac():
    eng.jacobi_begin(K, 0.0)
    eng.run(batch=8, max_launches=0)


t = ev_time(jac, 3)
print(f"jacobi: {t / (K + 1):.1f} us per sweep ({24 * N / (t / (K + 1)) / 1e3:.0f} GB/s at 24 B/pt)")

xp, yp = bb.zeros_pitched(), bb.zeros_pitched()
xp.copy_(torch.rand_like(xp))
t = ev_time(lambda: eng.apply(0, xp, yp), 50)
print(f"spmv: {t:.1f} us  ({16 * N / t / 1e3:.0f} GB/s at 16 B/pt)")
