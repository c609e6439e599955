"""Timeline of the persistent CG kernel (BS_TRACE build): per sweep, the
spread of tile-done / partials / barrier-release stamps across CTAs."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2009_12638_b200 as bs  # noqa: E402
from paper_2009_12638_b200 import _lib  # noqa: E402
from paper_2009_12638_b200.linalg import single_block_engine  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
its = int(sys.argv[2]) if len(sys.argv) > 2 else 12
op = bs.StencilOperator(n, n, n)
b = bs.seeded_rhs(op.num_rows, 0, device="cuda")
eng = single_block_engine(op, b.device, history_cap=64)
lib = eng.lib
nctas = eng.num_ctas
bs.cg_solve(op, b, torch.zeros_like(b), bs.InnerSolverSpec("cg", its, 0.0))
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (24 * 4 * 512))()
_lib.check(lib.bs_ptrace_read(buf))
t = np.frombuffer(buf, dtype=np.uint64).reshape(24, 4, 512)[:, :, :nctas].astype(np.int64)
order = np.argsort(t[:, 0, 0])  # ring buffer: sort sweeps by start time
t = t[order]
t0 = t[0, 0].min()
rel = (t - t0) / 1e3
prev_release = rel[0, 0].min()
for sw in range(0, 24):
    if rel[sw, 0].max() <= 0:
        continue
    st, done, part, rel_ = rel[sw]
    print(f"sweep {sw:2d}: start {st.min():8.1f}..{st.max():8.1f}  tiles-done med {np.median(done):8.1f} "
          f"max {done.max():8.1f}  partials max {part.max():8.1f}  released {rel_.min():8.1f}..{rel_.max():8.1f}"
          f"  | sweep {rel_.max() - prev_release:6.1f} us, tail {done.max() - np.median(done):5.1f}, "
          f"barrier {rel_.min() - part.max():5.1f}, fill->done {np.median(done) - st.max():6.1f}")
    prev_release = rel_.max()
