"""BS_TRACE build: per-CTA stamps of one residual sweep (bs_residual) at n^3."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2009_12638_b200 as bs  # noqa: E402
from paper_2009_12638_b200 import _lib  # noqa: E402
from paper_2009_12638_b200.linalg import single_block_engine  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
op = bs.StencilOperator(n, n, n)
b = bs.seeded_rhs(op.num_rows, 0, device="cuda")
eng = single_block_engine(op, b.device, history_cap=8)
eng.blocks[0].put("b", b)
lib = eng.lib
nctas = eng.num_ctas
for _ in range(3):
    eng.residual()
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (5 * nctas))()
_lib.check(lib.bs_trace_read(buf, nctas))
t = np.frombuffer(buf, dtype=np.uint64).reshape(5, nctas).astype(np.int64)[:4]
rel = (t - t[0].min()) / 1e3
for i, nm in enumerate(["entry", "first-data", "last-plane", "done"]):
    print(f"  {nm:11s} min {rel[i].min():8.2f}  med {np.median(rel[i]):8.2f}  max {rel[i].max():8.2f} us")
