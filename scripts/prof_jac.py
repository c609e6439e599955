"""Point-Jacobi sweeps and a residual sweep at n^3 in launch mode (one kernel
per sweep, visible to ncu; the default graph path hides them in a device loop)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2009_12638_b200 as bs  # noqa: E402
from paper_2009_12638_b200.linalg import single_block_engine  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
op = bs.StencilOperator(n, n, n)
b = bs.seeded_rhs(op.num_rows, 0, device="cuda")
eng = single_block_engine(op, b.device, history_cap=256)
eng.lib.bs_timing(eng.ctx, 1, None, None)
bb = eng.blocks[0]
bb.put("b", b)
bb.put("x", torch.zeros_like(b))
eng.residual()
eng.jacobi_begin(10, 0.0)
eng.run(batch=1, max_launches=0)
torch.cuda.synchronize()
print("ok")
