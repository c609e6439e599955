"""One 256^3 config-2 CG solve for ncu (sweep kernels launched from the host)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2009_12638_b200 as bs  # noqa: E402
from paper_2009_12638_b200.linalg import single_block_engine  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
its = int(sys.argv[2]) if len(sys.argv) > 2 else 20
op = bs.StencilOperator(n, n, n)
b = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, n ** 3)).cuda()
eng = single_block_engine(op, b.device, history_cap=its)
eng.lib.bs_timing(eng.ctx, 1, None, None)  # launch mode: one kernel launch per sweep
x, rep = bs.cg_solve(op, b, torch.zeros_like(b), bs.InnerSolverSpec("cg", its, 0.0), batch=4)
torch.cuda.synchronize()
print("its", rep.iterations_used, rep.stop_reason)
