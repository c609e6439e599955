"""One short 256^3 CG solve through the persistent kernel (for ncu)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2009_12638_b200 as bs  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
its = int(sys.argv[2]) if len(sys.argv) > 2 else 20
op = bs.StencilOperator(n, n, n)
b = bs.seeded_rhs(op.num_rows, 0, device="cuda")
x, rep = bs.cg_solve(op, b, torch.zeros_like(b), bs.InnerSolverSpec("cg", its, 0.0))
torch.cuda.synchronize()
print("its", rep.iterations_used, rep.stop_reason)
