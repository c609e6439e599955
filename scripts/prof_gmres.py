"""One GMRES(m) cycle on an n^3 single block (for ncu launch lists / timing)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2009_12638_b200 as bs  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
m = int(sys.argv[2]) if len(sys.argv) > 2 else 30
op = bs.StencilOperator(n, n, n)
b = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, n ** 3)).cuda()
spec = bs.InnerSolverSpec("gmres", m, 0.0, m)
bs.gmres_solve(op, b, torch.zeros_like(b), spec)  # warm-up (allocates the basis)
torch.cuda.synchronize()
t0 = time.perf_counter()
x, rep = bs.gmres_solve(op, b, torch.zeros_like(b), spec)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
N = n ** 3
# Arnoldi step j moves 32 + 24 (j+1) B/pt (SpMV 16, j+1 MGS passes, normalisation)
alg = sum(32 + 24 * (j + 1) for j in range(m)) * N
print(f"gmres({m}) n={n}: {rep.iterations_used} its, {dt*1e3:.1f} ms, {N*m/dt/1e9:.2f} Gpts/s, "
      f"algorithmic {alg/dt/1e9:.0f} GB/s ({alg/dt/1e9/6469.6:.2f} of HBM peak)")
