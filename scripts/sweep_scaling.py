"""Per-launch CG sweep times vs grid depth (256 x 256 x nz): separates the
fixed per-launch cost from the streaming rate."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
import paper_2009_12638_b200 as bs  # noqa: E402
from paper_2009_12638_b200.linalg import single_block_engine  # noqa: E402

its = 60
for spec in (sys.argv[1:] or ["16", "32", "64", "128", "256", "512"]):
    dims = [int(v) for v in spec.split("x")]
    nx, ny, nz = dims if len(dims) == 3 else (256, 256, dims[0])
    op = bs.StencilOperator(nx, ny, nz)
    n = op.num_rows
    b = bs.seeded_rhs(n, 0, device="cuda")
    eng = single_block_engine(op, b.device, history_cap=its)
    lib = eng.lib
    lib.bs_timing(eng.ctx, 1, None, None)
    bs.cg_solve(op, b, torch.zeros_like(b), bs.InnerSolverSpec("cg", 5, 0.0), batch=4)  # warm
    ms = (ctypes.c_double * 3)()
    cnt = (ctypes.c_longlong * 3)()
    lib.bs_timing(eng.ctx, 1, ms, cnt)  # reset counters
    bs.cg_solve(op, b, torch.zeros_like(b), bs.InnerSolverSpec("cg", its, 0.0), batch=4)
    lib.bs_timing(eng.ctx, 1, ms, cnt)
    s1 = ms[1] / cnt[1] * 1e3
    s2 = ms[2] / cnt[2] * 1e3
    print(f"{nx}x{ny}x{nz:4d} pts={n/1e6:6.1f}M  S1 {s1:7.1f} us ({40*n/s1/1e3:6.0f} GB/s)  "
          f"S2 {s2:7.1f} us ({24*n/s2/1e3:6.0f} GB/s)  ctas={eng.num_ctas}")
    eng.close()
    from paper_2009_12638_b200 import linalg
    linalg._ENGINES.clear()
