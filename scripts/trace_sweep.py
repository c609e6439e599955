"""Where does a CG sweep's time go?  Needs a BS_TRACE build (BS_LIB=...):
per-CTA entry / first-stage / last-plane / epilogue-done stamps of the last
S1 and S2 launches of a short 256^3 CG run (launch mode)."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2009_12638_b200 as bs  # noqa: E402
from paper_2009_12638_b200 import _lib  # noqa: E402
from paper_2009_12638_b200.linalg import single_block_engine  # noqa: E402

dims = [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "256").split("x")]
nx, ny, nz = dims if len(dims) == 3 else (256, 256, dims[0])
op = bs.StencilOperator(nx, ny, nz)
b = bs.seeded_rhs(op.num_rows, 0, device="cuda")
eng = single_block_engine(op, b.device, history_cap=64)
lib = eng.lib
lib.bs_trace_read.argtypes = [ctypes.c_void_p, ctypes.c_int]
nctas = eng.num_ctas
lib.bs_timing(eng.ctx, 1, None, None)
for its in (3, 4):  # odd/even: the last launch is S2 after 3 its... read after each
    bs.cg_solve(op, b, torch.zeros_like(b), bs.InnerSolverSpec("cg", its, 0.0), batch=1)
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * (5 * nctas))()
    _lib.check(lib.bs_trace_read(buf, nctas))
    t = np.frombuffer(buf, dtype=np.uint64).reshape(5, nctas).astype(np.int64)
    sm = t[4]
    t = t[:4]
    t0 = t[0].min()
    rel = (t - t0) / 1e3
    names = ["entry", "first-data", "last-plane", "done"]
    print(f"nz={nz} its={its} ctas={nctas}")
    for i, nm in enumerate(names):
        print(f"  {nm:11s} min {rel[i].min():7.2f}  med {np.median(rel[i]):7.2f}  max {rel[i].max():7.2f} us")
    d_fill, d_stream, d_epi = rel[1] - rel[0], rel[2] - rel[1], rel[3] - rel[2]
    print(f"  per CTA (median): fill {np.median(d_fill):6.2f}  stream {np.median(d_stream):7.2f}  "
          f"epilogue {np.median(d_epi):6.2f} us;  SM-time busy {(rel[3] - rel[0]).sum():.0f} us "
          f"over {len(set(t[0].tolist()) and set(sm.tolist()))} SMs x {rel[3].max():.1f} us span")
    tiles_x = (nx + 31) // 32
    ix = np.arange(nctas) % tiles_x
    iy = np.arange(nctas) // tiles_x
    lp = rel[2]
    print("  by x-tile :", " ".join(f"{lp[ix == v].mean():6.1f}" for v in range(tiles_x)))
    q = np.array_split(np.arange(iy.max() + 1), 8)
    print("  by y-band :", " ".join(f"{lp[np.isin(iy, g)].mean():6.1f}" for g in q))
    smb = np.array_split(np.arange(sm.max() + 1), 8)
    print("  by SM band:", " ".join(f"{lp[np.isin(sm, g)].mean():6.1f}" for g in smb))
    print("  by SM parity:", " ".join(f"{lp[sm % 2 == v].mean():6.1f}" for v in range(2)))
    per_sm = np.bincount(sm, minlength=sm.max() + 1)
    share = per_sm[sm]
    for k in sorted(set(share.tolist())):
        sel = share == k
        print(f"  CTAs sharing an SM = {k}: n={sel.sum():3d}  last-plane mean {rel[2][sel].mean():7.2f} "
              f"min {rel[2][sel].min():7.2f} max {rel[2][sel].max():7.2f}")
