"""Per-window averages over a full config-2 solve in the persistent kernel
(BS_TRACE build): S1/S2 fill->done, tail, barrier and the SM clock (from
clock64 vs globaltimer of CTA 0 across a sweep)."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2009_12638_b200 as bs  # noqa: E402
from paper_2009_12638_b200 import _lib  # noqa: E402
from paper_2009_12638_b200.linalg import single_block_engine  # noqa: E402

SW, CT = 2048, 296
n = 256
op = bs.StencilOperator(n, n, n)
b = bs.seeded_rhs(op.num_rows, 0, device="cuda")
eng = single_block_engine(op, b.device, history_cap=5000)
nctas = eng.num_ctas
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 1):
    bs.cg_solve(op, b, torch.zeros_like(b), bs.InnerSolverSpec("cg", 5000, 1e-8))
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (SW * 5 * CT))()
_lib.check(eng.lib.bs_ptrace_read(buf))
t = np.frombuffer(buf, dtype=np.uint64).reshape(SW, 5, CT)[:, :, :nctas].astype(np.int64)
nsw = 1 + 2 * 856 + 1
t = t[:nsw]
st, done, part, rel = (t[:, i] / 1e3 for i in range(4))
clk = t[:, 4, 0] & ((1 << 48) - 1)
sm = t[0, 4] >> 48
mhz = np.diff(clk) / np.diff(t[:, 0, 0]) * 1e3
for lo in range(1, nsw - 2, 200):
    idx = np.arange(lo, min(lo + 200, nsw - 2))
    for kind, sel in (("S1", idx[idx % 2 == 1]), ("S2", idx[idx % 2 == 0])):
        fd = np.median(done[sel], axis=1) - st[sel].max(axis=1)
        tail = done[sel].max(axis=1) - np.median(done[sel], axis=1)
        bar = rel[sel].min(axis=1) - part[sel].max(axis=1)
        spread = st[sel].max(axis=1) - st[sel].min(axis=1)
        epi = part[sel].max(axis=1) - done[sel].max(axis=1)
        red = st[sel + 1].min(axis=1) - rel[sel].max(axis=1)
        period = st[sel + 1].max(axis=1) - st[sel].max(axis=1)
        print(f"sweeps {lo:4d}-{idx[-1]:4d} {kind}: fill->done {fd.mean():6.1f}  tail {tail.mean():5.1f}  "
              f"barrier {bar.mean():5.1f}  start-spread {spread.mean():4.1f}  epi {epi.mean():4.1f}  reduce {red.mean():4.1f}  "
              f"period {period.mean():6.1f}  SM MHz {mhz[sel].mean():6.0f}")

# which CTAs finish late: lateness vs. how many CTAs share the SM
sel = np.arange(1, nsw - 2)
late = (done[sel] - np.median(done[sel], axis=1, keepdims=True)).mean(axis=0)
share = np.array([(sm == s).sum() for s in sm])
for c in (1, 2):
    m = share == c
    if m.any():
        print(f"CTAs sharing an SM with {c - 1} other: {m.sum():3d}  mean lateness {late[m].mean():5.2f} us  "
              f"max {late[m].max():5.2f}")
order = np.argsort(late)[::-1][:12]
print("latest CTAs (cta, sm, share, lateness):", [(int(i), int(sm[i]), int(share[i]), round(float(late[i]), 2)) for i in order])
# lateness by tile column (ix = tile % tiles_x; S2 walks the tiles in reverse order)
tx = 256 // 32 if n == 256 else None
if tx:
    for kind, sel in (("S1", np.arange(1, nsw - 2, 2)), ("S2", np.arange(2, nsw - 2, 2))):
        lt = (done[sel] - np.median(done[sel], axis=1, keepdims=True)).mean(axis=0)
        tiles = np.arange(nctas) if kind == "S1" else nctas - 1 - np.arange(nctas)
        print(kind, "lateness by tile ix:", [round(float(lt[tiles % tx == i].mean()), 2) for i in range(tx)])
        iy = tiles // tx
        print(kind, "lateness by tile iy (first/last 4):", [round(float(lt[iy == i].mean()), 2) for i in (0, 1, 2, 3, 28, 29, 30, 31)])
