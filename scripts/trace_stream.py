"""Per-sweep structure of the streaming persistent CG kernel (BS_TRACE build,
BS_LIB=...): one 512^2 x NZ slab (the per-GPU work of config 3 at 8 GPUs) or
NSLAB slabs, CG 100 iterations.  Stamps per sweep and CTA: 0 ring ready,
1 last tile done, 3 barrier passed, 2 reduction done."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_12638_b200 as bs  # noqa: E402
from paper_2009_12638_b200.engine import BlockEngine  # noqa: E402
from paper_2009_12638_b200.problems import Box  # noqa: E402

SW, CT = 2048, 448
n, nz, nslab = 512, int(os.environ.get("NZ", "64")), int(os.environ.get("NSLAB", "1"))
dev = torch.device("cuda", 0)
owned = [Box((0, 0, s * nz), (n, n, (s + 1) * nz)) for s in range(nslab)]
eng = BlockEngine((n, n, nz * nslab), owned, 0, dev, history_cap=100)
for bb in eng.blocks:
    bb.b.copy_(torch.rand_like(bb.b))
for rep in range(2):
    for bb in eng.blocks:
        bb.x.zero_()
    eng.cg_begin(100, 0.0, "rhs")
    eng.run(max_launches=0)
    torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (SW * 8 * CT))()
eng.lib.bs_strace_read(buf)
t = np.frombuffer(buf, dtype=np.uint64).reshape(SW, 8, CT).astype(np.int64)
nsw = 1 + 2 * 100
ncta = int((t[1, 0] > 0).sum())
t = t[:nsw, :, :ncta]
S = [t[:, i] / 1e3 for i in range(7)]
clk = t[:, 7, 0] & ((1 << 48) - 1)
mhz = np.diff(clk) / np.diff(t[:, 0, 0]) * 1e3
print(f"{nslab} slab(s) {n}x{n}x{nz}, {eng.num_ctas} tiles, {ncta} CTAs (traced); per-CTA medians of phase lengths in us")
for kind, sel in (("S1", np.arange(1, nsw - 1, 2)), ("S2", np.arange(2, nsw - 1, 2))):
    st, done = S[0][sel], S[1][sel]
    stream = np.median(done, axis=1) - st.max(axis=1)
    tail = done.max(axis=1) - np.median(done, axis=1)
    ph = {name: np.median(S[j][sel] - S[i][sel], axis=1).mean() for name, i, j in
          (("inval+arrive", 1, 2), ("spin", 2, 3), ("load-sum", 3, 4), ("tree", 4, 5), ("transition", 5, 6))}
    nxt = (S[0][sel + 1] - S[6][sel]).mean()
    period = st.max(axis=1)
    period = (S[0][sel + 1].max(axis=1) - period).mean()
    print(f"{kind}: stream {stream.mean():6.1f} tail {tail.mean():5.1f} " +
          " ".join(f"{k} {v:5.2f}" for k, v in ph.items()) +
          f" ->next {nxt:5.2f} period {period:6.1f}  SM {mhz[sel].mean():5.0f} MHz")
