"""Per-rank proxy of config 3 at 8/N GPUs on one GPU: the inner solves of
NSLAB (default 1) 512^2 x 64 slabs — the per-GPU work of config 3 at 8/NSLAB
GPUs — CG with 100 iterations each (what every config-3 inner solve runs),
repeated; CUDA events around each solve on its stream.  BS_PERSIST selects
the run path (0 graph, 1 default)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_12638_b200.engine import BlockEngine  # noqa: E402
from paper_2009_12638_b200.problems import Box  # noqa: E402

n, nz, nslab = 512, int(os.environ.get("NZ", "64")), int(os.environ.get("NSLAB", "1"))
reps = int(os.environ.get("REPS", "10"))
dev = torch.device("cuda", 0)
owned = [Box((0, 0, s * nz), (n, n, (s + 1) * nz)) for s in range(nslab)]
eng = BlockEngine((n, n, nz * nslab), owned, 0, dev, history_cap=100)
g = torch.Generator(device=dev).manual_seed(0)
for bb in eng.blocks:
    bb.b.uniform_(-1.0, 1.0, generator=g)
st = torch.cuda.current_stream(dev)
ts = []
for i in range(reps + 2):
    for bb in eng.blocks:
        bb.x.zero_()
    eng.cg_begin(100, 0.0, "rhs")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    eng.run(max_launches=0)
    e1.record(st)
    torch.cuda.synchronize()
    if i >= 2:
        ts.append(e0.elapsed_time(e1) / 1e3)
    eng.flush()
its = eng.reports()[0].iterations_used
t = float(np.median(ts))
N = n * n * nz * nslab
hbm = 6544.3
print(f"BS_PERSIST={os.environ.get('BS_PERSIST', '1')} {nslab} slab(s) {n}x{n}x{nz}: {its} its, solve {1e3 * t:.3f} ms, "
      f"{N * its / t / 1e9:.2f} Gpts/s, frac {N * (64 * its + 32 - 24) / t / 1e9 / hbm:.3f} (INIT + its)", flush=True)
