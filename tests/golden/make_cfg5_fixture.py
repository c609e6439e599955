"""Full-size parity fixture for config 5's weak-scaling companion
(BASELINE.json configs[4]): 512^3 grid, Dirichlet u = 1 on the
z_lo face and 0 elsewhere, block_grid (2, 2, 2) with a 2-plane overlap
(L1-dilated regions of 17,171,200 points, 1/m weights), inner GMRES(30) to
tol 1e-3 relative to ||r0||, synchronous sweeps, paper residual mode.  The
first ``SWEEPS`` sweeps are computed by the oracle's matrix-free overlap
restatement (``oracle.blocksolve_oracle.outer_solve_boxes``), pinned bit for
bit to the CSR oracle (itself pinned to the unmodified reference) by
``tests/test_oracle_golden.py::test_box_oracle_equals_csr_oracle``.

Writes tests/golden/cfg5_512.json (counts, local residuals, estimates,
per-block checksums) and cfg5_512.npz (the gathered iterate at 8192 seeded
points after every sweep).  About 30 minutes on 3 worker processes:

    python tests/golden/make_cfg5_fixture.py
"""

from __future__ import annotations

import json
import multiprocessing as mp
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

from oracle import blocksolve_oracle as O  # noqa: E402

N = int(os.environ.get("CFG5_N", "512"))
BG = (2, 2, 2)
OVERLAP = 2
INNER = dict(kind="gmres", max_iterations=30, tolerance=1e-3, restart=30, basis="initial")
SWEEPS = 2
FACES = {"z_lo": 1.0}
OUT = Path(__file__).resolve().parent


def main():
    t0 = time.time()
    b = O.dirichlet_rhs(N, N, N, FACES)
    idx = np.unique(np.random.default_rng(54321).integers(0, N ** 3, 8192, dtype=np.int64))
    meta = {"n": N, "block_grid": list(BG), "overlap": OVERLAP, "faces": FACES,
            "inner": ["gmres", 30, 1e-3], "restart": 30, "basis": "initial", "residual_check_mode": "paper",
            "sweeps": [], "generator": "tests/golden/make_cfg5_fixture.py (oracle.outer_solve_boxes)"}
    samples = []

    def on_sweep(rec):
        sol = np.zeros((N, N, N))
        for box, xo in zip(rec["boxes"], rec["owned"]):
            (x0, y0, z0), (x1, y1, z1) = box
            sol[z0:z1, y0:y1, x0:x1] = xo.reshape(z1 - z0, y1 - y0, x1 - x0)
        samples.append(sol.ravel()[idx].copy())
        meta["sweeps"].append({"k": rec["k"], "its": rec["its"], "locals": rec["locals"],
                               "estimate": rec["estimate"],
                               "block_sum": [float(np.sum(xo)) for xo in rec["owned"]],
                               "block_sumsq": [float(np.sum(xo * xo)) for xo in rec["owned"]],
                               "elapsed_s": time.time() - t0})
        print(f"sweep {rec['k']}: its {rec['its']} estimate {rec['estimate']:.17g} ({time.time() - t0:.0f} s)",
              flush=True)

    with mp.get_context("fork").Pool(int(os.environ.get("CFG5_PROCS", "3"))) as pool:
        O.outer_solve_boxes((N, N, N), b, BG, OVERLAP, INNER, SWEEPS, pool=pool, on_sweep=on_sweep)
    tag = f"cfg5_{N}"
    np.savez_compressed(OUT / f"{tag}.npz", idx=idx, samples=np.stack(samples))
    with open(OUT / f"{tag}.json", "w") as fh:
        json.dump(meta, fh, indent=1)
    print(f"done in {time.time() - t0:.0f} s")


if __name__ == "__main__":
    main()
