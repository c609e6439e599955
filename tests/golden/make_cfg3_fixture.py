"""Full-size parity fixture for config 3 (BASELINE.json configs[2]).

512^3 grid, seeded rhs U[-1, 1] (default_rng(0), x-fastest), zero Dirichlet
boundary, x0 = 0, block_grid (1, 1, 8) = eight z-slabs of 64 planes, inner
CG(100, tol 1e-3 relative to ||r0||), synchronous sweeps, paper residual
mode.  The first ``SWEEPS`` sweeps are computed by the oracle's matrix-free
slab restatement (``oracle.blocksolve_oracle.outer_solve_slabs``), which is
pinned bit for bit to the CSR oracle (itself pinned to the unmodified
reference) by ``tests/test_oracle_golden.py::test_slab_oracle_equals_csr_oracle``.
The reference itself cannot build a 512^3 operator (>60 GB).

Writes ``tests/golden/cfg3_512.json`` (counts, local residuals, estimates,
per-slab checksums) and ``tests/golden/cfg3_512.npz`` (the iterate at 8192
seeded sample points after every sweep).  About 10 minutes on 8 cores:

    python tests/golden/make_cfg3_fixture.py
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

N = 512
NSLABS = 8
MAX_ITS = 100
TOL = 1e-3
SWEEPS = 3
NSAMPLE = 8192
OUT = Path(__file__).resolve().parent


def sample_indices(n: int = N, count: int = NSAMPLE) -> np.ndarray:
    """Fixed sample points: every slab's two face planes are over-represented
    (they carry the coupling), the rest uniform."""
    rng = np.random.default_rng(12345)
    return np.unique(rng.integers(0, n ** 3, count, dtype=np.int64))


def main():
    t0 = time.time()
    b = O.seeded_rhs(N ** 3, 0)
    idx = sample_indices()
    meta = {"n": N, "nslabs": NSLABS, "inner": ["cg", MAX_ITS, TOL], "basis": "initial",
            "residual_check_mode": "paper", "seed": 0, "sweeps": [],
            "generator": "tests/golden/make_cfg3_fixture.py (oracle.outer_solve_slabs)"}
    samples = []

    def on_sweep(rec):
        x = np.concatenate([xx.ravel() for xx in rec["x"]])
        samples.append(x[idx].copy())
        meta["sweeps"].append({
            "k": rec["k"], "its": rec["its"], "locals": rec["locals"], "estimate": rec["estimate"],
            "slab_sum": [float(np.sum(xx)) for xx in rec["x"]],
            "slab_sumsq": [float(np.sum(xx * xx)) for xx in rec["x"]],
            "elapsed_s": time.time() - t0})
        print(f"sweep {rec['k']}: its {rec['its']} estimate {rec['estimate']:.17g} "
              f"({time.time() - t0:.0f} s)", flush=True)

    with mp.get_context("fork").Pool(min(NSLABS, os.cpu_count() or 1)) as pool:
        O.outer_solve_slabs((N, N, N), b, NSLABS, MAX_ITS, TOL, "initial", SWEEPS, pool=pool, on_sweep=on_sweep)
    np.savez_compressed(OUT / "cfg3_512.npz", idx=idx, samples=np.stack(samples))
    with open(OUT / "cfg3_512.json", "w") as fh:
        json.dump(meta, fh, indent=1)
    print(f"done in {time.time() - t0:.0f} s")


if __name__ == "__main__":
    main()
