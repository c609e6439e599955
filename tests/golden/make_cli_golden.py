"""Golden outputs of the UNMODIFIED reference CLI (``blocksolve run / sweep /
compare``, /root/reference/pkg/src/blocksolve/cli.py) for small sync
configurations, for the device CLI's parity tests (tests/test_cli.py).

    python tests/golden/make_cli_golden.py

Writes tests/golden/cli/: the traces and summaries of a ``run`` and of a
``sweep``, and the table + CSV of a ``compare`` over traces of different
configurations.  Replay execution, so the trace's time column is the outer
iteration index and the files are deterministic.
"""

from __future__ import annotations

import contextlib
import io
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, "/root/reference/pkg/src")
from blocksolve.cli import main  # noqa: E402  (reference, read-only)

OUT = Path(__file__).resolve().parent / "cli"
# Configurations whose traces are numerically stable: a dot-product
# reassociation (OpenBLAS -> pairwise) moves the reference's own per-sweep
# estimates by <= 1.3e-10 relative here.  (With fixed 10 CG iterations on
# 12 x 12 x 6 blocks it moves them by 4.7e-4 after 18 sweeps: chaotic
# amplification of roundoff by the inner solver, not a property of either
# implementation.)
RUN = ["--nx", "12", "--ny", "12", "--nz", "12", "--gz", "2", "--inner", "cg", "--inner-its", "40",
       "--tol", "1e-6", "--boundary", "faces:z_lo=1,x_hi=0.5"]
SWEEP = ["--nx", "12", "--ny", "12", "--nz", "12", "--inner", "cg", "--inner-its", "40", "--tol", "1e-6",
         "--axis", "block_grid", "--values", "1,1,2;1,2,2;2,2,2"]


def call(argv):
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        code = main(argv)
    return code, buf.getvalue()


def main_():
    OUT.mkdir(exist_ok=True)
    os.chdir(OUT)
    meta = {}
    code, text = call(["run"] + RUN + ["--out", "run_trace.csv"])
    meta["run"] = {"argv": RUN, "code": code, "stdout": text, "trace": "run_trace.csv"}
    code, text = call(["run"] + RUN + ["--inner-its", "4", "--max-outer", "7", "--out", "run_capped.csv"])
    meta["run_capped"] = {"argv": RUN + ["--inner-its", "4", "--max-outer", "7"], "code": code, "stdout": text,
                          "trace": "run_capped.csv"}
    code, text = call(["sweep"] + SWEEP + ["--out", "sweep.csv", "--summary-out", "sweep_summary.csv"])
    meta["sweep"] = {"argv": SWEEP, "code": code, "stdout": text, "summary": "sweep_summary.csv",
                     "traces": sorted(p.name for p in OUT.glob("sweep_block_grid_*.csv"))}
    traces = ["run_trace.csv", "run_capped.csv"] + meta["sweep"]["traces"]
    code, text = call(["compare"] + traces + ["--reference", "sweep_block_grid_1x1x2.csv", "--out", "compare.csv"])
    meta["compare"] = {"traces": traces, "reference": "sweep_block_grid_1x1x2.csv", "code": code, "stdout": text,
                       "csv": "compare.csv"}
    (OUT / "cli_golden.json").write_text(json.dumps(meta, indent=1))
    print(json.dumps({k: v["code"] for k, v in meta.items()}))


if __name__ == "__main__":
    main_()
