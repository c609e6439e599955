"""Device path of the experiment harness.

``python -m paper_2009_12638_b200 run --nx 64 --ny 64 --nz 64 --gz 2 --inner cg
--inner-its 50 --tolerance-basis initial --tol 1e-6 --out trace.csv``

Mirrors the reference ``blocksolve`` harness (cli.py:263-586): the
subcommands ``run`` (one solve), ``sweep`` (one solve per value of an axis:
block_grid, inner_max_its, overlap or mode, everything else — seed included —
fixed; cli.py:390-424) and ``compare`` (iteration counts, rates and ratios of
residual traces against a reference trace; cli.py:440-517), the same flags,
the optional ``--config key=value`` file layered under the flags, the same
CSV trace schema and the same exit codes (0 converged, 2 stopped on the
outer-iteration cap, 1 on any configuration or solver error).  Additions:
``--tolerance-basis`` and ``--device``.  ``mode=baseline`` runs the inner
solver alone on the whole grid (cli.py:268-290).  Every solve runs on the
GPU; ``compare`` only reads CSV files.
"""

from __future__ import annotations

import argparse
import sys
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .errors import ConfigurationError, DeviceError, ProtocolError, SolverBreakdownError
from .inner_solvers import InnerSolverSpec, solve
from .multisplit import DelayModel, OuterConfig, ResidualTrace, TraceRow, outer_solve
from .problems import FACES, DirichletBoundary, Grid3D, build_laplace_3d

DEFAULTS = {
    "nx": "8", "ny": "8", "nz": "8", "boundary": "faces:x_lo=1", "gx": "1", "gy": "1", "gz": "1",
    "overlap": "0", "inner": "gmres", "inner_its": "10", "inner_tol": "0", "restart": "", "mode": "sync",
    "R": "100", "tol": "1e-6", "max_outer": "5000", "residual_mode": "paper", "true_res_every": "10",
    "exec": "replay", "out": "trace.csv", "tolerance_basis": "rhs", "device": "cuda", "delay": "none",
    "seed": "0",
}
AXES = ("block_grid", "inner_max_its", "overlap", "mode")


def _int(raw: str, key: str) -> int:
    try:
        return int(raw)
    except ValueError:
        raise ConfigurationError(f"{key}: invalid integer {raw!r}") from None


def _float(raw: str, key: str) -> float:
    try:
        return float(raw)
    except ValueError:
        raise ConfigurationError(f"{key}: invalid number {raw!r}") from None


def boundary_from(raw: str) -> DirichletBoundary:
    """``const:v`` or ``faces:x_lo=1,y_hi=0.5`` (cli.py:111-127)."""
    if raw.startswith("const:"):
        return DirichletBoundary.constant(_float(raw[len("const:"):], "boundary"))
    if raw.startswith("faces:"):
        faces = {}
        for item in filter(None, raw[len("faces:"):].split(",")):
            name, _, value = item.partition("=")
            if name not in FACES:
                raise ConfigurationError(f"boundary: unknown face {name!r}")
            faces[name] = _float(value, "boundary")
        return DirichletBoundary(faces)
    raise ConfigurationError(f"boundary: expected const:v or faces:name=v,... got {raw!r}")


def parse_delay(raw: str, seed: int) -> DelayModel:
    """``none``, ``fixed:d``, ``uniform:lo:hi`` or ``jitter:lo:hi`` (cli.py:82-100)."""
    parts = raw.split(":")
    kind = parts[0]
    try:
        if kind == "none" and len(parts) == 1:
            return DelayModel(seed=seed)
        if kind == "fixed" and len(parts) == 2:
            return DelayModel("fixed", fixed=int(parts[1]), seed=seed)
        if kind == "uniform" and len(parts) == 3:
            return DelayModel("uniform", low=int(parts[1]), high=int(parts[2]), seed=seed)
        if kind in ("jitter", "drop_free_jitter") and len(parts) == 3:
            return DelayModel("drop_free_jitter", low=int(parts[1]), high=int(parts[2]), seed=seed)
    except ValueError:
        raise ConfigurationError(f"delay: invalid delay bounds in {raw!r}") from None
    raise ConfigurationError(f"delay: expected none, fixed:d, uniform:lo:hi or jitter:lo:hi, got {raw!r}")


def read_config_file(path: str) -> dict:
    out = {}
    with open(path) as fh:
        for n, line in enumerate(fh, 1):
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            key, sep, value = line.partition("=")
            if not sep:
                raise ConfigurationError(f"config: line {n} is not key=value: {line!r}")
            out[key.strip()] = value.strip()
    return out


def resolve_config(file_path=None, flags=None) -> dict:
    """Defaults < config file < flags, validated (cli.py:162-186)."""
    cfg = dict(DEFAULTS)
    if file_path:
        file_cfg = read_config_file(file_path)
        unknown = sorted(set(file_cfg) - set(DEFAULTS))
        if unknown:
            raise ConfigurationError(f"{unknown[0]}: unknown configuration key")
        cfg.update(file_cfg)
    cfg.update({k: v for k, v in (flags or {}).items() if k in DEFAULTS and v is not None})
    if cfg["mode"] not in ("baseline", "sync", "async"):
        raise ConfigurationError(f"mode: unknown mode {cfg['mode']!r}")
    if cfg["residual_mode"] not in ("paper", "true"):
        raise ConfigurationError(f"residual_mode: unknown mode {cfg['residual_mode']!r}")
    if cfg["exec"] not in ("replay", "threads"):
        raise ConfigurationError(f"exec: unknown execution {cfg['exec']!r}")
    return cfg


@dataclass
class RunSummary:
    """One run's outcome, consistent with the trace it wrote (cli.py:251-260)."""

    outer_iterations: int
    total_inner_iterations: int
    iterations_per_second: float | None
    final_true_residual: float
    converged: bool
    trace_path: str


def run_config(cfg: dict) -> RunSummary:
    """Execute one configured solve on the GPU and write its CSV trace."""
    grid = Grid3D(_int(cfg["nx"], "nx"), _int(cfg["ny"], "ny"), _int(cfg["nz"], "nz"), boundary_from(cfg["boundary"]))
    problem = build_laplace_3d(grid)
    restart = None if cfg["restart"] == "" else _int(cfg["restart"], "restart")
    mode = cfg["mode"]
    rate = None
    if mode == "baseline":
        spec = InnerSolverSpec(cfg["inner"], _int(cfg["max_outer"], "max_outer"), _float(cfg["tol"], "tol"), restart)
        x, rep = solve(problem.matrix, problem.rhs, np.zeros(grid.num_unknowns), spec,
                       tolerance_basis=cfg["tolerance_basis"])
        if rep.stop_reason == "breakdown":
            raise SolverBreakdownError(0, rep.iterations_used, "baseline solver breakdown")
        from .linalg import residual_norms

        final = residual_norms(problem.matrix, x, problem.rhs)[1]
        rows = [TraceRow(i, float(i), rel, None, 1, 0) for i, rel in enumerate(rep.residual_history)]
        if rows:
            rows[-1].true_residual = final
        trace, converged, outer, inner = ResidualTrace(rows), rep.stop_reason == "tolerance_met", \
            rep.iterations_used, rep.iterations_used
    else:
        config = OuterConfig(
            block_grid=(_int(cfg["gx"], "gx"), _int(cfg["gy"], "gy"), _int(cfg["gz"], "gz")),
            overlap=_int(cfg["overlap"], "overlap"),
            inner=InnerSolverSpec(cfg["inner"], _int(cfg["inner_its"], "inner_its"),
                                  _float(cfg["inner_tol"], "inner_tol"), restart),
            mode=mode, buffer_slots=_int(cfg["R"], "R"), tol=_float(cfg["tol"], "tol"),
            max_outer=_int(cfg["max_outer"], "max_outer"), residual_check_mode=cfg["residual_mode"],
            true_residual_interval=_int(cfg["true_res_every"], "true_res_every"), execution=cfg["exec"],
            tolerance_basis=cfg["tolerance_basis"], device=cfg["device"],
            delay=parse_delay(cfg["delay"], _int(cfg["seed"], "seed")))
        res = outer_solve(problem, config)
        trace, converged, outer = res.trace, res.converged, res.outer_iterations
        inner = sum(r.inner_iterations for r in trace.rows)
        final = res.final_true_residual
        elapsed = trace.rows[-1].time if trace.rows else 0.0
        if cfg["exec"] == "threads" and elapsed > 0:  # wall-clock times only in threads mode
            rate = outer / elapsed
    trace.write_csv(cfg["out"])
    return RunSummary(outer, inner, rate, final, converged, cfg["out"])


def run(cfg: dict) -> tuple:
    """Execute one solve; returns (exit code, summary text)."""
    s = run_config(cfg)
    return (0 if s.converged else 2), format_summary(s)


def format_summary(s: RunSummary) -> str:
    rate = f"{s.iterations_per_second:.2f} it/s" if s.iterations_per_second is not None else "-"
    return "\n".join([
        f"{'outer iterations':<24}{s.outer_iterations}",
        f"{'total inner iterations':<24}{s.total_inner_iterations}",
        f"{'iteration rate':<24}{rate}",
        f"{'final true residual':<24}{s.final_true_residual:.6e}",
        f"{'converged':<24}{'yes' if s.converged else 'no (max_outer reached)'}",
        f"{'trace':<24}{s.trace_path}",
    ])


# ------------------------------------------------------------------ sweep


def axis_values(axis: str, raw: str) -> list:
    """Parsed values of a sweep axis (cli.py:334-356): block grids as
    ``gx,gy,gz`` separated by ``;``, integers or modes as comma lists."""
    if axis not in AXES:
        raise ConfigurationError(f"axis: must be one of {', '.join(AXES)}")
    if axis == "block_grid":
        grids = []
        for item in raw.split(";"):
            dims = [p for p in item.split(",") if p]
            if len(dims) != 3:
                raise ConfigurationError(f"values: block grid {item!r} is not gx,gy,gz")
            grids.append(tuple(_int(d, "values") for d in dims))
        return grids
    items = [p for p in raw.split(",") if p]
    if axis == "mode":
        bad = [m for m in items if m not in ("baseline", "sync", "async")]
        if bad:
            raise ConfigurationError(f"values: unknown mode {bad[0]!r}")
        return items
    return [_int(p, "values") for p in items]


def axis_tag(axis: str, value) -> str:
    return "x".join(str(v) for v in value) if axis == "block_grid" else str(value)


def with_axis(cfg: dict, axis: str, value) -> dict:
    out = dict(cfg)
    if axis == "block_grid":
        out["gx"], out["gy"], out["gz"] = (str(v) for v in value)
    elif axis == "inner_max_its":
        out["inner_its"] = str(value)
    else:
        out[axis] = str(value)
    return out


def sweep(cfg: dict, axis: str, values_raw: str) -> list:
    """One solve per axis value; the trace of value v goes to
    ``<stem>_<axis>_<tag><suffix>`` next to ``out`` (cli.py:390-406)."""
    values = axis_values(axis, values_raw)
    out = Path(cfg["out"])
    results = []
    for v in values:
        tag = axis_tag(axis, v)
        c = with_axis(cfg, axis, v)
        c["out"] = str(out.with_name(f"{out.stem}_{axis}_{tag}{out.suffix}"))
        results.append((tag, run_config(c)))
    return results


def format_sweep(axis: str, results: list) -> str:
    lines = [f"{axis:<16}{'outer':>8}{'inner':>10}{'final_true_residual':>22}{'converged':>11}"]
    for tag, s in results:
        lines.append(f"{tag:<16}{s.outer_iterations:>8}{s.total_inner_iterations:>10}"
                     f"{s.final_true_residual:>22.6e}{'yes' if s.converged else 'no':>11}")
    return "\n".join(lines)


def sweep_csv(axis: str, results: list) -> str:
    rows = [f"{axis},outer_iterations,total_inner_iterations,final_true_residual,converged"]
    rows += [f"{tag},{s.outer_iterations},{s.total_inner_iterations},{format(s.final_true_residual, '.17g')},"
             f"{int(s.converged)}" for tag, s in results]
    return "\n".join(rows) + "\n"


# ------------------------------------------------------------------ compare


def trace_stats(path: str) -> dict:
    """Outer iterations, elapsed time, rate and final residuals of one trace
    (cli.py:440-457)."""
    trace = ResidualTrace.read_csv(path)
    if not trace.rows:
        raise ValueError(f"{path}: trace holds no rows")
    first, last = trace.rows[0], trace.rows[-1]
    elapsed = last.time - first.time
    trues = [r.true_residual for r in trace.rows if r.true_residual is not None]
    its = last.outer_iteration + 1
    return {"trace": path, "iterations": its, "elapsed": elapsed, "rate": its / elapsed if elapsed > 0 else None,
            "final_estimated": last.estimated_residual, "final_true": trues[-1] if trues else None}


def compare(paths: list, reference: str | None = None) -> list:
    """Per trace: iterations, rate, final residuals and the iteration / time
    ratios against the reference trace (the first by default; cli.py:460-481)."""
    stats = [trace_stats(p) for p in paths]
    ref_path = paths[0] if reference is None else reference
    ref = next((s for s in stats if s["trace"] == ref_path), None)
    if ref is None:
        raise ConfigurationError(f"reference: {ref_path!r} is not among the traces")
    rows = []
    for s in stats:
        row = {k: s[k] for k in ("trace", "iterations", "rate", "final_estimated", "final_true")}
        row["iteration_ratio"] = s["iterations"] / ref["iterations"]
        row["time_ratio"] = s["elapsed"] / ref["elapsed"] if ref["elapsed"] > 0 else None
        rows.append(row)
    return rows


def format_compare(rows: list) -> str:
    def opt(v, spec):
        return spec.format(v) if v is not None else "-"

    lines = [f"{'trace':<32}{'iters':>8}{'rate':>10}{'final_est':>14}{'final_true':>14}"
             f"{'iter_ratio':>12}{'time_ratio':>12}"]
    for r in rows:
        lines.append(f"{r['trace']:<32}{r['iterations']:>8}{opt(r['rate'], '{:.4g}'):>10}"
                     f"{r['final_estimated']:>14.4e}{opt(r['final_true'], '{:.4e}'):>14}"
                     f"{r['iteration_ratio']:>12.4f}{opt(r['time_ratio'], '{:.4f}'):>12}")
    return "\n".join(lines)


def compare_csv(rows: list) -> str:
    def num(v):
        return "" if v is None else format(v, ".17g")

    out = ["trace,iterations,rate,final_estimated,final_true,iteration_ratio,time_ratio"]
    for r in rows:
        out.append(",".join([r["trace"], str(r["iterations"]), num(r["rate"]), num(r["final_estimated"]),
                             num(r["final_true"]), num(r["iteration_ratio"]), num(r["time_ratio"])]))
    return "\n".join(out) + "\n"


# ------------------------------------------------------------------ entry point


def _config_flags(p: argparse.ArgumentParser) -> None:
    p.add_argument("--config", default=None, help="key=value file, flags override it")
    for key in DEFAULTS:
        p.add_argument("--" + key.replace("_", "-") if key != "R" else "--R", dest=key, default=None)


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="paper_2009_12638_b200",
                                 description="Two-stage block-Jacobi experiments on the GPU")
    sub = ap.add_subparsers(dest="cmd", required=True)
    _config_flags(sub.add_parser("run", help="one solve on the GPU, CSV trace"))
    sp = sub.add_parser("sweep", help="one solve per value of an axis")
    _config_flags(sp)
    sp.add_argument("--axis", required=True, help="|".join(AXES))
    sp.add_argument("--values", required=True, help="comma list (block grids gx,gy,gz separated by ';')")
    sp.add_argument("--summary-out", default=None, help="also write the sweep summary as CSV")
    cp = sub.add_parser("compare", help="compare residual traces")
    cp.add_argument("traces", nargs="+")
    cp.add_argument("--reference", default=None, help="reference trace (default: the first)")
    cp.add_argument("--out", default=None, help="also write the comparison as CSV")
    return ap


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        if args.cmd == "compare":
            rows = compare(args.traces, args.reference)
            print(format_compare(rows))
            if args.out:
                Path(args.out).write_text(compare_csv(rows))
            return 0
        cfg = resolve_config(args.config, vars(args))
        if args.cmd == "run":
            code, text = run(cfg)
            print(text)
            return code
        results = sweep(cfg, args.axis, args.values)
        print(format_sweep(args.axis, results))
        if args.summary_out:
            Path(args.summary_out).write_text(sweep_csv(args.axis, results))
        return 0 if all(s.converged for _, s in results) else 2
    except (ConfigurationError, ProtocolError, SolverBreakdownError, DeviceError, ValueError, OSError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
