"""Device path of the experiment harness.

``python -m paper_2009_12638_b200 run --nx 64 --ny 64 --nz 64 --gz 2 --inner cg
--inner-its 50 --tolerance-basis initial --tol 1e-6 --out trace.csv``

Mirrors the reference ``blocksolve run`` (cli.py:263-332, 538-586): the same
flags, the optional ``--config key=value`` file layered under the flags, the
same CSV trace schema and the same exit codes (0 converged, 2 stopped on the
outer-iteration cap, 1 on any configuration or solver error).  Additions:
``--tolerance-basis`` and ``--device``.  ``mode=baseline`` runs the inner
solver alone on the whole grid (cli.py:268-290).
"""

from __future__ import annotations

import argparse
import sys

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


def run(cfg: dict) -> tuple:
    """Execute one solve; returns (exit code, summary text)."""
    grid = Grid3D(_int(cfg["nx"], "nx"), _int(cfg["ny"], "ny"), _int(cfg["nz"], "nz"), boundary_from(cfg["boundary"]))
    problem = build_laplace_3d(grid)
    restart = None if cfg["restart"] == "" else _int(cfg["restart"], "restart")
    mode = cfg["mode"]
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
    trace.write_csv(cfg["out"])
    summary = "\n".join([
        f"{'outer iterations':<24}{outer}",
        f"{'total inner iterations':<24}{inner}",
        f"{'final true residual':<24}{final:.6e}",
        f"{'converged':<24}{'yes' if converged else 'no (max_outer reached)'}",
        f"{'trace':<24}{cfg['out']}",
    ])
    return (0 if converged else 2), summary


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="paper_2009_12638_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    rp = sub.add_parser("run", help="one solve on the GPU, CSV trace")
    rp.add_argument("--config", default=None, help="key=value file, flags override it")
    for key in DEFAULTS:
        rp.add_argument("--" + key.replace("_", "-"), dest=key, default=None)
    args = ap.parse_args(argv)
    try:
        cfg = dict(DEFAULTS)
        if args.config:
            file_cfg = read_config_file(args.config)
            unknown = set(file_cfg) - set(DEFAULTS)
            if unknown:
                raise ConfigurationError(f"{sorted(unknown)[0]}: unknown configuration key")
            cfg.update(file_cfg)
        cfg.update({k: v for k, v in vars(args).items() if k in DEFAULTS and v is not None})
        if cfg["mode"] not in ("baseline", "sync", "async"):
            raise ConfigurationError(f"mode: unknown mode {cfg['mode']!r}")
        code, text = run(cfg)
    except (ConfigurationError, ProtocolError, SolverBreakdownError, DeviceError, ValueError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1
    print(text)
    return code


if __name__ == "__main__":
    sys.exit(main())
