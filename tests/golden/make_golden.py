"""Generate golden vectors by running the UNMODIFIED reference ``blocksolve``.

Run in the build container (where ``/root/reference`` exists):

    python tests/golden/make_golden.py

Writes ``tests/golden/golden.npz`` (arrays) and ``tests/golden/golden.json``
(scalars, iteration counts, residual histories, traces).  The GPU box never
runs this script; tests read only the committed fixtures.
"""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from blocksolve import (  # noqa: E402  (reference, read-only)
    DirichletBoundary,
    Grid3D,
    InnerSolverSpec,
    LinearProblem,
    OuterConfig,
    block_system,
    build_laplace_3d,
    cg_solve,
    decompose,
    gmres_solve,
    iteration_operator,
    jacobi_solve,
    outer_solve,
    power_iteration,
    spmv,
)

OUT = Path(__file__).resolve().parent
arrays: dict[str, np.ndarray] = {}
meta: dict = {}


def wide_x(rng, n):
    """Wide-dynamic-range vector: exposes any change of summation order."""
    return rng.standard_normal(n) * np.exp(rng.uniform(-20, 20, n))


def seeded(n, seed=0):
    return np.random.default_rng(seed).uniform(-1.0, 1.0, n)


def problem(nx, ny, nz, faces=None, rhs=None):
    grid = Grid3D(nx, ny, nz, DirichletBoundary(faces or {}))
    base = build_laplace_3d(grid)
    if rhs is None:
        return base
    return LinearProblem(base.matrix, rhs, grid)


def add_report(key, x, rep):
    arrays[key + "/x"] = x
    meta[key] = dict(
        iterations_used=rep.iterations_used,
        final_relative_residual=rep.final_relative_residual,
        stop_reason=rep.stop_reason,
        residual_history=[float(h) for h in rep.residual_history],
    )


def main():
    rng = np.random.default_rng(20240917)

    # -- operator assembly + rhs folding (problems.py:123-175)
    faces = {"x_lo": 1.0, "y_hi": 0.5, "z_lo": 2.0, "x_hi": -0.25}
    p = problem(5, 4, 3, faces)
    arrays["assembly/offsets"] = p.matrix.row_offsets
    arrays["assembly/cols"] = p.matrix.col_indices
    arrays["assembly/vals"] = p.matrix.values
    arrays["assembly/rhs"] = p.rhs
    meta["assembly"] = dict(shape=[5, 4, 3], faces=faces)

    # callable face (problems.py:67-71)
    pc = build_laplace_3d(Grid3D(3, 4, 2, DirichletBoundary(
        {"y_lo": lambda i, k: 0.5 * i + k, "z_hi": 1.5})))
    arrays["assembly_callable/rhs"] = pc.rhs

    # -- global SpMV, bitwise (linalg.py:178-194)
    for shape in ((6, 5, 4), (16, 16, 16), (7, 1, 3)):
        pr = problem(*shape)
        x = wide_x(rng, pr.grid.num_unknowns)
        key = "spmv/%dx%dx%d" % shape
        arrays[key + "/x"] = x
        arrays[key + "/y"] = spmv(pr.matrix, x)

    # -- block-system SpMV (principal submatrix on extended regions)
    for shape, bg, ov in (((8, 8, 8), (1, 1, 2), 0), ((8, 8, 8), (2, 2, 2), 2),
                          ((9, 7, 6), (2, 1, 3), 1), ((6, 6, 6), (3, 2, 1), 0)):
        pr = problem(*shape)
        dec = decompose(pr.grid, bg, ov)
        key = "blocksys/%dx%dx%d_%d%d%d_o%d" % (shape + bg + (ov,))
        arrays[key + "/cover"] = dec.cover_counts
        meta[key] = dict(shape=list(shape), block_grid=list(bg), overlap=ov,
                         neighbors=[list(n) for n in dec.neighbors])
        for b in range(dec.num_blocks):
            a_ii, coupling = block_system(pr, dec, b)
            x = wide_x(rng, a_ii.num_rows)
            arrays[f"{key}/{b}/ext"] = dec.extended_indices[b]
            arrays[f"{key}/{b}/x"] = x
            arrays[f"{key}/{b}/y"] = spmv(a_ii, x)
            arrays[f"{key}/{b}/coupling"] = np.asarray(coupling, dtype=np.float64).reshape(-1, 3)

    # -- CG (inner_solvers.py:102-146)
    for n, tol, seed in ((12, 1e-8, 0), (20, 1e-10, 1), (32, 1e-8, 0)):
        pr = problem(n, n, n, rhs=seeded(n ** 3, seed))
        x, rep = cg_solve(pr.matrix, pr.rhs, np.zeros(n ** 3), InnerSolverSpec("cg", 10 * n, tol))
        add_report(f"cg/{n}_seed{seed}", x, rep)
    # warm start, capped iterations
    n = 10
    pr = problem(n, n, n, {"z_lo": 1.0})
    x0 = rng.uniform(-1, 1, n ** 3)
    arrays["cg/warm/x0"] = x0
    x, rep = cg_solve(pr.matrix, pr.rhs, x0, InnerSolverSpec("cg", 17, 1e-3))
    add_report("cg/warm", x, rep)
    # r0-relative basis via the wrapper of SURVEY §8(c)
    r0 = pr.rhs - spmv(pr.matrix, x0)
    tol_prime = 1e-3 * (float(np.linalg.norm(r0)) / float(np.linalg.norm(pr.rhs)))
    x, rep = cg_solve(pr.matrix, pr.rhs, x0, InnerSolverSpec("cg", 200, tol_prime))
    add_report("cg/warm_initial", x, rep)
    meta["cg/warm_initial"]["tol_prime"] = tol_prime

    # -- GMRES (inner_solvers.py:149-243)
    for n, its, tol, restart in ((8, 200, 1e-10, 10), (10, 30, 1e-3, 30), (6, 40, 0.0, 7)):
        pr = problem(n, n, n, {"x_lo": 1.0, "y_hi": 0.5})
        x, rep = gmres_solve(pr.matrix, pr.rhs, np.zeros(n ** 3),
                             InnerSolverSpec("gmres", its, tol, restart))
        add_report(f"gmres/{n}_{its}_{restart}", x, rep)

    # -- point Jacobi (inner_solvers.py:75-99)
    pr = problem(10, 10, 10, {"x_lo": 1.0, "z_hi": 0.5})
    x, rep = jacobi_solve(pr.matrix, pr.rhs, np.zeros(1000), InnerSolverSpec("jacobi", 400, 1e-3))
    add_report("jacobi/10_tol", x, rep)
    pr = problem(9, 6, 4, rhs=seeded(216, 2))
    x0 = wide_x(rng, 216)
    arrays["jacobi/9x6x4_maxit/x0"] = x0
    x, rep = jacobi_solve(pr.matrix, pr.rhs, x0, InnerSolverSpec("jacobi", 25, 0.0))
    add_report("jacobi/9x6x4_maxit", x, rep)
    for shape in ((7, 1, 3), (1, 1, 5), (1, 1, 1)):  # rows whose leading neighbour is an upper one
        n = shape[0] * shape[1] * shape[2]
        pr = problem(*shape, rhs=seeded(n, 4))
        x, rep = jacobi_solve(pr.matrix, pr.rhs, np.zeros(n), InnerSolverSpec("jacobi", 12, 0.0))
        add_report("jacobi/%dx%dx%d" % shape, x, rep)
    pr = problem(4, 4, 4, rhs=np.zeros(64))
    x, rep = jacobi_solve(pr.matrix, pr.rhs, np.zeros(64), InnerSolverSpec("jacobi", 5, 0.0))
    add_report("jacobi/zero_rhs", x, rep)

    # -- spectral diagnostics (linalg.py:243-276, multisplit.py:800-830)
    def est_meta(e):
        return dict(radius=e.radius, iterations_used=e.iterations_used, converged=e.converged)

    meta["power/diag123"] = est_meta(power_iteration(lambda v: np.array([1.0, 2.0, 3.0]) * v, 3, tol=1e-12,
                                                     seed=1))
    lap8 = problem(8, 8, 8).matrix
    meta["power/jacobi_8"] = est_meta(power_iteration(lambda v: v - spmv(lap8, v) / 6.0, 512, tol=1e-10,
                                                      seed=1))
    pr = problem(4, 4, 4, {"x_lo": 1.0, "y_hi": 0.5})
    apply_map, dim = iteration_operator(pr, decompose(pr.grid, (2, 1, 1), 0))
    arrays["itop/4_211_o0/matrix"] = np.stack([apply_map(e) for e in np.eye(dim)], axis=1)
    for n, bg, ov in ((4, (2, 1, 1), 0), (4, (2, 2, 1), 1), (8, (2, 1, 1), 0), (8, (4, 1, 1), 0),
                      (6, (1, 1, 3), 0), (6, (2, 2, 2), 1)):
        pr = problem(n, n, n, {"x_lo": 1.0, "y_hi": 0.5})
        dec = decompose(pr.grid, bg, ov)
        apply_map, dim = iteration_operator(pr, dec)
        key = "itop/%d_%d%d%d_o%d" % ((n,) + bg + (ov,))
        meta[key] = dict(dim=dim, **est_meta(power_iteration(apply_map, dim, tol=1e-10, seed=0)))

    # -- outer sync traces (multisplit.py:742-797)
    cases = {
        # config-1 shape at reduced size: z_lo=1, 2 z-slabs, CG(50) fixed its
        "outer/cfg1_16_fixed": dict(n=16, faces={"z_lo": 1.0}, bg=(1, 1, 2), ov=0,
                                    inner=("cg", 50, 0.0), tol=1e-6, mode="paper"),
        # literal config-1 semantics (rhs-relative inner tol): stalls
        "outer/cfg1_16_literal": dict(n=16, faces={"z_lo": 1.0}, bg=(1, 1, 2), ov=0,
                                      inner=("cg", 50, 1e-2), tol=1e-6, mode="paper",
                                      max_outer=40),
        # config-3 shape: 4 z-slabs, seeded rhs, CG fixed its, both modes
        "outer/cfg3_16_paper": dict(n=16, seed=0, bg=(1, 1, 4), ov=0,
                                    inner=("cg", 10, 0.0), tol=1e-8, mode="paper"),
        "outer/cfg3_16_true": dict(n=16, seed=0, bg=(1, 1, 4), ov=0,
                                   inner=("cg", 10, 0.0), tol=1e-8, mode="true"),
        # boxes in x and y (rows with several couplings)
        "outer/box_12_222": dict(n=12, seed=3, bg=(2, 2, 2), ov=0,
                                 inner=("cg", 8, 0.0), tol=1e-7, mode="paper"),
        # config-5 shape: 2x2x2 cubes, overlap 2, GMRES one cycle
        "outer/cfg5_12_o2": dict(n=12, faces={"z_lo": 1.0}, bg=(2, 2, 2), ov=2,
                                 inner=("gmres", 10, 0.0), tol=1e-8, mode="paper"),
        "outer/o1_10_211": dict(n=10, seed=5, bg=(2, 1, 1), ov=1,
                                inner=("cg", 6, 0.0), tol=1e-7, mode="true"),
        # point-Jacobi inner solves: slabs (box path) and an overlapping split
        "outer/jac_10_112": dict(n=10, seed=6, bg=(1, 1, 2), ov=0,
                                 inner=("jacobi", 20, 0.0), tol=1e-6, mode="paper"),
        "outer/jac_8_221_o1": dict(n=8, faces={"z_lo": 1.0}, bg=(2, 2, 1), ov=1,
                                   inner=("jacobi", 15, 0.0), tol=1e-6, mode="true"),
    }
    for key, c in cases.items():
        n = c["n"]
        if "seed" in c:
            pr = problem(n, n, n, rhs=seeded(n ** 3, c["seed"]))
        else:
            pr = problem(n, n, n, c["faces"])
        kind, its, itol = c["inner"]
        cfg = OuterConfig(block_grid=c["bg"], overlap=c["ov"],
                          inner=InnerSolverSpec(kind, its, itol), tol=c["tol"],
                          max_outer=c.get("max_outer", 5000),
                          residual_check_mode=c["mode"])
        res = outer_solve(pr, cfg)
        arrays[key + "/solution"] = res.solution
        arrays[key + "/rhs"] = pr.rhs
        meta[key] = dict(
            case={k: (list(v) if isinstance(v, tuple) else v) for k, v in c.items()},
            converged=res.converged, outer_iterations=res.outer_iterations,
            final_true_residual=res.final_true_residual,
            trace=[[r.outer_iteration, r.time, r.estimated_residual, r.true_residual,
                    r.inner_iterations, r.max_halo_staleness] for r in res.trace.rows],
        )

    np.savez_compressed(OUT / "golden.npz", **arrays)
    with open(OUT / "golden.json", "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)
    print("wrote", len(arrays), "arrays,", len(meta), "meta entries")


if __name__ == "__main__":
    os.chdir("/tmp")
    main()
