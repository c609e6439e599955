#!/usr/bin/env python
"""Benchmark: time-to-solution and stencil Gpts/s of the 7-point CG solve.

Workload (BASELINE.json configs[1], "config 2"): 256^3 fp64 grid, 7-point
Laplacian with zero Dirichlet boundary, seeded rhs uniform[-1, 1]
(default_rng(0), x-fastest), x0 = 0, CG to relative residual 1e-8 — 856
iterations, identical to the reference.  One *step* = one complete solve.

  value   whole-job stencil throughput, N * iterations / time (Gpts/s), with
          rhs and x0 resident in HBM (device tensors through the public
          ``cg_solve`` API); K timed solves bracketed by CUDA events.
  e2e     the same metric through the same public call with pinned HOST
          buffers: H2D of b and x0 and D2H of x inside the timed region.
  roofline  the dominant kernel of the timed region, ``k_cg_persistent`` (one
          cooperative launch runs a whole solve): algorithmic bytes per launch
          N * (64 * iterations + 32) / its CUDA-event duration on the
          launching stream.  Supplemental: the two CG sweeps launched one by
          one (launch mode) with an event pair around every launch.

Multi-GPU (torchrun, one rank per GPU): the single-block solve does not
shard, so ranks run independent replicas ("replicas only", scaling weak).

``--impl reference`` times the oracle's restatement of the reference CPU
path (CSR reduceat SpMV + numpy CG, oracle/blocksolve_oracle.py) on the
host, on a bounded sample of CG iterations of the same problem.
"""

from __future__ import annotations

import os

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")  # the port runs one thread; say so

import argparse
import ctypes
import json
import math
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "time-to-solution & stencil Gpts/s, 3D Laplace 7-pt block-Jacobi+CG, 1-8 GPU"
UNIT = "Gpts/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--tol", type=float, default=1e-8)
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--cpu-its", type=int, default=48, help="CG iterations in the CPU sample (~10-20 s)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--transport", default="nccl", choices=["nccl", "p2p"],
                    help="cross-GPU halo transport of the sharded outer workloads")
    ap.add_argument("--max-outer", type=int, default=100000,
                    help="outer-sweep cap of the supplemental workloads (bounded runs at full size)")
    ap.add_argument("--workload", default="config2", choices=["config2", "config3", "config4", "config5"],
                    help="config2 (default, the bench line); config3/4/5 = outer block-Jacobi solves (supplemental)")
    return ap.parse_args()


def workload(n, tol):
    return {"workload": f"config2: {n}^3 single-block CG to rel {tol:g}, seeded rhs U[-1,1] (seed 0), x0=0",
            "grid": [n, n, n], "tol": tol, "dtype_bytes": 8,
            "l2": "inputs larger than L2 (5 fp64 vectors of %d MB each vs 126 MB L2)" % (n ** 3 * 8 // 2 ** 20)}


class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(kernel_key):
    """Per-launch DRAM bytes of a kernel from a committed ncu --set full capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            return json.load(fh).get(kernel_key)
    except Exception:
        return None


def cpu_port_sample(n, its, tol):
    """The oracle's CSR restatement of the reference CG, timed on the host with
    the SpMV (83% of the reference's time) row-split over every core."""
    from oracle import blocksolve_oracle as O

    b = O.seeded_rhs(n ** 3, 0)
    t0 = time.perf_counter()
    a = O.laplace_csr(n, n, n)
    build_s = time.perf_counter() - t0
    cores = os.cpu_count() or 1
    apply = O.ThreadedCSR(a, cores)
    t0 = time.perf_counter()
    _, rep = O.cg(apply, b, np.zeros(n ** 3), its, tol)
    dt = time.perf_counter() - t0
    return {"value": n ** 3 * rep.iterations_used / dt / 1e9, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"{rep.iterations_used} CG iterations (+1 initial SpMV) of the {n}^3 config-2 solve, "
                      f"CSR reduceat SpMV row-split over {cores} threads + numpy CG vector ops "
                      f"(oracle restatement), OPENBLAS_NUM_THREADS=1; CSR build {build_s:.1f}s untimed; "
                      f"{dt:.1f}s timed",
            "seconds": dt}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import blocksolve_oracle as O

    n = args.n
    b = O.seeded_rhs(n ** 3, 0)
    a = O.laplace_csr(n, n, n)
    cores = os.cpu_count() or 1
    apply = O.ThreadedCSR(a, cores)
    its = max(1, int(args.cpu_its) // 3)
    x0 = np.zeros(n ** 3)
    for _ in range(args.warmup):
        O.cg(apply, b, x0, its, args.tol)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        _, rep = O.cg(apply, b, x0, its, args.tol)
        times.append(time.perf_counter() - t0)
    total = sum(times)
    value = n ** 3 * its * args.steps / total / 1e9
    sample = (f"each step = {its} CG iterations (+1 initial SpMV) of the {n}^3 config-2 solve; "
              f"oracle port of the reference CPU path (CSR reduceat SpMV row-split over {cores} threads, "
              f"numpy CG vector ops)")
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload(n, args.tol), "impl": "reference",
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "extrapolated_time_to_solution_s": 856 * n ** 3 / (value * 1e9)}
    print(json.dumps(line), flush=True)


def run_b200(args):
    import torch
    import torch.distributed as dist

    import paper_2009_12638_b200 as bs
    from paper_2009_12638_b200 import _lib
    from paper_2009_12638_b200.linalg import single_block_engine

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            dist.barrier()

    n = args.n
    N = n ** 3
    lib = _lib.load()
    op = bs.StencilOperator(n, n, n)
    spec = bs.InnerSolverSpec("cg", 20000, args.tol)
    b_host = np.random.default_rng(0).uniform(-1.0, 1.0, N)
    b = torch.from_numpy(b_host).to(dev)
    x0 = torch.zeros_like(b)
    eng = single_block_engine(op, dev, history_cap=spec.max_iterations)

    def step():
        return bs.cg_solve(op, b, x0, spec, batch=args.batch)

    for _ in range(args.warmup):
        x, rep = step()
    torch.cuda.synchronize(dev)
    its_ref = rep.iterations_used

    # ---- value: device-resident inputs, production path (device-side CUDA-graph loop)
    stream = torch.cuda.current_stream(dev)
    barrier()
    torch.cuda.synchronize(dev)
    launches0 = lib.bs_launch_count()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    its_total = 0
    with ClockSampler(local) as clocks:
        start.record(stream)
        for _ in range(args.steps):
            x, rep = step()
            its_total += rep.iterations_used
        end.record(stream)
        torch.cuda.synchronize(dev)
    launches = lib.bs_launch_count() - launches0
    elapsed = start.elapsed_time(end) / 1e3
    t = torch.tensor([elapsed], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    elapsed_max = float(t.item())
    value = world * N * its_total / elapsed_max / 1e9

    # ---- per-kernel CUDA events: the same K solves with the sweep kernels
    # launched from the host, an event pair around every launch
    ms = (ctypes.c_double * 3)()
    cnt = (ctypes.c_longlong * 3)()
    lib.bs_timing(eng.ctx, 1, None, None)
    torch.cuda.synchronize(dev)
    k_start, k_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    k_start.record(stream)
    for _ in range(args.steps):
        step()
    k_end.record(stream)
    torch.cuda.synchronize(dev)
    launch_mode_s = k_start.elapsed_time(k_end) / 1e3
    lib.bs_timing(eng.ctx, -1, ms, cnt)
    lib.bs_timing(eng.ctx, 0, None, None)

    # ---- the dominant kernel: the persistent CG kernel, one launch per solve,
    # timed alone with CUDA events on its stream (engine-level calls, so the
    # bracket holds only the control reset, the launch and the 32-byte
    # control read-back)
    bb = eng.blocks[0]
    k_ms = []
    for i in range(args.steps + 1):
        bb.put("b", b)
        bb.put("x", x0)
        eng.cg_begin(spec.max_iterations, spec.tolerance, "rhs")
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        eng.run(batch=args.batch, max_launches=0)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        eng.flush()
        if i:  # the first one is a warm-up
            k_ms.append(e0.elapsed_time(e1))
    k_us = 1e3 * statistics.mean(k_ms)
    persist_bytes = N * (64 * its_ref + 32)  # INIT 24 + first S1 16 + S2 24 + 64/it + verify 32

    hbm, peak_src = peaks()
    steps = args.steps
    s1_bytes = steps * N * (40 * (its_ref - 1) + 16)
    s2_bytes = steps * N * 24 * its_ref
    s1_ms, s2_ms, r_ms = ms[1], ms[2], ms[0]
    s1_gbs = s1_bytes / (s1_ms / 1e3) / 1e9 if s1_ms > 0 else None
    s2_gbs = s2_bytes / (s2_ms / 1e3) / 1e9 if s2_ms > 0 else None
    cg_bytes = steps * N * (64 * its_ref + 32)  # + INIT and verify residual sweeps
    cg_gbs = cg_bytes / elapsed / 1e9

    # ---- e2e: pinned host buffers through the same public call
    e2e = None
    if not args.no_e2e:
        b_pin = torch.from_numpy(b_host).pin_memory()
        x0_pin = torch.zeros(N, dtype=torch.float64).pin_memory()
        out_pin = torch.empty(N, dtype=torch.float64).pin_memory()
        bs.cg_solve(op, b_pin, x0_pin, spec, batch=args.batch, out=out_pin)
        barrier()
        torch.cuda.synchronize(dev)
        e_start, e_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e_its = 0
        e_start.record(stream)
        for _ in range(args.steps):
            _, rep_e = bs.cg_solve(op, b_pin, x0_pin, spec, batch=args.batch, out=out_pin)
            e_its += rep_e.iterations_used
        e_end.record(stream)
        torch.cuda.synchronize(dev)
        te = torch.tensor([e_start.elapsed_time(e_end) / 1e3], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": world * N * e_its / float(te.item()) / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": 2 * N * 8, "d2h_bytes_per_step": N * 8 + its_ref * 8,
               "ms_per_step": 1e3 * float(te.item()) / args.steps}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_port_sample(n, args.cpu_its, args.tol)
        cpu.pop("seconds", None)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * elapsed_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: seeded rhs U[-1,1] default_rng(0), x-fastest (SURVEY 8d)",
            "config": dict(workload(n, args.tol), parallelism="replicas" if world > 1 else "single GPU",
                           iterations_per_solve=its_ref),
            "time_to_solution_s": elapsed_max / args.steps,
            "iterations_per_solve": its_ref,
            "roofline": {"bound": "hbm", "kernel": "k_cg_persistent (whole CG solve, one cooperative launch)",
                         "achieved": persist_bytes / (k_us * 1e-6) / 1e9, "peak": hbm, "peak_source": peak_src,
                         "unit": "GB/s", "frac": persist_bytes / (k_us * 1e-6) / 1e9 / hbm,
                         "traffic": ncu_traffic("k_cg_persistent"),
                         "algorithmic_bytes_per_launch": persist_bytes,
                         "algorithmic_bytes_per_point": f"64 per iteration + 32 ({its_ref} iterations)",
                         "launches": len(k_ms), "avg_launch_us": k_us},
            "roofline_s1_launch_mode": {"achieved": s1_gbs, "frac": (s1_gbs / hbm) if s1_gbs else None,
                                        "bytes_per_point": "40 (first iteration 16)",
                                        "traffic": ncu_traffic("k_sweep_s1"),
                                        "avg_launch_us": 1e3 * s1_ms / max(1, cnt[1])},
            "roofline_s2_launch_mode": {"achieved": s2_gbs, "frac": (s2_gbs / hbm) if s2_gbs else None,
                                        "bytes_per_point": 24, "avg_launch_us": 1e3 * s2_ms / max(1, cnt[2])},
            "roofline_cg_iteration": {"achieved": cg_gbs, "frac": cg_gbs / hbm, "bytes_per_point": 64,
                                      "note": "whole cg_solve call (arm, kernel, flush, reports, result copy): 64 B/pt/it + 32 B/pt"},
            "resid_sweep_ms_total": r_ms,
            "launch_mode_time_to_solution_s": launch_mode_s / args.steps,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


OUTER_WORKLOADS = {
    # BASELINE.json configs[2..4]; inner tolerances in the r0-relative basis (the
    # literal rhs-relative reading stalls on the reference)
    "config3": dict(block_grid=(1, 1, 8), inner=("cg", 100, 1e-3), mode="sync", tol=1e-8, overlap=0,
                    faces=None, basis="initial", every=1),
    "config4": dict(block_grid=(1, 1, 8), inner=("cg", 20, 0.0), mode="async", tol=1e-8, overlap=0,
                    faces=None, basis="rhs", every=10),
    "config5": dict(block_grid=(2, 2, 2), inner=("gmres", 30, 1e-3), mode="sync", tol=1e-8, overlap=2,
                    faces={"z_lo": 1.0}, basis="initial", every=1),
}


def region_sizes(n, block_grid, overlap):
    """Points of each block's extended region: the owned box dilated `overlap`
    times by the 7-point stencil (an L1 ball, problems.py:178-190) clipped to
    the n^3 grid, counted analytically (SURVEY §8 notation N_b)."""
    from paper_2009_12638_b200.problems import _split_ranges

    sizes = []
    gx, gy, gz = block_grid
    for bz in range(gz):
        for by in range(gy):
            for bx in range(gx):
                counts = []
                for g, bi in ((gx, bx), (gy, by), (gz, bz)):
                    lo, hi = _split_ranges(n, g)[bi]
                    # c[k]: coordinates at distance k outside [lo, hi) on this axis
                    counts.append([hi - lo] + [int(lo - k >= 0) + int(hi - 1 + k < n) for k in range(1, overlap + 1)])
                cx, cy, cz = counts
                sizes.append(sum(cx[a] * cy[b] * cz[c] for a in range(overlap + 1) for b in range(overlap + 1)
                                 for c in range(overlap + 1) if a + b + c <= overlap))
    return sizes


def run_outer_workload(args):
    """Supplemental: time-to-solution of the outer block-Jacobi configs on this
    box (1 GPU: all blocks on one device; torchrun N>1: config3 sharded)."""
    import torch
    import torch.distributed as dist

    import paper_2009_12638_b200 as bs

    w = OUTER_WORKLOADS[args.workload]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    n = args.n
    N = n ** 3
    grid = bs.Grid3D(n, n, n, bs.DirichletBoundary(w["faces"] or {}))
    if w["faces"]:
        prob = bs.build_laplace_3d(grid)
    else:
        prob = bs.LinearProblem(bs.StencilOperator(n, n, n), np.random.default_rng(0).uniform(-1.0, 1.0, N), grid)
    kind, its, itol = w["inner"]
    cfg = bs.OuterConfig(block_grid=w["block_grid"], overlap=w["overlap"], inner=bs.InnerSolverSpec(kind, its, itol),
                         mode=w["mode"], tol=w["tol"], max_outer=args.max_outer, tolerance_basis=w["basis"],
                         residual_check_every=w["every"], execution="threads" if w["mode"] == "async" else "replay")
    from paper_2009_12638_b200.distributed import outer_solve_distributed

    def solve():
        if world > 1:
            return outer_solve_distributed(prob, cfg, transport=args.transport)
        return bs.outer_solve(prob, cfg)

    for _ in range(args.warmup):
        solve()
    times, results = [], []
    for _ in range(args.steps):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        res = solve()
        torch.cuda.synchronize(dev)
        times.append(time.perf_counter() - t0)
        results.append(res)
    t = torch.tensor([sum(times) / len(times)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    tts = float(t.item())
    res = results[-1]
    total_its = int(sum(sum(row) for row in res.inner_iterations_per_block))
    nb = int(np.prod(w["block_grid"]))
    pts_its = N * total_its / nb if w["overlap"] == 0 else None
    if w["overlap"] == 0:
        # sum over sweeps and blocks of N_b (64 its_b + 64)
        alg = sum((N / nb) * (64 * i + 64) for row in res.inner_iterations_per_block for i in row)
    elif kind == "gmres":
        # Arnoldi step j of a GMRES(m) cycle moves 32 + 24 (j + 1)
        # B/pt (SpMV, j + 1 MGS passes, normalisation) over the block's region
        # (N_b = owned box dilated by the overlap), + 64 B/pt outer overhead
        sizes = region_sizes(n, w["block_grid"], w["overlap"])
        m = 30

        def block_bytes(its):
            return sum(32 + 24 * ((j % m) + 1) for j in range(its)) + 64

        alg = sum(sizes[b] * block_bytes(i) for row in res.inner_iterations_per_block for b, i in enumerate(row))
    else:
        alg = None
    hbm = peaks()[0]
    if rank == 0:
        line = {"metric": METRIC + " (supplemental: " + args.workload + ")", "workload": args.workload,
                "grid": [n, n, n], "n_gpus": world, "config": {k: (list(v) if isinstance(v, tuple) else v)
                                                             for k, v in w.items()},
                "time_to_solution_s": tts, "outer_sweeps": res.outer_iterations, "converged": res.converged,
                "seconds_per_sweep": tts / max(1, res.outer_iterations), "max_outer": args.max_outer,
                "estimates": [row.estimated_residual for row in res.trace.rows][-3:],
                "final_true_residual": res.final_true_residual, "inner_iterations_total": total_its,
                "stencil_gpts_per_s": (pts_its / tts / 1e9) if pts_its else None,
                "hbm_fraction": (alg / tts / 1e9 / (hbm * world)) if alg else None,
                "dtype": "f64", "data": "synthetic" if not w["faces"] else "Dirichlet z_lo=1"}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    elif args.workload != "config2":
        run_outer_workload(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
