#!/usr/bin/env python
"""Benchmark: time-to-solution and stencil Gpts/s of block-Jacobi + CG.

Workload (BASELINE.json configs[2], "config 3" — the configuration the
metric is quoted on): 512^3 fp64 grid, 7-point Laplacian, zero Dirichlet
boundary, seeded rhs U[-1, 1] (default_rng(0), x-fastest), x0 = 0; block
Jacobi over eight z-slabs of 64 planes (block_grid (1, 1, 8), overlap 0),
inner CG(100, tol 1e-3 relative to ||r0||), synchronous sweeps, outer tol
1e-8 on the paper residual (multisplit.py:742-797, 544-640).  At N GPUs
(--gpus N: torchrun, one rank per GPU; spawned here when WORLD_SIZE is
unset) rank r owns slabs [8r/N, 8(r+1)/N) — 8/4/2/1 blocks per GPU — and the
problem is fixed (strong scaling).

One *step* = one outer sweep: the halo exchange, residual sweep, global
reduction and termination test of sweep k-1 plus the inner CG solves of
sweep k — all inside ONE complete solve through the public ``outer_solve``
(``outer_solve_distributed`` at N > 1), called with the host numpy rhs:

  value     N_b * sum(inner its) / time over the K timed sweeps W..W+K-1
            (inputs resident in HBM by then), CUDA events on the solve's
            stream bracketed by a barrier + synchronize, max over ranks.
  e2e       the same metric over the whole call: host rhs -> H2D (1 GiB) ->
            solve to 1e-8 -> D2H of the 1 GiB solution; time_to_solution_s.
  roofline  the dominant kernel, the inner solve: one cooperative launch
            per sweep (k_cg_stream: every block of the GPU, many tiles per
            CTA), CUDA events around it on its stream; algorithmic bytes per
            launch = sum_b N_b (64 its_b - 24) (64 B/pt per CG
            iteration; the first sweep 1 of a solve reads no p_old / x).
  halo      CUDA events around the halo exchange of every timed sweep: the
            pack kernel (N = 1: against HBM) / pack + peer put (p2p) or pack +
            NCCL (N > 1: against NVLink).
  cpu_baseline  the oracle's restatement of the reference CPU path (CSR
            reduceat SpMV row-split over the host threads + numpy CG) on one
            512^2 x 64 slab, a bounded sample of CG iterations, extrapolated.
  config2   secondary: 256^3 single-block CG to 1e-8 (the kernel check of
            round 1), N = 1 only.

``--impl reference`` times the same oracle port (the reference is pure
Python and has no GPU path) on the same config, one step =
a bounded sample of CG iterations on one slab.  ``--workload config4 /
config5`` run the supplemental asynchronous / overlapping outer configs.
"""

from __future__ import annotations

import os

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")  # the port threads its SpMV itself

import argparse
import ctypes
import json
import math
import socket
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
NVLINK_GBS = 900.0  # NVLink 5 per direction per GPU (B200_PROFILING.md)
# inner CG iterations of the complete config-3 solve (3464 sweeps x 8 blocks x
# 100; identical at 1/2/4/8 GPUs) — used only to extrapolate CPU rates
CFG3_TOTAL_ITS = 2771200

WORKLOADS = {
    # BASELINE.json configs[2..4]; inner tolerances in the r0-relative basis (the
    # literal rhs-relative reading stalls on the reference)
    "config3": dict(n=512, block_grid=(1, 1, 8), inner=("cg", 100, 1e-3), mode="sync", tol=1e-8, overlap=0,
                    faces=None, basis="initial", every=1),
    "config4": dict(n=512, block_grid=(1, 1, 8), inner=("cg", 20, 0.0), mode="async", tol=1e-8, overlap=0,
                    faces=None, basis="rhs", every=10),
    "config5": dict(n=512, block_grid=(2, 2, 2), inner=("gmres", 30, 1e-3), mode="sync", tol=1e-8, overlap=2,
                    faces={"z_lo": 1.0}, basis="initial", every=1),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20, help="timed outer sweeps")
    ap.add_argument("--warmup", type=int, default=5, help="untimed outer sweeps before them (>= 1)")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="config3", choices=["config3", "config2", "config4", "config5"])
    ap.add_argument("--n", type=int, default=0, help="grid size (default: the workload's)")
    ap.add_argument("--max-outer", type=int, default=100000, help="outer-sweep cap (bounded runs)")
    ap.add_argument("--transport", default="auto", choices=["auto", "nccl", "p2p"],
                    help="cross-GPU halo transport (auto: p2p peer puts when every GPU pair has peer access)")
    ap.add_argument("--cpu-its", type=int, default=40, help="CG iterations of the CPU-baseline sample")
    ap.add_argument("--ref-its", type=int, default=16, help="CG iterations per reference-arm step")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-config2", action="store_true")
    return ap.parse_args()


def grid_n(args) -> int:
    if args.n:
        return args.n
    return 256 if args.workload == "config2" else WORKLOADS[args.workload]["n"]


def workload_config(args) -> dict:
    """The config dict of the bench line — identical in both arms."""
    n = grid_n(args)
    if args.workload == "config2":
        return {"workload": f"config2: {n}^3 single-block CG to rel 1e-08, seeded rhs U[-1,1] (seed 0), x0=0",
                "grid": [n, n, n], "tol": 1e-8, "dtype_bytes": 8,
                "l2": "inputs larger than L2 (5 fp64 vectors of %d MB vs 126 MB L2)" % (n ** 3 * 8 // 2 ** 20)}
    w = WORKLOADS[args.workload]
    nb = int(np.prod(w["block_grid"]))
    kind, its, tol = w["inner"]
    return {"workload": (f"{args.workload}: {n}^3 {w['mode']} block-Jacobi, block_grid {tuple(w['block_grid'])}, "
                         f"overlap {w['overlap']}, inner {kind.upper()}({its}, {tol:g} rel. "
                         f"{'r0' if w['basis'] == 'initial' else 'rhs'}), outer tol {w['tol']:g} (paper residual), "
                         f"seeded rhs U[-1,1] seed 0, x0=0; one step = one outer sweep"),
            "grid": [n, n, n], "block_grid": list(w["block_grid"]), "overlap": w["overlap"],
            "inner": [kind, its, tol], "tolerance_basis": w["basis"], "outer_tol": w["tol"],
            "residual_check_mode": "paper", "residual_check_every": w["every"], "dtype_bytes": 8,
            "parallelism": f"{nb} blocks over {args.gpus} GPU(s), one process per GPU",
            "l2": f"inputs larger than L2 (per block 5 fp64 vectors of {n ** 3 // nb * 8 // 2 ** 20} MB; "
                  f"{n ** 3 * 8 * 5 // 2 ** 30} GiB resident vs 126 MB L2)"}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons, timestamped, sampled every 200 ms."""

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
            self.lines.append((time.time(), line.strip()))

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self, t0=None, t1=None):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ts, line in self.lines:
            if t0 is not None and not (t0 <= ts <= t1 + 0.25):
                continue
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
    """DRAM bytes (read + write) per algorithmic byte of a kernel, from a
    committed ``ncu --set full`` capture (profiles/ncu_traffic.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            return json.load(fh).get(kernel_key)
    except Exception:
        return None


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


# ---------------------------------------------------------------- CPU legs (oracle port)


def cpu_slab_sample(n, nslabs, its, tol, basis):
    """The oracle's restatement of the reference CPU path (CSR reduceat SpMV,
    row-split over every host thread, + numpy CG vector ops) timed on slab 0
    of the sweep-0 block system (rhs = b on the slab)."""
    from oracle import blocksolve_oracle as O

    nzb = n // nslabs
    nb = n * n * nzb
    b = np.random.default_rng(0).uniform(-1.0, 1.0, nb)  # the first n*n*nzb draws = slab 0 of the seeded rhs
    t0 = time.perf_counter()
    a = O.laplace_csr(n, n, nzb)  # slab principal submatrix (problems.py:362-406)
    build_s = time.perf_counter() - t0
    cores = os.cpu_count() or 1
    apply = O.ThreadedCSR(a, cores)
    O.cg(apply, b, np.zeros(nb), 2, 0.0)  # page in
    t0 = time.perf_counter()
    _, rep = O.cg(apply, b, np.zeros(nb), its, tol, basis)
    dt = time.perf_counter() - t0
    return {"value": nb * rep.iterations_used / dt / 1e9, "cores": cores, "kind": "port", "seconds": dt,
            "its": rep.iterations_used, "build_s": build_s, "points": nb}


def run_reference(args):
    """--impl reference: the oracle port of the reference CPU path on the same
    config; rank 0 only (the others exit without work)."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    from oracle import blocksolve_oracle as O

    n = grid_n(args)
    cores = os.cpu_count() or 1
    if args.workload == "config2":
        nb, label = n ** 3, f"the {n}^3 config-2 system"
        a = O.laplace_csr(n, n, n)
        b = np.random.default_rng(0).uniform(-1.0, 1.0, nb)
        total_pts_its = 856 * nb
    else:
        w = WORKLOADS[args.workload]
        nslabs = w["block_grid"][2]
        nzb = n // nslabs
        nb, label = n * n * nzb, f"slab 0 ({n}x{n}x{nzb}) of the sweep-0 block system"
        a = O.laplace_csr(n, n, nzb)
        b = np.random.default_rng(0).uniform(-1.0, 1.0, nb)
        total_pts_its = CFG3_TOTAL_ITS * nb
    apply = O.ThreadedCSR(a, cores)
    its = max(1, args.ref_its)
    x0 = np.zeros(nb)
    for _ in range(args.warmup):
        O.cg(apply, b, x0, its, 0.0)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        _, rep = O.cg(apply, b, x0, its, 0.0)
        times.append(time.perf_counter() - t0)
        assert rep.iterations_used == its
    total = sum(times)
    value = nb * its * args.steps / total / 1e9
    sample = (f"each step = {its} CG iterations (+1 initial SpMV) on {label}; oracle port of the reference CPU "
              f"path (CSR reduceat SpMV row-split over {cores} threads, numpy CG vector ops)")
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
            "scaling": "strong" if args.workload != "config2" else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": workload_config(args), "impl": "reference",
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "extrapolated_time_to_solution_s": total_pts_its / (value * 1e9),
            "extrapolation": "inner point-iterations of the complete solve (the device run's counts, identical in "
                             "sync mode) / this rate"}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- device arm


class SweepProbe:
    """Measurement hooks of the sync sweep loop (sync_driver.run_sync): K
    timed sweeps W..W+K-1 bracketed by barrier + synchronize + CUDA events on
    the solve's stream, plus event pairs around every timed inner solve and
    halo exchange."""

    def __init__(self, torch, dev, warmup, steps, barrier, lib):
        self.torch = torch
        self.stream = torch.cuda.current_stream(dev)
        self.dev = dev
        self.warmup, self.steps = max(1, warmup), steps
        self.barrier = barrier
        self.lib = lib
        self.pairs = {"solve": [], "exchange": [], "resid": []}
        self.open = {}
        self.its = []  # per timed sweep: global per-block counts
        self.t_start = self.t_end = None
        self.h0 = self.h1 = None
        self.l0 = self.l1 = 0
        self.eng = None
        self.path = None

    def attach(self, eng):
        self.eng = eng

    def _ev(self):
        e = self.torch.cuda.Event(enable_timing=True)
        e.record(self.stream)
        return e

    def timed(self, k):
        return self.warmup <= k < self.warmup + self.steps

    def begin(self, phase, k):
        if self.timed(k):
            self.open[phase] = self._ev()

    def end(self, phase, k):
        if phase in self.open:
            self.pairs[phase].append((self.open.pop(phase), self._ev()))

    def sweep(self, k, its):
        if self.timed(k):
            self.its.append(list(its))
        if k == self.warmup - 1:
            self.barrier()
            self.torch.cuda.synchronize(self.dev)
            self.t_start = self._ev()
            self.h0 = time.time()
            self.l0 = self.lib.bs_launch_count()
        if k == self.warmup + self.steps - 1:
            self.t_end = self._ev()
            self.torch.cuda.synchronize(self.dev)
            self.h1 = time.time()
            self.l1 = self.lib.bs_launch_count()
            self.path = getattr(self.eng, "run_path", None)
            self.barrier()

    def elapsed_s(self):
        return self.t_start.elapsed_time(self.t_end) / 1e3

    def durations_s(self, phase):
        return [a.elapsed_time(b) / 1e3 for a, b in self.pairs[phase]]


def spawn_ranks(args):
    """--gpus N without WORLD_SIZE: re-launch under torchrun, one rank per GPU."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


def run_config3(args):
    import torch
    import torch.distributed as dist

    import paper_2009_12638_b200 as bs
    from paper_2009_12638_b200 import _lib
    from paper_2009_12638_b200.distributed import block_range, outer_solve_distributed

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench: --gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(v):
        t = torch.tensor([float(v)], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    w = WORKLOADS["config3"]
    n = grid_n(args)
    N = n ** 3
    nslabs = w["block_grid"][2]
    Nb = N // nslabs
    lib = _lib.load()
    b_host = np.random.default_rng(0).uniform(-1.0, 1.0, N)
    prob = bs.LinearProblem(bs.StencilOperator(n, n, n), b_host, bs.Grid3D(n, n, n))
    kind, its, itol = w["inner"]
    cfg = bs.OuterConfig(block_grid=w["block_grid"], overlap=0, inner=bs.InnerSolverSpec(kind, its, itol),
                         mode="sync", tol=w["tol"], max_outer=args.max_outer, tolerance_basis=w["basis"],
                         residual_check_mode="paper", residual_check_every=1)
    transport = args.transport
    probe = SweepProbe(torch, dev, args.warmup, args.steps, barrier, lib)
    stream = torch.cuda.current_stream(dev)
    barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(local) as clocks:
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        h0 = time.perf_counter()
        e0.record(stream)
        if world > 1:
            res = outer_solve_distributed(prob, cfg, transport=transport, probe=probe)
        else:
            res = bs.outer_solve(prob, cfg, probe=probe)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        wall = time.perf_counter() - h0
    solve_s = max_over_ranks(e0.elapsed_time(e1) / 1e3)
    if probe.t_end is None:
        raise SystemExit(f"bench: the solve ended after {res.outer_iterations} sweeps, before the "
                         f"{probe.warmup}+{probe.steps} warm-up + timed sweeps")
    elapsed = max_over_ranks(probe.elapsed_s())
    timed_its = sum(sum(row) for row in probe.its)
    value = Nb * timed_its / elapsed / 1e9
    total_its = int(sum(sum(row) for row in res.inner_iterations_per_block))

    # roofline of the dominant kernel: this rank's inner solves (one launch each)
    mine = block_range(nslabs, rank, world)
    solve_bytes = sum(Nb * (64 * row[g] - 24 * (row[g] > 0)) for row in probe.its for g in mine)
    solve_s_list = probe.durations_s("solve")
    hbm, peak_src = peaks()
    kernel_s = sum(solve_s_list)
    achieved = solve_bytes / kernel_s / 1e9
    traffic_ratio = ncu_traffic("cfg3_inner_solve")
    kernel = {"stream": "k_cg_stream: the inner CG of every block of this GPU as one cooperative launch per sweep "
                        "(256 CTAs, one reduction lane each, tiles streamed through one ring)",
              "persistent": "k_cg_persistent: the inner CG as one cooperative launch per sweep (one tile per CTA)",
              "graph": "the inner CG of every block of this GPU as one CUDA-graph launch per sweep: "
                       "WHILE{k_sweep<S1>, k_sweep<S2>} (444 CTAs, tiles handed out dynamically)"}.get(probe.path, probe.path)
    roofline = {"bound": "hbm", "kernel": kernel, "run_path": probe.path,
                "achieved": achieved, "peak": hbm, "peak_source": peak_src, "unit": "GB/s", "frac": achieved / hbm,
                "traffic": (traffic_ratio * solve_bytes / len(solve_s_list)) if traffic_ratio else None,
                "traffic_source": "profiles/ncu_traffic.json (ncu --set full dram__bytes per algorithmic byte)"
                if traffic_ratio else None,
                "algorithmic_bytes_per_launch": solve_bytes / len(solve_s_list),
                "algorithmic_bytes_per_point": "64 per CG iteration - 24 per solve (SURVEY 8(d))",
                "launches": len(solve_s_list), "avg_launch_us": 1e6 * kernel_s / len(solve_s_list),
                "share_of_step": kernel_s / probe.elapsed_s()}
    # halo exchange: local planes by the pack kernel, cross-rank by p2p puts / NCCL
    plane = n * n * 8
    nif = nslabs - 1
    cross = sum(1 for i in range(nif) if (i in mine) != (i + 1 in mine) and (i in mine or i + 1 in mine))
    local_if = sum(1 for i in range(nif) if i in mine and i + 1 in mine)
    ex = probe.durations_s("exchange")
    ex_avg = sum(ex) / len(ex) if ex else None
    halo = {"planes_per_sweep_local": 2 * local_if, "planes_per_sweep_sent_remote": cross,
            "plane_bytes": plane, "avg_us": 1e6 * ex_avg if ex_avg else None,
            "share_of_step": (sum(ex) / probe.elapsed_s()) if ex else None,
            "transport": "local pack kernel" if world == 1 else transport}
    if ex_avg:
        if world == 1:
            moved = 2 * 2 * local_if * plane  # read + write per plane
            halo.update({"achieved_gbs": moved / ex_avg / 1e9, "vs": "HBM", "frac": moved / ex_avg / 1e9 / hbm})
        else:
            halo.update({"achieved_gbs": cross * plane / ex_avg / 1e9, "vs": "NVLink 900 GB/s per direction",
                         "frac": cross * plane / ex_avg / 1e9 / NVLINK_GBS})
    # where a step goes on this rank: device time of the three phases (CUDA events on the solve's
    # stream) and the rest — the host round trip per sweep (one report read, the scalar reduction and the
    # stop decision, with the device idle) plus launch gaps
    rs = probe.durations_s("resid")
    step_s = probe.elapsed_s() / len(probe.its)
    phases = {"inner_solve_ms": 1e3 * kernel_s / len(solve_s_list),
              "halo_exchange_ms": 1e3 * ex_avg if ex_avg else 0.0,
              "residual_sweep_ms": 1e3 * sum(rs) / len(rs) if rs else 0.0}
    rest = 1e3 * step_s - sum(phases.values())
    breakdown = dict(phases, host_and_gaps_ms=rest, host_and_gaps_share=rest / (1e3 * step_s),
                     note="per outer sweep on rank 0; residual sweep = re-arm + k_sweep<RESID> (local residual, "
                          "true residual on owned rows, next rhs / r0)")
    clock = clocks.summary(probe.h0, probe.h1)
    config2 = None
    if world == 1 and not args.no_config2:
        config2 = config2_check(args, torch, dev, bs, lib)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        s = cpu_slab_sample(n, nslabs, args.cpu_its, itol, w["basis"])
        cpu = {"value": s["value"], "unit": UNIT, "cores": s["cores"], "kind": "port",
               "sample": f"{s['its']} CG iterations (+1 initial SpMV) on slab 0 ({n}x{n}x{n // nslabs}, "
                         f"{s['points']} points) of the sweep-0 block system: CSR reduceat SpMV row-split over "
                         f"{s['cores']} threads + numpy CG (oracle restatement of the reference CPU path), "
                         f"OPENBLAS_NUM_THREADS=1; CSR build {s['build_s']:.1f}s untimed; {s['seconds']:.1f}s timed",
               "extrapolated_time_to_solution_s": Nb * total_its / (s["value"] * 1e9),
               "extrapolation": "this rate over the complete solve's inner point-iterations"}
    if rank == 0:
        converged = bool(res.converged)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": len(probe.its),
            "warmup": probe.warmup, "ms_per_step": 1e3 * elapsed / len(probe.its), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: seeded rhs U[-1,1] default_rng(0), x-fastest (SURVEY 8d)",
            "config": workload_config(args),
            "time_to_solution_s": solve_s if converged else None,
            "bounded_solve_s": None if converged else solve_s,
            "converged": converged, "outer_sweeps": res.outer_iterations,
            "inner_iterations_total": total_its, "final_true_residual": res.final_true_residual,
            "final_estimate": res.trace.rows[-1].estimated_residual,
            "solve_rate_gpts": Nb * total_its / solve_s / 1e9,
            "hbm_fraction_solve": Nb * sum(64 * i + 64 for row in res.inner_iterations_per_block for i in row)
            / solve_s / 1e9 / (hbm * world),
            "roofline": roofline, "halo": halo, "breakdown": breakdown,
            "cpu_baseline": cpu,
            "e2e": {"value": Nb * total_its / solve_s / 1e9, "unit": UNIT, "h2d_bytes_per_step": N * 8,
                    "d2h_bytes_per_step": N * 8,
                    "step": "one complete solve: outer_solve(host numpy rhs) -> host numpy solution",
                    "seconds": solve_s, "host_wall_s": wall},
            "gpu_launches": int(probe.l1 - probe.l0),
            "clocks": clock,
            "config2": config2,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def config2_check(args, torch, dev, bs, lib, steps=5, warmup=3):
    """Secondary: 256^3 single-block CG to 1e-8 (856 its), device-resident
    inputs through cg_solve; the persistent kernel timed alone with events."""
    from paper_2009_12638_b200.linalg import single_block_engine

    n = 256
    N = n ** 3
    op = bs.StencilOperator(n, n, n)
    spec = bs.InnerSolverSpec("cg", 20000, 1e-8)
    b = torch.from_numpy(np.random.default_rng(0).uniform(-1.0, 1.0, N)).to(dev)
    x0 = torch.zeros_like(b)
    stream = torch.cuda.current_stream(dev)
    for _ in range(warmup):
        _, rep = bs.cg_solve(op, b, x0, spec)
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    its = 0
    for _ in range(steps):
        _, rep = bs.cg_solve(op, b, x0, spec)
        its += rep.iterations_used
    e1.record(stream)
    torch.cuda.synchronize(dev)
    t = e0.elapsed_time(e1) / 1e3
    eng = single_block_engine(op, dev, history_cap=spec.max_iterations)
    bb = eng.blocks[0]
    k_ms = []
    for i in range(steps + 1):
        bb.put("b", b)
        bb.put("x", x0)
        eng.cg_begin(spec.max_iterations, spec.tolerance, "rhs")
        a, c = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        eng.run(max_launches=0)
        c.record(stream)
        torch.cuda.synchronize(dev)
        eng.flush()
        if i:
            k_ms.append(a.elapsed_time(c))
    hbm, _ = peaks()
    kbytes = N * (64 * rep.iterations_used + 32)
    k_s = statistics.mean(k_ms) / 1e3
    return {"workload": "config2: 256^3 single-block CG to rel 1e-8, seeded rhs, x0=0",
            "iterations": rep.iterations_used, "time_to_solution_s": t / steps, "value": N * its / t / 1e9,
            "unit": UNIT, "kernel": "k_cg_persistent", "kernel_us": 1e6 * k_s,
            "roofline_frac": kbytes / k_s / 1e9 / hbm, "traffic": ncu_traffic("k_cg_persistent")}


def run_config2_line(args):
    """--workload config2: round 1's bench line (single-block CG), N = 1."""
    import torch

    import paper_2009_12638_b200 as bs
    from paper_2009_12638_b200 import _lib

    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0")))
    torch.cuda.set_device(dev)
    r = config2_check(args, torch, dev, bs, _lib.load(), steps=args.steps, warmup=args.warmup)
    print(json.dumps({"metric": METRIC + " (config2 kernel check)", "value": r["value"], "unit": UNIT,
                      "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "dtype": "f64",
                      "config": workload_config(args), **r}), flush=True)


# ---------------------------------------------------------------- supplemental outer workloads


def region_sizes(n, block_grid, overlap):
    """N_b of every block: its extended region (SURVEY §8 notation)."""
    from paper_2009_12638_b200.problems import Grid3D, decompose, region_size

    decomp = decompose(Grid3D(n, n, n), block_grid, overlap)
    return [region_size((n, n, n), box, overlap) for box in decomp.owned]


def run_outer_workload(args):
    """Supplemental: time-to-solution of configs 4 (async) and 5 (overlapping
    GMRES) on this box (1 GPU: all blocks on one device; torchrun: sharded)."""
    import torch
    import torch.distributed as dist

    import paper_2009_12638_b200 as bs

    w = WORKLOADS[args.workload]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    n = grid_n(args)
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

    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    res = outer_solve_distributed(prob, cfg, transport=args.transport) if world > 1 else bs.outer_solve(prob, cfg)
    torch.cuda.synchronize(dev)
    t = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    tts = float(t.item())
    total_its = int(sum(sum(row) for row in res.inner_iterations_per_block))
    nb = int(np.prod(w["block_grid"]))
    if w["overlap"] == 0:
        alg = sum((N / nb) * (64 * i + 64) for row in res.inner_iterations_per_block for i in row)
        gpts = N * total_its / nb / tts / 1e9
    else:
        # Arnoldi step j of a GMRES(m) cycle moves 32 + 24 (j + 1)
        # B/pt over the block's region (N_b = owned box dilated by the overlap)
        sizes = region_sizes(n, w["block_grid"], w["overlap"])
        m = 30

        def block_bytes(k):
            return sum(32 + 24 * ((j % m) + 1) for j in range(k)) + 64

        alg = sum(sizes[b] * block_bytes(i) for row in res.inner_iterations_per_block for b, i in enumerate(row))
        gpts = sum(sizes[b] * i for row in res.inner_iterations_per_block for b, i in enumerate(row)) / tts / 1e9
    hbm = peaks()[0]
    if rank == 0:
        print(json.dumps({
            "metric": METRIC + " (supplemental: " + args.workload + ")", "workload": args.workload,
            "grid": [n, n, n], "n_gpus": world, "config": {k: (list(v) if isinstance(v, tuple) else v)
                                                         for k, v in w.items()},
            "time_to_solution_s": tts, "outer_sweeps": res.outer_iterations, "converged": res.converged,
            "seconds_per_sweep": tts / max(1, res.outer_iterations), "max_outer": args.max_outer,
            "estimates": [row.estimated_residual for row in res.trace.rows][-3:],
            "final_true_residual": res.final_true_residual, "inner_iterations_total": total_its,
            "stencil_gpts_per_s": gpts, "hbm_fraction": alg / tts / 1e9 / (hbm * world),
            "dtype": "f64", "data": "synthetic" if not w["faces"] else "Dirichlet z_lo=1"}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        spawn_ranks(args)
    if args.workload == "config3":
        run_config3(args)
    elif args.workload == "config2":
        run_config2_line(args)
    else:
        run_outer_workload(args)


if __name__ == "__main__":
    main()
