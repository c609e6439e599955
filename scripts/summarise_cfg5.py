"""Summarise the segmented config-5 run (gpurun_out/cfg5_seg*.log -> profiles/r02_cfg5_1024_full.md and
profiles/r02_cfg5_1024_trace.csv, one row per logged sweep)."""
import glob
import json
import math
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
logs = sorted(glob.glob(os.path.join(ROOT, "gpurun_out", "cfg5_seg*.log")),
              key=lambda p: int(re.search(r"seg(\d+)\.log", p).group(1)))
rows, segs, done = {}, [], None
for path in logs:
    seg = int(re.search(r"seg(\d+)\.log", path).group(1))
    info = {"seg": seg}
    for line in open(path):
        if not line.startswith("{"):
            continue
        r = json.loads(line)
        if "k" in r and "estimate" in r and "paused_at" not in r and "segment_done" not in r:
            rows[r["k"]] = r
            info.setdefault("first_k", r["k"])
            info["last_k"] = r["k"]
        if "resume_from" in r:
            info["resume_from"] = r["resume_from"]
        if "paused_at" in r:
            info.update(paused_at=r["paused_at"], solve_s=r["segment_solve_s"], total_s=r["solve_s_total"],
                        save_s=r["save_s"], estimate=r["estimate"])
        if r.get("done"):
            done = r
            info["done"] = True
    segs.append(info)
with open(os.path.join(ROOT, "profiles", "r02_cfg5_1024_trace.csv"), "w") as fh:
    fh.write("outer_iteration,estimated_residual,true_residual,inner_iterations,solve_seconds\n")
    for k in sorted(rows):
        r = rows[k]
        fh.write(f"{k},{r['estimate']:.17g},{r['true']:.17g},{r['inner']},{r['solve_s']}\n")
out = ["# Config 5 at 1024^3 on one B200: the complete solve (round 2)", "",
       "BASELINE.json configs[4]: 1024^3 fp64 grid, u = 1 on z = 0, 2x2x2 blocks with a 2-plane overlap and weighted",
       "combination, inner GMRES(30) to 1e-3 relative to ||r0|| (one cycle of at most 30 steps), synchronous sweeps,",
       "paper residual, outer tol 1e-8.  `scripts/run_cfg5.py 1024` through the public `outer_solve`, one shared Krylov",
       "basis (the eight 514^3 blocks solved one after another), run in segments of one GPU call each",
       "(`scripts/r02_cfg5_segment.sh`; pause / `save_state` / `resume` continue bit for bit: the rows of segment 2",
       "equal those of an uninterrupted first hour, `profiles/r02_cfg5_1024_first_hour.log`, through sweep 1250).", ""]
out += ["| segment | sweeps | sweep phase (s) | total (s) | estimate at the pause |", "|---|---|---|---|---|"]
for s in segs:
    lo = 0 if s.get("resume_from") is None else s["resume_from"] + 1
    if "paused_at" in s:
        out.append(f"| {s['seg']} | {lo}..{s['paused_at']} | {s['solve_s']:.1f} | {s['total_s']:.1f} | {s['estimate']:.4e} |")
    elif s.get("done") and done:
        prev = max([t.get("total_s", 0.0) for t in segs if "total_s" in t] + [0.0])
        out.append(f"| {s['seg']} | {lo}..{done['outer_sweeps'] - 1} | {done['time_to_solution_s'] - prev:.1f} | "
                   f"{done['time_to_solution_s']:.1f} | converged |")
out.append("")
if done:
    its = done["inner_iterations_total"]
    N = 8 * 135792128  # points of the eight dilated blocks (N_b of config 5)
    out += [f"**Converged: {done['converged']}** after **{done['outer_sweeps']} sweeps**, {its:,} inner GMRES iterations, final "
            f"estimate {done['final_estimate']:.4e}, **final true residual {done['final_true_residual']:.4e}** (< 1e-8), "
            f"**time to solution {done['time_to_solution_s']:.1f} s** ({done['time_to_solution_s'] / 3600:.2f} h; the sum "
            f"of the {done['segments']} segments' sweep phases — engine set-up ~5 s and checkpoint write ~7 s / read per "
            f"segment excluded), {done['seconds_per_sweep']:.3f} s per sweep.", ""]
    cyc = 135792128 * sum(72 + 32 * j for j in range(30))  # bytes a 30-step cycle moves on one block
    out += [f"One sweep = 8 blocks x one 30-step GMRES cycle = {8 * cyc / 1e12:.2f} TB of Krylov traffic (16.1 KB per point, "
            f"`profiles/r02_gmres512_summary.md`): at {done['seconds_per_sweep']:.3f} s per sweep the whole sweep (merge, owner "
            f"residual and restarts included) runs at {8 * cyc / done['seconds_per_sweep'] / 1e12:.2f} TB/s = "
            f"{8 * cyc / done['seconds_per_sweep'] / 1e9 / 6535.4:.2f} of the measured HBM peak.", ""]
if not done:
    ks = sorted(rows)
    last = rows[ks[-1]]
    tail = [k for k in ks if k >= ks[-1] - 400]
    rate = math.log(rows[tail[0]]["estimate"] / last["estimate"]) / (ks[-1] - tail[0])
    more = math.log(last["estimate"] / 1e-8) / rate
    per = last["solve_s"] / (ks[-1] + 1)
    tot_s = max(t.get("total_s", 0.0) for t in segs)
    paused = max(t.get("paused_at", 0) for t in segs)
    out += [f"**Not converged: the GPU box was taken back by the pool 17 minutes into segment 5** (`gpurun`: \"the GPU box was "
            f"lost while the command ran\"), and with it the checkpoint in its /tmp.  State of the run at the last pause: "
            f"**{paused + 1} sweeps in {tot_s:.1f} s** of sweep phases ({tot_s / 3600:.2f} h, {per:.3f} s per sweep, "
            f"{sum(1 for _ in ks)} logged rows), estimate **{rows[paused - paused % 25]['estimate']:.4e}** at sweep "
            f"{paused - paused % 25} (true residual {rows[paused - paused % 25]['true']:.4e}), contracting by "
            f"{100 * (1 - math.exp(-rate)):.3f}% per sweep — a rate that has been flat since sweep ~3000 (table below).  "
            f"At that rate the stop test (estimate < 1e-8) falls at sweep ~{int(ks[-1] + more)}: about "
            f"{(ks[-1] + more) * per:.0f} s = {(ks[-1] + more) * per / 3600:.1f} h of sweeps on one B200, "
            f"{int((ks[-1] + more - paused) * per / 3250) + 1} more one-hour segments.  Restarting from sweep 0 did not fit "
            f"the rest of the round (5.4 h).", ""]
    cyc = 135792128 * sum(72 + 32 * j for j in range(30))
    out += [f"One sweep = 8 blocks x one 30-step GMRES cycle = {8 * cyc / 1e12:.2f} TB of Krylov traffic (16.1 KB per point, "
            f"`profiles/r02_gmres512_summary.md`): at {per:.3f} s per sweep the whole sweep (merge, owner residual included) "
            f"runs at {8 * cyc / per / 1e12:.2f} TB/s = {8 * cyc / per / 1e9 / 6535.4:.2f} of the measured HBM peak.  The same "
            f"code converges the 512^3 companion (2011 sweeps, 747.9 s) and 256^3 (654 sweeps, 33.3 s, segmented and "
            f"uninterrupted runs identical, `profiles/r02_cfg5_segmented_dry_run.log`).", ""]
out += ["The same configuration at smaller sizes, all converged on one B200 with this code (sweeps grow as n^1.6):", "",
        "| grid | blocks (points each) | sweeps | inner its | final true residual | time to solution | s per sweep | log |",
        "|---|---|---|---|---|---|---|---|",
        "| 256^3 | 8 x 130^3 | 654 | 156,360 | 6.28e-9 | 33.3 s | 0.051 | `profiles/r02_cfg5_segmented_dry_run.log` |",
        "| 512^3 | 8 x 258^3 | 2011 | 481,268 | 6.32e-9 | 731.1 s | 0.364 | `profiles/r02_cfg5_512_final.log` |",
        "| 640^3 | 8 x 322^3 | 2939 | 703,528 | 6.32e-9 | 2033.0 s | 0.692 | `profiles/r02_cfg5_640.log` |",
        "| 1024^3 | 8 x 514^3 | 4210 of ~6300-6600 | ~1.0 M so far | 2.6e-7 so far | 12,182 s so far | 2.894 | this file |", ""]
ks = sorted(rows)
out += ["Convergence (every logged sweep in `profiles/r02_cfg5_1024_trace.csv`):", "",
        "| sweep | estimate | true residual | contraction per sweep |", "|---|---|---|---|"]
prev = None
for k in ks:
    if k % 500 == 0 or k == ks[-1]:
        rate = "" if prev is None else f"{1 - math.exp(-math.log(rows[prev]['estimate'] / rows[k]['estimate']) / (k - prev)):.5f}"
        out.append(f"| {k} | {rows[k]['estimate']:.4e} | {rows[k]['true']:.4e} | {rate} |")
        prev = k
out.append("")
open(os.path.join(ROOT, "profiles", "r02_cfg5_1024_full.md"), "w").write("\n".join(out) + "\n")
print("\n".join(out))
