"""Config 5 (BASELINE.json configs[4]) to convergence on one GPU: n^3 grid
(default 1024), u = 1 on z_lo, block_grid (2, 2, 2), overlap 2, GMRES(30)
to 1e-3 relative to ||r0||, sync, paper residual, tol 1e-8.  At 1024^3 the
eight 514^3-point blocks share one Krylov basis (solved one after another,
bitwise the per-block numbers).  Progress (sweep, estimate, true residual,
inner its, elapsed) is flushed to stdout every LOG_EVERY sweeps, so a run cut
short still leaves its trace.

Segmented runs (a GPU call here lasts at most an hour, the solve several):
``SEG_BUDGET_S`` = seconds of process time after which the run pauses at the
next sweep boundary, writes the outer iterate (every block's x and halo
planes, ``BlockEngine.save_state``) to ``CKPT_DIR`` together with the trace so
far, and exits 0; the next call with ``RESUME=1`` restores it and continues
bit for bit (tests/test_gpu_checkpoint.py).  Times are accumulated over the
segments' solve phases (checkpoint I/O and set-up excluded, and reported)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_12638_b200 as bs  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
max_outer = int(sys.argv[2]) if len(sys.argv) > 2 else 100000
every = int(os.environ.get("LOG_EVERY", "50"))
budget = float(os.environ.get("SEG_BUDGET_S", "0"))
ckpt = os.environ.get("CKPT_DIR", "/tmp/cfg5_ckpt")
resume = os.environ.get("RESUME", "0") == "1"
t0 = time.perf_counter()

state = {"k": -1, "solve_s": 0.0, "inner": 0, "segments": 0, "rows": []}
if resume:
    meta = os.path.join(ckpt, "state.json")
    if not os.path.exists(meta):
        print(json.dumps({"error": "no checkpoint on this box", "ckpt": ckpt}), flush=True)
        sys.exit(3)
    with open(meta) as fh:
        state = json.load(fh)


class Log:
    paused_at = None

    def attach(self, eng):
        self.eng = eng
        self.t_solve = time.perf_counter()  # engine built, iterate restored: the sweeps start

    def begin(self, phase, k):
        pass

    def end(self, phase, k):
        pass

    def sweep(self, k, its):
        pass

    def trace(self, k, est, true_res, inner):
        state["rows"].append([k, est, true_res, inner])
        if k % every == 0:
            print(json.dumps({"k": k, "estimate": est, "true": true_res, "inner": inner,
                              "solve_s": round(state["solve_s"] + time.perf_counter() - self.t_solve, 2),
                              "elapsed_s": round(time.perf_counter() - t0, 2)}), flush=True)

    def pause(self, k):
        if not budget or time.perf_counter() - t0 < budget:
            return False
        seg = time.perf_counter() - self.t_solve
        t = time.perf_counter()
        self.eng.save_state(ckpt)
        state.update(k=k, solve_s=state["solve_s"] + seg, segments=state["segments"] + 1,
                     inner=sum(r[3] for r in state["rows"]))
        with open(os.path.join(ckpt, "state.json"), "w") as fh:
            json.dump(state, fh)
        print(json.dumps({"paused_at": k, "segment_solve_s": round(seg, 2), "solve_s_total": round(state["solve_s"], 2),
                          "save_s": round(time.perf_counter() - t, 2), "estimate": state["rows"][-1][1]}), flush=True)
        return True


grid = bs.Grid3D(n, n, n, bs.DirichletBoundary({"z_lo": 1.0}))
prob = bs.build_laplace_3d(grid)
cfg = bs.OuterConfig(block_grid=(2, 2, 2), overlap=2, inner=bs.InnerSolverSpec("gmres", 30, 1e-3, 30), mode="sync",
                     tol=1e-8, max_outer=max_outer, tolerance_basis="initial", residual_check_mode="paper")
print(json.dumps({"config": "config5", "n": n, "setup_s": round(time.perf_counter() - t0, 2),
                  "resume_from": state["k"] if resume else None}), flush=True)
log = Log()
res = bs.outer_solve(prob, cfg, probe=log, resume=(state["k"], ckpt) if resume else None)
if log.paused_at is not None:
    print(json.dumps({"segment_done": True, "next": "RESUME=1", "k": log.paused_at}), flush=True)
    sys.exit(0)
solve_s = state["solve_s"] + time.perf_counter() - log.t_solve
rows = state["rows"]
its = sum(r[3] for r in rows)
print(json.dumps({"done": True, "n": n, "converged": res.converged, "outer_sweeps": len(rows),
                  "inner_iterations_total": its, "final_estimate": rows[-1][1],
                  "final_true_residual": res.final_true_residual, "time_to_solution_s": solve_s,
                  "segments": state["segments"] + 1, "seconds_per_sweep": solve_s / len(rows),
                  "note": "time = sum of the segments' sweep phases (engine set-up, checkpoint write / read excluded)"
                  if state["segments"] else "one uninterrupted run"}), flush=True)
