"""Real multi-GPU runs (skipped unless the box has >= 2 GPUs): one process
per GPU over NCCL, the sharded synchronous sweep (distributed.py) with the
NCCL halo transport and with one-sided peer puts (p2p, cross-device CUDA IPC
with lazy peer access), compared bit for bit with the single-process solve
(counts, estimates, iterates) — the basis of "identical counts at 1/2/4/8
GPUs" (comm.py:332-365, 422-453 of the reference).  Also the bench's own
--gpus N spawning (n_gpus must equal N)."""

import json
import os
import socket
import subprocess
import sys
import tempfile

import numpy as np
import pytest

from oracle import blocksolve_oracle as O

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpu():
    import torch

    return torch.cuda.device_count()


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir, transport):
    sys.path.insert(0, ROOT)
    os.environ["LOCAL_RANK"] = str(rank)
    import torch

    import paper_2009_12638_b200 as bs
    from paper_2009_12638_b200.distributed import outer_solve_distributed

    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    torch.distributed.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                                         world_size=world, device_id=dev)
    n = 64
    b = O.seeded_rhs(n ** 3, 0)
    prob = bs.LinearProblem(bs.StencilOperator(n, n, n), b, bs.Grid3D(n, n, n))
    cfg = bs.OuterConfig(block_grid=(1, 1, 8), inner=bs.InnerSolverSpec("cg", 100, 1e-3), tol=1e-8,
                         tolerance_basis="initial", max_outer=60)
    res = outer_solve_distributed(prob, cfg, transport=transport)
    if rank == 0:
        np.savez(os.path.join(out_dir, f"mg_{transport}_{world}.npz"), solution=res.solution,
                 counts=np.asarray(res.inner_iterations_per_block),
                 est=np.asarray([r.estimated_residual for r in res.trace.rows]))
    torch.distributed.destroy_process_group()


@pytest.mark.timeout(900)
@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("transport", ["nccl", "p2p"])
def test_sharded_sweep_on_real_gpus_equals_single_process(transport, world):
    if _ngpu() < world:
        pytest.skip(f"needs {world} GPUs, the box has {_ngpu()}")
    import torch.multiprocessing as mp

    import paper_2009_12638_b200 as bs

    with tempfile.TemporaryDirectory() as tmp:
        mp.spawn(_worker, args=(world, _port(), tmp, transport), nprocs=world, join=True)
        got = np.load(os.path.join(tmp, f"mg_{transport}_{world}.npz"))
    n = 64
    b = O.seeded_rhs(n ** 3, 0)
    prob = bs.LinearProblem(bs.StencilOperator(n, n, n), b, bs.Grid3D(n, n, n))
    cfg = bs.OuterConfig(block_grid=(1, 1, 8), inner=bs.InnerSolverSpec("cg", 100, 1e-3), tol=1e-8,
                         tolerance_basis="initial", max_outer=60)
    ref = bs.outer_solve(prob, cfg)
    assert np.array_equal(got["counts"], np.asarray(ref.inner_iterations_per_block))
    assert np.array_equal(got["est"], np.asarray([r.estimated_residual for r in ref.trace.rows]))
    assert np.array_equal(got["solution"], ref.solution)


@pytest.mark.timeout(900)
def test_bench_spawns_its_ranks():
    """``bench.py --gpus 2`` without WORLD_SIZE launches two ranks itself and
    reports n_gpus = 2 on a bounded config-3 run."""
    if _ngpu() < 2:
        pytest.skip("needs 2 GPUs")
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--max-outer", "12",
                          "--steps", "5", "--warmup", "3", "--no-cpu", "--no-config2"],
                         capture_output=True, text=True, env=env, timeout=800, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["steps"] == 5 and line["scaling"] == "strong"
    assert line["halo"]["planes_per_sweep_sent_remote"] == 1
