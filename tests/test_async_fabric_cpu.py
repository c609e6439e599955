"""Host side of the multi-process asynchronous fabric (async_driver._Board
over node-shared memory, _Rendezvous = block threads + a gloo barrier),
exercised with two gloo processes on CPU: one-sided board writes are seen
by the other process, the +inf-until-published estimate, the confirmation
round's barrier across processes and threads, and flag hand-off."""

import math
import os
import socket
import tempfile
import threading

import numpy as np


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch

    from paper_2009_12638_b200.async_driver import _Board, _close_fabric, _shared_store

    torch.distributed.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                                         world_size=world)
    nb = 4
    local = [2 * rank, 2 * rank + 1]
    store, shm = _shared_store(nb, None)
    board = _Board(nb, len(local), store, None, multi=True)
    log = {}

    def block(b):
        # before every block published once the estimate is +inf (comm.py:455-527)
        log[(b, "inf")] = math.isinf(board.estimate())
        board.barrier.wait()
        board.local_sq[b] = float(b + 1)          # one-sided publish
        board.barrier.wait()
        log[(b, "est")] = board.estimate()        # every process sees every block
        if b == 3:
            board.confirm_requested = True
        board.barrier.wait()
        log[(b, "flag")] = board.confirm_requested
        board.confirm_sq[b] = float(10 * (b + 1))
        board.barrier.wait()
        log[(b, "sum")] = float(sum(board.confirm_sq[w] for w in range(nb)))

    threads = [threading.Thread(target=block, args=(b,)) for b in local]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    torch.distributed.barrier()
    np.save(os.path.join(out, f"fab_{rank}.npy"), np.asarray(
        [[log[(b, "inf")], log[(b, "est")], log[(b, "flag")], log[(b, "sum")]] for b in local], dtype=float))
    _close_fabric([], shm, True)
    torch.distributed.destroy_process_group()


def test_board_and_rendezvous_across_two_processes():
    import torch.multiprocessing as mp

    with tempfile.TemporaryDirectory() as tmp:
        mp.spawn(_worker, args=(2, _port(), tmp), nprocs=2, join=True)
        for rank in (0, 1):
            got = np.load(os.path.join(tmp, f"fab_{rank}.npy"))
            assert np.all(got[:, 0] == 1.0)
            assert np.allclose(got[:, 1], math.sqrt(1 + 2 + 3 + 4), rtol=0, atol=0)
            assert np.all(got[:, 2] == 1.0)
            assert np.all(got[:, 3] == 100.0)
