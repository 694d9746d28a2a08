"""Failure handling of the multi-GPU run (solver.CommGuard), on CPU.

The reference aborts its fabric when any rank fails, reports the first
failing rank (RankFailure) and bounds every wait by a 120 s timeout
(runtime.py:29, 133-144, 176-187, 345-364).  On B200s the waits are on CUDA
events of work that includes NCCL operations; CommGuard bounds them with the
communicator's async-error state, a failure notice in torch.distributed's
store and a deadline, and aborts the communicator on any of them.

Here the NCCL side is replaced by fakes (an event that never completes, a
recorded abort) and the notice travels between two real gloo processes.
"""

import os
import socket
import tempfile
import time

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1304_7654_b200.exceptions import CollectiveError, RankFailure, RunAborted
from paper_1304_7654_b200.solver import CommGuard


class NeverDone:
    def query(self):
        return False


class DoneAfter:
    def __init__(self, n):
        self.n = n

    def query(self):
        self.n -= 1
        return self.n < 0


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_timeout_aborts_and_raises_collective_error():
    aborted = []
    g = CommGuard(None, 0, None, timeout=0.2, async_error=lambda: None, abort=lambda: aborted.append(1))
    t0 = time.monotonic()
    with pytest.raises(CollectiveError, match="did not complete"):
        g.wait(NeverDone())
    assert 0.2 <= time.monotonic() - t0 < 5
    assert aborted == [1] and g.aborted


def test_async_error_aborts_and_raises():
    aborted = []
    g = CommGuard(None, 3, None, timeout=30, async_error=lambda: "NCCL asynchronous error: remote process exited",
                  abort=lambda: aborted.append(1))
    with pytest.raises(CollectiveError, match="rank 3: NCCL asynchronous error"):
        g.wait(NeverDone())
    assert aborted == [1]


def test_completed_work_passes():
    g = CommGuard(None, 0, None, timeout=5, async_error=lambda: None, abort=lambda: pytest.fail("abort"))
    g.wait(DoneAfter(10))
    assert not g.aborted


def _worker(rank, world, port, outdir):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    store = dist.distributed_c10d._get_default_store()
    aborted = []
    g = CommGuard(None, rank, store, timeout=30, async_error=lambda: None, abort=lambda: aborted.append(1))
    dist.barrier()
    result = "none"
    if rank == 1:
        # this rank fails: it posts the notice and aborts its communicator
        g.notify_failure()
        result = f"notified aborted={len(aborted)}"
    else:
        t0 = time.monotonic()
        try:
            g.wait(NeverDone())    # a collective the failed peer will never join
        except RankFailure as e:
            ok = isinstance(e.cause, RunAborted)
            result = f"rankfailure rank={e.rank} cause_ok={ok} aborted={len(aborted)} " \
                     f"fast={time.monotonic() - t0 < 10}"
    with open(os.path.join(outdir, f"r{rank}.txt"), "w") as fh:
        fh.write(result)
    dist.barrier()
    dist.destroy_process_group()


def test_peer_failure_notice_wakes_the_other_rank():
    """Two gloo processes: rank 1 fails; rank 0, waiting on work its peer
    will never complete, raises RankFailure(1, RunAborted) within seconds
    (not after the timeout) and aborts its own communicator."""
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_worker, args=(2, _free_port(), d), nprocs=2, join=True, start_method="spawn")
        r0 = open(os.path.join(d, "r0.txt")).read()
        r1 = open(os.path.join(d, "r1.txt")).read()
    assert r1 == "notified aborted=1"
    assert r0 == "rankfailure rank=1 cause_ok=True aborted=1 fast=True"
