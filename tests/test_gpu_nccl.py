"""NCCL plumbing of libhbgpu on the GPU box (one GPU: world size 1).

The pool gives one GPU per call, so the multi-GPU data path is validated by
the loopback transport (test_gpu_parity.py) and the gloo emulation
(test_layout_and_multirank.py); this file checks the NCCL side itself:
dlopen of libnccl, unique-id broadcast, communicator creation, the device
all-gather + rank-ordered fold used for the force history, and an engine
carrying a communicator.
"""

import ctypes
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.fixture
def world1(cuda):
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{_free_port()}", rank=0, world_size=1)
    yield dist
    dist.destroy_process_group()


def test_comm_allgather_and_ordered_fold(world1):
    import torch
    from paper_1304_7654_b200 import native
    from paper_1304_7654_b200.solver import make_comm
    lib = native.load()
    comm = make_comm(0, 1, torch.cuda.current_device())
    try:
        src = torch.arange(12, dtype=torch.float64, device="cuda") * 0.5
        dst = torch.empty(12, dtype=torch.float64, device="cuda")
        s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        native.check(lib.hbgpu_comm_allgather(comm, ctypes.c_void_p(src.data_ptr()),
                                              ctypes.c_void_p(dst.data_ptr()), 12, s), "allgather")
        torch.cuda.synchronize()
        assert torch.equal(src, dst)
        stacked = torch.stack([src, src * 3, -src]).contiguous()
        out = torch.empty(12, dtype=torch.float64, device="cuda")
        native.check(lib.hbgpu_ordered_fold(ctypes.c_void_p(stacked.data_ptr()), 3, 12,
                                            ctypes.c_void_p(out.data_ptr()), s), "fold")
        torch.cuda.synchronize()
        want = (stacked[0].cpu().numpy() + stacked[1].cpu().numpy()) + stacked[2].cpu().numpy()
        assert np.array_equal(out.cpu().numpy(), want)
    finally:
        native.check(lib.hbgpu_comm_destroy(comm), "destroy")


def test_engine_with_communicator_matches_oracle(world1, oracle_mod):
    import torch
    from paper_1304_7654_b200 import build_cut_plan, build_topology, partition_blocks, tc2_mini
    from paper_1304_7654_b200.solver import DeviceRank, make_comm
    case = tc2_mini()
    topo = build_topology(case)
    part = partition_blocks(topo, 1)
    plan = build_cut_plan(topo, part, case.nharms, case.npde)
    comm = make_comm(0, 1, torch.cuda.current_device())
    dr = DeviceRank(case, topo, part, plan, comm=comm, max_iters=3)
    try:
        dr.prime()
        dr.iterate(3)
        torch.cuda.synchronize()
        got = dr.fields(0)
    finally:
        dr.close()
        from paper_1304_7654_b200 import native
        native.load().hbgpu_comm_destroy(comm)
    want = oracle_mod.run(case, 3)
    for b, q in want.fields.items():
        assert np.array_equal(got[b], q)
