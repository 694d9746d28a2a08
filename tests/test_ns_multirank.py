"""North-star physics sharded over ranks (§8 e).

The NS path splits a case's blocks over ranks (nsflow.ns_partition, the
proxy path's LPT rule).  Per RK stage each rank copies its local cut halos,
packs the halo values its peers need into one payload per peer, the payloads
move (NCCL on GPUs, gloo here), and each rank unpacks; the per-block residual
sums and per-face force products are kept at job-wide positions, summed over
ranks (exact: one contributor per entry) and folded as one rank's.

CPU: the split exchange plans (nsflow.HaloPlan) applied with numpy -- in one
process and between two gloo processes -- fill every halo exactly as the
single-rank plan does.  GPU: run_ns_ranks (the ranks' engines on one GPU, the
payloads moved by device copies) equals the single-rank run bit for bit --
fields with halos, residual norms, wall forces -- and the oracle.
"""

import os
import socket
import tempfile

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1304_7654_b200 import nsflow

SPLITS = [("C1", 8, 2), ("C1", 8, 4), ("C3", 32, 3), ("C4", 128, 8), ("C4", 128, 5)]


def _layout(case, blocks):
    off, n = {}, 0
    for b in sorted(blocks, key=lambda b: b.id):
        off[b.id] = n
        n += case.planes * 4 * (b.nj + 4) * (b.ni + 4)
    return off, n


def _apply(rows, pool, send, recv, nv):
    """hbgpu_halo on numpy arrays (kinds: 0 slot, 1 send buffer, 2 receive buffer)."""
    for r in rows:
        src = (pool, send, recv)[r["src_kind"]]
        dst = (pool, send)[r["dst_kind"]]
        e = np.arange(r["length"])[:, None]
        v = np.arange(nv)[None, :]
        dst[r["dst_off"] + e * r["dst_es"] + v * r["dst_vs"]] = src[r["src_off"] + e * r["src_es"] + v * r["src_vs"]]


def _single_rank(case, seed=5):
    off, n = _layout(case, case.blocks)
    pool = np.random.default_rng(seed).uniform(-1, 1, n)
    want = pool.copy()
    _apply(nsflow.HaloPlan(case, off).first, want, None, None, 4 * case.planes)
    return off, pool, want


def _rank_pool(case, owner, rank, goff, gpool):
    blocks = [b for b in case.blocks if owner[b.id] == rank]
    off, n = _layout(case, blocks)
    pool = np.empty(n)
    for b in blocks:
        m = case.planes * 4 * (b.nj + 4) * (b.ni + 4)
        pool[off[b.id]:off[b.id] + m] = gpool[goff[b.id]:goff[b.id] + m]
    return blocks, off, pool


def _check(case, goff, want, blocks, off, pool):
    for b in blocks:
        m = case.planes * 4 * (b.nj + 4) * (b.ni + 4)
        assert np.array_equal(pool[off[b.id]:off[b.id] + m], want[goff[b.id]:goff[b.id] + m]), f"block {b.id}"


@pytest.mark.parametrize("key,scale,nranks", SPLITS)
def test_split_exchange_fills_halos_like_one_rank(key, scale, nranks):
    case = nsflow.ns_workload(key, scale=scale)
    nv = 4 * case.planes
    goff, gpool, want = _single_rank(case)
    owner = nsflow.ns_partition(case, nranks)
    ranks = []
    for r in range(nranks):
        blocks, off, pool = _rank_pool(case, owner, r, goff, gpool)
        plan = nsflow.HaloPlan(case, off, owner, r)
        send, recv = np.zeros(max(1, plan.nsend)), np.zeros(max(1, plan.nrecv))
        _apply(plan.first, pool, send, None, nv)
        ranks.append((blocks, off, pool, plan, send, recv))
    assert any(rk[3].sends for rk in ranks), "the split must have remote cuts"
    for r, (blocks, off, pool, plan, send, recv) in enumerate(ranks):
        for q, o, c in plan.recvs:
            peer = ranks[q][3]
            so, sc = {p: (o2, c2) for p, o2, c2 in peer.sends}[r]
            assert sc == c
            recv[o:o + c] = ranks[q][4][so:so + sc]
        _apply(plan.unpack, pool, None, recv, nv)
        _check(case, goff, want, blocks, off, pool)


def test_partition_is_the_proxy_lpt_rule():
    case = nsflow.ns_workload("C3", scale=32)
    owner = nsflow.ns_partition(case, 3)
    assert [owner[b] for b in range(8)] == [0, 1, 2, 0, 1, 2, 0, 1]   # equal blocks: b mod G
    off, n = nsflow.wall_layout(case)
    assert n == 4 * 32 and [off[b] for b in range(4)] == [0, 32, 64, 96]   # bottom row of 4 walls


# ---- two gloo processes ---------------------------------------------------------------

def _worker(rank, world, port, outdir):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        import torch
        case = nsflow.ns_workload("C1", scale=8)
        nv = 4 * case.planes
        goff, gpool, want = _single_rank(case)
        owner = nsflow.ns_partition(case, world)
        blocks, off, pool = _rank_pool(case, owner, rank, goff, gpool)
        plan = nsflow.HaloPlan(case, off, owner, rank)
        send, recv = np.zeros(max(1, plan.nsend)), np.zeros(max(1, plan.nrecv))
        _apply(plan.first, pool, send, None, nv)
        ops, bufs = [], []
        for q, o, c in plan.sends:
            ops.append(dist.P2POp(dist.isend, torch.from_numpy(send[o:o + c].copy()), q))
        for q, o, c in plan.recvs:
            t = torch.empty(c, dtype=torch.float64)
            bufs.append((o, t))
            ops.append(dist.P2POp(dist.irecv, t, q))
        for req in dist.batch_isend_irecv(ops):
            req.wait()
        for o, t in bufs:
            recv[o:o + t.numel()] = t.numpy()
        _apply(plan.unpack, pool, None, recv, nv)
        _check(case, goff, want, blocks, off, pool)
        open(os.path.join(outdir, f"ok{rank}"), "w").close()
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_rank_exchange_over_gloo():
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_worker, args=(2, _free_port(), d), nprocs=2, join=True, start_method="spawn")
        assert os.path.exists(os.path.join(d, "ok0")) and os.path.exists(os.path.join(d, "ok1"))


# ---- GPU: the sharded run equals the single-rank run ------------------------------------

@pytest.mark.gpu
@pytest.mark.parametrize("key,scale,nranks", SPLITS)
def test_gpu_ranks_equal_single_rank_and_oracle(key, scale, nranks, cuda):
    import ns_oracle
    case = nsflow.ns_workload(key, scale=scale)
    iters = 4
    one = nsflow.run_ns(case, iters)
    got = nsflow.run_ns_ranks(case, iters, nranks)
    gf, of = got.fields(), one.fields()
    for b in of:
        assert np.array_equal(gf[b], of[b]), f"{key}/{nranks} block {b}"
    assert got.norm_history() == one.norm_history()
    assert np.array_equal(got.force_history(), one.force_history())
    want = ns_oracle.run(case, iters)
    for b, q in want.fields().items():
        assert np.array_equal(gf[b], q), f"{key}/{nranks} block {b} vs oracle"
    np.testing.assert_allclose(got.norm_history(), want.norms, rtol=1e-12, atol=0)
