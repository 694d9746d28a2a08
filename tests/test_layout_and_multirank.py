"""Device-layout tables and the multi-rank exchange schedule, on CPU.

tests/devemu.py executes the engine's schedule with numpy over the exact
tables libhbgpu consumes (face-target pool, priming / unpack directions,
per-peer send / receive segments).  Single-rank runs check the local
forwarding tables; world_size-2 runs over torch.distributed gloo check the
remote pack, the one-message-per-peer pairing, the unpack and the
rank-ordered force fold -- all bitwise against the single-rank oracle.
"""

import os
import socket
import tempfile

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from devemu import RankEmulator, run_schedule
from paper_1304_7654_b200 import (BlockSpec, build_cut_plan, build_topology, lattice_case,
                                  pair_case, partition_blocks, ring_case, tc_tiny)
from paper_1304_7654_b200.devlayout import build_rank_layout
from paper_1304_7654_b200.topology import CaseConfig, CutSide, CutSpec


def _self_cut_reversed():
    blk = BlockSpec(0, 12, 9, 0.5, 0.25, 0.05, body_faces=(("east", 0),))
    return CaseConfig(nharms=2, npde=4, iterations=3, dtau=0.0005, omega=1.0, nbody=1,
                      blocks=[blk], cuts=[CutSpec(CutSide(0, "north", 2, 7), CutSide(0, "south", 3, 8),
                                                  reversed=True)], name="self-cut-reversed")


SINGLE = {
    "tc-tiny": (tc_tiny, 3),
    "pair-reversed": (lambda: pair_case(6, 5, 2, h=0.2, dtau=0.01, reversed_cut=True, nbody=1,
                                        bodies=((1, "north", 0),)), 3),
    "self-cut-reversed": (_self_cut_reversed, 3),
    "lattice-3x2": (lambda: lattice_case(3, 2, 9, 7, 1, h=0.05, dtau=0.001, nbody=2,
                                         bodies=((0, "south", 0), (4, "north", 1))), 2),
}


def _no_remote(emu, slot):
    assert not emu.L.sends and not emu.L.recvs


@pytest.mark.parametrize("name", sorted(SINGLE))
def test_single_rank_tables_reproduce_oracle(name):
    build, iters = SINGLE[name]
    case = build()
    topo = build_topology(case)
    part = partition_blocks(topo, 1)
    plan = build_cut_plan(topo, part, case.nharms, case.npde)
    emu = run_schedule(RankEmulator(case, topo, part, plan, 0), iters, _no_remote)
    want = oracle.run(case, iters)
    for b, q in emu.fields().items():
        assert np.array_equal(q, want.fields[b]), f"block {b}"
    assert np.array_equal(emu.force_hist[-1], want.forces)


def test_layout_alignment_and_tiles():
    case = lattice_case(2, 2, 45, 19, 3, h=0.02, dtau=0.0005)
    topo = build_topology(case)
    part = partition_blocks(topo, 1)
    L = build_rank_layout(topo, part, build_cut_plan(topo, part, 3, 4), 0, case.planes, tile_rows=8)
    for k, b in enumerate(L.blocks):
        assert L.base[k] % 32 == 0 and L.pitch[k] % 8 == 0
        assert L.elem(b.id, 0, 0, 0, 1) % 8 == 0        # interior column 1: 64-B granule aligned
        assert L.pitch[k] >= b.ni + 2 + 7
        t = L.block_table[k]
        assert t["ntiles"] == t["tiles_i"] * t["tiles_j"]
        assert t["sxy_off"] % 4 == 0 and t["sxy_pitch"] >= b.ni
        sx, sy = L.sxy[k]
        from paper_1304_7654_b200.hbop import forcing_table
        assert np.array_equal(sx[None, :] * sy[:, None], forcing_table(b))
    assert len(L.tile_block) == L.total_tiles == sum(int(t) for t in L.block_table["ntiles"])
    # every face cell on a cut has exactly one pool target; west / east ones
    # are also covered by the first stage's post-pass directions
    assert np.count_nonzero(L.faces["ps"]) == sum(2 * c.length for c in topo.cuts)
    cols = sum(c.length for c in topo.cuts for side in (c.side_a, c.side_b)
               if side.face in ("west", "east"))
    assert int(L.post_dirs["length"].sum()) == cols > 0


# ---------------------------------------------------------------------------
# world_size 2 over gloo
# ---------------------------------------------------------------------------

MULTI = {
    "tc-tiny": (tc_tiny, 3),
    "pair-reversed": (lambda: pair_case(6, 5, 2, h=0.2, dtau=0.01, reversed_cut=True, nbody=1,
                                        bodies=((1, "north", 0),)), 2),
    "ring4": (lambda: ring_case(4, 7, 5, 1, h=0.1, dtau=0.002, nbody=2,
                                bodies=((0, "south", 0), (3, "north", 1))), 2),
    "lattice-3x2": (lambda: lattice_case(3, 2, 9, 7, 2, h=0.05, dtau=0.001, nbody=1,
                                         bodies=((1, "south", 0),)), 2),
}


def _gloo_exchange(emu, slot):
    ops = []
    for peer, off, count in emu.L.sends:
        import torch
        ops.append(dist.P2POp(dist.isend, torch.from_numpy(emu.sendbuf[off:off + count].copy()), peer))
    recv_bufs = []
    for peer, off, count in emu.L.recvs:
        import torch
        t = torch.empty(count, dtype=torch.float64)
        recv_bufs.append((off, t))
        ops.append(dist.P2POp(dist.irecv, t, peer))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    for off, t in recv_bufs:
        emu.recvbuf[off:off + t.numel()] = t.numpy()
    emu.halo(emu.L.unpack_dirs, slot)


def _worker(rank, world, port, name, outdir):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        build, iters = MULTI[name]
        case = build()
        topo = build_topology(case)
        part = partition_blocks(topo, world)
        plan = build_cut_plan(topo, part, case.nharms, case.npde)
        emu = run_schedule(RankEmulator(case, topo, part, plan, rank), iters, _gloo_exchange)
        fields = [None] * world
        dist.all_gather_object(fields, emu.fields())
        hists = [None] * world
        dist.all_gather_object(hists, emu.force_hist)
        if rank == 0:
            merged = {k: v for part_ in fields for k, v in part_.items()}
            forces = oracle.ordered_sum([h[-1] for h in hists])   # runtime.py:290-294 order
            np.savez(os.path.join(outdir, "out.npz"), forces=forces,
                     **{f"f{b}": q for b, q in merged.items()})
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("name", sorted(MULTI))
def test_two_rank_exchange_matches_single_rank_oracle(name):
    build, iters = MULTI[name]
    case = build()
    topo = build_topology(case)
    part = partition_blocks(topo, 2)
    plan = build_cut_plan(topo, part, case.nharms, case.npde)
    assert any(not c.local for c in plan.cuts), "case must have a remote cut"
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_worker, args=(2, _free_port(), name, d), nprocs=2, join=True,
                           start_method="spawn")
        got = np.load(os.path.join(d, "out.npz"))
        want = oracle.run(case, iters)
        for b, q in want.fields.items():
            assert np.array_equal(got[f"f{b}"], q), f"block {b}"
        assert np.array_equal(got["forces"], want.forces)


def test_peer_messages_pair_up():
    """Rank r's send segment to s has exactly the length of s's receive from r."""
    case = lattice_case(4, 2, 16, 8, 1, h=0.05, dtau=0.001)
    topo = build_topology(case)
    for world in (2, 4, 8):
        part = partition_blocks(topo, world)
        plan = build_cut_plan(topo, part, 1, 4)
        lay = [build_rank_layout(topo, part, plan, r, case.planes) for r in range(world)]
        for r in range(world):
            for peer, _, count in lay[r].sends:
                match = [c for p, _, c in lay[peer].recvs if p == r]
                assert match == [count]
            assert lay[r].sendbuf_elems == sum(c for _, _, c in lay[r].sends)


def test_paired_schedule_eligibility_and_band_segments():
    """Paired stages need P <= 9 and every block a whole number of strips;
    the band covers the first / last row of every row tile and the face
    columns that feed a cut (paired-kernel edge warp covers the rest)."""
    from paper_1304_7654_b200.devlayout import fused_eligible
    from paper_1304_7654_b200 import baseline_workload
    for key in ("C0", "C1", "C2", "C3", "C4"):
        case = baseline_workload(key).case
        topo = build_topology(case)
        part = partition_blocks(topo, 1)
        plan = build_cut_plan(topo, part, case.nharms, 4)
        L = build_rank_layout(topo, part, plan, 0, case.planes)
        # auto: paired stages only from FUSED_MIN_UNITS units per stage (C3, C4)
        assert L.fused == (key in ("C3", "C4")), key
        assert build_rank_layout(topo, part, plan, 0, case.planes, fused=True).fused, key
    case = lattice_case(2, 2, 45, 19, 3, h=0.02, dtau=0.0005)          # ragged strips
    topo = build_topology(case)
    assert not fused_eligible(topo.blocks, case.planes, 4)
    assert not fused_eligible(build_topology(lattice_case(2, 1, 256, 8, 5, h=0.02, dtau=0.0005)).blocks, 11, 1)
    case = lattice_case(3, 2, 256, 40, 2, h=0.01, dtau=0.0002)
    topo = build_topology(case)
    part = partition_blocks(topo, 1)
    L = build_rank_layout(topo, part, build_cut_plan(topo, part, 2, 4), 0, case.planes, tile_rows=16)
    segs = L.band_segs
    for k, b in enumerate(L.blocks):
        rows = sorted(int(s["j"]) for s in segs if s["block"] == k and s["dir"] == 0)
        want = sorted({r for j0 in range(1, b.nj + 1, 16) for r in (j0, min(j0 + 15, b.nj))})
        assert rows == want
        cols = sorted(int(s["i"]) for s in segs if s["block"] == k and s["dir"] != 0)
        face = L.block_table["face_off"][k]
        assert cols == sorted(c for c, fi in ((1, 2), (b.ni, 3)) if face[fi] >= 0)
        assert all(int(s["len"]) == (b.ni if s["dir"] == 0 else b.nj) for s in segs if s["block"] == k)
