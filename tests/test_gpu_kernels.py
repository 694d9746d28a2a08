"""Kernel-level parity on the GPU: each libhbgpu entry point vs the reference.

The residual / update drop-ins are compared bitwise with the reference's own
numba kernels' outputs (tests/golden/kernels.npz, sub-ranges included); the
halo and force kernels with the oracle; the hand-evaluated stencil and
divergence-location cases restate the reference's tests
(tests/test_hbcore.py:100-125, 202-210).
"""

import os

import numpy as np
import pytest

from paper_1304_7654_b200 import (BlockSpec, DivergenceError, build_cut_plan, build_topology,
                                  lattice_case, pair_case, partition_blocks, spectral_matrix)
from paper_1304_7654_b200.hbop import ADVECTION, NU
from paper_1304_7654_b200.topology import CaseConfig, CutSide, CutSpec, Topology

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _torch():
    import torch
    return torch


@pytest.mark.parametrize("tag", ["p3", "p5", "p9"])
def test_residual_and_update_bitwise_vs_reference_kernels(tag, cuda):
    from paper_1304_7654_b200 import blockops
    torch = _torch()
    g = np.load(os.path.join(GOLD, "kernels.npz"))
    ni, nj, nharms, h, omega = g[f"{tag}/meta"]
    ni, nj, nharms = int(ni), int(nj), int(nharms)
    planes = 2 * nharms + 1
    spec = BlockSpec(0, ni, nj, 10.0, 20.0, float(h))
    blk = blockops.BlockState(spec, planes)
    assert np.array_equal(blk.forcing.cpu().numpy(), g[f"{tag}/forcing"])
    deriv = spectral_matrix(nharms, float(omega))
    blk.q.copy_(torch.from_numpy(g[f"{tag}/q"]))
    assert np.array_equal(blockops.residual(blk, deriv), g[f"{tag}/resid_full"])
    blk.resid.zero_()
    blockops.residual_into(blk, deriv, 1, planes, 2, nj)
    assert np.array_equal(blk.resid.cpu().numpy(), g[f"{tag}/resid_sub"])
    # update with snapshot over the full interior
    blk.resid.copy_(torch.from_numpy(g[f"{tag}/resid_full"]))
    blk.q0.copy_(torch.from_numpy(g[f"{tag}/upd_q0"]))
    blockops.update_stage(blk, 0.0123, 0, planes, 1, nj + 1, snapshot=True)
    assert np.array_equal(blk.q.cpu().numpy(), g[f"{tag}/upd_snap_q"])
    assert np.array_equal(blk.q0.cpu().numpy(), g[f"{tag}/upd_snap_q0"])
    # sub-range update without snapshot
    blk.q.copy_(torch.from_numpy(g[f"{tag}/upd_q_before"]))
    blk.q0.copy_(torch.from_numpy(g[f"{tag}/upd_q0"]))
    blockops.update_stage(blk, 0.5, 0, planes, 2, nj)
    assert np.array_equal(blk.q.cpu().numpy(), g[f"{tag}/upd_sub_q"])


def test_residual_hand_stencil(cuda):
    from paper_1304_7654_b200 import blockops
    h = 0.2
    blk = blockops.BlockState(BlockSpec(0, 5, 5, 10.0, 20.0, h), 1)
    blk.forcing.zero_()
    blk.q[0, 0, 3, 3] = 1.0
    r = blockops.residual(blk, spectral_matrix(0, 1.0))[0, 0]
    nu_h2, adv = NU / (h * h), ADVECTION / (2 * h)
    assert r[2, 2] == 4.0 * nu_h2
    assert r[2, 1] == -nu_h2 + adv
    assert r[2, 3] == -nu_h2 - adv
    assert r[1, 2] == -nu_h2 and r[3, 2] == -nu_h2 and r[0, 0] == 0.0


def test_residual_uniform_field(cuda):
    from paper_1304_7654_b200 import blockops
    blk = blockops.BlockState(BlockSpec(0, 5, 5, 10.0, 20.0, 0.2), 3)
    blk.forcing.zero_()
    blk.q.fill_(7.25)
    assert np.abs(blockops.residual(blk, spectral_matrix(1, 1.0))).max() <= 1e-13


def test_update_detects_divergence_with_location(cuda):
    from paper_1304_7654_b200 import blockops
    blk = blockops.BlockState(BlockSpec(0, 5, 5, 10.0, 20.0, 0.2), 1)
    blk.q.fill_(1.0)
    blk.resid.zero_()
    blk.resid[0, 2, 1, 3] = float("inf")
    with pytest.raises(DivergenceError) as err:
        blockops.update_stage(blk, 1.0, 0, 1, 1, 6, snapshot=True)
    e = err.value
    assert (e.block, e.n, e.i, e.j, e.p) == (0, 0, 4, 2, 2)


def _seeded(field, seed=1000):
    torch = _torch()
    for b, bs in field.blocks.items():
        rng = np.random.default_rng(seed + b)
        bs.q.copy_(torch.from_numpy(rng.normal(size=tuple(bs.q.shape))))


def _self_cut_reversed():
    blk = BlockSpec(0, 12, 9, 0.5, 0.25, 0.05, body_faces=(("east", 0), ("south", 1)))
    return CaseConfig(nharms=2, npde=4, iterations=1, dtau=0.0005, omega=1.0, nbody=2, blocks=[blk],
                      cuts=[CutSpec(CutSide(0, "north", 2, 7), CutSide(0, "south", 3, 8), reversed=True)])


@pytest.mark.parametrize("builder", [
    lambda: lattice_case(3, 3, 7, 5, 1, h=0.1, dtau=0.01, nbody=1, bodies=((4, "west", 0),)),
    lambda: pair_case(6, 5, 2, h=0.2, dtau=0.01, reversed_cut=True, nbody=1, bodies=((1, "north", 0),)),
    _self_cut_reversed,
])
def test_exchange_halos_and_forces_vs_oracle(builder, cuda, oracle_mod):
    from paper_1304_7654_b200 import blockops
    case = builder()
    topo = build_topology(case)
    plan = build_cut_plan(topo, partition_blocks(topo, 1), case.nharms, case.npde)
    field = blockops.HarmonicField.allocate(topo.blocks, case.planes)
    _seeded(field)
    qs = {b: bs.q.cpu().numpy().copy() for b, bs in field.blocks.items()}
    blockops.exchange_halos(field, plan)
    oracle_mod.exchange(qs, topo.cuts)
    for b, bs in field.blocks.items():
        assert np.array_equal(bs.q.cpu().numpy(), qs[b]), f"block {b}"
    got = blockops.compute_forces(field, topo)
    want = oracle_mod.compute_forces(qs, topo.blocks, case.planes, topo.nbody)
    assert np.array_equal(np.stack([got.cl, got.cd, got.cm]), want)


def test_forces_no_bodies(cuda):
    from paper_1304_7654_b200 import blockops
    spec = BlockSpec(0, 4, 4, 0.0, 0.0, 0.25)
    field = blockops.HarmonicField.allocate([spec], 3)
    got = blockops.compute_forces(field, Topology(blocks=(spec,), cuts=(), nbody=0))
    assert got.cl.shape == (3, 0)


@pytest.mark.parametrize("ranks", [2, 3])
def test_exchange_halos_remote_cuts_vs_oracle(ranks, cuda, oracle_mod):
    """Block-level exchange_halos with remote cuts (exchange.py:382-402 with a
    rank context): each rank, a thread holding only its own blocks, packs its
    sends element-major, moves one payload per peer through a HaloContext
    (LoopbackHub here, NCCL on several GPUs) and unpacks; every halo must
    equal the all-local oracle exchange."""
    import threading
    from paper_1304_7654_b200 import blockops
    case = lattice_case(3, 2, 9, 6, 1, h=0.1, dtau=0.01)
    topo = build_topology(case)
    part = partition_blocks(topo, ranks)
    plan = build_cut_plan(topo, part, case.nharms, case.npde)
    assert any(not c.local for c in plan.cuts)
    full = blockops.HarmonicField.allocate(topo.blocks, case.planes)
    _seeded(full)
    qs = {b: bs.q.cpu().numpy().copy() for b, bs in full.blocks.items()}
    oracle_mod.exchange(qs, topo.cuts)
    fields = []
    for r in range(ranks):
        f = blockops.HarmonicField.allocate([topo.blocks[g] for g in part.blocks_of(r)], case.planes)
        for g, bs in f.blocks.items():
            bs.q.copy_(full.blocks[g].q)
        fields.append(f)
    hub = blockops.LoopbackHub(ranks)
    errors = []

    def rank_main(r):
        try:
            blockops.exchange_halos(fields[r], plan, blockops.HaloContext(r, hub=hub))
        except Exception as e:   # noqa: BLE001
            errors.append(e)
            hub.barrier.abort()

    threads = [threading.Thread(target=rank_main, args=(r,)) for r in range(ranks)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    for f in fields:
        for g, bs in f.blocks.items():
            assert np.array_equal(bs.q.cpu().numpy(), qs[g]), f"block {g}"
    with pytest.raises(Exception, match="HaloContext"):
        blockops.exchange_halos(fields[0], plan)
