"""Run-level parity: run_case on the GPU vs the CPU oracle, bitwise.

Fields (halos included), forces and the residual-norm history of the CUDA
path are compared with oracle/oracle.py, a restatement of the reference
pinned to the reference's own outputs (tests/test_oracle_golden.py).
Bar: bitwise for fields and forces; residual norms within 1e-12 relative
(tree vs exactly-rounded summation order; north_star allows 1e-10).
"""

import numpy as np
import pytest

from paper_1304_7654_b200 import (BlockSpec, CaseConfig, CutSide, CutSpec, DivergenceError, RankFailure,
                                  RunSpec, baseline_workload, lattice_case, pair_case,
                                  ring_case, run_case, stacked_pair_case, tc1_mini, tc2_mini,
                                  tc_tiny)

pytestmark = pytest.mark.gpu

NORM_RTOL = 1e-12


def assert_parity(got, want, label):
    for b in want.fields:
        g, w = got.fields[b], want.fields[b]
        if not np.array_equal(g, w):
            bad = np.argwhere(g != w)
            raise AssertionError(f"{label}: block {b} differs at {len(bad)} places, first {bad[0]}"
                                 f" got {g[tuple(bad[0])]!r} want {w[tuple(bad[0])]!r}")
    forces = np.stack([got.forces.cl, got.forces.cd, got.forces.cm])
    assert np.array_equal(forces, want.forces), f"{label}: forces differ"
    if want.norms:
        np.testing.assert_allclose(got.residual_norms, want.norms, rtol=NORM_RTOL, atol=0,
                                   err_msg=f"{label}: residual norms")


CASES = {
    "tc-tiny-8": (tc_tiny, 8, None),
    "pair-reversed": (lambda: pair_case(6, 5, 2, h=0.2, dtau=0.01, reversed_cut=True, nbody=1,
                                        bodies=((1, "north", 0),)), 6, None),
    "steady-nharms0": (lambda: CaseConfig(nharms=0, npde=4, iterations=12, dtau=0.01, omega=1.0,
                                          nbody=0, blocks=[BlockSpec(0, 6, 5, 0.3, -0.7, 0.2)],
                                          cuts=[]), 12, None),
    "stacked-ns": (lambda: stacked_pair_case(40, 7, 1, h=0.01, dtau=0.0001, nbody=1,
                                             bodies=((0, "south", 0),)), 4, None),
    "tc2-mini-3": (tc2_mini, 3, None),
    "tc1-mini-4": (tc1_mini, 4, None),
    "lattice-p7-ragged": (lambda: lattice_case(3, 2, 45, 19, 3, h=0.02, dtau=0.0005, nbody=2,
                                               bodies=((0, "south", 0), (4, "north", 1))), 5, None),
    "generic-p21": (lambda: ring_case(3, 33, 9, 10, h=0.05, dtau=0.0005, nbody=1,
                                      bodies=((2, "south", 0),)), 3, None),
}


@pytest.mark.parametrize("small", [None, False])
@pytest.mark.parametrize("name", sorted(CASES))
def test_run_case_matches_oracle(name, small, cuda, oracle_mod):
    """small=None: the auto schedule, the one-launch small kernel for these
    sizes (hb_small.cu); small=False: the per-stage TMA kernels."""
    build, iters, initial = CASES[name]
    case = build()
    got = run_case(RunSpec(case=case, ranks=1, iterations=iters, initial=initial, small=small))
    want = oracle_mod.run(case, iters, initial=initial)
    assert_parity(got, want, name)


@pytest.mark.parametrize("small", [None, False])
@pytest.mark.parametrize("key,iters", [("C0", 20), ("C1", 2), ("C2", 2)])
def test_baseline_workloads_match_oracle(key, iters, small, cuda, oracle_mod):
    wl = baseline_workload(key)
    got = run_case(RunSpec(case=wl.case, ranks=1, iterations=iters, initial=wl.initial, small=small))
    want = oracle_mod.run(wl.case, iters, initial=wl.initial)
    assert_parity(got, want, key)


@pytest.mark.parametrize("ni", [5, 41, 42, 43, 44, 45, 46, 47, 48, 193, 199, 255, 256, 257, 263])
def test_ragged_widths_match_oracle(ni, cuda, oracle_mod):
    """Every residue of ni mod 8 at both strip geometries (64 x 4 pdes below
    192 columns, 256 x 1 above): the TMA store extent ends on the 64-B boundary
    at or before cell ni, and the forwarded east halo cell ni+1 -- in the same
    granule as cell ni when ni % 8 != 0 -- must survive every stage."""
    case = ring_case(2, ni, 5, 1, h=0.05, dtau=0.0005, nbody=1, bodies=((1, "south", 0),))
    got = run_case(RunSpec(case=case, ranks=1, iterations=3, small=False))
    want = oracle_mod.run(case, 3)
    assert_parity(got, want, f"ring2-ni{ni}")


def test_graph_and_eager_identical(cuda):
    case = tc2_mini()
    a = run_case(RunSpec(case=case, ranks=1, iterations=3, use_graph=True))
    b = run_case(RunSpec(case=case, ranks=1, iterations=3, use_graph=False))
    assert a.field_bits_equal(b) and a.forces.equal_bits(b.forces)


@pytest.mark.parametrize("tile_rows", [8, 13, 64])
def test_tile_rows_invariance(tile_rows, cuda):
    case = lattice_case(2, 2, 70, 41, 2, h=0.02, dtau=0.0005)
    base = run_case(RunSpec(case=case, ranks=1, iterations=3, tile_rows=9))
    other = run_case(RunSpec(case=case, ranks=1, iterations=3, tile_rows=tile_rows))
    assert base.field_bits_equal(other)
    np.testing.assert_allclose(base.residual_norms, other.residual_norms, rtol=1e-13)


def test_rank_count_invariance_single_process(cuda):
    case = tc2_mini()
    one = run_case(RunSpec(case=case, ranks=1, iterations=3))
    eight = run_case(RunSpec(case=case, ranks=8, iterations=3))
    assert one.field_bits_equal(eight) and one.forces.equal_bits(eight.forces)


LOOPBACK = {
    "tc-tiny/2": (tc_tiny, 2, 4),
    "pair-reversed/2": (lambda: pair_case(6, 5, 2, h=0.2, dtau=0.01, reversed_cut=True, nbody=1,
                                          bodies=((1, "north", 0),)), 2, 3),
    "tc2-mini/8": (tc2_mini, 8, 2),
    "lattice-p7-ragged/3": (lambda: lattice_case(3, 2, 45, 19, 3, h=0.02, dtau=0.0005, nbody=2,
                                                 bodies=((0, "south", 0), (4, "north", 1))), 3, 3),
    "tc1-mini/4": (tc1_mini, 4, 2),
    "C1/4": (lambda: baseline_workload("C1").case, 4, 2),
}


@pytest.mark.parametrize("transport", ["loopback", "loopback-split"])
@pytest.mark.parametrize("name", sorted(LOOPBACK))
def test_loopback_multirank_matches_oracle(name, transport, cuda, oracle_mod):
    """Several ranks' engines on one GPU: remote cuts go through the fused
    pack, per-peer segments and unpack of the multi-GPU path, with device
    copies standing in for NCCL; the force history is folded in rank order.
    "loopback-split" runs every pass as the NCCL engine's overlapped
    schedule: boundary tiles + remote packs, then the transfer on a side
    stream concurrently with the interior tiles, then the unpack."""
    build, ranks, iters = LOOPBACK[name]
    case = build()
    initial = baseline_workload("C1").initial if name.startswith("C1") else None
    got = run_case(RunSpec(case=case, ranks=ranks, iterations=iters, transport=transport,
                           initial=initial))
    want = oracle_mod.run(case, iters, initial=initial)
    assert_parity(got, want, name)


def test_divergence_reports_reference_location(cuda, oracle_mod):
    case = pair_case(8, 6, 1, h=0.25, dtau=50.0, nbody=0)
    with pytest.raises(oracle_mod.OracleDivergence) as want:
        oracle_mod.run(case, 100)
    with pytest.raises(RankFailure) as got:
        run_case(RunSpec(case=case, ranks=1, iterations=100))
    w, g = want.value, got.value.cause
    assert (g.block, g.i, g.j, g.p, g.n) == (w.block, w.i, w.j, w.p, w.n)


def test_dtau_zero_is_identity(cuda):
    from paper_1304_7654_b200 import initial_values
    case = pair_case(4, 4, 1, h=0.25, dtau=0.0)
    res = run_case(RunSpec(case=case, ranks=1, iterations=3))
    want = initial_values(case.blocks[0], 3, 4, 0, 3, 1, 5)
    assert np.array_equal(res.fields[0][:, :, 1:5, 1:5], want)


# ---------------------------------------------------------------------------
# paired stages (hb_pair.cu): every tile-perimeter path -- strip edges, row
# tile edges, block faces across local / reversed / self / remote cuts
# ---------------------------------------------------------------------------

FUSED = {
    # name: (builder, iterations, tile_rows, ranks, transport)
    "lattice-256": (lambda: lattice_case(3, 2, 256, 40, 2, h=0.01, dtau=0.0002, nbody=2,
                                         bodies=((0, "south", 0), (4, "north", 1))), 3, 16, 1, "fold"),
    "lattice-256-rows1": (lambda: lattice_case(2, 2, 256, 7, 1, h=0.02, dtau=0.0005), 2, 1, 1, "fold"),
    "lattice-256-ragged-rows": (lambda: lattice_case(2, 1, 512, 37, 4, h=0.01, dtau=0.0002, nbody=1,
                                                     bodies=((1, "north", 0),)), 3, 10, 1, "fold"),
    "pair-64-pt4": (lambda: pair_case(64, 30, 3, h=0.02, dtau=0.0005, reversed_cut=True, nbody=1,
                                      bodies=((1, "north", 0),)), 3, 8, 1, "fold"),
    "ring-128-pt4": (lambda: ring_case(3, 128, 20, 2, h=0.02, dtau=0.0005, nbody=1,
                                       bodies=((2, "south", 0),)), 3, 7, 1, "fold"),
    "self-cut-512": (lambda: CaseConfig(nharms=4, npde=4, iterations=3, dtau=0.0001, omega=0.12, nbody=1,
                                        blocks=[BlockSpec(0, 512, 24, 0.0, 0.0, 0.01,
                                                          body_faces=(("south", 0),))],
                                        cuts=[CutSpec(CutSide(0, "east", 1, 24), CutSide(0, "west", 1, 24))]),
                     3, 9, 1, "fold"),
    "lattice-256-loopback4": (lambda: lattice_case(2, 2, 256, 24, 2, h=0.01, dtau=0.0002, nbody=1,
                                                   bodies=((3, "north", 0),)), 3, 8, 4, "loopback"),
    "lattice-256-split4": (lambda: lattice_case(2, 2, 256, 24, 2, h=0.01, dtau=0.0002, nbody=1,
                                                bodies=((3, "north", 0),)), 3, 8, 4, "loopback-split"),
    "lattice-3x2-split2": (lambda: lattice_case(3, 2, 256, 40, 4, h=0.01, dtau=0.0002, nbody=1,
                                                bodies=((4, "north", 0),)), 2, 8, 2, "loopback-split"),
    "C1-loopback2": (lambda: baseline_workload("C1").case, 2, None, 2, "loopback"),
    "nj1-p1": (lambda: CaseConfig(nharms=0, npde=4, iterations=4, dtau=0.001, omega=1.0, nbody=1,
                                  blocks=[BlockSpec(0, 512, 1, 0.0, 0.0, 0.01, body_faces=(("north", 0),))],
                                  cuts=[CutSpec(CutSide(0, "east", 1, 1), CutSide(0, "west", 1, 1))]),
               4, None, 1, "fold"),
    "nj2-stacked": (lambda: stacked_pair_case(256, 2, 1, h=0.01, dtau=0.0002, nbody=1,
                                              bodies=((1, "north", 0),)), 3, 1, 1, "fold"),
}


@pytest.mark.parametrize("name", sorted(FUSED))
def test_paired_stages_match_oracle_and_single_stages(name, cuda, oracle_mod):
    from paper_1304_7654_b200 import build_topology, partition_blocks, build_cut_plan
    from paper_1304_7654_b200.devlayout import build_rank_layout
    build, iters, tile_rows, ranks, transport = FUSED[name]
    case = build()
    topo = build_topology(case)
    part = partition_blocks(topo, 1)
    lay = build_rank_layout(topo, part, build_cut_plan(topo, part, case.nharms, 4), 0, case.planes, tile_rows,
                            fused=True)
    assert lay.fused, "case must take the paired-stage path"
    initial = baseline_workload("C1").initial if name.startswith("C1") else None
    got = run_case(RunSpec(case=case, ranks=ranks, iterations=iters, tile_rows=tile_rows, initial=initial,
                           transport=transport, fused=True))
    single = run_case(RunSpec(case=case, ranks=ranks, iterations=iters, tile_rows=tile_rows, initial=initial,
                              transport=transport, fused=False, small=False))
    want = oracle_mod.run(case, iters, initial=initial)
    assert_parity(got, want, name)
    assert got.field_bits_equal(single) and got.forces.equal_bits(single.forces)
    np.testing.assert_allclose(got.residual_norms, single.residual_norms, rtol=1e-13)


def test_paired_stages_divergence_location(cuda, oracle_mod):
    """A blow-up inside a pair reports the reference's (stage, cell)."""
    case = lattice_case(2, 1, 256, 12, 1, h=0.01, dtau=5.0)
    with pytest.raises(oracle_mod.OracleDivergence) as want:
        oracle_mod.run(case, 100)
    with pytest.raises(RankFailure) as got:
        run_case(RunSpec(case=case, ranks=1, iterations=100, fused=True))
    w, g = want.value, got.value.cause
    assert (g.block, g.i, g.j, g.p, g.n) == (w.block, w.i, w.j, w.p, w.n)


def test_paired_graph_and_eager_identical(cuda):
    case = lattice_case(2, 2, 256, 20, 2, h=0.01, dtau=0.0002, nbody=1, bodies=((1, "north", 0),))
    a = run_case(RunSpec(case=case, ranks=1, iterations=3, tile_rows=8, use_graph=True, fused=True))
    b = run_case(RunSpec(case=case, ranks=1, iterations=3, tile_rows=8, use_graph=False, fused=True))
    assert a.field_bits_equal(b) and a.forces.equal_bits(b.forces)
    np.testing.assert_allclose(a.residual_norms, b.residual_norms, rtol=1e-13)


MANY_TILES = {
    # 4 blocks x 2 strips x 4 pdes x 5 row tiles = 160 tiles
    "lattice-512": (lambda: lattice_case(2, 2, 512, 40, 2, h=0.01, dtau=0.0002, nbody=1,
                                         bodies=((3, "north", 0),)), 3, 8),
    # 64-column strips x 4 pdes (PT = 4), reversed cut
    "pair-64-pt4": (lambda: pair_case(64, 30, 3, h=0.02, dtau=0.0005, reversed_cut=True, nbody=1,
                                      bodies=((1, "north", 0),)), 3, 4),
    # self-cut: a block's own strips feed each other's halos
    "self-cut-768": (lambda: CaseConfig(nharms=4, npde=4, iterations=3, dtau=0.0001, omega=0.12, nbody=1,
                                        blocks=[BlockSpec(0, 768, 23, 0.0, 0.0, 0.01,
                                                          body_faces=(("south", 0),))],
                                        cuts=[CutSpec(CutSide(0, "east", 1, 23), CutSide(0, "west", 1, 23))]),
                     3, 5),
}


@pytest.mark.parametrize("limit", [1, 3])
@pytest.mark.parametrize("fused", [True, False])
@pytest.mark.parametrize("name", sorted(MANY_TILES))
def test_many_tiles_per_cta_match_oracle(name, fused, limit, cuda, oracle_mod, monkeypatch):
    """With HBGPU_GRID_LIMIT CTAs every CTA walks many tiles, as at full size
    (C4: 1024 tiles on 148 CTAs), and the strips of one row tile are not
    processed together (limit 1: strictly one after another).  This covers
    the rings' hand-over from tile to tile and the in-place pass B, where a
    strip must not read q0 at its neighbour's edge column from HBM."""
    monkeypatch.setenv("HBGPU_GRID_LIMIT", str(limit))
    build, iters, tile_rows = MANY_TILES[name]
    case = build()
    got = run_case(RunSpec(case=case, ranks=1, iterations=iters, tile_rows=tile_rows, fused=fused, small=False))
    want = oracle_mod.run(case, iters)
    assert_parity(got, want, f"{name} fused={fused} limit={limit}")


# ---------------------------------------------------------------------------
# run control: early divergence stop, iteration capacity, hazard -> strict rerun
# ---------------------------------------------------------------------------

def test_divergence_stops_the_loop_early(cuda, oracle_mod):
    """A 500-iteration run that diverges in its first iterations stops
    within one polling chunk (the reference raises at the failing stage,
    hbcore.py:273-276) and reports the reference's location."""
    from paper_1304_7654_b200 import solver
    case = lattice_case(2, 1, 256, 12, 1, h=0.01, dtau=5.0)
    with pytest.raises(oracle_mod.OracleDivergence) as want:
        oracle_mod.run(case, 500)
    with pytest.raises(RankFailure) as got:
        run_case(RunSpec(case=case, ranks=1, iterations=500))
    w, g = want.value, got.value.cause
    assert (g.block, g.i, g.j, g.p, g.n) == (w.block, w.i, w.j, w.p, w.n)
    chunk = solver.POLL_MAX
    assert solver.LAST_RUN["iterations_issued"] <= w.iteration + 1 + 2 * chunk < 500


def test_engine_refuses_iterations_past_max_iters(cuda):
    """sumsq and force_hist hold max_iters rows: the engine refuses to issue
    more iterations (include/hbgpu.h hbgpu_engine_iterate) until rewound."""
    from paper_1304_7654_b200.solver import DeviceRank
    from paper_1304_7654_b200 import build_topology, partition_blocks, build_cut_plan
    case = tc_tiny()
    topo = build_topology(case)
    part = partition_blocks(topo, 1)
    dr = DeviceRank(case, topo, part, build_cut_plan(topo, part, case.nharms, 4), max_iters=2)
    try:
        dr.prime()
        dr.iterate(2)
        assert dr.iterations_done() == 2
        with pytest.raises(RuntimeError, match="max_iters"):
            dr.iterate(1)
        with pytest.raises(RuntimeError, match="max_iters"):
            dr.iterate(1, use_graph=False)
        dr.reset_counters()
        assert dr.iterations_done() == 0
        dr.iterate(2, use_graph=False)
        import torch
        torch.cuda.synchronize()
        assert int(dr.iter.item()) == 2
    finally:
        dr.close()


@pytest.mark.parametrize("scale", [1.5, 1.0])
def test_huge_initial_value_reruns_strict_and_matches_oracle(scale, cuda, oracle_mod):
    """The paired kernel's DFMA 4c - w is the reference's rounding only for
    |c| < 2^1022.  A state holding a larger finite value sets a hazard key
    (engine prime scan / stage outputs) and run_case repeats the run on the
    strict single-stage kernels, so the outcome is the reference's: here
    the divergence the overflowing 4c causes, at the reference's cell."""
    from paper_1304_7654_b200 import solver
    case = lattice_case(2, 1, 256, 12, 1, h=0.01, dtau=0.0002)
    big = scale * 2.0 ** 1022

    def initial(spec, planes, npde):
        ic = oracle_mod.initial_values(spec, planes, npde)
        if spec.id == 1:
            ic[1, 2, 5, 17] = big
            ic[1, 2, 5, 16] = 2.9 * big   # 4c - w stays finite in one rounding
        return ic

    before = solver.STRICT_RERUNS[0]
    try:
        want = oracle_mod.run(case, 3, initial=initial)
        want_err = None
    except oracle_mod.OracleDivergence as e:
        want_err = e
    if want_err is None:
        got = run_case(RunSpec(case=case, ranks=1, iterations=3, initial=initial, fused=True))
        assert_parity(got, want, "huge")
    else:
        with pytest.raises(RankFailure) as got:
            run_case(RunSpec(case=case, ranks=1, iterations=3, initial=initial, fused=True))
        g = got.value.cause
        assert (g.block, g.i, g.j, g.p, g.n) == (want_err.block, want_err.i, want_err.j, want_err.p,
                                                 want_err.n)
    assert solver.STRICT_RERUNS[0] == before + 1


def test_stage_output_hazard_is_recorded(cuda, oracle_mod):
    """In-kernel hazard keys.  One cell of q = 2^1021 (below the prime
    scan's 2^1022) with coef = dtau/4 = 1 and nu_h2 = 1.25: stage 1 is
    exact and finite everywhere, but writes -2^1023 at that cell (and
    1.875 * 2^1022 east of it).  Stage 2's 4c then overflows -- in the
    reference a DivergenceError at stage 2, which the paired kernel's DFMA
    4c - w would only match by luck.  The paired kernel must flag the stage-1
    outputs of magnitude >= 2^1022 (hazard key, global stage 1) so that
    run_case repeats the run on the strict kernels, whose outcome is the
    reference's."""
    import torch
    from paper_1304_7654_b200 import solver
    from paper_1304_7654_b200.solver import DeviceRank
    from paper_1304_7654_b200 import build_topology, partition_blocks, build_cut_plan
    case = lattice_case(2, 1, 256, 12, 1, h=0.2, dtau=4.0)

    def initial(spec, planes, npde):
        ic = oracle_mod.initial_values(spec, planes, npde)
        if spec.id == 1:
            ic[0, 0, 5, 100] = 2.0 ** 1021
        return ic

    with pytest.raises(oracle_mod.OracleDivergence) as want:
        oracle_mod.run(case, 1, initial=initial)
    w = want.value
    assert (w.iteration, w.stage) == (0, 1)
    topo = build_topology(case)
    part = partition_blocks(topo, 1)
    dr = DeviceRank(case, topo, part, build_cut_plan(topo, part, case.nharms, 4), initial=initial,
                    tile_rows=12, max_iters=1, fused=True)
    try:
        assert dr.fused
        dr.prime()
        dr.iterate(1, use_graph=False)
        torch.cuda.synchronize()
        assert dr.divergence() == (1, True, 1, 101, 6, 0, 0)
    finally:
        dr.close()
    before = solver.STRICT_RERUNS[0]
    with pytest.raises(RankFailure) as got:
        run_case(RunSpec(case=case, ranks=1, iterations=1, initial=initial, fused=True))
    g = got.value.cause
    assert (g.block, g.i, g.j, g.p, g.n) == (w.block, w.i, w.j, w.p, w.n)
    assert solver.STRICT_RERUNS[0] == before + 1


def test_run_diverges_with_rank_in_error(cuda):
    """The reference's run_case wraps a rank's DivergenceError in a
    RankFailure naming the rank (runtime.py:359-364; its
    tests/test_driver_cli.py:30-36 asserts exactly this)."""
    case = pair_case(4, 4, 1, h=0.25, dtau=50.0)
    for ranks in (1, 2):
        with pytest.raises(RankFailure) as err:
            run_case(RunSpec(case=case, ranks=ranks, iterations=50))
        assert isinstance(err.value.cause, DivergenceError)
        assert err.value.rank in range(ranks)


@pytest.mark.parametrize("name", ["tc1-mini-4", "lattice-p7-ragged", "stacked-ns"])
def test_small_schedule_equals_stage_kernels(name, cuda):
    """The one-launch small schedule and the per-stage TMA kernels agree
    bitwise (fields, forces) and on the norms (rtol 1e-13), over several
    iterations and through the status poller's chunks."""
    build, iters, initial = CASES[name]
    case = build()
    a = run_case(RunSpec(case=case, ranks=1, iterations=iters + 3, small=True))
    b = run_case(RunSpec(case=case, ranks=1, iterations=iters + 3, small=False))
    assert a.field_bits_equal(b) and a.forces.equal_bits(b.forces)
    np.testing.assert_allclose(a.residual_norms, b.residual_norms, rtol=1e-13)
    from paper_1304_7654_b200 import solver
    assert solver.LAST_RUN["small"] is False


def test_small_schedule_divergence_location(cuda, oracle_mod):
    case = pair_case(8, 6, 1, h=0.25, dtau=50.0, nbody=0)
    with pytest.raises(oracle_mod.OracleDivergence) as want:
        oracle_mod.run(case, 100)
    with pytest.raises(RankFailure) as got:
        run_case(RunSpec(case=case, ranks=1, iterations=100, small=True))
    w, g = want.value, got.value.cause
    assert (g.block, g.i, g.j, g.p, g.n) == (w.block, w.i, w.j, w.p, w.n)
