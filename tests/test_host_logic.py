"""Host-side logic of the drop-in vs the reference (CPU only).

Case grammar, topology validation, LPT partition, cut plan and message
forecasts must equal the reference's (goldens in tests/golden/host.json,
produced by tests/golden/make_golden.py from the reference itself); the
spectral operator follows the reference's own tests (test_hbcore.py:24-87).
"""

import json
import os

import numpy as np
import pytest

from paper_1304_7654_b200 import (BUILDERS, BlockSpec, CapacityError, ConfigError, DomainError,
                                  RKScheme, Topology, TopologyError, baseline_workload, build_cut_plan,
                                  build_topology, case_text, cut2500, load_builtin, pair_case,
                                  parse_case, partition_blocks, predicted_message_count, ring_case,
                                  spectral_matrix, stacked_pair_case, tc1_mini, tc2_mini, tc_tiny)
from paper_1304_7654_b200.cutplan import ExchangeMode, ExchangeStrategy
from paper_1304_7654_b200.topology import CaseConfig, CutRole, CutSide, CutSpec, cut_role

GOLD = os.path.join(os.path.dirname(__file__), "golden")
with open(os.path.join(GOLD, "host.json")) as fh:
    HOST = json.load(fh)


def _reversed_pair():
    return pair_case(6, 5, 2, h=0.2, dtau=0.01, reversed_cut=True, nbody=1,
                     bodies=((1, "north", 0),), name="pair-reversed")


def _self_cut():
    blk = BlockSpec(0, 24, 10, 0.0, 0.0, 0.05, body_faces=(("south", 0),))
    return CaseConfig(nharms=4, npde=4, iterations=5, dtau=0.0005, omega=0.12, nbody=1,
                      blocks=[blk], cuts=[CutSpec(CutSide(0, "east", 1, 10), CutSide(0, "west", 1, 10))],
                      name="self-cut")


def _self_cut_reversed():
    blk = BlockSpec(0, 12, 9, 0.5, 0.25, 0.05)
    return CaseConfig(nharms=2, npde=4, iterations=5, dtau=0.0005, omega=1.0, nbody=0,
                      blocks=[blk], cuts=[CutSpec(CutSide(0, "north", 2, 7), CutSide(0, "south", 3, 8),
                                                  reversed=True)], name="self-cut-reversed")


CASES = {
    "tc-tiny": tc_tiny, "tc1-mini": tc1_mini, "tc2-mini": tc2_mini, "cut2500": cut2500,
    "pair-reversed": _reversed_pair, "self-cut": _self_cut, "self-cut-reversed": _self_cut_reversed,
    "ring5": lambda: ring_case(5, 8, 4, 1, h=0.1, dtau=0.01),
    "stacked": lambda: stacked_pair_case(12, 3, 2, h=0.1, dtau=0.01, nbody=1, bodies=((1, "north", 0),)),
    "C0": lambda: baseline_workload("C0").case, "C1": lambda: baseline_workload("C1").case,
    "C2": lambda: baseline_workload("C2").case, "C3": lambda: baseline_workload("C3").case,
    "C4": lambda: baseline_workload("C4").case,
}


def _plan_rows(plan):
    return [[d.cut_index, d.direction, d.sender_rank, d.recv_rank, d.src_block, d.src_face,
             d.src_lo, d.src_hi, d.src_reversed, d.dst_block, d.dst_face, d.dst_lo, d.dst_hi,
             d.dst_reversed, d.length, d.local] for d in plan.directions()]


@pytest.mark.parametrize("name", sorted(CASES))
def test_case_text_matches_reference_rendering(name):
    case = CASES[name]()
    assert case_text(case) == HOST["cases"][name]["case_text"]
    again = parse_case(case_text(case), name=case.name)
    assert case_text(again) == case_text(case)


@pytest.mark.parametrize("name", sorted(CASES))
def test_partition_plan_and_forecast_match_reference(name):
    case = CASES[name]()
    topo = build_topology(case)
    gold = HOST["cases"][name]
    for ranks_s, want in gold["partitions"].items():
        ranks = int(ranks_s)
        part = partition_blocks(topo, ranks)
        assert list(part.rank_of_block) == want
        plan = build_cut_plan(topo, part, case.nharms, case.npde)
        assert _plan_rows(plan) == gold["plans"][ranks_s]
        agg = predicted_message_count(plan, ExchangeStrategy(ExchangeMode.AGGREGATED_CUT))
        per = predicted_message_count(plan, ExchangeStrategy(ExchangeMode.PER_ELEMENT))
        assert [agg.messages, agg.nbytes, per.messages, per.nbytes] == gold["forecast"][ranks_s]


def test_lpt_partition_unequal_blocks_matches_reference():
    blocks = tuple(BlockSpec(id=k, ni=c // 2, nj=2, x0=0.0, y0=float(k), h=1.0)
                   for k, c in enumerate([8, 4, 4, 12, 6, 6, 2]))
    topo = Topology(blocks=blocks, cuts=(), nbody=0)
    for ranks_s, want in HOST["lpt"].items():
        assert list(partition_blocks(topo, int(ranks_s)).rank_of_block) == want


def test_capacity_error_when_more_ranks_than_blocks():
    topo = build_topology(tc_tiny())
    with pytest.raises(CapacityError):
        partition_blocks(topo, 3)
    with pytest.raises(CapacityError):
        partition_blocks(topo, 0)


@pytest.mark.parametrize("name", sorted(HOST["parse_errors"]))
def test_parse_errors_match_reference(name):
    kind, text, message = HOST["parse_errors"][name]
    try:
        build_topology(parse_case(text, source="t.cfg"))
        got = ("ok", "")
    except (ConfigError, TopologyError, KeyError) as exc:
        got = (type(exc).__name__, str(exc))
    assert got == (kind, message)


def test_builtin_catalog_round_trips():
    assert set(BUILDERS) == {"tc-tiny", "tc1-mini", "tc2-mini", "cut2500", "tc1-full", "tc2-full"}
    topo = build_topology(load_builtin("tc1-full"))
    assert topo.nblocks == 512 and topo.total_cells() == 262144
    assert build_topology(load_builtin("tc2-full")).total_cells() == 4194304


def test_cut_roles():
    case = tc_tiny()
    topo = build_topology(case)
    part = partition_blocks(topo, 2)
    cut = topo.cuts[0]
    assert cut_role(part, cut, 0) is CutRole.RECV_SIDE
    assert cut_role(part, cut, 1) is CutRole.SEND_SIDE
    one = partition_blocks(topo, 1)
    assert cut_role(one, cut, 0) is CutRole.BOTH_LOCAL


# ---------------------------------------------------------------------------
# spectral operator (reference tests/test_hbcore.py:24-87, acceptance criterion 5)
# ---------------------------------------------------------------------------

def _fft_derivative(samples, omega):
    n = samples.size
    k = np.fft.fftfreq(n, d=1.0 / n)
    return np.real(np.fft.ifft(np.fft.fft(samples) * 1j * k * omega))


def test_spectral_antisymmetric_exactly_and_row_sums():
    for nh in range(9):
        d = spectral_matrix(nh, 1.0).matrix
        assert np.array_equal(d, -d.T)
        if nh:
            assert np.abs(d.sum(axis=1)).max() <= 1e-14


def test_spectral_circulant_structure_the_stage_kernel_shares_products_on():
    """The fused stage kernel computes D[m+k][m]*q[m] once and subtracts it for
    row m-k: exact only if the reference's D is bitwise antisymmetric circulant."""
    from paper_1304_7654_b200.hbop import circulant_antisymmetric
    for nh in range(64):
        for omega in (1.0, 0.12, 2.3, 1e-3):
            assert circulant_antisymmetric(spectral_matrix(nh, omega).matrix)
    gold = np.load(os.path.join(os.path.dirname(__file__), "golden", "kernels.npz"))
    for key in ("p3/dmat", "p5/dmat", "p9/dmat"):       # the reference's own matrices
        assert circulant_antisymmetric(gold[key])
    bent = spectral_matrix(4, 1.0).matrix.copy()
    bent[3, 1] = np.nextafter(bent[3, 1], 9.0)
    assert not circulant_antisymmetric(bent)


@pytest.mark.parametrize("nharms", range(1, 9))
def test_spectral_derivative_vs_fft(nharms):
    omega = 2.3
    d = spectral_matrix(nharms, omega)
    t = np.arange(d.planes) * d.period / d.planes
    for k in range(1, nharms + 1):
        assert np.abs(d.matrix @ np.cos(k * omega * t) + k * omega * np.sin(k * omega * t)).max() <= 1e-10
        assert np.abs(d.matrix @ np.sin(k * omega * t) - k * omega * np.cos(k * omega * t)).max() <= 1e-10
        assert np.abs(d.matrix @ np.cos(k * omega * t)
                      - _fft_derivative(np.cos(k * omega * t), omega)).max() <= 1e-10


def test_spectral_and_rk_validation():
    assert spectral_matrix(0, 2.0).matrix.shape == (1, 1)
    with pytest.raises(DomainError):
        spectral_matrix(-1, 1.0)
    with pytest.raises(DomainError):
        spectral_matrix(1, 0.0)
    with pytest.raises(DomainError):
        RKScheme(dtau=-1.0)
    with pytest.raises(DomainError):
        RKScheme(dtau=0.1, alphas=(0.5, 0.5))
    assert RKScheme(0.4).stage_coefficients() == [0.25 * 0.4, (1.0 / 3.0) * 0.4, 0.5 * 0.4, 1.0 * 0.4]


def test_spectral_matrix_bits_match_reference_fixture():
    g = np.load(os.path.join(GOLD, "kernels.npz"))
    for tag, nh in (("p3", 1), ("p5", 2), ("p9", 4)):
        assert np.array_equal(spectral_matrix(nh, 1.3).matrix, g[f"{tag}/dmat"])


def test_forcing_factorisation_is_bit_exact():
    """ap[n][p] * sxy[j, i] reproduces the reference forcing array bitwise."""
    import oracle
    from paper_1304_7654_b200.hbop import forcing_amplitudes, forcing_table
    spec = BlockSpec(0, 37, 19, 10.0, 20.0, 0.05)
    ref = oracle.forcing_values(spec, 9)
    ap, sxy = forcing_amplitudes(9), forcing_table(spec)
    mine = ap[:, :, None, None] * sxy[None, None]
    assert np.array_equal(mine.view(np.uint64), ref.view(np.uint64))   # signed zeros too


def test_baseline_workloads_shapes():
    sizes = {k: baseline_workload(k) for k in ("C0", "C1", "C2", "C3", "C4")}
    assert sizes["C0"].case.planes == 3 and sizes["C0"].case.iterations == 100
    assert build_topology(sizes["C1"].case).total_cells() == 4 * 256 * 128
    assert sizes["C2"].case.planes == 9 and len(sizes["C2"].case.cuts) == 1
    assert sizes["C3"].units_per_iteration == 8 * 1024 * 512 * 7 * 4
    assert sizes["C4"].units_per_iteration == 64 * 1024 * 1024 * 9 * 4
    ic = sizes["C1"].initial(sizes["C1"].case.blocks[2], 5)
    assert ic.shape == (5, 4, 128, 256)
    qinf0 = 1.0
    assert np.all(np.abs(ic[:, 0] / qinf0 - 1.0) <= 0.01 + 1e-15)


def test_tile_rows_follow_the_stage_kernel_grid():
    """The single-stage kernel runs two CTAs per SM up to SMALL_P_MAX planes
    (hb_stage.cu stage_ctas_per_sm), the paired kernel always one: the tile
    rows are chosen for that grid."""
    from paper_1304_7654_b200 import baseline_workload, devlayout

    c1 = baseline_workload("C1").case
    tpd = devlayout.choose_tile_pdes(c1.blocks)
    assert devlayout.stage_grid_ctas(c1.blocks, c1.planes, tpd, None) == 2 * devlayout.GRID_CTAS
    assert devlayout.stage_grid_ctas(c1.blocks, c1.planes, tpd, True) == devlayout.GRID_CTAS   # paired
    rows = devlayout.choose_tile_rows(c1.blocks, tpd, 2 * devlayout.GRID_CTAS)
    tiles = sum(-(-b.nj // rows) * devlayout.tiles_per_row(c1.blocks, tpd)[b.id] for b in c1.blocks)
    assert tiles <= 2 * devlayout.GRID_CTAS < 2 * tiles          # one wave, more than half the CTAs busy
    c2 = baseline_workload("C2").case                             # P = 9: one CTA per SM
    assert devlayout.stage_grid_ctas(c2.blocks, c2.planes, devlayout.choose_tile_pdes(c2.blocks), None) \
        == devlayout.GRID_CTAS
    c3 = baseline_workload("C3").case                             # paired by size
    assert devlayout.stage_grid_ctas(c3.blocks, c3.planes, devlayout.choose_tile_pdes(c3.blocks), None) \
        == devlayout.GRID_CTAS
