"""Per-rank counters against the reference's acceptance
criteria 1, 2, 7, 8 and its exchange-counter test (tests/test_acceptance.py:
70-245, tests/test_exchange.py:195-206), on CPU: the counters are a pure
function of the plan and the strategies."""

import pytest

from paper_1304_7654_b200 import (ExchangeMode, ExchangeStrategy, RunSpec, build_cut_plan,
                                  build_topology, cut2500, partition_blocks, predicted_message_count,
                                  tc1_mini, tc_tiny)
from paper_1304_7654_b200.outio import WriteMode, all_layouts
from paper_1304_7654_b200.solver import ForceReduceStrategy, ReduceMode, rank_counters


def _counters(case, ranks, iterations, targets=(), **kw):
    spec = RunSpec(case=case, ranks=ranks, iterations=iterations, **kw)
    topo = build_topology(case)
    part = partition_blocks(topo, ranks)
    plan = build_cut_plan(topo, part, case.nharms, case.npde)
    layouts = all_layouts(topo, case.nharms) if targets else ()
    act = iterations * (12 if kw.get("activation") == "per-loop" else 1) + len(targets)
    return rank_counters(plan, spec, part, iterations, act, layouts, list(targets)), plan


@pytest.mark.parametrize("mode", list(ExchangeMode))
def test_messages_equal_forecast_per_direction(mode):
    strategy = ExchangeStrategy(mode)
    cs, plan = _counters(tc_tiny(), 2, 0, exchange=strategy)     # one (priming) exchange
    fc = predicted_message_count(plan, strategy)
    assert sum(c.msgs_sent for c in cs) == fc.total_messages
    assert sum(c.bytes_sent for c in cs) == fc.total_bytes
    for c in cs:       # one cut, one sender per direction
        assert (c.msgs_sent, c.bytes_sent, c.msgs_received) == (fc.messages, fc.nbytes, fc.messages)


def test_criterion_1_collectives_30_vs_1():
    case = tc1_mini()
    for mode, want in ((ReduceMode.PER_BODY_PER_HARMONIC, 30), (ReduceMode.SINGLE_BUFFER, 1)):
        cs, _ = _counters(case, 2, 2, reduce=ForceReduceStrategy(mode))
        assert all(c.collective_calls == want * 2 for c in cs)


def test_criterion_2_per_element_5000_vs_1():
    case = cut2500()
    for mode, want in ((ExchangeMode.PER_ELEMENT, 5000), (ExchangeMode.AGGREGATED_CUT, 1)):
        cs, _ = _counters(case, 2, 0, exchange=ExchangeStrategy(mode))
        assert all(c.msgs_sent == want for c in cs)
    a, _ = _counters(case, 2, 0, exchange=ExchangeStrategy(ExchangeMode.PER_ELEMENT))
    b, _ = _counters(case, 2, 0)
    assert sum(c.bytes_sent for c in a) == sum(c.bytes_sent for c in b)


def test_criterion_7_activations_120_vs_10():
    for mode, want in (("per-loop", 120), ("hoisted", 10)):
        cs, _ = _counters(tc_tiny(), 2, 10, activation=mode, threads=4)
        assert all(c.team_activations == want for c in cs)


def test_criterion_8_write_ops():
    case = tc_tiny()
    topo = build_topology(case)
    records = 2 * topo.nblocks * case.planes
    for mode, want in ((WriteMode.PER_VALUE, records * (2 + 4 * 4 * 4)), (WriteMode.BUFFERED, records * 3)):
        cs, _ = _counters(case, 2, 1, targets=[("/unused", mode)])
        assert sum(c.write_ops for c in cs) == want


def test_counters_of_the_tiny_record():
    """test_driver_cli.py:60-73: 17 exchanges for 4 iterations, 1 cut."""
    cs, _ = _counters(tc_tiny(), 2, 4)
    assert sum(c.msgs_sent for c in cs) == 2 * 17
    assert sum(c.bytes_sent for c in cs) == 2 * 17 * 4 * 12 * 8
    assert all(c.collective_calls == 4 and c.team_activations == 4 for c in cs)


def test_device_counters_report_what_the_device_moves():
    """The reference counters follow the strategy (per-element: 2L messages
    per direction); the device_* fields record what the device path moves:
    one aggregated payload per peer and exchange, the same bytes."""
    case = cut2500()
    for mode in ExchangeMode:
        cs, plan = _counters(case, 2, 3, exchange=ExchangeStrategy(mode), transport="loopback")
        exchanges = 4 * 3 + 1
        for c in cs:
            assert c.device_msgs == exchanges          # one peer
            assert c.device_bytes == c.bytes_sent       # the same payload bytes
            assert c.device_collectives == 0
    cs, _ = _counters(case, 2, 3, exchange=ExchangeStrategy(ExchangeMode.PER_ELEMENT))   # "fold"
    assert all(c.device_msgs == 0 and c.device_bytes == 0 for c in cs)
    assert all(c.msgs_sent == 5000 * 13 for c in cs)
