"""Pin the CPU oracle (oracle/) to the reference's own outputs.

tests/golden/ holds vectors produced by running the reference `hbproxy`
itself (tests/golden/make_golden.py).  The oracle must reproduce them bit for
bit; only then is it trusted as the checker of the CUDA path.

Run-level goldens depend on the host's numpy sin/cos bits (initial state and
forcing are transcendental).  Each fixture records the hash of the inputs it
was generated from; on a host whose numpy produces different input bits the
comparison is skipped (the GPU-vs-oracle parity tests still run there, both
sides consuming the same host inputs).
"""

import hashlib
import json
import os

import numpy as np
import pytest

import oracle
from paper_1304_7654_b200 import baseline_workload, pair_case, tc1_mini, tc2_mini, tc_tiny
from paper_1304_7654_b200.topology import BlockSpec, CaseConfig, CutSide, CutSpec

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _load_json(name):
    with open(os.path.join(GOLD, name)) as fh:
        return json.load(fh)


FPS = _load_json("fingerprints.json")


def _steady():
    return CaseConfig(nharms=0, npde=4, iterations=12, dtau=0.01, omega=1.0, nbody=0,
                      blocks=[BlockSpec(0, 6, 5, 0.3, -0.7, 0.2)], cuts=[], name="steady")


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


RUNS = {
    "tc-tiny-8": (tc_tiny, None),
    "pair-reversed-6": (_reversed_pair, None),
    "steady-12": (_steady, None),
    "self-cut-5": (_self_cut, None),
    "self-cut-reversed-5": (_self_cut_reversed, None),
    "tc1-mini-20": (tc1_mini, None),
    "tc2-mini-10": (tc2_mini, None),
    "C0-seeded-10": (lambda: baseline_workload("C0").case, "C0"),
}


def input_hash(case, initial=None):
    h = hashlib.sha256()
    planes = 2 * case.nharms + 1
    for spec in sorted(case.blocks, key=lambda s: s.id):
        ic = initial(spec, planes, 4) if initial is not None else oracle.initial_values(spec, planes)
        h.update(np.ascontiguousarray(ic).tobytes())
        h.update(oracle.forcing_values(spec, planes).tobytes())
    h.update(oracle.spectral_matrix(case.nharms, case.omega).tobytes())
    return h.hexdigest()[:16]


def _host_matches(name, case, initial):
    if input_hash(case, initial) != FPS[name]["input_hash"]:
        pytest.skip(f"{name}: this host's numpy sin/cos bits differ from the fixture's")


@pytest.mark.parametrize("name", sorted(RUNS))
def test_oracle_run_matches_reference_fingerprint(name, oracle_mod):
    build, wl = RUNS[name]
    case = build()
    initial = baseline_workload(wl).initial if wl else None
    _host_matches(name, case, initial)
    res = oracle_mod.run(case, FPS[name]["iterations"], initial=initial, record_norms=False)
    assert oracle_mod.fingerprint(res.fields, res.forces) == FPS[name]["fingerprint"]
    peak = max(np.abs(q).max() for q in res.fields.values())
    assert peak == FPS[name]["max_abs_q"]


@pytest.mark.parametrize("name", ["tc-tiny-8", "pair-reversed-6", "steady-12", "self-cut-5",
                                  "self-cut-reversed-5", "C0-seeded-10"])
def test_oracle_full_arrays_match_reference(name, oracle_mod):
    build, wl = RUNS[name]
    case = build()
    initial = baseline_workload(wl).initial if wl else None
    _host_matches(name, case, initial)
    gold = np.load(os.path.join(GOLD, "runs.npz"))
    res = oracle_mod.run(case, FPS[name]["iterations"], initial=initial)
    for b, q in res.fields.items():
        assert np.array_equal(q, gold[f"{name}/field/{b}"]), f"block {b}"
    assert np.array_equal(res.forces, gold[f"{name}/forces"])


def test_tc1_mini_100_iterations_master_oracle(oracle_mod):
    """The reference's acceptance criterion 4 baseline (100 tc1-mini iterations)."""
    name = "tc1-mini-100"
    case = tc1_mini()
    _host_matches(name, case, None)
    res = oracle_mod.run(case, 100, record_norms=False)
    assert oracle_mod.fingerprint(res.fields, res.forces) == FPS[name]["fingerprint"]
    assert round(max(np.abs(q).max() for q in res.fields.values()), 3) == 0.208


@pytest.mark.parametrize("tag", ["p3", "p5", "p9"])
def test_oracle_kernels_bitwise_vs_reference(tag, oracle_mod):
    g = np.load(os.path.join(GOLD, "kernels.npz"))
    ni, nj, nharms, h, _ = g[f"{tag}/meta"]
    ni, nj, nharms = int(ni), int(nj), int(nharms)
    planes = 2 * nharms + 1
    q = g[f"{tag}/q"].copy()
    src, dmat = g[f"{tag}/forcing"], g[f"{tag}/dmat"]
    out = np.zeros((planes, 4, nj, ni))
    oracle_mod.residual_into(q, dmat, src, h, out, 0, planes, 1, nj + 1)
    assert np.array_equal(out, g[f"{tag}/resid_full"])
    out[:] = 0.0
    oracle_mod.residual_into(q, dmat, src, h, out, 1, planes, 2, nj)
    assert np.array_equal(out, g[f"{tag}/resid_sub"])
    # update with snapshot on the full residual
    resid = g[f"{tag}/resid_full"]
    q0 = g[f"{tag}/upd_q0"].copy()
    acc = oracle_mod.update(q, q0, resid, 0.0123, True, 0, planes, 1, nj + 1)
    assert acc == 0.0
    assert np.array_equal(q, g[f"{tag}/upd_snap_q"])
    assert np.array_equal(q0, g[f"{tag}/upd_snap_q0"])
    # sub-range update without snapshot
    q = g[f"{tag}/upd_q_before"].copy()
    q0 = g[f"{tag}/upd_q0"].copy()
    oracle_mod.update(q, q0, resid, 0.5, False, 0, planes, 2, nj)
    assert np.array_equal(q, g[f"{tag}/upd_sub_q"])


def test_oracle_spectral_matrix_bits_vs_reference(oracle_mod):
    g = np.load(os.path.join(GOLD, "kernels.npz"))
    for tag, nh in (("p3", 1), ("p5", 2), ("p9", 4)):
        assert np.array_equal(oracle_mod.spectral_matrix(nh, 1.3), g[f"{tag}/dmat"])


def test_oracle_divergence_location_like_reference(oracle_mod):
    """hbcore._raise_divergence: lexicographically first non-finite (n, p, j, i)."""
    q = np.zeros((3, 4, 7, 7))
    q[1, 2, 3, 4] = np.nan
    q[1, 3, 1, 1] = np.inf
    q[2, 0, 1, 1] = np.nan
    assert oracle_mod.divergence_location(q) == (4, 3, 2, 1)


def test_oracle_ordered_sum_is_rank_ordered(oracle_mod):
    bufs = [np.array([1e16, 1.0]), np.array([1.0, 1e16]), np.array([-1e16, -1e16])]
    acc = oracle_mod.ordered_sum(bufs)
    want = (bufs[0] + bufs[1]) + bufs[2]
    assert np.array_equal(acc, want)


@pytest.mark.parametrize("name", sorted(RUNS))
def test_lean_oracle_matches_reference_fingerprint(name, oracle_mod):
    """The memory-lean driver (q and q0 only, forcing on the fly, 2-row
    residual scratch; used for C3/C4 at full size) reproduces the reference's
    own fingerprints bit for bit."""
    build, wl = RUNS[name]
    case = build()
    initial = baseline_workload(wl).initial if wl else None
    _host_matches(name, case, initial)
    res = oracle_mod.run(case, FPS[name]["iterations"], initial=initial, record_norms=False, lean=True)
    assert oracle_mod.fingerprint(res.fields, res.forces) == FPS[name]["fingerprint"]


@pytest.mark.parametrize("name,iters", [("tc1-mini-20", 20), ("self-cut-5", 5), ("C0-seeded-10", 10)])
def test_lean_oracle_equals_full_oracle(name, iters, oracle_mod):
    """Same fields bitwise and the same per-iteration norms (rtol 1e-13: the
    lean driver sums R**2 per block with a compensated accumulator, the full
    one with math.fsum) on any host, fixtures or not."""
    build, wl = RUNS[name]
    case = build()
    initial = baseline_workload(wl).initial if wl else None
    full = oracle_mod.run(case, iters, initial=initial)
    lean = oracle_mod.run(case, iters, initial=initial, lean=True)
    for b in full.fields:
        assert np.array_equal(full.fields[b], lean.fields[b]), f"block {b}"
    assert np.array_equal(full.forces, lean.forces)
    np.testing.assert_allclose(lean.norms, full.norms, rtol=1e-13, atol=0)


def test_lean_oracle_divergence_like_full(oracle_mod):
    case = pair_case(8, 6, 1, h=0.25, dtau=50.0, nbody=0)
    errs = []
    for lean in (False, True):
        with pytest.raises(oracle_mod.OracleDivergence) as ei:
            oracle_mod.run(case, 100, lean=lean)
        e = ei.value
        errs.append((e.iteration, e.stage, e.block, e.i, e.j, e.p, e.n))
    assert errs[0] == errs[1]
