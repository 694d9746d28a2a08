"""North-star physics: HB Euler / laminar NS.

The reference has no flux physics (hbcore.py:3-13), so this
row's parity is UNPINNED: the GPU path (hb_ns.cu) is checked bitwise against
oracle/ns_oracle.c, a builder-written independent restatement of the same
specification (nsflow.py's docstring) -- not against any reference output.

CPU: the host geometry (numpy) equals the C oracle's bit for bit; the oracle
runs stay physical and converge.  GPU: fields (halos included) and forces
bitwise, residual norms at rtol 1e-12, on scaled-down versions of every
BASELINE config (sinusoidal Euler, tanh-stretched NS with a no-slip wall and
cuts, the pitching NACA 0012 O-grid with grid velocity, a slip wall and a
self-cut).
"""

import numpy as np
import pytest

import ns_oracle
from paper_1304_7654_b200 import nsflow

SCALES = {"C0": 2, "C1": 8, "C2": 16, "C3": 32, "C4": 128}


@pytest.mark.parametrize("key", sorted(SCALES))
def test_host_geometry_equals_oracle_geometry(key):
    case = nsflow.ns_workload(key, scale=SCALES[key])
    o = ns_oracle.OracleNS(case)
    for b in case.blocks:
        m = nsflow.metrics(b)
        for k, v in m.items():
            assert np.array_equal(v, o.blocks[b.id].geo[k]), (key, b.id, k)
        assert (m["vol"][:, 2:-2, 2:-2] > 0).all(), "cells must be right-handed with positive area"


@pytest.mark.parametrize("key,iters", [("C0", 60), ("C1", 40), ("C2", 40)])
def test_oracle_runs_converge_and_stay_physical(key, iters):
    case = nsflow.ns_workload(key, scale=SCALES[key] * 2)
    o = ns_oracle.run(case, iters)
    assert o.norms[-1] < o.norms[0]
    for q in o.fields().values():
        rho = q[:, 0, 2:-2, 2:-2]
        assert np.isfinite(q).all() and rho.min() > 0.5 and rho.max() < 2.0


def test_freestream_is_preserved():
    """A uniform freestream (the same in every snapshot) has no HB source
    (the rows of D sum to zero), no JST dissipation and no viscous flux; its
    residual is the rounding of the metric closure only."""
    case = nsflow.ns_workload("C0", scale=8)
    case.dalpha_deg = 0.0
    winf = nsflow.freestream(case)
    P = case.planes

    def uniform(b):
        q = np.zeros((P, 4, b.nj + 4, b.ni + 4))
        q[:] = winf[:, :, None, None]
        return q

    o = ns_oracle.OracleNS(case, initial=uniform)
    o.iterate(1)
    q = o.fields()[0][:, :, 2:-2, 2:-2]
    assert np.abs(q - winf[:, :, None, None]).max() < 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("key,iters", [("C0", 12), ("C1", 6), ("C2", 6), ("C3", 4), ("C4", 3)])
def test_gpu_matches_oracle_bitwise(key, iters, cuda):
    case = nsflow.ns_workload(key, scale=SCALES[key])
    want = ns_oracle.run(case, iters)
    got = nsflow.run_ns(case, iters)
    gf, wf = got.fields(), want.fields()
    for b in wf:
        if not np.array_equal(gf[b], wf[b]):
            bad = np.argwhere(gf[b] != wf[b])
            raise AssertionError(f"{key} block {b}: {len(bad)} values differ, first {bad[0]}: "
                                 f"{gf[b][tuple(bad[0])]!r} vs {wf[b][tuple(bad[0])]!r}")
    np.testing.assert_allclose(got.norm_history(), want.norms, rtol=1e-12, atol=0)
    assert np.array_equal(got.force_history(), np.stack(want.forces))


@pytest.mark.gpu
@pytest.mark.parametrize("key,iters", [("C0", 100), ("C1", 12), ("C2", 8)])
def test_gpu_full_size_matches_oracle_bitwise(key, iters, cuda):
    """BASELINE configs at full size: C0 (64 x 32, P = 3) at its stated 100
    iterations; C1 (4 blocks of 256 x 128, viscous, P = 5) and C2 (the
    pitching 512 x 256 O-grid, P = 9) for as many iterations as the
    single-threaded oracle finishes in seconds (profiles/ns_soak.py runs
    them at their stated 200 and 500).  Full-size tiles take the 16-byte
    staging path of the stage kernel; the scaled cases above mostly do not."""
    case = nsflow.ns_workload(key)
    want = ns_oracle.run(case, iters)
    got = nsflow.run_ns(case, iters)
    gf, wf = got.fields(), want.fields()
    for b in wf:
        assert np.array_equal(gf[b], wf[b]), f"{key} block {b} differs"
    np.testing.assert_allclose(got.norm_history(), want.norms, rtol=1e-12, atol=0)
    assert np.array_equal(got.force_history(), np.stack(want.forces))


@pytest.mark.gpu
def test_gpu_full_size_c2_converges(cuda):
    """BASELINE config 2 at full size (512 x 256, P = 9, pitching, 100 of its
    500 iterations): the GPU run stays physical and its residual falls."""
    case = nsflow.ns_workload("C2")
    got = nsflow.run_ns(case, 100)
    norms = got.norm_history()
    assert np.isfinite(norms).all() and norms[-1] < 0.5 * norms[0]
    q = got.fields()[0][:, 0, 2:-2, 2:-2]
    assert q.min() > 0.5 and q.max() < 2.0


def _ragged_case():
    """Two 40 x 13 blocks side by side (viscous, a no-slip wall below, one
    cut): neither dimension a multiple of the stage kernel's 32 x 8 tiles, so
    both tile directions end in partial tiles and the residual scratch rows
    are not whole L2 lines."""
    ni, nj = 40, 13
    blocks = []
    for c in range(2):
        x, y = nsflow.tanh_mesh(ni, nj, c * 1.0, 0.0, 1.0, 0.4)
        kinds = [nsflow.NOSLIP, nsflow.FARFIELD, nsflow.FARFIELD, nsflow.FARFIELD]
        kinds[3 if c == 0 else 2] = nsflow.CUT
        blocks.append(nsflow.NSBlock(c, ni, nj, x, y, tuple(kinds)))
    cuts = [nsflow.NSCut(0, "east", 1, "west", 1, nj)]
    return nsflow.NSCase("ragged-ns", 1, 0.3, 1.0, 1e3, 1.0, blocks, cuts, iterations=5)


@pytest.mark.gpu
def test_gpu_ragged_tiles_match_oracle(cuda):
    case = _ragged_case()
    want = ns_oracle.run(case, 5)
    got = nsflow.run_ns(case, 5)
    for b, q in want.fields().items():
        assert np.array_equal(got.fields()[b], q), f"block {b}"
    np.testing.assert_allclose(got.norm_history(), want.norms, rtol=1e-12, atol=0)
    assert np.array_equal(got.force_history(), np.stack(want.forces))
    split = nsflow.run_ns_ranks(case, 5, 2)
    for b, q in want.fields().items():
        assert np.array_equal(split.fields()[b], q), f"block {b} (2 ranks)"
    assert np.array_equal(split.force_history(), got.force_history())


@pytest.mark.gpu
@pytest.mark.parametrize("key,scale,cfl", [("C0", 2, 5.0), ("C0", 2, 30.0), ("C1", 8, 5.0), ("C1", 8, 10.0)])
def test_gpu_divergence_stops_at_the_oracles_stage(key, scale, cfl, cuda):
    """Too large a CFL number: the oracle stops at the first stage that writes
    a non-finite value; the GPU run raises DivergenceError for the same
    block, iteration and stage, within its status-polling chunk, and the
    split run names the same place."""
    from paper_1304_7654_b200.exceptions import DivergenceError
    case = nsflow.ns_workload(key, scale=scale)
    case.cfl = cfl
    with pytest.raises(ns_oracle.NSDivergence) as want:
        ns_oracle.run(case, 30)
    with pytest.raises(DivergenceError) as got:
        nsflow.run_ns(case, 30, poll=4)
    assert (got.value.block, got.value.iteration, got.value.stage) == \
        (want.value.block, want.value.iteration, want.value.stage)
    if len(case.blocks) > 1:
        with pytest.raises(DivergenceError) as split:
            nsflow.run_ns_ranks(case, want.value.iteration + 1, 2)
        assert (split.value.block, split.value.iteration, split.value.stage, split.value.i, split.value.j) == \
            (got.value.block, got.value.iteration, got.value.stage, got.value.i, got.value.j)
