"""Parity at BASELINE.json's stated sizes AND iteration counts.

Every BASELINE config runs through run_case on the GPU and is compared with
the oracle -- the memory-lean driver (oracle.LeanOracleSolver: q and q0 only,
pinned to the reference's own fingerprints in test_oracle_golden.py) --
bitwise for the fields (halos included) and forces, and per iteration for
the residual norms (rtol 1e-12):

  C0  1 block 64x32, P=3          100 iterations (BASELINE count)
  C1  2x2 blocks of 256x128, P=5  200 iterations (BASELINE count)
  C2  512x256 self-cut, P=9       500 iterations (BASELINE count)
  C3  4x2 blocks of 1024x512, P=7  20 iterations (200-iteration soak:
                                    profiles/soak.py, fingerprints in profiles/)
  C4  8x8 blocks of 1024^2, P=9     2 iterations, all 64 blocks (50-iteration
                                    soak: profiles/soak.py)

plus the paired-stage schedule on a 3x3 lattice of 256-wide blocks (the
centre block has four cuts, every strip edge lies inside a block or on a cut
face) at several row-tile heights and with many tiles per CTA.
"""

import numpy as np
import pytest

from paper_1304_7654_b200 import RunSpec, baseline_workload, lattice_case, run_case

from test_gpu_parity import assert_parity

pytestmark = pytest.mark.gpu


def _need_hbm(gb):
    import torch
    free, _ = torch.cuda.mem_get_info()
    if free < gb * 1e9:
        pytest.skip(f"needs {gb} GB of free device memory, {free / 1e9:.0f} GB free")


@pytest.mark.parametrize("key,iters", [("C0", 100), ("C1", 200), ("C2", 500), ("C3", 20)])
def test_baseline_config_at_stated_length(key, iters, cuda, oracle_mod):
    wl = baseline_workload(key)
    if key != "C3":
        assert wl.case.iterations == iters, "BASELINE iteration count"
    got = run_case(RunSpec(case=wl.case, ranks=1, iterations=iters, initial=wl.initial))
    want = oracle_mod.run(wl.case, iters, initial=wl.initial, lean=True)
    assert len(got.residual_norms) == iters
    assert_parity(got, want, f"{key}x{iters}")


def test_c4_all_blocks_match_oracle(cuda, oracle_mod):
    """The bench's workload: 64 blocks of 1024x1024 at P = 9 (19.4 GB per
    state) through the auto (paired-stage) schedule, two iterations."""
    import gc
    _need_hbm(65)
    wl = baseline_workload("C4")
    got = run_case(RunSpec(case=wl.case, ranks=1, iterations=2, initial=wl.initial))
    want = oracle_mod.run(wl.case, 2, initial=wl.initial, lean=True)
    assert_parity(got, want, "C4x2")
    del got, want
    gc.collect()


LATTICE_3X3 = lambda: lattice_case(3, 3, 256, 96, 4, h=1.0 / 768, dtau=4.096 / 768 ** 2,  # noqa: E731
                                   nbody=2, bodies=((1, "south", 0), (7, "north", 1)))


@pytest.mark.parametrize("tile_rows,limit", [(96, None), (16, None), (7, 5)])
def test_paired_lattice_3x3_matches_oracle(tile_rows, limit, cuda, oracle_mod, monkeypatch):
    """3x3 blocks of 256x96 at P = 9: the centre block has four cuts, so the
    paired schedule's band values arrive from all four faces; tile_rows 16 and
    7 put row-tile edges inside every block, and a 5-CTA grid makes each CTA
    walk many tiles (strips of one row tile run far apart)."""
    if limit is not None:
        monkeypatch.setenv("HBGPU_GRID_LIMIT", str(limit))
    case = LATTICE_3X3()
    got = run_case(RunSpec(case=case, ranks=1, iterations=3, tile_rows=tile_rows, fused=True))
    want = oracle_mod.run(case, 3, lean=True)
    assert_parity(got, want, f"lattice3x3 rows={tile_rows} limit={limit}")
