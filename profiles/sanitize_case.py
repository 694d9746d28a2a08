"""Small many-tiles cases for compute-sanitizer (racecheck / synccheck).

Paired schedule (pair + band kernels) and single stages on a 2x2 lattice of
256 x 24 blocks, P = 9, 8-row tiles, with the persistent grid capped at 3 CTAs
(HBGPU_GRID_LIMIT, set by the caller) so every CTA walks many tiles through
its TMA / mbarrier rings; each run is checked bitwise against the oracle.

  HBGPU_GRID_LIMIT=3 compute-sanitizer --tool racecheck python profiles/sanitize_case.py
"""
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [REPO, os.path.join(REPO, "oracle")]

import numpy as np  # noqa: E402

import oracle  # noqa: E402  (the checker)
from paper_1304_7654_b200 import RunSpec, lattice_case, run_case  # noqa: E402

case = lattice_case(2, 2, 256, 24, 4, h=0.01, dtau=0.0002, nbody=1, bodies=((3, "north", 0),))
want = oracle.run(case, 2, lean=True)
for fused in (True, False):
    got = run_case(RunSpec(case=case, ranks=1, iterations=2, tile_rows=8, fused=fused, use_graph=False))
    for b in want.fields:
        assert np.array_equal(got.fields[b], want.fields[b]), f"fused={fused} block {b}"
    print(f"fused={fused}: bitwise equal to the oracle", flush=True)
